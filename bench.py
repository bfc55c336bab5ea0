#!/usr/bin/env python
"""FlashSparse-on-B200 benchmark (BASELINE.json metric: effective GFLOP/s =
2*nnz*N / t, plus the HBM-roofline fraction).

Workload (BASELINE.json configs[2], the north star's target): SpMM FP16,
N = 128, on a Reddit-shaped synthetic power-law graph (Chung-Lu, 232,965
nodes, ~115 M nnz, uniform [-1,1) values, seeded) -- generated on the GPU,
converted CSR -> ME-BCRS once on the GPU (timed separately as encode_ms).
One step = one SpMM over the resident ME-BCRS and dense B (the hot path).
L2 is flushed (256 MB write) before every timed step.

  python bench.py [--gpus N --steps K --warmup W] [--impl reference]

N > 1 (torchrun, one rank per GPU): row windows are sharded into contiguous
ranges balanced by nnz; B is broadcast once over NCCL (timed separately);
each rank runs its shard; the step time is the max over ranks (strong
scaling of one graph).  --impl reference times the reference's own CPU
implementation (oracle/_ref: the unmodified reference headers) on bounded
samples of the same workload, on all host cores, rank 0 only.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# mma.sync (HMMA) peak measured on B200 by tools/mma_peak.cu, TFLOP/s.
MMA_SYNC_PEAK_TFLOPS = {"fp16": 554.6, "tf32": 277.7}
# Hardware L2 -> SM gather peak (random 256-byte rows, LDG.128 only), as last
# measured by tools/l2_gather_peak on a B200 (profiles/r2_l2_gather_peak.json);
# bench.py re-measures it in the run and uses this only when the probe is missing.
L2_GATHER_PEAK_GBS = 18953.9
METRIC = "SpMM/SDDMM effective GFLOP/s (2·nnz·N) and % HBM roofline at 1/2/4/8 B200"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=100)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--n", type=int, default=128)
    p.add_argument("--precision", default="fp16", choices=["fp16", "tf32"])
    p.add_argument("--workload", default="c3", choices=["c3", "c1"])
    p.add_argument("--e2e-steps", type=int, default=9)
    p.add_argument("--cpu-seconds", type=float, default=15.0, help="CPU-baseline sample budget")
    p.add_argument("--quick", action="store_true", help="kernel timing only (for ncu runs)")
    return p.parse_args()


# ------------------------------------------------------------------ helpers
def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


class NvmlClockSampler:
    """SM clock and throttle reasons sampled every 10 ms through NVML during
    the timed region (the nvidia-smi loop needs longer to start than a
    sub-second timed region lasts)."""

    # nvmlClocksEventReason* bits
    BITS = {"sw_power_cap": 0x4, "hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40}
    lead_s = 0.0

    def __init__(self, device):
        import pynvml

        self.nv = pynvml
        pynvml.nvmlInit()
        props = torch.cuda.get_device_properties(device)
        try:
            bus = f"{props.pci_domain_id:08x}:{props.pci_bus_id:02x}:{props.pci_device_id:02x}.0"
            self.h = pynvml.nvmlDeviceGetHandleByPciBusId(bus)
        except Exception:
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device)
        self.max = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        self.sm, self.reasons, self.run, self.t = [], 0, False, None

    def _loop(self):
        nv = self.nv
        while self.run:
            self.sm.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
            try:
                self.reasons |= nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            except Exception:
                self.reasons |= nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
            time.sleep(0.01)

    def start(self):
        self.run = True
        self.t = threading.Thread(target=self._loop, daemon=True)
        self.t.start()

    def stop(self):
        self.run = False
        self.t.join(1)
        return {"sm_mhz": statistics.median(self.sm) if self.sm else None, "sm_max_mhz": self.max,
                "reasons": sorted(k for k, b in self.BITS.items() if self.reasons & b), "samples": len(self.sm),
                "sampler": "nvml 10 ms"}


def clock_sampler(device):
    try:
        return NvmlClockSampler(device)
    except Exception:
        return ClockSampler(device)


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    lead_s = 0.15
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device, self.proc, self.lines = device, None, []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                          "-lms", "50", "-i", str(self.device)], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.12)
        self.proc.terminate()
        try:
            self.proc.wait(2)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                mx = float(f[1])
            except ValueError:
                continue
            for nm, val in zip(names, f[3:7]):
                if val.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def small_configs(device):
    """BASELINE configs[0]/[1] (4096^2, 16 nnz/row): launch-latency-bound, so
    timed as CUDA-graph replays of 200 back-to-back calls (us per call)."""
    import paper_2412_11007_b200.tcsparse as T
    from paper_2412_11007_b200 import _abi, graphs as G

    # the reference's own C1 inputs (generate.hpp restated in graphs.py;
    # tests/test_graphs.py pins them to the golden hashes): seed 1, real mode
    rows = cols = 4096
    rp, ci, v = (torch.from_numpy(x.view("int32") if x.dtype.kind == "u" else x).to(device)
                 for x in G.reference_random_csr(rows, cols, 16.0 / 4096, 1, "real"))
    nnz = ci.numel()
    csr = T.CsrMatrix(rows, cols, rp, ci, v)
    out = {}
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def timed(fn, reps=200):
        fn()
        torch.cuda.synchronize()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        graph = None
        try:
            with torch.cuda.stream(s):
                fn()
            torch.cuda.synchronize()
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph, stream=s):
                for _ in range(reps):
                    fn()
        except Exception:
            graph = None
            torch.cuda.synchronize()
        e0.record()
        if graph is not None:
            graph.replay()
        else:
            for _ in range(reps):
                fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) * 1e3 / reps, graph is not None

    peak, _ = peaks()
    for pname, prec, dt in (("fp16", T.Precision.fp16, torch.float16), ("tf32", T.Precision.tf32, torch.float32)):
        me = T.encode_mebcrs(csr, prec)
        W, nv = me.num_windows, me.num_vectors
        vw = 2 if dt == torch.float16 else 4
        vwA = 2 if me.value_dtype == _abi.TCS_DTYPE_F16 else 4
        B = torch.from_numpy(G.reference_random_dense(cols, 128, 2, "real")).to(device=device, dtype=dt)
        C = torch.empty(rows, 128, device=device)
        us, g = timed(lambda: T.spmm(me, B, T.KernelConfig(prec), out=C))
        balg = bytes_alg_spmm(W, nv, rows, 128, vwA, vw)
        out[f"c1_spmm_{pname}_n128_us"] = round(us, 2)
        out[f"c1_spmm_{pname}_gflops"] = round(2.0 * nnz * 128 / (us * 1e-6) / 1e9, 1)
        out[f"c1_spmm_{pname}_roofline"] = {"bytes_alg": balg, "frac": round(balg / (us * 1e-6) / 1e9 / peak, 4),
                                            "us_at_peak": round(balg / (peak * 1e9) * 1e6, 2),
                                            "dram": _with_frac(dram_traffic(f"c1_{pname}_n128_g1"), us / 1e3)}
        A = torch.from_numpy(G.reference_random_dense(rows, 32, 3, "real")).to(device=device, dtype=dt)
        Bt = torch.from_numpy(G.reference_random_dense(cols, 32, 4, "real")).to(device=device, dtype=dt)
        ov = torch.empty(8 * me.num_vectors, device=device)
        ops = T.SddmmOperands(me, A, Bt)
        us2, g2 = timed(lambda: T.sddmm(ops, T.KernelConfig(prec), out_values=ov))
        sbalg = bytes_alg_sddmm(W, nv, rows, 32, vwA, vw)
        out[f"c2_sddmm_{pname}_k32_us"] = round(us2, 2)
        out[f"c2_sddmm_{pname}_gflops"] = round(2.0 * nnz * 32 / (us2 * 1e-6) / 1e9, 1)
        out[f"c2_sddmm_{pname}_roofline"] = {"bytes_alg": sbalg, "frac": round(sbalg / (us2 * 1e-6) / 1e9 / peak, 4),
                                             "us_at_peak": round(sbalg / (peak * 1e9) * 1e6, 2),
                                             "dram": _with_frac(dram_traffic(f"c2_sddmm_{pname}_f32_g1"), us2 / 1e3)}
        out["graph_captured"] = bool(g and g2)
        me.free()
    t = []
    for _ in range(5):  # conversion synchronises (data-dependent sizes): eager timing
        e0.record()
        m = T.encode_mebcrs(csr, T.Precision.fp16)
        e1.record()
        torch.cuda.synchronize()
        t.append(e0.elapsed_time(e1) * 1e3)
        m.free()
    out["c2_encode_fp16_us"] = round(sorted(t)[len(t) // 2], 1)
    out["nnz"] = int(nnz)
    return out


def layer_configs(device):
    """BASELINE configs[3]/[4] on this GPU (reported beside the headline, not
    the metric): the GCN layer on the ogbn-products-shaped graph (F = 128)
    and the AGNN layer on R-MAT scale 23 (F = 32).  CUDA events, L2 flushed
    before every timed call, median of 5."""
    import paper_2412_11007_b200.layers as L
    import paper_2412_11007_b200.tcsparse as T
    from paper_2412_11007_b200 import graphs as G

    flush = torch.empty(64 << 20, dtype=torch.int32, device=device)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def timed(fn, reps=5):
        fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(reps):
            flush.zero_()
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        return round(sorted(ts)[len(ts) // 2], 3)

    out = {}
    peak, _ = peaks()

    def roof(bytes_alg, bytes_min, ms, key):
        d = {"bytes_alg": bytes_alg, "frac": round(bytes_alg / (ms / 1e3) / 1e9 / peak, 4)}
        if bytes_min is not None:
            d["bytes_min"] = bytes_min
            d["frac_bytes_min"] = round(bytes_min / (ms / 1e3) / 1e9 / peak, 4)
        d["dram"] = _with_frac(dram_traffic(key), ms)
        return d

    rows, _, rp, ci, _ = G.power_law_csr(G.C4_PRODUCTS, values="real", device=device)
    W = torch.randn(128, 128, device=device).half() / 128 ** 0.5
    H = torch.randn(rows, 128, device=device).half()
    gcn = L.GCNLayer(rows, rp, ci, W)
    adj = gcn.adj
    HW = (H @ W).contiguous()
    Cf = torch.empty(rows, 128, device=device)
    spmm_ms = timed(lambda: T.spmm(adj, HW, gcn.cfg, out=Cf))
    nv, Wn = adj.num_vectors, adj.num_windows
    out["c4_gcn"] = {"nodes": rows, "nnz": int(ci.numel()), "adjacency": "D^-1/2 (A + I) D^-1/2", "F": 128,
                     "degree_cap": f"Chung-Lu hub weight cap {G.C4_PRODUCTS.cap:g}x mean weight (SURVEY 8(d))",
                     "layer_ms": timed(lambda: gcn(H)), "precision": "fp16", "path": "cuBLAS GEMM + tcs_spmm",
                     "spmm_ms": spmm_ms,
                     "spmm_roofline": roof(bytes_alg_spmm(Wn, nv, rows, 128, 2, 2),
                                           bytes_alg_spmm(Wn, nv, rows, 128, 2, 2) - nv * 128 * 2 + rows * 128 * 2,
                                           spmm_ms, "c4_fp16_n128_g1")}
    del gcn, H, HW, Cf, adj, rp, ci
    torch.cuda.empty_cache()
    rows, _, rp, ci, _ = G.rmat_csr(G.C5_RMAT, values="real", device=device)
    H = torch.randn(rows, 32, device=device)
    agnn = L.AGNNLayer(rows, rp, ci, beta=1.0)
    mask = agnn.mask
    nv, Wn = mask.num_vectors, mask.num_windows
    Hh = H.half().contiguous()
    Cf = torch.empty(rows, 32, device=device)
    sp_ms = timed(lambda: T.spmm(mask, Hh, agnn.cfg, out=Cf))
    ov = torch.empty(8 * nv, device=device)
    ops = T.SddmmOperands(mask, Hh, Hh)
    sd_ms = timed(lambda: T.sddmm(ops, agnn.mask_cfg, out_values=ov))
    out["c5_agnn"] = {"nodes": rows, "nnz": int(ci.numel()), "F": 32, "layer_ms": timed(lambda: agnn(H)),
                      "precision": "fp16", "path": "rows_normalize (f16 copy) + tcs_agnn_attend (one pass, static mask)",
                      "spmm_n32_ms": sp_ms,
                      "spmm_n32_roofline": roof(bytes_alg_spmm(Wn, nv, rows, 32, 2, 2),
                                                bytes_alg_spmm(Wn, nv, rows, 32, 2, 2) - nv * 32 * 2 + rows * 32 * 2,
                                                sp_ms, "c5_fp16_n32_g1"),
                      "sddmm_f32_static_mask_ms": sd_ms,
                      "sddmm_f32_roofline": roof(bytes_alg_sddmm(Wn, nv, rows, 32, 2, 2, pattern_bytes=nv), None,
                                                 sd_ms, "c5_sddmm_fp16_f32_g1")}
    del agnn, H, Hh, Cf, ov, ops, mask, rp, ci
    torch.cuda.empty_cache()
    return out


def dram_traffic(key):
    """ncu-measured DRAM bytes per launch of the dominant kernel for this
    config (profiles/traffic.json, written by tools/traffic_from_ncu.py from
    a `ncu --set full` capture).  `current` says whether the kernel sources
    the capture was taken on are the ones in this tree."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            tj = json.load(f)
    except Exception:
        return None
    e = tj.get(key)
    if not isinstance(e, dict):
        return None
    out = {k: e[k] for k in ("bytes_per_launch", "l2_hit_pct", "source") if k in e}
    out["current"] = e.get("csrc_sha") == csrc_sha()
    return out


def _with_frac(dram, ms):
    """dram_traffic() plus the measured DRAM bytes / time against the HBM peak."""
    if not dram:
        return None
    return dict(dram, frac_dram=round(dram["bytes_per_launch"] / (ms / 1e3) / 1e9 / peaks()[0], 4))


def csrc_sha():
    import hashlib

    h = hashlib.sha256()
    d = os.path.join(ROOT, "paper_2412_11007_b200", "csrc")
    for name in sorted(os.listdir(d)):
        with open(os.path.join(d, name), "rb") as f:
            h.update(name.encode() + f.read())
    return h.hexdigest()[:16]


def l2_gather_peak():
    """Hardware L2 -> SM gather peak measured now by tools/l2_gather_peak
    (random 256-B rows of a 60 MB table, LDG.128 only, best over memory-level
    parallelism and occupancy)."""
    exe = os.path.join(ROOT, "tools", "l2_gather_peak")
    try:
        r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
        d = json.loads(r.stdout.strip().splitlines()[-1])
        return {"peak_gbs": float(d["l2_gather_peak_gbs"]), "source": "measured in this run (tools/l2_gather_peak)"}
    except Exception:
        return {"peak_gbs": L2_GATHER_PEAK_GBS, "source": "profiles/r2_l2_gather_peak.json (probe unavailable)"}


def bytes_alg_spmm(W, nv, rows, N, vwA, vwB):
    """row pointers + column indices + sparse values (no padding)
    + one N-wide dense row per stored vector + the fp32 C write."""
    return 4 * (W + 1) + 4 * nv + 8 * nv * vwA + nv * N * vwB + 4 * rows * N


def bytes_alg_sddmm(W, nv, rows, F, vwA, vwB, pattern_bytes=None, vo=4):
    """row pointers + column indices + the mask pattern (its
    stored values, or 1 liveness byte per vector) + the A rows once + one
    F-wide Bt row per stored vector + the 8 output values per vector."""
    P = 8 * nv * vwA if pattern_bytes is None else pattern_bytes
    return 4 * (W + 1) + 4 * nv + P + rows * F * vwB + nv * F * vwB + 8 * nv * vo


# --------------------------------------------------------------- workloads
def build_graph(args, device):
    from paper_2412_11007_b200 import graphs as G

    if args.workload == "c3":
        rows, cols, rp, ci, v = G.power_law_csr(G.C3_REDDIT, values="real", device=device)
        desc = "C3 SpMM on Reddit-shaped synthetic power-law graph (Chung-Lu alpha=1.2, hub cap 60x mean)"
    else:
        rows = cols = 4096
        rp, ci, v = (torch.from_numpy(x.view("int32") if x.dtype.kind == "u" else x).to(device)
                     for x in G.reference_random_csr(rows, cols, 16.0 / 4096, 1, "real"))
        desc = "C1 SpMM on the reference's generate_random_sparse_real(4096, 4096, 16/4096, seed 1)"
    return rows, cols, rp, ci, v, desc


# ---------------------------------------------------------------- ours
def run_ours(args, rank, world, device):
    import paper_2412_11007_b200.tcsparse as T
    from paper_2412_11007_b200 import _abi, distributed as D, graphs as G

    prec = T.Precision.fp16 if args.precision == "fp16" else T.Precision.tf32
    N = args.n
    rows, cols, rp, ci, v, desc = build_graph(args, device)
    nnz_total = int(ci.numel())
    shard = D.shard_of(D.shard_windows(rp, rows, world), rank, rows)  # nnz-balanced window range
    lrp, lci, lv = D.local_rows(rp, ci, v, shard)
    l_rows = shard.rows
    local_csr = T.CsrMatrix(l_rows, cols, lrp, lci, lv)
    del rp, ci, v

    # dense operand: generated on rank 0, broadcast over NCCL (timed separately)
    dt = torch.float16 if prec == T.Precision.fp16 else torch.float32
    B = G.dense(cols, N, 3, values="real", dtype=dt, device=device) if rank == 0 else \
        torch.empty(cols, N, dtype=dt, device=device)
    bcast_ms = 0.0
    if world > 1:
        torch.distributed.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        D.broadcast_dense(B, src=0)
        e1.record()
        torch.cuda.synchronize()
        bcast_ms = e0.elapsed_time(e1)

    # CSR -> ME-BCRS on the GPU (timed once, after one warm-up conversion)
    me = T.encode_mebcrs(local_csr, prec)
    me.free()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    me = T.encode_mebcrs(local_csr, prec)
    e1.record()
    torch.cuda.synchronize()
    encode_ms = e0.elapsed_time(e1)
    nv, W = me.num_vectors, me.num_windows
    nnz_local = local_csr.nnz
    # tensor work the kernel issues: one MMA k-step per kin vectors of a
    # window (16 FP16 / 8 TF32, residue steps padded), 8 rows x N features
    rp_host = np.empty(W + 1, np.uint32)
    rc = _abi.load().tcs_mebcrs_download(C.byref(me._h), rp_host.ctypes.data, None, None,
                                         C.c_void_p(torch.cuda.current_stream().cuda_stream))
    assert rc == 0, _abi.load().tcs_last_error()
    kin = 16 if prec == T.Precision.fp16 else 8
    tensor_flops = 2.0 * 8 * kin * N * float(((np.diff(rp_host.astype(np.int64)) + kin - 1) // kin).sum())

    out = torch.empty(l_rows, N, dtype=torch.float32, device=device)
    cfg = T.KernelConfig(prec)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.int32, device=device)  # 256 MB > 126 MB L2
    for _ in range(args.warmup):
        flush.zero_()
        T.spmm(me, B, cfg, out=out)
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    sampler = clock_sampler(device.index if device.index is not None else 0)
    sampler.start()
    time.sleep(sampler.lead_s)  # nvidia-smi loop start-up; NVML samples at once
    l0 = T.launch_count()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    torch.cuda.synchronize()
    for a, b in evs:
        flush.zero_()
        a.record()
        T.spmm(me, B, cfg, out=out)
        b.record()
    torch.cuda.synchronize()
    launches = T.launch_count() - l0
    clocks = sampler.stop()
    times = [a.elapsed_time(b) for a, b in evs]
    step_ms = sum(times) / len(times)
    t = torch.tensor([step_ms], dtype=torch.float64, device=device)
    if world > 1:
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        torch.distributed.barrier()
    step_ms_max = float(t.item())

    # back-to-back (no flush) for reference
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10):
        T.spmm(me, B, cfg, out=out)
    b.record()
    torch.cuda.synchronize()
    b2b_ms = a.elapsed_time(b) / 10

    # instruction-path comparison (north star: mma.sync weighed against tcgen05)
    paths = {}
    if not args.quick:
        for path in ("mma_sync", "tcgen05"):
            pc = T.KernelConfig(prec, path=path)
            try:
                T.spmm(me, B, pc, out=out)
            except T.TcsError:
                continue
            ts = []
            for _ in range(10):
                flush.zero_()
                a.record()
                T.spmm(me, B, pc, out=out)
                b.record()
                torch.cuda.synchronize()
                ts.append(a.elapsed_time(b))
            paths[path] = round(sum(ts) / len(ts), 4)

    # the same SpMM in TF32 (BASELINE configs: C3 TF32 N = 64/128/256): its own
    # ME-BCRS (f32 values, k = 4) and an f32 dense operand, L2 flushed per call
    tf32 = None
    if not args.quick and prec == T.Precision.fp16:
        me32 = T.encode_mebcrs(local_csr, T.Precision.tf32)
        B32 = G.dense(cols, N, 3, values="real", dtype=torch.float32, device=device)
        c32 = T.KernelConfig(T.Precision.tf32)
        T.spmm(me32, B32, c32, out=out)
        ts = []
        for _ in range(10):
            flush.zero_()
            a.record()
            T.spmm(me32, B32, c32, out=out)
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        ms32 = sorted(ts)[len(ts) // 2]
        b32 = bytes_alg_spmm(me32.num_windows, me32.num_vectors, l_rows, N, 4, 4)
        tf32 = {"N": N, "ms": round(ms32, 4), "gflops": round(2.0 * nnz_local * N / (ms32 / 1e3) / 1e9, 1),
                "bytes_alg_per_launch": b32, "frac": round(b32 / (ms32 / 1e3) / 1e9 / peaks()[0], 4),
                "kernel": "tf32_pack_kernel + spmm_tf32p_kernel<2> (mma.sync m16n8k8 on the 2.5-byte packed operand)",
                "dram": _with_frac(dram_traffic("c3_tf32_n128_g1") if N == 128 and world == 1 else None, ms32)}
        me32.free()
        del B32

    # SDDMM on the same pattern (BASELINE metric covers SpMM/SDDMM; F = 32 as configs[1])
    sddmm = None
    if True:
        F = 32
        Ad = G.dense(l_rows, F, 4, values="real", dtype=dt, device=device)
        Btd = G.dense(cols, F, 5, values="real", dtype=dt, device=device)
        ov = torch.empty(8 * nv, dtype=torch.float32, device=device)
        ops = T.SddmmOperands(me, Ad, Btd)
        def sd_time(c):
            T.sddmm(ops, c, out_values=ov)
            ts = []
            for _ in range(10):
                flush.zero_()
                a.record()
                T.sddmm(ops, c, out_values=ov)
                b.record()
                torch.cuda.synchronize()
                ts.append(a.elapsed_time(b))
            return sum(ts) / len(ts)
        sd_ms = sd_time(cfg)
        # TCS_CFG_STATIC_MASK: the mask's sampling rule read from cached
        # liveness bytes (1 B per vector instead of its 8 stored values)
        sd_static_ms = sd_time(T.KernelConfig(prec, static_mask=True))
        vA = 2 if me.value_dtype == _abi.TCS_DTYPE_F16 else 4
        vB = 2 if dt == torch.float16 else 4
        sd_bytes = 4 * (W + 1) + 4 * nv + 8 * nv * vA + l_rows * F * vB + nv * F * vB + 8 * nv * 4
        peak_, _ = peaks()
        sddmm = {"F": F, "ms": round(sd_ms, 4), "gflops": round(2.0 * nnz_local * F / (sd_ms / 1e3) / 1e9, 1),
                 "bytes_alg_per_launch": sd_bytes, "achieved_gbs": round(sd_bytes / (sd_ms / 1e3) / 1e9, 1),
                 "frac": round(sd_bytes / (sd_ms / 1e3) / 1e9 / peak_, 4), "out": "f32 ME-BCRS values",
                 "dram": _with_frac(dram_traffic(f"{args.workload}_sddmm_{args.precision}_f{F}_g{world}"), sd_ms),
                 "ms_static_mask": round(sd_static_ms, 4),
                 "gflops_static_mask": round(2.0 * nnz_local * F / (sd_static_ms / 1e3) / 1e9, 1)}
        del Ad, Btd, ov

    vwA = 2 if me.value_dtype == _abi.TCS_DTYPE_F16 else 4
    vwB = 2 if dt == torch.float16 else 4
    balg = bytes_alg_spmm(W, nv, l_rows, N, vwA, vwB)
    bmin = 4 * (W + 1) + 4 * nv + 8 * nv * vwA + cols * N * vwB + 4 * l_rows * N
    peak, peak_src = peaks()
    achieved = balg / (step_ms / 1e3) / 1e9

    e2e = None
    if not args.quick:
        e2e = run_e2e(args, T, _abi, local_csr, B, l_rows, cols, N, prec, device, world)

    res = {"rank": rank, "nnz": nnz_local, "nv": nv, "W": W, "step_ms": step_ms, "encode_ms": encode_ms,
           "bytes_alg": balg, "bytes_min": bmin, "achieved": achieved, "tensor_flops": tensor_flops}
    gathered = [res]
    if world > 1:
        gathered = [None] * world
        torch.distributed.all_gather_object(gathered, res)
    if rank != 0:
        return None
    value = 2.0 * nnz_total * N / (step_ms_max / 1e3) / 1e9
    dram = dram_traffic(f"{args.workload}_{args.precision}_n{N}_g{world}")
    gather_bytes = nv * N * vwB  # the B-row gathers alone: what the L2 probe measures
    l2 = l2_gather_peak() if rank == 0 and not args.quick else {"peak_gbs": L2_GATHER_PEAK_GBS,
                                                                 "source": "profiles/r2_l2_gather_peak.json"}
    line = {
        "metric": METRIC, "value": round(value, 2), "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(step_ms_max, 4), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": args.precision, "data": "synthetic",
        "config": {"workload": desc + f", {args.precision.upper()} N={N}", "nodes": rows, "nnz": nnz_total,
                   "nv_8x1": sum(g["nv"] for g in gathered), "N": N, "precision": args.precision,
                   "values": "uniform [-1,1) (seeded)", "l2": "flushed before every timed step (256 MB write)",
                   "parallelism": f"row-window shards x{world} (nnz-balanced), B broadcast over NCCL",
                   "backend": os.environ.get("TCS_BENCH_BACKEND", "none")},
        # Contract fields: achieved = ALGORITHMIC bytes / kernel
        # time, against the measured HBM copy peak.  frac > 1 because B (60 MB
        # in f16) is L2-resident: the B-row gathers are served by L2, not HBM.
        # The resource that binds is the L2 -> SM gather path (l2_gather);
        # measured DRAM traffic (dram) is close to bytes_min.
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 4),
                     "traffic": dram["bytes_per_launch"] if dram else None, "peak_source": peak_src,
                     "bytes_alg_per_launch": balg, "bytes_min_per_launch": bmin,
                     "frac_bytes_min": round(bmin / (step_ms / 1e3) / 1e9 / peak, 4),
                     "kernel": ("spmm_f16_kernel<2,8> (mma.sync; L2-prefetch instance when B <= 80 MB) + claim-counter "
                                "memset + spmm_reduce_split") if prec == 0 else
                               "tf32_pack_kernel + spmm_tf32p_kernel<2> (mma.sync on the 2.5-byte packed operand)",
                     "binding_resource": ("l2_gather (L1 data pipe: one LDG + one SHFL wavefront per 128 B)" if prec == 0
                                          else "gather latency (long-scoreboard; 16 warps/SM at 117 registers)"),
                     "dram": _with_frac(dram, step_ms),
                     "l2_gather": {"gather_bytes_per_launch": gather_bytes,
                                   "achieved_gbs": round(gather_bytes / (step_ms / 1e3) / 1e9, 1),
                                   "peak_gbs": l2["peak_gbs"], "peak_source": l2["source"],
                                   "frac": round(gather_bytes / (step_ms / 1e3) / 1e9 / l2["peak_gbs"], 4)},
                     # the legacy tensor path this kernel uses (HMMA), against its
                     # measured peak; the tcgen05 bf16 peak for scale
                     "tensor_pipe": {"issued_tflop_per_launch": round(tensor_flops / 1e12, 4),
                                     "achieved_tflops": round(tensor_flops / (step_ms / 1e3) / 1e12, 2),
                                     "peak_mma_sync_tflops": MMA_SYNC_PEAK_TFLOPS[args.precision],
                                     "frac": round(tensor_flops / (step_ms / 1e3) / 1e12
                                                   / MMA_SYNC_PEAK_TFLOPS[args.precision], 4),
                                     "frac_of_tcgen05_bf16_peak": round(tensor_flops / (step_ms / 1e3) / 1e12
                                                                        / 1693.0, 4),
                                     "peak_source": "tools/mma_peak.cu (profiles/r1s4_mma_sync_peak.txt)"}},
        "gpu_launches": launches,
        "clocks": clocks,
        "encode_ms": round(max(g["encode_ms"] for g in gathered), 3),
        "back_to_back_ms": round(b2b_ms, 4),
        "path_ms": paths,
        "tf32": tf32,
        "sddmm": sddmm,
        "broadcast_ms": round(bcast_ms, 3),
        "shards": [{"nnz": g["nnz"], "nv": g["nv"], "step_ms": round(g["step_ms"], 4)} for g in gathered],
    }
    if e2e:
        line["e2e"] = e2e
    return line


def run_e2e(args, T, _abi, local_csr, B, rows, cols, N, prec, device, world):
    """Same metric through the reference-facing C-ABI call with HOST buffers:
    tcs_spmm_csr_host (ref CLI pipeline: encode_mebcrs + spmm) -- H2D of the
    CSR and f32 B, GPU conversion, SpMM, D2H of C, every step."""
    lib = _abi.load()
    rp = local_csr.row_ptr.cpu().pin_memory()
    ci = local_csr.col_idx.cpu().pin_memory()
    vals = local_csr.values.cpu().pin_memory()
    Bh = B.float().cpu().pin_memory()
    Ch = torch.empty(rows, N, dtype=torch.float32).pin_memory()
    csr = _abi.tcs_csr(rows, cols, local_csr.nnz, rp.data_ptr(), ci.data_ptr(), vals.data_ptr())
    cfg = _abi.tcs_kernel_config(int(prec), 8, 1, 0)
    stream = torch.cuda.current_stream()
    sp = C.c_void_p(stream.cuda_stream)
    rc = lib.tcs_spmm_csr_host(C.byref(csr), int(prec), Bh.data_ptr(), N, Ch.data_ptr(), C.byref(cfg), None, sp)
    assert rc == 0, lib.tcs_last_error()
    times = []
    for _ in range(args.e2e_steps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        rc = lib.tcs_spmm_csr_host(C.byref(csr), int(prec), Bh.data_ptr(), N, Ch.data_ptr(), C.byref(cfg), None, sp)
        b.record(stream)
        torch.cuda.synchronize()
        assert rc == 0, lib.tcs_last_error()
        times.append(a.elapsed_time(b))
    # median: one step in ~50 can catch a host-side stall (a 31 ms outlier
    # among 21 ms steps was seen); every step is listed in step_ms
    ms = sorted(times)[len(times) // 2]
    # link check: plain pinned H2D of the same CSR bytes in this process state
    d_ci = torch.empty_like(ci, device=device)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    d_ci.copy_(ci, non_blocking=True)
    b.record(stream)
    torch.cuda.synchronize()
    h2d_gbs = ci.numel() * 4 / (a.elapsed_time(b) / 1e3) / 1e9
    del d_ci
    t = torch.tensor([ms], dtype=torch.float64, device=device)
    nnz = torch.tensor([local_csr.nnz], dtype=torch.float64, device=device)
    if world > 1:
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        torch.distributed.all_reduce(nnz)
    h2d = (rows + 1) * 4 + local_csr.nnz * 8 + cols * N * 4
    d2h = rows * N * 4
    return {"value": round(2.0 * float(nnz.item()) * N / (float(t.item()) / 1e3) / 1e9, 2), "unit": "GFLOP/s",
            "ms_per_step": round(float(t.item()), 3), "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
            "step_ms": [round(x, 2) for x in times], "pinned_h2d_gbs": round(h2d_gbs, 1),
            "call": "tcs_spmm_csr_host (host CSR + host f32 B -> host f32 C; GPU encode + SpMM)"}


# ----------------------------------------------------------- reference arm
_HOST_GRAPH = {}


def host_graph(args, device):
    """The workload's CSR and dense operands on the host (built once)."""
    from paper_2412_11007_b200 import graphs as G

    key = (args.workload, args.precision, args.n)
    if key not in _HOST_GRAPH:
        rows, cols, rp, ci, v, _ = build_graph(args, device)
        dt = torch.float16 if args.precision == "fp16" else torch.float32
        g = {"rows": rows, "cols": cols, "rp": rp.cpu().numpy().view(np.uint32),
             "ci": ci.cpu().numpy().view(np.uint32), "v": v.cpu().numpy(),
             # the same operands run_ours uses (seeded), as f32 host arrays
             "B": np.ascontiguousarray(G.dense(cols, args.n, 3, values="real", dtype=dt, device=device)
                                       .float().cpu().numpy()),
             "A": np.ascontiguousarray(G.dense(rows, 32, 4, values="real", dtype=dt, device=device)
                                       .float().cpu().numpy()),
             "Bt": np.ascontiguousarray(G.dense(cols, 32, 5, values="real", dtype=dt, device=device)
                                        .float().cpu().numpy())}
        del rp, ci, v
        _HOST_GRAPH.clear()
        _HOST_GRAPH[key] = g
    return _HOST_GRAPH[key]


def reference_sample_runner(args, device, op="spmm"):
    """Returns (run_step(budget_s) -> (flops, seconds, nnz), description,
    threads).  Each step: the reference's encode_mebcrs + spmm (or + sddmm,
    F = 32) -- oracle/_ref, the unmodified reference headers, timed inside
    the shim around the reference calls only -- over disjoint 64-row slices
    (8 windows) spread over the workload, one slice per host thread."""
    import oracle as O

    g = host_graph(args, device)
    rows, cols, rp_h, ci_h, v_h = g["rows"], g["cols"], g["rp"], g["ci"], g["v"]
    N = args.n if op == "spmm" else 32
    threads = max(1, min(os.cpu_count() or 1, 64))
    prec = 0 if args.precision == "fp16" else 1
    lib = O.ref()
    dense = lib.ref_dense_new(cols, N, (g["B"] if op == "spmm" else g["Bt"]).ctypes.data_as(O._f32p))
    nslices = (rows + 63) // 64
    stride = max(1, nslices // 997)  # spread slices over the whole graph
    state = {"next": 0}
    lock = threading.Lock()

    def one_slice(idx):
        r0 = (idx * stride % nslices) * 64
        r1 = min(rows, r0 + 64)
        b, e = int(rp_h[r0]), int(rp_h[r1])
        srp = (rp_h[r0:r1 + 1] - rp_h[r0]).astype(np.uint32)
        sci = np.ascontiguousarray(ci_h[b:e])
        sv = np.ascontiguousarray(v_h[b:e])
        up = O._u32p
        if op == "spmm":
            Cm = np.empty((r1 - r0, N), np.float32)
            secs = lib.ref_time_encode_spmm(r1 - r0, cols, srp.ctypes.data_as(up), sci.ctypes.data_as(up),
                                            sv.ctypes.data_as(O._f32p), prec, dense, Cm.ctypes.data_as(O._f32p))
        else:
            As = np.ascontiguousarray(g["A"][r0:r1])
            cap = 8 * (e - b) + 64
            out = np.empty(cap, np.float32)
            secs = lib.ref_time_encode_sddmm(r1 - r0, cols, srp.ctypes.data_as(up), sci.ctypes.data_as(up),
                                             sv.ctypes.data_as(O._f32p), prec, As.ctypes.data_as(O._f32p), N,
                                             dense, out.ctypes.data_as(O._f32p), cap)
        assert secs >= 0
        return e - b, secs

    def run_step(budget_s):
        done = {"nnz": 0}
        t0 = time.perf_counter()

        def worker():
            while time.perf_counter() - t0 < budget_s:
                with lock:
                    idx = state["next"]
                    state["next"] += 1
                n, _ = one_slice(idx)
                with lock:
                    done["nnz"] += n

        ths = [threading.Thread(target=worker) for _ in range(threads)]
        for th in ths:
            th.start()
        for th in ths:
            th.join()
        secs = time.perf_counter() - t0
        return 2.0 * done["nnz"] * N, secs, done["nnz"]

    what = "spmm" if op == "spmm" else "sddmm (F=32, f32 output)"
    desc = (f"reference encode_mebcrs+{what} (oracle/_ref, -O3, unmodified headers) on 64-row slices "
            f"(8 windows) spread over the graph, {threads} threads")
    return run_step, desc, threads


def run_reference(args, rank, world, device):
    if rank != 0:
        return None
    run_step, desc, threads = reference_sample_runner(args, device)
    budget = max(0.5, min(4.0, 150.0 / max(1, args.steps + args.warmup)))
    for _ in range(args.warmup):
        run_step(budget)
    flops = secs = 0.0
    for _ in range(args.steps):
        f, s, _ = run_step(budget)
        flops += f
        secs += s
    value = flops / secs / 1e9
    return {"impl": "reference", "metric": METRIC, "value": round(value, 5), "unit": "GFLOP/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(secs / args.steps * 1e3, 2),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": args.precision,
            "data": "synthetic",
            "config": {"workload": "C3 SpMM on Reddit-shaped synthetic power-law graph" if args.workload == "c3"
                       else "C1 SpMM uniform 4096x4096", "N": args.n, "precision": args.precision},
            "cpu_baseline": {"value": round(value, 5), "unit": "GFLOP/s", "cores": threads, "kind": "reference",
                             "sample": desc + f", {budget:.1f}s per step"},
            "e2e": {"value": round(value, 5), "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def restatement_baseline(args, device, budget_s):
    """BASELINE.md / SURVEY §8(d) item 2: the CPU restatement of the reference
    semantics (oracle/oracle.cpp: ordered CSR loop with RNE operands, OpenMP
    over rows) on all host cores -- SpMM at N and SDDMM at F = 32 -- over a
    row sample sized to ~budget_s each.  Returns GFLOP/s per op."""
    import oracle as O

    g = host_graph(args, device)
    lib = O.lib()
    cores = os.cpu_count() or 1
    lib.orc_set_num_threads(cores)  # torchrun exports OMP_NUM_THREADS=1
    m = O.Csr(g["rows"], g["cols"], g["rp"], g["ci"], g["v"])
    prec = 0 if args.precision == "fp16" else 1
    rng = np.random.default_rng(7)
    out = {"cores": int(lib.orc_num_threads()), "kind": "port",
           "what": "oracle/oracle.cpp CSR-form restatement (bit-exact with the reference), OpenMP"}
    for op in ("spmm", "sddmm"):
        frac = 0.002
        while True:
            sel = np.sort(rng.choice(g["rows"], max(1, int(g["rows"] * frac)), replace=False)).astype(np.uint64)
            nnz = int((g["rp"][sel.astype(np.int64) + 1].astype(np.int64) - g["rp"][sel.astype(np.int64)]).sum())
            t0 = time.perf_counter()
            if op == "spmm":
                O.spmm_csr_rows(m, g["B"], prec, rows=sel)
                flops = 2.0 * nnz * g["B"].shape[1]
            else:
                # dot products only: the ME-BCRS output slots are a parity
                # concern, not part of the timed work
                O.sddmm_csr_rows(m, prec, None, None, g["A"], g["Bt"], rows=sel)
                flops = 2.0 * nnz * 32
            secs = time.perf_counter() - t0
            if secs > budget_s / 4 or frac >= 1.0:
                break
            frac = min(1.0, frac * max(2.0, budget_s / max(secs, 1e-3) / 2))
        out[op] = {"value": round(flops / secs / 1e9, 4), "unit": "GFLOP/s", "rows": int(sel.size), "nnz": nnz,
                   "seconds": round(secs, 3)}
    return out


def cpu_baseline(args, device):
    run_step, desc, threads = reference_sample_runner(args, device)
    run_step(1.0)
    f, s, nnz = run_step(args.cpu_seconds)
    out = {"value": round(f / s / 1e9, 5), "unit": "GFLOP/s", "cores": threads, "kind": "reference",
           "sample": desc + f", {s:.1f}s wall, {nnz} nnz"}
    # the reference's SDDMM (sddmm.hpp:84) on the same pattern, F = 32
    run_sd, desc_sd, _ = reference_sample_runner(args, device, op="sddmm")
    run_sd(0.5)
    f, s, nnz = run_sd(max(2.0, args.cpu_seconds / 3))
    out["sddmm"] = {"value": round(f / s / 1e9, 5), "unit": "GFLOP/s", "cores": threads, "kind": "reference",
                    "sample": desc_sd + f", {s:.1f}s wall, {nnz} nnz"}
    out["restatement"] = restatement_baseline(args, device, max(2.0, args.cpu_seconds / 3))
    return out


def _free_port() -> int:
    import socket

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def relaunch(args) -> int:
    """`bench.py --gpus N` without torchrun: start N ranks (one per GPU)
    under torch.distributed.run on this node and forward their output.  The
    rank count is visible to the driver through NCCL_DEBUG=INFO (stderr)."""
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    ngpu = torch.cuda.device_count() if torch.cuda.is_available() else 0
    if ngpu < args.gpus and "TCS_DIST_BACKEND" not in env:
        # NCCL refuses two ranks on one device: with fewer GPUs than ranks the
        # sharded path still runs (gloo, ranks share devices round-robin) as a
        # functional check; the line says so in config.backend.
        env["TCS_DIST_BACKEND"] = "gloo"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd, env=env)


def main():
    args = parse()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(relaunch(args))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}; using WORLD_SIZE", file=sys.stderr)
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # TCS_DIST_BACKEND=gloo runs the multi-rank path with every rank on the
    # GPUs there are (ranks share a device round-robin): a functional check
    # of the sharded bench on a 1-GPU box; its timings mean nothing.
    backend = os.environ.get("TCS_DIST_BACKEND", "nccl")
    os.environ["TCS_BENCH_BACKEND"] = backend if world > 1 else "none"
    if args.impl == "reference":
        # the reference arm is host-only: rank 0 runs it, the other ranks exit
        # 0 without work (no process group needed)
        if rank == 0:
            dev = torch.device("cuda", 0) if torch.cuda.is_available() else torch.device("cpu")
            print(json.dumps(run_reference(args, rank, world, dev)), flush=True)
        return
    if not torch.cuda.is_available():
        backend = "gloo"
    if torch.cuda.is_available():
        local = local % torch.cuda.device_count() if backend != "nccl" else local
    if world > 1:
        if torch.cuda.is_available():
            torch.cuda.set_device(local)
        if backend == "nccl":
            torch.distributed.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            torch.distributed.init_process_group(backend)
    device = torch.device("cuda", local) if torch.cuda.is_available() else torch.device("cpu")
    line = run_ours(args, rank, world, device)
    if line is not None and world == 1 and not args.quick:
        line["small_configs"] = small_configs(device)
        line["layer_configs"] = layer_configs(device)
        line["cpu_baseline"] = cpu_baseline(args, device)
    if line is not None:
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
