"""Regenerate tests/golden/golden.json from the REFERENCE itself.

Runs here only (needs oracle/_ref/libtcsref.so, built by `make -C oracle`
from /root/reference/proj/include).  Inputs come from the reference's own
generators (cases.GEN = oracle.Ref); outputs from the reference's
encode_mebcrs / spmm / sddmm (inc/mebcrs.hpp:80, inc/spmm.hpp:173,
inc/sddmm.hpp:84).  Only hashes (sha256, first 128 bits) and counters are
stored, so the fixture stays small; tests rebuild inputs with the oracle
generators and must reproduce both the input and the output hashes.

    PYTHONPATH=. python tests/golden/make_golden.py
"""
from __future__ import annotations

import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
sys.path.insert(0, HERE)

import numpy as np  # noqa: E402

import oracle as O  # noqa: E402
import cases  # noqa: E402


def record(case: cases.Case) -> dict:
    R = O.Ref
    m = case.csr
    rec = {"rows": m.rows, "cols": m.cols, "nnz": m.nnz,
           "csr": cases.sha(m.row_ptr, m.col_idx, m.values)}
    for key in ("B", "A", "Bt", "D"):
        arr = getattr(case, key)
        if arr is not None:
            rec[key] = {"shape": list(arr.shape), "sha": cases.sha(arr)}
    for p in case.precisions:
        tag = "fp16" if p == 0 else "tf32"
        me = R.encode_mebcrs(m, p)
        rec[f"me_{tag}"] = {"nv": me.nv, "sha": cases.sha(me.row_pointers, me.column_indices, me.values),
                            "rp_sha": cases.sha(me.row_pointers), "ci_sha": cases.sha(me.column_indices)}
        if case.B is not None:
            Cm, cnt = R.spmm(me, case.B)
            rec[f"spmm_{tag}"] = {"sha": cases.sha(Cm), "mma": cnt}
            # 16x1 ablation (inc/spmm.hpp:187-257) on the 16-row partition (inc/partition.hpp:40-66)
            prp, pci = R.partition_windows(m, 16, O.K_OF[p])
            C16, cnt16 = R.spmm_baseline16(m, case.B, p)
            rec[f"b16_{tag}"] = {"nv": int(pci.shape[0]), "part_sha": cases.sha(prp, pci), "sha": cases.sha(C16),
                                 "mma": cnt16}
        # SR-BCRS padded ablation format (inc/srbcrs.hpp:40-72) and its SpMM (inc/spmm.hpp:181)
        sr = R.encode_srbcrs(m, p)
        rec[f"sr_{tag}"] = {"np": int(sr.column_indices.shape[0]),
                            "sha": cases.sha(sr.row_pointer_pairs, sr.column_indices, sr.values)}
        if case.B is not None:
            Csr_, cnt_sr = R.spmm_srbcrs(sr, case.B)
            rec[f"sr_{tag}"].update({"spmm_sha": cases.sha(Csr_), "mma": cnt_sr})
        if case.A is not None:
            out, cnt = R.sddmm(me, case.A, case.Bt)
            rec[f"sddmm_{tag}"] = {"sha": cases.sha(out), "mma": cnt}
            if case.D is not None:
                chained = O.MeBcrs(me.rows, me.cols, p, me.row_pointers, me.column_indices, out)
                Cc, cnt2 = R.spmm(chained, case.D)
                rec[f"chain_{tag}"] = {"sha": cases.sha(Cc), "mma": cnt2}
    return rec


def main():
    cases.GEN = O.Ref
    t0 = time.time()
    golden = {"generated_by": "tests/golden/make_golden.py (reference via oracle/_ref)", "cases": {}}
    todo = list(cases.kat_cases())
    p2 = cases.acceptance2_params()
    todo += [cases.acceptance2_case(i, p2) for i in range(200)]
    p6 = cases.acceptance6_params()
    todo += [cases.acceptance6_case(i, p6) for i in range(100)]
    todo += [cases.c1_case(False), cases.c1_case(True)]
    for c in todo:
        golden["cases"][c.name] = record(c)
    # rounding known answers (tests/test_tcu_emu.cpp:68-98) + random bit patterns
    rng = np.random.default_rng(2412)
    bits = rng.integers(0, 2**32, size=4096, dtype=np.uint64).astype(np.uint32)
    xs = bits.view(np.float32)
    f16 = np.array([O.Ref.round_fp16(float(x)) for x in xs], np.float32)
    t32 = np.array([O.Ref.round_tf32(float(x)) for x in xs], np.float32)
    golden["rounding"] = {"seed": 2412, "n": 4096, "fp16_sha": cases.sha(f16), "tf32_sha": cases.sha(t32)}
    golden["sddmm_offsets"] = {"b8x8": [O.Ref.sddmm_output_offsets(l, 0) for l in range(32)],
                               "b8x4": [O.Ref.sddmm_output_offsets(l, 1) for l in range(32)]}
    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(golden, f, indent=1, sort_keys=True)
    print(f"wrote {len(golden['cases'])} cases in {time.time() - t0:.1f}s")


if __name__ == "__main__":
    main()
