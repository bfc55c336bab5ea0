"""Write profiles/traffic.json (the DRAM bytes per launch bench.py reports as
roofline.traffic / roofline.dram) from `ncu --set full` captures.

  python tools/traffic_from_ncu.py KEY=REPORT[:KERNEL_REGEX] ...   (REPORT: .ncu-rep or raw .csv)

KEY is bench.py's config key (c3_fp16_n128_g1, c4_fp16_n128_g1,
c5_fp16_n32_g1, c5_sddmm_fp16_f32_g1, ...).  For each report the launches
whose name matches KERNEL_REGEX (default: any) are summed per capture
(dram__bytes_read.sum + dram__bytes_write.sum over the kernels of one
operator call, e.g. the SpMM kernel and its split-window reduce).  The file
records the kernel-source hash (bench.csrc_sha) so bench.py can tell whether
the capture was taken on the sources in the tree."""
import csv
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def metrics(report):
    # an .ncu-rep, or its `--page raw --csv` export (what gpu_profiles.sh keeps)
    if report.endswith(".csv"):
        out = open(report).read()
    else:
        out = subprocess.run(["ncu", "-i", report, "--page", "raw", "--csv", "--metrics",
                              "dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,"
                              "gpu__time_duration.sum"], capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
    res = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")]}
        for m in ("dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct",
                  "gpu__time_duration.sum"):
            i = hdr.index(m)
            v = float(r[i].replace(",", ""))
            if m.startswith("dram"):
                v *= scale.get(units[i], 1)
            d[m] = v
        res.append(d)
    return res


def main(argv):
    import bench

    path = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(path) as f:
            tj = json.load(f)
    except Exception:
        tj = {}
    tj["_source"] = ("ncu --set full --clock-control none (cold cache, one call): dram__bytes_read.sum + "
                     "dram__bytes_write.sum over the kernels of one operator call, bytes per call; "
                     "written by tools/traffic_from_ncu.py")
    for arg in argv:
        key, spec = arg.split("=", 1)
        report, _, rx = spec.partition(":")
        ks = [k for k in metrics(report) if re.search(rx or ".", k["kernel"])]
        if not ks:
            raise SystemExit(f"{report}: no kernel matches {rx!r}")
        dram = sum(k["dram__bytes_read.sum"] + k["dram__bytes_write.sum"] for k in ks)
        main_k = max(ks, key=lambda k: k["gpu__time_duration.sum"])
        tj[key] = {"bytes_per_launch": int(dram), "l2_hit_pct": round(main_k["lts__t_sector_hit_rate.pct"], 1),
                   "kernels": [k["kernel"].split("(")[0] for k in ks], "source": os.path.relpath(report, ROOT),
                   "csrc_sha": bench.csrc_sha()}
        print(key, tj[key])
    with open(path, "w") as f:
        json.dump(tj, f, indent=1)


if __name__ == "__main__":
    main(sys.argv[1:])
