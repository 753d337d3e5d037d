"""DRAM traffic per roofline unit from `ncu --set full` raw CSV exports
(`ncu -i X.ncu-rep --page raw --csv > X_raw.csv`), written to
profiles/ncu_traffic.json for bench.py's roofline "traffic" field.

    python scripts/ncu_traffic.py --k4 profiles/rN/ncu_k4_raw.csv --k3 profiles/rN/ncu_k3_raw.csv

Units (must match engine.KernelProfiler's names and per-unit bytes):
  "K4 w4_swiglu_gemv+down_gemv"  one expert's decode FFN = one SwiGLU GEMV
                                 launch + one down GEMV launch (first of each)
  "K3 w4_grouped_ffn (tcgen05)"  one expert's grouped FFN = GEMM1 + GEMM2
                                 (+ split reduce if captured)
traffic = dram__bytes_read.sum + dram__bytes_write.sum, bytes.
"""
import argparse
import csv
import json
import re
from pathlib import Path

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1024, "MB": 1 << 20, "GB": 1 << 30}


def launches(path):
    rows = list(csv.reader(open(path)))
    h, units = rows[0], rows[1]
    ki = h.index("Kernel Name")
    out = []
    for r in rows[2:]:
        if len(r) < len(h):
            continue
        b = 0.0
        for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            i = h.index(m)
            b += float(r[i].replace(",", "")) * SCALE.get(units[i], 1)
        t = h.index("gpu__time_duration.sum")
        out.append({"kernel": re.sub(r"\(.*", "", r[ki]), "dram_bytes": b,
                    "us": float(r[t].replace(",", "")) * (1e-3 if units[t] == "ns" else 1.0)})
    return out


def first(ls, pat):
    return next((x for x in ls if re.search(pat, x["kernel"])), None)


ap = argparse.ArgumentParser()
ap.add_argument("--k4")
ap.add_argument("--k3")
ap.add_argument("--out", default="profiles/ncu_traffic.json")
a = ap.parse_args()
res = json.loads(Path(a.out).read_text()) if Path(a.out).exists() else {}
if a.k4:
    ls = launches(a.k4)
    fused = first(ls, r"expert_fused_v6")
    if fused:                                    # K4 v6: one launch is one expert
        parts = [fused]
    else:
        sw = first(ls, r"staged_mma_swiglu|staged_gemv_kernel<2|mma_gemv_kernel<2|swiglu_gemv")
        dn = first(ls, r"staged_gemv_kernel<1|mma_gemv_kernel<1|down_gemv")
        parts = [x for x in (sw, dn) if x]
    res["K4 w4_swiglu_gemv+down_gemv"] = {"bytes_per_unit": sum(x["dram_bytes"] for x in parts),
                                          "launches": parts, "source": a.k4}
if a.k3:
    ls = launches(a.k3)
    parts = [x for x in (first(ls, r"w4_gemm_kernel<2"), first(ls, r"w4_gemm_kernel<1"),
                         first(ls, r"split_reduce")) if x]
    res["K3 w4_grouped_ffn (tcgen05)"] = {"bytes_per_unit": sum(x["dram_bytes"] for x in parts),
                                          "launches": parts, "source": a.k3}
Path(a.out).write_text(json.dumps(res, indent=1) + "\n")
print(json.dumps(res, indent=1))
