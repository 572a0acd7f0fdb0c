"""Summarise an ncu launch list (gpu__time_duration per launch) into per-kernel shares of
the ST-block step: only this library's kernels (gemm / fmha / layer_norm / run_copy / p2p)."""
import csv, io, json, sys
from collections import defaultdict

def load(path):
    txt = open(path).read()
    txt = txt[txt.index('"ID"'):]
    return list(csv.DictReader(io.StringIO(txt)))

def kind(name):
    for k in ("gemm_bf16_tc_kernel<192, 0>", "gemm_bf16_tc_kernel<192, 1>", "gemm_bf16_tc_kernel<256, 2>",
              "gemm_bf16_tc_kernel<256, 0>", "fmha_pair_kernel", "fmha_bf16_tc_kernel", "layer_norm", "run_copy",
              "p2p_barrier", "gemm_bf16_tc_kernel"):
        if k in name:
            return k
    return None

rows = [r for r in load(sys.argv[1]) if r["Metric Name"] == "gpu__time_duration.sum"]
per = defaultdict(list)
for r in rows:
    k = kind(r["Kernel Name"])
    if k:
        per[k].append(float(r["Metric Value"]) / 1e3)
tot = sum(sum(v) for v in per.values())
print(f"{'kernel':36s} {'launches':>8s} {'avg us':>9s} {'share':>7s}")
out = {}
for k, v in sorted(per.items(), key=lambda kv: -sum(kv[1])):
    print(f"{k:36s} {len(v):8d} {sum(v)/len(v):9.1f} {sum(v)/tot:7.1%}")
    out[k] = {"launches": len(v), "avg_us": sum(v) / len(v), "share": sum(v) / tot}
if len(sys.argv) > 2:
    json.dump(out, open(sys.argv[2], "w"), indent=1)
