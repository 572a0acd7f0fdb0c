"""Summarise an ncu launch list (gpu__time_duration per launch) into per-kernel shares of
the ST-block step: only this library's kernels (gemm / fmha / layer_norm / run_copy / p2p)."""
import csv, io, json, re, sys
from collections import defaultdict

def load(path):
    txt = open(path).read()
    txt = txt[txt.index('"ID"'):]
    return list(csv.DictReader(io.StringIO(txt)))

EPI = {"0": "plain", "1": "+residual", "2": "+GELU", "3": "LN folded", "4": "LN folded+GELU", "5": "+residual, remote rows"}
ROLE = {"3": "QKV_S/QKV_T", "1": "PROJ_S/PROJ_T/FC2", "4": "FC1", "2": "FC1 (raw weights)", "0": "QKV (raw weights)",
        "5": "PROJ_S/FC2 (fused switch)"}


def kind(name):
    m = re.search(r"gemm_bf16_tc_kernel<(\d+), (\d+)(?:, \d+)?>", name)
    if m:
        return f"gemm BN={m.group(1)} {EPI.get(m.group(2), m.group(2))} [{ROLE.get(m.group(2), '?')}]"
    for k in ("fmha_pt_kernel", "fmha_seq_kernel", "fmha_split_kernel", "fmha_pair_kernel", "fmha_bf16_tc_kernel", "fmha_bwd_kernel",
              "row_partials", "row_stats", "layer_norm", "ln_bwd", "wgrad_reduce", "colsum", "transpose", "attn_bwd_dvec",
              "dq_convert", "run_copy", "p2p_barrier",
              "p2p_put", "fold_ln_weights"):
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
