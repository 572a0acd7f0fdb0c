"""Per-kernel times of ONE training step from an ncu launch list (gpu__time_duration.sum, serialised,
cold L2): the last forward_train + backward in the list (bench.py --config train --steps 1)."""
import csv, io, re, sys

txt = open(sys.argv[1]).read()
txt = txt[txt.index('"ID"'):]
rows = [r for r in csv.DictReader(io.StringIO(txt)) if r["Metric Name"] == "gpu__time_duration.sum"]
names = [r["Kernel Name"] for r in rows]
# the step starts at the last forward LayerNorm preceded by the bench's flat.zero_ fill of a previous bwd
# a step starts at LN1: LayerNorm -> QKV GEMM -> the spatial FMHA (fmha_pt_kernel)
starts = [i for i, n in enumerate(names) if "layer_norm_bf16_vec_kernel" in n and i + 2 < len(names)
          and "fmha_pt_kernel" in names[i + 2]]
s0 = starts[1] if len(starts) >= 3 else starts[0]  # a warm-up step (the list may end mid-step)
step = rows[s0:]
# stop before the next forward (if any)
out, tot = [], 0.0
for i, r in enumerate(step):
    if i > 0 and i in [j - s0 for j in starts]:
        break
    us = float(r["Metric Value"].replace(",", "")) / 1e3
    k = r["Kernel Name"]
    m = re.search(r"gemm_bf16_tc_kernel<(\d+), (\d+), (\d+)>", k)
    short = f"gemm<BN={m.group(1)},EPI={m.group(2)},MAJ={m.group(3)}>" if m else re.sub(r"\(.*", "", k).replace("void ", "").replace("dsp::<unnamed>::", "")
    out.append((short, us))
    tot += us
for s, us in out:
    print(f"{us:9.1f} us  {100 * us / tot:5.1f} %  {s}")
print(f"{tot:9.1f} us  total (serialised under ncu)")
