"""Per-CUDA-source-line instruction and stall shares from an
`ncu --page source --csv --print-source cuda,sass` export (the per-line
rows carry the aggregated metrics; the source text may break the CSV
quoting, so metric columns are taken from the right):
    python tools/ncu_cuda_lines.py file.csv source.cu [top]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(r for r in rows if r and r[0] == "Line No")
n_metrics = len(hdr) - 4
ii = hdr.index("Instructions Executed") - 4
si = hdr.index("Warp Stall Sampling (All Samples)") - 4
src = open(sys.argv[2]).read().splitlines() if len(sys.argv) > 2 else []
out = []
for r in rows:
    if not r or not r[0].isdigit():
        continue
    m = r[-n_metrics:]
    try:
        n = int(m[ii]) if m[ii] not in ("-", "") else 0
        s = int(m[si]) if m[si] not in ("-", "") else 0
    except ValueError:
        continue
    out.append((int(r[0]), n, s))
tot_i = sum(n for _, n, _ in out) or 1
tot_s = sum(s for _, _, s in out) or 1
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
print(f"instructions {tot_i}, stall samples {tot_s}")
for ln, n, s in sorted(out, key=lambda x: -x[1])[:top]:
    text = src[ln - 1].strip()[:96] if 0 < ln <= len(src) else ""
    print(f"{ln:>5} inst {n / tot_i:6.1%} stall {s / tot_s:6.1%}  {text}")
