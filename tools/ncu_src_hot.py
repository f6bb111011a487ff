"""Hot spots of an `ncu --page source --csv` SASS listing: instructions
executed and stall samples per basic-block-ish region (split at branch
targets), plus the opcode mix.  python tools/ncu_src_hot.py file.csv [top]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
body = [r for r in rows[2:] if len(r) == len(hdr)]
tot_i = sum(int(r[ix["Instructions Executed"]] or 0) for r in body)
tot_s = sum(int(r[ix["Warp Stall Sampling (All Samples)"]] or 0) for r in body)
print(f"instructions {tot_i}  samples {tot_s}")
ops = collections.Counter()
for r in body:
    op = r[ix["Source"]].split()[0] if r[ix["Source"]].split() else "?"
    if op.startswith("@"):
        op = r[ix["Source"]].split()[1]
    ops[op.split(".")[0]] += int(r[ix["Instructions Executed"]] or 0)
print("mix:", ", ".join(f"{k} {v / tot_i:.1%}" for k, v in ops.most_common(14)))
# regions: consecutive rows with equal execution count
regs = []
for r in body:
    n = int(r[ix["Instructions Executed"]] or 0)
    s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    if regs and regs[-1][2] == n:
        regs[-1][1] = r[ix["Address"]]
        regs[-1][3] += n
        regs[-1][4] += s
        regs[-1][5] += 1
        regs[-1][6][r[ix["Source"]].split()[0]] += 1
    else:
        regs.append([r[ix["Address"]], r[ix["Address"]], n, n, s, 1, collections.Counter({r[ix["Source"]].split()[0]: 1})])
top = int(sys.argv[2]) if len(sys.argv) > 2 else 12
for g in sorted(regs, key=lambda g: -g[3])[:top]:
    print(f"{g[0][-5:]}-{g[1][-5:]} n={g[5]:4d} x{g[2]:>9d} inst {g[3] / tot_i:6.1%} stall {g[4] / max(tot_s, 1):6.1%} "
          + " ".join(f"{k}:{v}" for k, v in g[6].most_common(6)))
