"""Instruction mix of the innermost loops of one kernel in a built .so
(cuobjdump -sass), e.g. to count a u-loop step's DFMA / FSEL / LDS:

    python tools/sass_loops.py paper_2303_10672_b200/lib/libpvi_b200.so 'k_b_fact_qw4IdLb1ELb1E'
"""
import collections
import re
import subprocess
import sys


def functions(so):
    out = subprocess.run(["cuobjdump", "-sass", so], capture_output=True, text=True).stdout
    cur, body = None, []
    for line in out.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            if cur:
                yield cur, body
            cur, body = m.group(1), []
            continue
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
        if m and cur:
            body.append((int(m.group(1), 16), m.group(2).strip()))
    if cur:
        yield cur, body


def loops(body):
    out = []
    for a, op in body:
        m = re.search(r"BRA (0x[0-9a-f]+)", op)
        if m and int(m.group(1), 16) < a:
            t = int(m.group(1), 16)
            ins = [o for x, o in body if t <= x <= a]
            mix = collections.Counter(re.sub(r"^@!?U?P[T0-9]+\s+", "", o).split()[0].split(".")[0] for o in ins)
            out.append((hex(t), hex(a), len(ins), mix))
    return out


if __name__ == "__main__":
    so, pat = sys.argv[1], sys.argv[2]
    for name, body in functions(so):
        if pat in name:
            print(name, len(body), "instructions")
            for t, a, n, mix in loops(body):
                if mix.get("DFMA", 0) >= 32:
                    print(f"  loop {t}..{a}: {n} instr", dict(mix.most_common(10)))
