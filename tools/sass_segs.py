"""Instruction / stall-sample totals per straight-line SASS segment of an ncu source page."""
import csv
import sys


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    hdr = rows[1]
    idx = {h: i for i, h in enumerate(hdr)}
    data = rows[2:]
    ie, ss = idx["Instructions Executed"], idx["Warp Stall Sampling (All Samples)"]
    thr = float(sys.argv[2]) if len(sys.argv) > 2 else 0.01
    segs, cur = [], None
    for i, r in enumerate(data):
        n, s = float(r[ie] or 0), float(r[ss] or 0)
        if cur and n == cur[4]:
            cur[1] = i; cur[2] += n; cur[3] += s
        else:
            if cur:
                segs.append(cur)
            cur = [i, i, n, s, n]
    segs.append(cur)
    tot = sum(x[2] for x in segs)
    tots = sum(x[3] for x in segs)
    print(f"total instr {tot:.0f} samples {tots:.0f}")
    for a, b, n, s, per in segs:
        if n > tot * thr or s > tots * thr:
            print(f"{a:5d}-{b:5d} x{per:8.0f} len {b - a + 1:4d} instr {n:9.0f} ({100 * n / tot:4.1f}%) "
                  f"samples {s:5.0f} ({100 * s / max(tots, 1):4.1f}%)  {data[a][1].strip()[:40]}")


if __name__ == "__main__":
    main()
