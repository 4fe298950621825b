"""Summarise an ncu SASS source page (--page source --csv --print-source sass):
instruction counts and stall samples per region of consecutive instructions."""
import csv
import sys


def main():
    path = sys.argv[1]
    rows = list(csv.reader(open(path)))
    hdr = rows[1]
    idx = {h: i for i, h in enumerate(hdr)}
    data = rows[2:]
    ie = idx["Instructions Executed"]
    ss = idx["Warp Stall Sampling (All Samples)"]
    stall_cols = [h for h in hdr if h.startswith("stall_")]
    tot_i = sum(float(r[ie] or 0) for r in data)
    tot_s = sum(float(r[ss] or 0) for r in data)
    print(f"instructions executed {tot_i:.0f}, samples {tot_s:.0f}")
    agg = {h: sum(float(r[idx[h]] or 0) for r in data) for h in stall_cols}
    for h, v in sorted(agg.items(), key=lambda x: -x[1])[:10]:
        print(f"  {h:32s} {v:8.0f} ({100 * v / max(tot_s, 1):.1f}%)")
    # windows of 32 instructions
    W = int(sys.argv[2]) if len(sys.argv) > 2 else 64
    wins = []
    for s in range(0, len(data), W):
        chunk = data[s:s + W]
        wins.append((sum(float(r[ss] or 0) for r in chunk), sum(float(r[ie] or 0) for r in chunk), s, chunk))
    print("hottest windows (samples, instr, first address):")
    for smp, ins, s, chunk in sorted(wins, key=lambda x: -x[0])[:12]:
        top = max(chunk, key=lambda r: float(r[ss] or 0))
        print(f"  {smp:7.0f} {ins:9.0f}  @{chunk[0][0]}  top: {top[1][:60]} ({top[ss]})")


if __name__ == "__main__":
    main()
