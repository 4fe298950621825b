"""Aggregate an ncu report's stall samples / executed instructions per CUDA source line.

usage: python tools/ncu_lines.py report.ncu-rep [top]
"""
import csv
import subprocess
import sys


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    func, recs, fname = None, {}, None
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r[0] == "Function Name":
            func = r[1]
            recs.setdefault(func, [])
            continue
        if r[0] == "Line No":
            continue
        if r[0] and func is not None and len(r) > 7:
            try:
                recs[func].append((int(r[4]), int(r[7]), f"{fname}:{r[0]}", r[1].strip()[:100]))
            except ValueError:
                pass
    for f, v in recs.items():
        tot = sum(x[0] for x in v) or 1
        inst = sum(x[1] for x in v) or 1
        print(f"== {f[:110]}\n   samples={tot} warp-inst={inst}")
        for s, i, ln, src in sorted(v, reverse=True)[:top]:
            print(f"{100 * s / tot:5.1f}% inst {100 * i / inst:5.1f}%  {ln:24s} {src}")


if __name__ == "__main__":
    main()
