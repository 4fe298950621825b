"""SASS listing + opcode histogram of one kernel of an object file (evidence for which
memory and tensor instructions the hot kernel actually uses).
usage: python tools/sass_listing.py build/obj/inst_v9.o '_ZN4lvk915louver_layer_v9ILi128ELi4ELb0E' out_prefix"""
import collections
import re
import subprocess
import sys

GROUPS = {
    "tensor (legacy mma.sync)": ("HMMA",),
    "tensor (tcgen05)": ("UTCHMMA", "UTCQMMA", "UTCMMA", "UTCBAR", "LDTM", "STTM"),
    "TMA / bulk copy": ("UTMALDG", "UTMASTG", "UBLKCP", "UTMAPF", "UBLKPF"),
    "cp.async (LDGSTS)": ("LDGSTS",),
    "mbarrier (SYNCS)": ("SYNCS",),
    "ldmatrix": ("LDSM",),
    "shared ld/st": ("LDS", "STS"),
    "global ld/st": ("LDG", "STG"),
    "atomics": ("ATOM", "ATOMS", "RED", "ATOMG", "REDG"),
    "fp32": ("FADD", "FMUL", "FFMA", "FMNMX", "FSETP", "FADD2", "FMUL2", "FFMA2"),
    "sfu": ("MUFU",),
}


def main():
    obj, name, out = sys.argv[1], sys.argv[2], sys.argv[3]
    sass = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True, check=True).stdout
    blocks = re.split(r"\n\s*Function : ", sass)
    body = next(b for b in blocks if b.startswith(name))
    fn = body.splitlines()[0].strip()
    ops = collections.Counter()
    lines = []
    for ln in body.splitlines():
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(@!?U?P\w+\s+)?([A-Z0-9_]+)(\.[A-Z0-9_.]+)?", ln)
        if m:
            ops[m.group(3)] += 1
            lines.append(ln.rstrip())
    with open(out + "_sass.txt", "w") as f:
        f.write(f"// {fn}\n// cuobjdump -sass {obj}\n")
        f.write("\n".join(lines) + "\n")
    with open(out + "_sass_summary.txt", "w") as f:
        f.write(f"kernel {fn}\nstatic instructions: {sum(ops.values())}\n\nby group:\n")
        for g, mn in GROUPS.items():
            f.write(f"  {g:28s} {sum(ops[m] for m in mn):6d}  ({', '.join(f'{m} {ops[m]}' for m in mn if ops[m])})\n")
        f.write("\nall opcodes:\n")
        for k, v in ops.most_common():
            f.write(f"  {k:12s} {v:6d}\n")
    print(open(out + "_sass_summary.txt").read()[:1500])


if __name__ == "__main__":
    main()
