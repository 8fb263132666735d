"""Instruction-mix summary of the hot kernels in the built libnmfb200.so (cuobjdump -sass):
the opcodes that prove the data path (UTMALDG / UBLKCP = TMA, SYNCS = mbarrier, DMMA = FP64
tensor cores, DFMA, LDGSTS = cp.async, LDS/LDG widths).

python scripts/sass_mix.py [substring ...] > profiles/r02_sass_mix.txt
"""
import collections
import re
import subprocess
import sys

LIB = "paper_2101_08431_b200/libnmfb200.so"
WANT = ("UTMALDG", "UBLKCP", "UTCHMMA", "UTCMMA", "LDTM", "DMMA", "DFMA", "DADD", "DMUL", "FFMA",
        "HMMA", "SYNCS", "LDGSTS", "LDS", "LDG", "STG", "STS", "BAR", "SHFL", "MUFU")


def main(filters):
    txt = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
    cur, mix = None, {}
    for line in txt.splitlines():
        m = re.match(r"\s+Function : (\S+)", line)
        if m:
            cur = m.group(1)
            mix[cur] = collections.Counter()
            continue
        m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]+)", line)
        if m and cur:
            op = m.group(1)
            base = op.split(".")[0]
            if base in WANT:
                mix[cur][op if base in ("LDS", "LDG", "STG", "DMMA", "SYNCS", "UTMALDG") else base] += 1
    names = subprocess.run(["c++filt"], input="\n".join(mix), capture_output=True,
                           text=True).stdout.splitlines()
    for mangled, name in zip(mix, names):
        if filters and not any(f in name for f in filters):
            continue
        c = mix[mangled]
        if not c:
            continue
        short = re.sub(r"\(.*", "", name.replace("(anonymous namespace)::", ""))
        print(f"{short}")
        print("   " + ", ".join(f"{k} {v}" for k, v in sorted(c.items())))


if __name__ == "__main__":
    main(sys.argv[1:])
