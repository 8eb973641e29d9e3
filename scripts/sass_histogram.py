"""Opcode histogram of the built sm_100a objects (cuobjdump -sass), per
kernel family: evidence for TMA (UTMALDG / UTMASTG / UBLKCP), mbarriers
(SYNCS), clusters (UCGABAR, distributed shared memory) and the FP mix.
    python scripts/sass_histogram.py > profiles/r02_sass_histogram.txt"""
import re
import subprocess
import sys
from collections import Counter, defaultdict
from pathlib import Path

LIB = Path(__file__).resolve().parents[1] / "paper_2303_12529_b200" / "_lib"
KEY = ["UTMALDG", "UTMASTG", "UBLKCP", "UTMACCTL", "SYNCS", "UCGABAR", "UTCMMA", "UTCHMMA", "UTCQMMA", "LDTM",
       "STTM", "HMMA", "FFMA", "FADD", "FMUL", "DFMA", "DADD", "DMUL", "LDS", "STS", "LDG", "STG", "SHFL", "BAR",
       "ATOMS", "ATOMG", "REDG", "LDGSTS"]


def family(name):
    for tag in ("TF1Op", "TF2Op", "TA1Op", "TA2Op", "TMaskRowsOp", "TColsOp", "A3Op", "F1COp", "F1Op", "F2Op",
                "A1Op", "A2Op", "MaskRowsOp", "ColsOp", "RowsOp"):
        if tag in name:
            kind = "k_pass_tma" if "k_pass_tma" in name else "k_pass_cluster" if "k_pass_cluster" in name else "k_pass"
            return f"{kind}<{tag}>"
    m = re.search(r"(k_[a-z0-9_]+)", name)
    return m.group(1) if m else name[:60]


def main():
    hist = defaultdict(Counter)
    for obj in sorted(LIB.glob("*.o")):
        out = subprocess.run(["cuobjdump", "-sass", str(obj)], capture_output=True, text=True).stdout
        cur = None
        for line in out.splitlines():
            m = re.match(r"\s+Function : (\S+)", line)
            if m:
                cur = (obj.name, family(m.group(1)))
                continue
            m = re.match(r"\s+/\*[0-9a-f]{4}\*/\s+(@!?U?P\d+\s+)?([A-Z0-9_]+)", line)
            if m and cur:
                op = m.group(2).split(".")[0]
                hist[cur][next((k for k in KEY if op.startswith(k)), op)] += 1
    print("static SASS opcode counts per kernel family (cuobjdump -sass of paper_2303_12529_b200/_lib/*.o)")
    print(f"{'object':18s} {'kernel':34s} " + " ".join(f"{k:>7s}" for k in KEY))
    for (obj, fam), c in sorted(hist.items()):
        if sum(c.values()) == 0:
            continue
        print(f"{obj:18s} {fam[:34]:34s} " + " ".join(f"{c.get(k, 0):7d}" for k in KEY))


if __name__ == "__main__":
    sys.exit(main())
