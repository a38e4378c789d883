"""Static SASS of libtangram.so (cuobjdump -sass): per kernel, the instruction
count, the opcode mix that matters for a byte-moving kernel (global / shared
memory, cp.async LDGSTS, TMA/bulk UBLKCP/UTMALDG/UTMASTG, 32-bit integer
multiply-add of the murmur mix, funnel shifts).  K3 (relocate_bulk_kernel)
shows its bulk copies (UBLKCP) and mbarrier ops (SYNCS); the load kernel's
staging is LDGSTS, its hash the IMAD/SHF/LOP3 mix.

    python tools/sass_counts.py > profiles/r02_sass_counts.json
"""
import collections
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ["LDG", "STG", "LDS", "STS", "LDGSTS", "UBLKCP", "UTMALDG", "UTMASTG", "SYNCS", "IMAD", "IMAD.WIDE", "IADD3",
        "SHF", "LOP3", "ATOMG", "RED", "BRA", "BAR", "SHFL"]


def main():
    so = os.path.join(ROOT, "paper_2512_01357_b200", "libtangram.so")
    sass = subprocess.run(["cuobjdump", "-sass", so], capture_output=True, text=True).stdout
    out = {}
    for m in re.finditer(r"Function : (\S+)\n(.*?)(?=\n\s*Function : |\Z)", sass, re.S):
        name, body = m.group(1), m.group(2)
        demangled = subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()
        short = re.sub(r"tg::\(anonymous namespace\)::", "", demangled)
        ops = re.findall(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", body)
        c = collections.Counter(o.split(".")[0] for o in ops)
        full = collections.Counter(ops)
        row = {"instructions": len(ops)}
        for k in KEYS:
            row[k] = full[k] if "." in k else c[k]
        out[short[:160]] = row
    json.dump({"source": "cuobjdump -sass paper_2512_01357_b200/libtangram.so (sm_100a), static counts",
               "kernels": out}, sys.stdout, indent=1)


if __name__ == "__main__":
    main()
