"""Per-kernel SASS instruction summary of libklsgpu.so (cuobjdump -sass):
the TMA / mbarrier / tensor-core / fp64 mnemonics that show which engine a
kernel uses.  Writes profiles/sass_<tag>.json.

    python scripts/sass_summary.py r02
"""
import json
import os
import re
import subprocess
import sys
from collections import Counter, defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ("UBLKCP", "UTMALDG", "UTMASTG", "SYNCS", "DMMA", "DFMA", "DADD", "DMUL", "LDGSTS",
        "LDG", "STG", "LDS", "STS", "SHFL", "RED", "ATOM", "BAR", "MEMBAR")


def main():
    tag = sys.argv[1] if len(sys.argv) > 1 else "latest"
    lib = os.path.join(ROOT, "paper_2104_01253_b200", "libklsgpu.so")
    out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
    per = defaultdict(Counter)
    fn = None
    for ln in out.splitlines():
        m = re.match(r"\s*Function : (\S+)", ln)
        if m:
            fn = m.group(1)
            continue
        if fn is None:
            continue
        m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[A-Z0-9_.]+)?", ln)
        if m:
            op = m.group(1)
            for k in KEYS:
                if op == k or op.startswith(k + "."):
                    per[fn][k] += 1
            per[fn]["_total"] += 1
    demangled = {}
    names = list(per)
    try:
        dm = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True,
                            text=True).stdout.splitlines()
        demangled = dict(zip(names, dm))
    except Exception:
        pass
    res = {}
    for f, c in per.items():
        name = demangled.get(f, f).replace("(anonymous namespace)::", "")
        name = re.sub(r"^void ", "", re.sub(r"\(.*", "", name))
        res.setdefault(name, Counter()).update(c)
    summary = {k: dict(v) for k, v in sorted(res.items())}
    path = os.path.join(ROOT, "profiles", f"sass_{tag}.json")
    with open(path, "w") as f:
        json.dump({"library": "paper_2104_01253_b200/libklsgpu.so (sm_100a)",
                   "command": "cuobjdump -sass | per-function mnemonic counts",
                   "kernels": summary}, f, indent=1)
    for k, v in summary.items():
        if any(v.get(x) for x in ("UBLKCP", "UTMALDG", "DMMA")):
            print(k, {x: v.get(x, 0) for x in ("UBLKCP", "UTMALDG", "SYNCS", "DMMA", "DFMA")})


if __name__ == "__main__":
    main()
