"""SASS op-count evidence for profiles/: which kernels of libswitchback_b200.so issue tcgen05 MMAs
(UTC*MMA), TMEM loads (LDTM), TMA loads / stores / reduce-stores (UTMALDG / UTMASTG / UTMAREDG),
bulk copies (UBLKCP) and fp64 math, from `cuobjdump -sass` of the built library.

    python tools/sass_summary.py r02     -> profiles/r02_sass_summary.md
"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2304_13013_b200", "libswitchback_b200.so")
OPS = ["UTCIMMA", "UTCQMMA", "UTCHMMA", "UTCBAR", "LDTM", "UTMALDG", "UTMASTG", "UTMAREDG", "UTMAPF", "UBLKCP",
       "SYNCS", "DFMA", "DMUL", "DADD", "MUFU", "IDP", "REDG", "ATOMG"]


def demangle(names):
    r = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True)
    return r.stdout.splitlines()


def main(tag):
    sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True, check=True).stdout
    per = collections.OrderedDict()
    cur = None
    for line in sass.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            cur = m.group(1)
            per[cur] = collections.Counter()
            continue
        if cur is None:
            continue
        m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", line)
        if m:
            op = m.group(1)
            for k in OPS:
                if op == k or op.startswith(k + "_") or (k in ("SYNCS",) and op.startswith(k)):
                    per[cur][k] += 1
    names = list(per)
    pretty = dict(zip(names, demangle(names)))
    totals = collections.Counter()
    for c in per.values():
        totals.update(c)
    out = os.path.join(ROOT, "profiles", f"{tag}_sass_summary.md")
    with open(out, "w") as f:
        f.write(f"# {tag}: SASS op counts of `libswitchback_b200.so` (`cuobjdump -sass`, `tools/sass_summary.py`)\n\n")
        f.write("Static instruction counts per kernel (not dynamic). UTCIMMA = tcgen05.mma kind::i8, UTCQMMA = "
                "kind::f8f6f4, UTCHMMA = kind::f16, LDTM = tcgen05.ld, UTMALDG / UTMASTG / UTMAREDG = TMA tensor "
                "load / store / reduce-store, UBLKCP = cp.async.bulk, SYNCS = mbarrier ops.\n\n")
        f.write(f"{len(per)} kernels. Library totals: " + ", ".join(f"{k} {totals[k]}" for k in OPS if totals[k]) + "\n\n")
        f.write("| kernel | " + " | ".join(OPS) + " |\n|---|" + "---|" * len(OPS) + "\n")
        for n, c in per.items():
            if not any(c[k] for k in OPS[:10]):
                continue  # list only kernels that touch the tensor core / TMEM / TMA
            short = pretty[n].replace("(anonymous namespace)::", "")
            short = re.sub(r"\(.*", "", short)[:110]
            f.write(f"| `{short}` | " + " | ".join(str(c[k]) if c[k] else "" for k in OPS) + " |\n")
    print(out, dict(totals))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "r02")
