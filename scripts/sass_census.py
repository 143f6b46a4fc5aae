"""SASS census of the built library: per kernel, the count of the Blackwell-native
instructions that prove the tcgen05 / TMEM / TMA path (B200_PROFILING.md):

  UTCHMMA  tcgen05.mma (kind::tf32)          UTMALDG  TMA tensor load (cp.async.bulk.tensor)
  LDTM     tcgen05.ld (TMEM -> registers)    UTCBAR   tcgen05.commit (mbarrier arrive)
  UTMASTG  TMA tensor store                  FFMA     CUDA-core FP32 FMA (SIMT kernels)

  python scripts/sass_census.py [lib.so] > profiles/sass_census.md
"""
import collections
import re
import subprocess
import sys

OPS = ("UTCHMMA", "UTMALDG", "LDTM", "UTCBAR", "UTMASTG", "FFMA")


def demangle(name):
    m = re.search(r"(_ZN.*)$", name)
    if not m:
        return name
    out = subprocess.run(["c++filt", m.group(1)], capture_output=True, text=True).stdout.strip()
    out = re.sub(r"\(anonymous namespace\)::|ptb::", "", out)
    return out.split("(")[0] if out else name


def main():
    lib = sys.argv[1] if len(sys.argv) > 1 else "paper_1606_04884_b200/lib/libpt_b200.so"
    sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True,
                          check=True).stdout
    counts = collections.OrderedDict()
    fn = None
    for line in sass.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            fn = demangle(m.group(1))
            counts.setdefault(fn, collections.Counter())
            continue
        if fn is None:
            continue
        for tok in line.split():
            op = tok.split(".")[0]
            if op in OPS:
                counts[fn][op] += 1
    print(f"# SASS census of `{lib}` (cuobjdump -sass, sm_100a)\n")
    print("| kernel | " + " | ".join(OPS) + " |")
    print("|---|" + "---|" * len(OPS))
    tot = collections.Counter()
    for fn, c in sorted(counts.items()):
        if not any(c[o] for o in OPS):
            continue
        tot.update(c)
        print(f"| `{fn}` | " + " | ".join(str(c[o]) for o in OPS) + " |")
    print("| **total** | " + " | ".join(f"**{tot[o]}**" for o in OPS) + " |")


if __name__ == "__main__":
    main()
