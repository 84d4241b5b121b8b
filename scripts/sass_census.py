"""SASS instruction census of the built library (static counts per kernel):
    python scripts/sass_census.py > profiles/r02_sass_summary.md"""
import re
import subprocess
import sys
from pathlib import Path

LIB = Path(__file__).resolve().parent.parent / "paper_2412_01523_b200" / "_lib" / "libflexsp_b200.so"
OPS = ["UTCHMMA", "LDTM", "STTM", "UTMALDG", "UTMAPF", "UBLKCP", "UGETNEXTWORKID", "USETMAXREG",
       "SYNCS", "MUFU.EX2", "REDG", "LDG", "STG", "LDS", "STS"]


def main():
    lib = sys.argv[1] if len(sys.argv) > 1 else str(LIB)
    sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True,
                          check=True).stdout
    dem = subprocess.run(["cu++filt"], input="\n".join(re.findall(r"Function : (\S+)", sass)),
                         capture_output=True, text=True).stdout.splitlines()
    names = iter(dem)
    counts, cur = {}, None
    for line in sass.splitlines():
        if "Function : " in line:
            cur = next(names, line.split()[-1])
            cur = re.sub(r"^void ", "", cur)
            cur = cur.replace("fsp::(anonymous namespace)::", "").replace("fsp::<unnamed>::", "")
            cur = cur.replace("(bool)0", "false").replace("(bool)1", "true")
            cur = re.sub(r"\((?:int|unsigned int|long)\)", "", cur).split("(")[0]
            counts[cur] = {o: 0 for o in OPS}
            continue
        m = re.match(r"\s*/\*[0-9a-f]+\*/\s+(?:@!?U?P\w+\s+)?([A-Z0-9_.]+)", line)
        if cur and m:
            op = m.group(1)
            for o in OPS:
                if op == o or op.startswith(o + "."):
                    counts[cur][o] += 1
    print("# SASS instruction census of libflexsp_b200.so (cuobjdump -sass, sm_100a)\n")
    print("Static instruction counts per kernel (not executed counts): the tensor-core "
          "(UTCHMMA), TMEM (LDTM/STTM), TMA tensor (UTMALDG/UTMAPF), bulk-copy (UBLKCP), "
          "cluster-launch-control (UGETNEXTWORKID) and register-reallocation (USETMAXREG) "
          "instructions that show which hardware paths each kernel uses. "
          "Regenerate: `python scripts/sass_census.py`.\n")
    print("| kernel | " + " | ".join(OPS) + " |")
    print("|---|" + "---:|" * len(OPS))
    for k, c in counts.items():
        print(f"| `{k}` | " + " | ".join(str(c[o]) for o in OPS) + " |")


if __name__ == "__main__":
    main()
