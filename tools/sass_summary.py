"""SASS instruction counts per kernel of libdmtk_gpu.so (evidence that the
streaming MTTKRP issues FP64 tensor-core DMMA fed by TMA on sm_100a).

python tools/sass_summary.py > profiles/sass_summary.txt
"""
import collections
import os
import re
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OPS = ("DMMA", "UTMALDG", "UTMAPF", "SYNCS", "DFMA", "LDGSTS")


def main():
    so = os.path.join(ROOT, "paper_1708_08976_b200", "libdmtk_gpu.so")
    out = subprocess.run(["cuobjdump", "-sass", so], capture_output=True, text=True, check=True).stdout
    print("# SASS instruction counts per kernel of paper_1708_08976_b200/libdmtk_gpu.so (cuobjdump -sass, sm_100a)")
    print("# DMMA = FP64 tensor-core MMA 8x8x4; UTMALDG = TMA tile load; UTMAPF = TMA descriptor prefetch;")
    print("# SYNCS = mbarrier operations; DFMA = FP64 FMA (tail columns, small kernels); LDGSTS = cp.async")
    for f in re.split(r"\n\s+Function : ", out)[1:]:
        name = f.split("\n", 1)[0].strip()
        dem = subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()
        c = collections.Counter({op: len(re.findall(r"\b" + op + r"[.\s]", f)) for op in OPS})
        if c["DMMA"] or c["UTMALDG"] or "gen_dist" in dem or "mt64" in dem or "krp_level" in dem:
            print(dem)
            print("    " + "  ".join(f"{k}={c[k]}" for k in OPS))


if __name__ == "__main__":
    main()
