"""SASS evidence per kernel from the in-tree objects (cuobjdump): the instructions that prove
TMA bulk copies (UBLKCP: S.G = global->shared loads in the apply, G.S = shared->global stores in
the lattice fill), mbarriers (SYNCS.*), packed fp32x2 math (FADD2/FMUL2/FFMA2) and 16-byte
vector memory ops. Usage: python tools/sass_evidence.py > profiles/<round>/sass_evidence.txt"""
import os
import re
import subprocess
from collections import Counter

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OBJ = os.path.join(ROOT, "paper_2012_08208_b200", "build")
PAT = re.compile(r"\b(UBLKCP\.[A-Z.]+|SYNCS\.[A-Z0-9.]+|FADD2|FMUL2|FFMA2|FENCE\.VIEW\.ASYNC\.S|LDS\.128|"
                 r"STG\.E\.128|LDG\.E\.128|LDG\.E\.ENL2\.256[A-Z.]*|DSQRT|MUFU\.RSQ64H|VIMNMX3\.U32|SHF\.L\.W\.U32\.HI|MATCH\.ANY|"
                 r"ACQBULK|DEPBAR)\b")
# the instances config 5 (and config 3 for the stencil) runs
KERNELS = {"k_spmvILi1ELi8ELi8E": "k_spmv<1,8,8> sensitivity (config 5)",
           "k_spmvILi0ELi8ELi8E": "k_spmv<0,8,8> density (config 5)", "k_tpass": "k_tpass (sensitivity t pass)",
           "k_cl_countILi3E": "k_cl_count<3> (group count)", "k_cl_fill3ILi3ELi3E": "k_cl_fill3<3,3> (group fill, config 5)",
           "k_cl_fill4ILi2ELi2E": "k_cl_fill4<2,2> (group fill, small unions: config 4)",
           "k_countILi3ELi4E": "k_count<3,4> (per-bin)", "k_fillILi3ELi4E": "k_fill<3,4> (per-bin)",
           "k_lat_fill_exactILi3E": "k_lat_fill_exact<3>", "k_lat_rowsILi3ELb1E": "k_lat_rows<3,fill>",
           "k_stencilILi1ELi3ELi1E": "k_stencil<1,3,1>", "k_latticeILi1ELi3ELi1ELi6E": "k_lattice<1,3,1,6>"}


def main():
    for obj in ("apply.o", "build.o", "cl_build.o", "lattice_build.o", "stencil.o"):
        sass = subprocess.run(["cuobjdump", "-sass", os.path.join(OBJ, obj)], capture_output=True, text=True).stdout
        cur, counts = None, {}
        for line in sass.splitlines():
            if "Function : " in line:
                name = line.split("Function : ")[1].strip()
                cur = next((v for k, v in KERNELS.items() if k in name), None)
                if cur:
                    counts.setdefault(cur, Counter())
                continue
            if cur:
                for m in PAT.findall(line):
                    counts[cur][m] += 1
        for k, c in counts.items():
            if c:
                print(f"== {obj}: {k}")
                for ins, n in sorted(c.items()):
                    print(f"  {n:6d}  {ins}")


if __name__ == "__main__":
    main()
