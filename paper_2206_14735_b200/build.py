"""Build the in-tree CUDA extension ``_gsb.so`` for sm_100a (B200).

    python -m paper_2206_14735_b200.build

The library is a plain C-ABI shared object (include/gsb.h) loaded with
ctypes; it is built in-tree so it travels with the repo snapshot.
"""

from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
SRC = os.path.join(CSRC, "gsb.cu")
INST = os.path.join(CSRC, "gsb_step_inst.cu")
DEPS = sorted(glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.cu"))) + [
    os.path.join(ROOT, "include", "gsb.h")]
OUT = os.path.join(HERE, "_gsb.so")
OBJDIR = os.path.join(ROOT, "build", "obj")
# one translation unit per (dtype, levels, geometry width, colour width)
STEP_UNITS = [("f446", "float", 4, 4, 6), ("d446", "double", 4, 4, 6),
              ("f222", "float", 2, 2, 2), ("d222", "double", 2, 2, 2)]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    # keep every separately-rounded multiply/add of the reference separate;
    # fused multiply-adds are written explicitly where intended
    "--fmad=false",
    "-Xcompiler", "-fPIC",
]


def nvcc():
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.isabs(cand) and os.path.exists(cand) or not os.path.isabs(cand)):
            return cand
    return "nvcc"


def needs_build():
    if not os.path.exists(OUT):
        return True
    t = os.path.getmtime(OUT)
    return any(os.path.getmtime(p) > t for p in [SRC] + DEPS)


def build(force=False, verbose=False):
    if not force and not needs_build():
        return OUT
    os.makedirs(OBJDIR, exist_ok=True)
    extra = ["-Xptxas", "-v"] if verbose else []
    extra += os.environ.get("GSB_NVCC_EXTRA", "").split()  # A/B builds (e.g. -DGSB_SPLIT_TRUNC)
    jobs = [([nvcc()] + NVCC_FLAGS + extra + ["-c", "-o", os.path.join(OBJDIR, "gsb.o"), SRC])]
    for tag, t, nl, cg, cc in STEP_UNITS:
        jobs.append([nvcc()] + NVCC_FLAGS + extra + [
            f"-DGSB_T={t}", f"-DGSB_NL={nl}", f"-DGSB_CG={cg}", f"-DGSB_CC={cc}",
            f"-DGSB_ENTRY=gsb_step_{tag}", "-c", "-o", os.path.join(OBJDIR, f"step_{tag}.o"), INST])
    procs = [subprocess.Popen(j, cwd=ROOT, stdout=subprocess.PIPE, stderr=subprocess.STDOUT,
                              text=True) for j in jobs]
    logs = []
    failed = False
    for p in procs:
        out, _ = p.communicate()
        logs.append(out)
        failed |= p.returncode != 0
    if failed or verbose:
        sys.stderr.write("\n".join(logs))
    if failed:
        raise RuntimeError("nvcc failed building _gsb.so")
    objs = [os.path.join(OBJDIR, "gsb.o")] + [os.path.join(OBJDIR, f"step_{u[0]}.o")
                                              for u in STEP_UNITS]
    tmp = OUT + ".tmp"
    res = subprocess.run([nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared",
                          "-o", tmp] + objs, cwd=ROOT, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc link failed for _gsb.so")
    os.replace(tmp, OUT)
    return OUT


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(OUT)
