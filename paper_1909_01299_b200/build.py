"""Build the sm_100a C-ABI library in-tree: paper_1909_01299_b200/_lib/liblfds.so.

nvcc cross-compiles for B200 (no GPU needed).  The CUDA runtime is linked statically so
the library does not depend on which libcudart the host process (torch) loaded; it uses
the device's primary context, the same one torch uses, so torch streams are valid here.
"""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "_lib", "liblfds.so")
SOURCES = ["lfds_kernels.cu", "lfds_peak.cu", "lfds_margin.cu", "lfds_zsolve.cu", "lfds_proj.cu", "lfds_xform.cu", "lfds_dst.cu", "lfds_modal.cu", "lfds_krylov.cu", "lfds_host.cpp", "lfds_eig.cpp", "lfds_ml.cpp", "lfds_mw.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-Xcompiler", "-O3", "-cudart", "static", "--expt-relaxed-constexpr"]


def needs_build():
    if not os.path.exists(OUT):
        return True
    t = os.path.getmtime(OUT)
    deps = [os.path.join(SRC, f) for f in os.listdir(SRC)] + [os.path.join(HERE, "..", "include", "lfds.h")]
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(force=False, verbose=False):
    if not force and not needs_build():
        return OUT
    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    objs = [os.path.join(HERE, "_lib", s + ".o") for s in SOURCES]
    cmds = [[NVCC] + FLAGS + ["-c", os.path.join(SRC, s), "-o", o] for s, o in zip(SOURCES, objs)]
    if verbose:
        for cmd in cmds:
            print(" ".join(cmd))
    # translation units compile in parallel (one nvcc process each)
    procs = [subprocess.Popen(cmd) for cmd in cmds]
    codes = [p.wait() for p in procs]
    if any(codes):
        raise subprocess.CalledProcessError(next(c for c in codes if c), "nvcc")
    cmd = [NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-cudart", "static",
           "-o", OUT] + objs
    if verbose:
        print(" ".join(cmd))
    subprocess.run(cmd, check=True)
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
