"""Build libsc.so in-tree: nvcc for sm_100a (CUDA sources) + g++ (host C++), linked
with a static CUDA runtime.  Called by __graft_entry__.build() and the tests."""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.environ.get("SC_BUILD_OUT", os.path.join(HERE, "libsc.so"))   # experiments: variant builds
BUILD = os.path.join(HERE, "_build" + os.environ.get("SC_BUILD_TAG", ""))
DEFS = os.environ.get("SC_NVCC_DEFS", "").split()   # experiments: e.g. -DSOLVE_NT=256
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CU = ["setup.cu", "step.cu", "solve.cu"]
CPP = ["rules.cpp", "factor.cpp", "partition.cpp", "nccl.cpp", "api.cpp"]


def _run(cmd):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
        raise RuntimeError("build failed: " + " ".join(cmd[:3]))
    return r.stdout + r.stderr


def sources():
    return [os.path.join(CSRC, f) for f in CU + CPP] + [
        os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".h", ".cuh"))] + [
        os.path.join(HERE, "..", "include", "sc.h")]


def up_to_date():
    if not os.path.exists(OUT):
        return False
    t = os.path.getmtime(OUT)
    return all(os.path.getmtime(s) <= t for s in sources())


def build(force=False, verbose=False):
    if not force and up_to_date():
        return OUT
    os.makedirs(BUILD, exist_ok=True)
    objs = []
    logs = []
    for f in CU:
        o = os.path.join(BUILD, f + ".o")
        logs.append(_run([NVCC, *ARCH, *DEFS, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
                          "--expt-relaxed-constexpr", "-Xptxas", "-v", "-c", os.path.join(CSRC, f), "-o", o]))
        objs.append(o)
    for f in CPP:
        o = os.path.join(BUILD, f + ".o")
        logs.append(_run([NVCC, *ARCH, *DEFS, "-O3", "-std=c++17", "-Xcompiler", "-fPIC,-fopenmp,-ffp-contract=off",
                          "-c", os.path.join(CSRC, f), "-o", o]))
        objs.append(o)
    tmp = OUT + ".tmp"
    _run([NVCC, *ARCH, "-shared", "-cudart", "static", "-o", tmp, *objs, "-Xcompiler", "-fopenmp", "-lgomp", "-ldl"])
    os.replace(tmp, OUT)
    if verbose:
        print("\n".join(logs))
    return OUT


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(OUT)
