"""Build libaci.so in-tree with nvcc for sm_100a (called by __graft_entry__.build())."""
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SRC = [os.path.join(HERE, "csrc", f) for f in ("aci.cu", "gemm.cu", "prrlu.cu")]
HDR = [os.path.join(HERE, "csrc", f) for f in ("aci_common.cuh", "gemm_kernel.cuh", "prrlu_rook.cuh")] + [
    os.path.join(ROOT, "include", "aci.h")]
LIB = os.path.join(HERE, "libaci.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17", "-shared",
         "-Xcompiler", "-fPIC", "-Xptxas", "-v", "-I", os.path.join(ROOT, "include")]


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(f) > t for f in SRC + HDR)


PEAK_SRC = os.path.join(HERE, "csrc", "peak_probe.cu")
PEAK_LIB = os.path.join(HERE, "libaci_peak.so")


def build_peak(force: bool = False) -> str:
    """libaci_peak.so: the FP64 DMMA / DFMA loops bench.py measures its roofline peaks with."""
    deps = [PEAK_SRC, os.path.join(HERE, "csrc", "prrlu.cu"), os.path.join(HERE, "csrc", "prrlu_rook.cuh")] + HDR
    if force or not os.path.exists(PEAK_LIB) or any(os.path.getmtime(f) > os.path.getmtime(PEAK_LIB) for f in deps):
        cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17", "-shared",
               "-Xcompiler", "-fPIC", "-I", os.path.join(HERE, "csrc"), "-I", os.path.join(ROOT, "include"),
               "-o", PEAK_LIB, PEAK_SRC, "-lcudart"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            if os.path.exists(PEAK_LIB):
                os.remove(PEAK_LIB)
            raise RuntimeError("nvcc failed (peak probe):\n" + r.stderr[-2000:])
    return PEAK_LIB


def build(force: bool = False, verbose: bool = False) -> str:
    """Compile the translation units of libaci.so in parallel (nvcc -c each), then link."""
    if force or stale():
        objdir = os.path.join(HERE, "build")
        os.makedirs(objdir, exist_ok=True)
        cflags = [f for f in FLAGS if f != "-shared"]
        procs = []
        for src in SRC:
            obj = os.path.join(objdir, os.path.basename(src) + ".o")
            procs.append((obj, subprocess.Popen([NVCC] + cflags + ["-c", "-o", obj, src], stdout=subprocess.PIPE,
                                                stderr=subprocess.PIPE, text=True)))
        logs, failed = [], []
        for obj, p in procs:
            out, err = p.communicate()
            logs.append(err)
            if p.returncode != 0:
                failed.append(out + err)
        if not failed:
            r = subprocess.run([NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", LIB]
                               + [o for o, _ in procs] + ["-lcudart"], capture_output=True, text=True)
            if r.returncode != 0:
                failed.append(r.stdout + r.stderr)
        if failed:
            if os.path.exists(LIB):
                os.remove(LIB)  # never leave a stale library behind a failed build
            errs = "\n".join(l for f in failed for l in f.splitlines() if "error" in l.lower())
            raise RuntimeError("nvcc failed:\n" + errs)
        with open(os.path.join(HERE, "ptxas.log"), "w") as f:
            f.write("".join(logs))
        if verbose:
            print("".join(logs))
    return LIB


EXAMPLE_SRC = os.path.join(ROOT, "examples", "aci_example.c")
EXAMPLE_BIN = os.path.join(ROOT, "examples", "aci_example")


def build_example() -> str:
    """Compile examples/aci_example.c (plain C against include/aci.h and libaci.so)."""
    build()
    cmd = ["gcc", "-O2", "-I", os.path.join(ROOT, "include"), EXAMPLE_SRC, "-L", HERE, "-laci",
           "-Wl,-rpath," + HERE, "-lm", "-o", EXAMPLE_BIN]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    return EXAMPLE_BIN


if __name__ == "__main__":
    build(force=True, verbose=False)
    build_peak(force=True)
    print(LIB)
