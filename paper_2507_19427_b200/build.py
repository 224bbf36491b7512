"""Build the sm_100a C-ABI library in-tree (paper_2507_19427_b200/libafdk.so).

nvcc cross-compiles for sm_100a without a GPU.  The library links the CUDA
runtime statically and resolves cuTensorMapEncodeTiled through
cudaGetDriverEntryPoint, so loading it needs no libcuda at link time and
the .so can be dlopen'ed on a CPU-only box to check its exports.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libafdk.so")

CU_SOURCES = [
    "afdk_api.cu",
    "mfa_decode.cu",
    "mfa_decode_fp8.cu",
    "mfa_decode_mtp.cu",
    "linear.cu",
    "linear_mx.cu",
    "moe_gemm_mx.cu",
    "moe_gemm_mx2.cu",
    "moe_gemm_bf16.cu",
    "moe_ffn_mx_fused.cu",
    "mfa_layer.cu",
    "moe_route.cu",
    "moe_gemm.cu",
    "moe_ffn.cu",
    "exchange.cu",
    "afd_measured.cu",
    "pipeline_model.cpp",
    "afd_runtime.cu",
    "nvls.cu",
]
CXX_SOURCES: list[str] = []

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "--expt-relaxed-constexpr",
    "-Xcompiler", "-fPIC",
    "-Xptxas", "-v",
    "-I", os.path.join(ROOT, "include"),
]


def _stale(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(verbose: bool = False, force: bool = False) -> str:
    objdir = os.path.join(HERE, "_obj")
    os.makedirs(objdir, exist_ok=True)
    headers = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".h", ".cuh", ".hpp"))]
    headers += [os.path.join(ROOT, "include", h) for h in ("afdk.h", "afd_b200.hpp", "afd_compat.hpp")]
    objs = []
    for src in CU_SOURCES + CXX_SOURCES:
        path = os.path.join(CSRC, src)
        obj = os.path.join(objdir, src + ".o")
        objs.append(obj)
        if force or _stale(obj, [path] + headers):
            cmd = [NVCC, *NVCC_FLAGS, "-c", path, "-o", obj]
            res = subprocess.run(cmd, capture_output=True, text=True)
            if verbose or res.returncode != 0:
                sys.stderr.write(" ".join(cmd) + "\n" + res.stdout + res.stderr)
            if res.returncode != 0:
                raise RuntimeError(f"nvcc failed for {src}")
    if force or _stale(OUT, objs):
        cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", OUT, *objs,
               "-cudart", "static", "-lrt", "-ldl", "-lpthread"]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            sys.stderr.write(" ".join(cmd) + "\n" + res.stdout + res.stderr)
            raise RuntimeError("link failed")
    build_demo(force)
    build_afd_demo(force)
    build_ref_demo(force)
    return OUT


DEMO_SRC = os.path.join(ROOT, "tests", "cpp", "stage_times_demo.cpp")
DEMO_OUT = os.path.join(ROOT, "tests", "cpp", "stage_times_demo")


def build_demo(force: bool = False) -> str:
    """C++ consumer of the host API (afd_b200.hpp), linked against libafdk.so."""
    deps = [DEMO_SRC, OUT, os.path.join(ROOT, "include", "afd_b200.hpp")]
    if force or _stale(DEMO_OUT, deps):
        cmd = ["g++", "-std=c++20", "-O2", "-I", os.path.join(ROOT, "include"), DEMO_SRC, "-o", DEMO_OUT,
               "-L", HERE, "-lafdk", f"-Wl,-rpath,{HERE}", "-Wl,-rpath,$ORIGIN/../../paper_2507_19427_b200"]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            sys.stderr.write(" ".join(cmd) + "\n" + res.stdout + res.stderr)
            raise RuntimeError("demo build failed")
    return DEMO_OUT


AFD_DEMO_SRC = os.path.join(ROOT, "tests", "cpp", "afd_cpp_demo.cpp")
AFD_DEMO_OUT = os.path.join(ROOT, "tests", "cpp", "afd_cpp_demo")
CUDA_HOME = os.environ.get("CUDA_HOME", "/usr/local/cuda")


def build_afd_demo(force: bool = False) -> str:
    """The AFD runtime driven from C++ alone (fork per rank, file rendezvous),
    linked against libafdk.so and the static CUDA runtime for its own buffers."""
    deps = [AFD_DEMO_SRC, OUT, os.path.join(ROOT, "include", "afdk.h")]
    if force or _stale(AFD_DEMO_OUT, deps):
        cmd = ["g++", "-std=c++17", "-O2", "-Wall", "-I", os.path.join(ROOT, "include"), "-I",
               os.path.join(CUDA_HOME, "include"), AFD_DEMO_SRC, "-o", AFD_DEMO_OUT, "-L", HERE, "-lafdk",
               "-L", os.path.join(CUDA_HOME, "lib64"), "-lcudart_static", "-lrt", "-ldl", "-lpthread",
               f"-Wl,-rpath,{HERE}", "-Wl,-rpath,$ORIGIN/../../paper_2507_19427_b200"]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            sys.stderr.write(" ".join(cmd) + "\n" + res.stdout + res.stderr)
            raise RuntimeError("AFD C++ demo build failed")
    return AFD_DEMO_OUT


REF_INCLUDE = os.environ.get("AFD_REFERENCE_INCLUDE", "/root/reference/proj/include")
REF_LIB = os.path.join(ROOT, "oracle", "_ref", "libafdref.so")
REF_DEMO_SRC = os.path.join(ROOT, "tests", "cpp", "stage_times_ref_demo.cpp")
REF_DEMO_OUT = os.path.join(ROOT, "tests", "cpp", "stage_times_ref_demo")


def build_ref_demo(force: bool = False) -> str | None:
    """The drop-in proof: the C++ host API compiled against the REFERENCE's own
    headers (AFD_B200_USE_REFERENCE_HEADERS) and linked with the reference's
    own library (oracle/_ref/libafdref.so) + libafdk.so.  Built only where the
    reference tree is present (this container); the binary travels to the GPU
    box with the snapshot (rpaths are $ORIGIN-relative)."""
    if not (os.path.isdir(REF_INCLUDE) and os.path.exists(REF_LIB)):
        return None
    deps = [REF_DEMO_SRC, OUT, REF_LIB, os.path.join(ROOT, "include", "afd_b200.hpp")]
    if force or _stale(REF_DEMO_OUT, deps):
        cmd = ["g++", "-std=c++20", "-O2", "-DAFD_B200_USE_REFERENCE_HEADERS", "-I", REF_INCLUDE, "-I",
               os.path.join(ROOT, "include"), REF_DEMO_SRC, "-o", REF_DEMO_OUT, "-L", HERE, "-lafdk",
               "-L", os.path.dirname(REF_LIB), "-lafdref",
               "-Wl,-rpath,$ORIGIN/../../paper_2507_19427_b200", "-Wl,-rpath,$ORIGIN/../../oracle/_ref"]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            sys.stderr.write(" ".join(cmd) + "\n" + res.stdout + res.stderr)
            raise RuntimeError("reference-headers demo build failed")
    return REF_DEMO_OUT


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))
