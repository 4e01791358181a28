"""Build libfj.so (the C-ABI library) in-tree for sm_100a with nvcc."""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
SO = os.path.join(HERE, "libfj.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

def _nccl_include():
    """nccl.h for the TYPES only (libnccl.so.2 is dlopen'ed at fj_comm_init): torch's pip NCCL."""
    try:
        import nvidia.nccl
        return os.path.join(list(nvidia.nccl.__path__)[0], "include")
    except Exception:
        return "/usr/include"


FLAGS = [
    "-O3", "-std=c++17", "-lineinfo",
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-Xcompiler", "-fPIC,-O3", "-shared", "-cudart", "static",
    "--expt-relaxed-constexpr", "-DCCCL_IGNORE_DEPRECATED_API",
    "-Xcompiler", "-Wno-deprecated-declarations",
]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def source_hash() -> str:
    """Identity of the CUDA sources a libfj.so is built from (csrc/*.cu, *.cuh, include/fj.h): keys
    the ncu evidence in profiles/ncu_traffic.json so bench.py never attaches a stale capture."""
    import hashlib
    h = hashlib.sha256()
    files = sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cuh")))
    for f in files + [os.path.join(ROOT, "include", "fj.h")]:
        h.update(os.path.basename(f).encode())
        h.update(open(f, "rb").read())
    return h.hexdigest()[:16]


def needs_build() -> bool:
    """Rebuild when libfj.so is missing or was built from other sources (content hash recorded
    beside it at build time), or when a source is newer than it."""
    if not os.path.exists(SO):
        return True
    hp = SO + ".srchash"
    if not os.path.exists(hp) or open(hp).read().strip() != source_hash():
        return True
    t = os.path.getmtime(SO)
    deps = sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + [os.path.join(ROOT, "include", "fj.h"), __file__]
    return any(os.path.getmtime(p) > t for p in deps)


def build(force: bool = False, verbose: bool = False, so: str = SO, defines=()) -> str:
    """Compile every csrc/*.cu and link `so`.  `defines` (e.g. ["FJ_ITEMS=16"]) are tuning-knob
    variants for A/B builds (tools/build_variant.py); the default build uses none."""
    if not force and so == SO and not needs_build():
        return SO
    objs = []
    tag = "" if not defines else "_" + "_".join(d.replace("=", "") for d in defines)
    # variant objects live outside the repo (they are not shipped to the GPU box)
    bdir = os.path.join(HERE, "build") if not defines else os.path.join("/tmp", "fj_build" + tag)
    os.makedirs(bdir, exist_ok=True)
    procs = []
    for src in sources():
        obj = os.path.join(bdir, os.path.basename(src) + ".o")
        cmd = [NVCC, *[f for f in FLAGS if f != "-shared"], *[f"-D{d}" for d in defines], "-c", src, "-o", obj,
               "-I", os.path.join(ROOT, "include"), "-I", _nccl_include()]
        if verbose:
            cmd += ["-Xptxas", "-v"]
        procs.append((subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT), src))
        objs.append(obj)
    failed = False
    for p, src in procs:
        out, _ = p.communicate()
        if out:
            sys.stderr.write(out.decode())
        if p.returncode != 0:
            failed = True
            sys.stderr.write(f"nvcc failed on {src}\n")
    if failed:
        raise RuntimeError("libfj build failed")
    tmp = so + ".tmp"
    subprocess.check_call([NVCC, "-shared", "-cudart", "static", "-gencode", "arch=compute_100a,code=sm_100a",
                           *objs, "-o", tmp, "-ldl"])
    os.replace(tmp, so)
    if so == SO and not defines:
        with open(SO + ".srchash", "w") as f:
            f.write(source_hash() + "\n")
    return so


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(SO)
