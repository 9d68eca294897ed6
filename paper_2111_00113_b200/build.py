"""Build libsks.so (the C-ABI of include/sks.h) in-tree with nvcc for sm_100a.

    python -m paper_2111_00113_b200.build [--force]

Sources: paper_2111_00113_b200/csrc/*.cu.  Output: paper_2111_00113_b200/libsks.so,
linked against the CUDA runtime (shared) and the torch-bundled NCCL 2.28.
"""
import glob
import hashlib
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libsks.so")
OBJ = os.path.join(HERE, "_build")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2", "-Xptxas", "-warn-spills"]
# experiments only (e.g. SKS_NVCC_EXTRA="-DZM_ZS_FORCE=2"); part of the build digest
FLAGS += [f for f in os.environ.get("SKS_NVCC_EXTRA", "").split() if f]


def nccl_dir():
    try:
        import nvidia.nccl as nn  # type: ignore
        d = list(nn.__path__)[0]
        if os.path.exists(os.path.join(d, "include", "nccl.h")):
            return d
    except Exception:
        pass
    for cand in glob.glob(os.path.join(sys.prefix, "lib", "python3*", "site-packages", "nvidia", "nccl")):
        if os.path.exists(os.path.join(cand, "include", "nccl.h")):
            return cand
    raise RuntimeError("NCCL (torch-bundled nvidia/nccl) not found")


def _digest(paths):
    h = hashlib.sha256()
    for p in sorted(paths):
        h.update(p.encode())
        with open(p, "rb") as f:
            h.update(f.read())
    h.update(" ".join(ARCH + FLAGS).encode())
    return h.hexdigest()


def build(force: bool = False, verbose: bool = False) -> str:
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    deps = srcs + glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h")) + \
        [os.path.join(ROOT, "include", "sks.h")]
    dig = _digest(deps)
    stamp = OUT + ".sha256"
    if not force and os.path.exists(OUT) and os.path.exists(stamp) and open(stamp).read() == dig:
        return OUT
    nd = nccl_dir()
    os.makedirs(OBJ, exist_ok=True)
    inc = ["-I" + os.path.join(nd, "include"), "-I" + os.path.join(ROOT, "include")]

    def comp(src):
        obj = os.path.join(OBJ, os.path.basename(src).replace(".cu", ".o"))
        cmd = [NVCC] + ARCH + FLAGS + inc + ["-c", src, "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError("nvcc failed for %s:\n%s\n%s" % (src, r.stdout, r.stderr))
        if verbose and (r.stderr.strip() or r.stdout.strip()):
            print(r.stderr, r.stdout)
        return obj

    with ThreadPoolExecutor(max_workers=min(8, len(srcs))) as ex:
        objs = list(ex.map(comp, srcs))
    libdir = os.path.join(nd, "lib")
    cmd = [NVCC] + ARCH + ["-shared", "-cudart", "shared", "-o", OUT + ".tmp"] + objs + [
        "-L" + libdir, "-l:libnccl.so.2", "-L/usr/local/cuda/lib64",
        "-Xlinker", "-rpath=" + libdir, "-Xlinker", "-rpath=/usr/local/cuda/lib64"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("link failed:\n%s\n%s" % (r.stdout, r.stderr))
    os.replace(OUT + ".tmp", OUT)
    with open(stamp, "w") as f:
        f.write(dig)
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
