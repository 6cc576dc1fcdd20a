"""Builds libllama_b200.so in-tree with nvcc for sm_100a (no JIT, no torch
extension machinery): every .cu/.cpp under csrc/ -> one shared library with a
plain C ABI (include/llama_b200.h)."""
import glob
import hashlib
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(ROOT, "build")
LIB = os.path.join(HERE, "libllama_b200.so")
STAMP = LIB + ".stamp"  # content hash of the sources + flags the library was built from
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler", "-Wall",
         "-I" + os.path.join(ROOT, "include"), "-I" + CSRC, "-I" + BUILD, "-I/usr/local/cuda/include"]


# device sources compiled at plan time by NVRTC (jit.cpp), embedded as strings
JIT_EMBED = [("kJitParamsSrc", "jit_params.h"), ("kJitKernelSrc", "jit_kernel.cuh"),
             ("kJitKernel2dSrc", "jit_kernel2d.cuh")]


def _write_embed():
    """build/jit_embed.inc: the NVRTC-compiled device sources as C++ raw strings."""
    os.makedirs(BUILD, exist_ok=True)
    out = []
    for name, fn in JIT_EMBED:
        with open(os.path.join(CSRC, fn)) as f:
            text = f.read()
        assert ')LLBJIT"' not in text
        out.append(f'static const char {name}[] = R"LLBJIT({text})LLBJIT";\n')
    path = os.path.join(BUILD, "jit_embed.inc")
    data = "".join(out)
    if not os.path.exists(path) or open(path).read() != data:
        with open(path, "w") as f:
            f.write(data)


def _sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))


def _deps():
    return _sources() + sorted(glob.glob(os.path.join(CSRC, "*.hpp")) + glob.glob(os.path.join(CSRC, "*.cuh"))
                               + [os.path.join(ROOT, "include", "llama_b200.h")])


def source_hash():
    h = hashlib.sha256(" ".join(ARCH + FLAGS[:3]).encode())
    for f in _deps():
        h.update(os.path.basename(f).encode())
        with open(f, "rb") as fh:
            h.update(fh.read())
    return h.hexdigest()


def up_to_date():
    """True when the library exists and was built from the current sources
    (content hash, not mtimes: a snapshot copied to another box keeps it)."""
    if not os.path.exists(LIB) or not os.path.exists(STAMP):
        return False
    with open(STAMP) as f:
        return f.read().strip() == source_hash()


def build(force=False, verbose=False):
    if not force and up_to_date():
        return LIB
    os.makedirs(BUILD, exist_ok=True)
    digest = source_hash()
    _write_embed()

    def compile_one(src):
        obj = os.path.join(BUILD, os.path.basename(src) + ".o")
        cmd = [NVCC] + ARCH + FLAGS + ["-c", src, "-o", obj]
        if src.endswith(".cu"):
            cmd += ["-Xptxas", "-v"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        return src, obj, cmd, r

    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        results = list(ex.map(compile_one, _sources()))
    objs = []
    log = []
    for src, obj, cmd, r in results:
        log.append(" ".join(cmd) + "\n" + r.stdout + r.stderr)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError(f"nvcc failed on {src}")
        objs.append(obj)
    tmp = LIB + f".tmp{os.getpid()}"
    cmd = [NVCC] + ARCH + ["-shared", "-o", tmp] + objs + ["-ldl"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("link failed")
    os.replace(tmp, LIB)
    with open(STAMP, "w") as f:
        f.write(digest + "\n")
    with open(os.path.join(BUILD, "build.log"), "w") as f:
        f.write("\n".join(log))
    if verbose:
        print("\n".join(log))
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
