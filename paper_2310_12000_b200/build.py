"""Build the in-tree CUDA library ``libvlgpx.so`` for sm_100a with nvcc.

Usage:  python -m paper_2310_12000_b200.build   (or __graft_entry__.build())

Objects are compiled in parallel into a per-checkout directory under the
system temp dir (``VLGPX_BUILD_DIR`` overrides it) and linked into ``paper_2310_12000_b200/libvlgpx.so`` (git-ignored, but shipped
to the GPU box by gpurun because it lives in the tree).
"""

from __future__ import annotations

import concurrent.futures as cf
import hashlib
import os
import shutil
import subprocess
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
# object files live outside the tree (only the linked library travels to the GPU box)
OUT_DIR = os.environ.get("VLGPX_BUILD_DIR") or os.path.join(
    tempfile.gettempdir(), "vlgpx_build_" + hashlib.sha1(HERE.encode()).hexdigest()[:10], "_build")
LIB = os.path.join(HERE, "libvlgpx.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC,-O3,-pthread", "--expt-relaxed-constexpr",
          "-I", os.path.join(HERE, "..", "include")]


def nvcc():
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def sources():
    return sorted(f for f in os.listdir(CSRC) if f.endswith((".cu", ".cpp")))


def _includes(path, seen):
    """Transitive quoted includes of a source file (csrc/ and include/)."""
    if path in seen or not os.path.exists(path):
        return
    seen.add(path)
    with open(path) as fh:
        for line in fh:
            line = line.strip()
            if line.startswith("#include \""):
                name = line.split('"')[1]
                for base in (CSRC, os.path.join(HERE, "..", "include")):
                    _includes(os.path.join(base, name), seen)


def _compile(src, verbose_ptxas=False, defines=(), out_dir=OUT_DIR):
    obj = os.path.join(out_dir, src + ".o")
    path = os.path.join(CSRC, src)
    deps = set()
    _includes(path, deps)
    deps = sorted(deps)
    if os.path.exists(obj) and os.path.getmtime(obj) >= max(os.path.getmtime(d) for d in deps):
        return obj, ""
    cmd = [nvcc(), *ARCH, *COMMON, *[f"-D{d}" for d in defines], "-c", path, "-o", obj]
    if src.endswith(".cpp"):
        cmd[1:1] = ["-x", "cu"]  # host sources share the device headers
    if verbose_ptxas and src.endswith(".cu"):
        cmd.insert(1, "-Xptxas=-v")
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    return obj, r.stderr


def build(verbose=False, jobs=None, defines=(), lib=LIB, only=None):
    """``defines`` builds a variant library into its own object directory; with ``only``
    (source names) just those sources are compiled with the defines and every other object
    is taken from the default build (A/B experiments on one kernel family)."""
    out_dir = OUT_DIR if not defines else OUT_DIR + "_" + "_".join(d.replace("=", "") for d in defines)
    os.makedirs(out_dir, exist_ok=True)
    srcs = sources()
    jobs = jobs or min(len(srcs), os.cpu_count() or 4)

    def one(s):
        if only is not None and s not in only:
            return _compile(s, verbose, (), OUT_DIR)
        return _compile(s, verbose, defines, out_dir)

    with cf.ThreadPoolExecutor(jobs) as ex:
        results = list(ex.map(one, srcs))
    objs = [o for o, _ in results]
    if verbose:
        for (o, log), s in zip(results, srcs):
            if log:
                print(f"--- {s}\n{log}")
    newest = max(os.path.getmtime(o) for o in objs)
    if not (os.path.exists(lib) and os.path.getmtime(lib) >= newest):
        cmd = [nvcc(), *ARCH, "-shared", "-o", lib, *objs, "-lcudart", "-lcusolver", "-Xcompiler", "-pthread"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    return lib


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
