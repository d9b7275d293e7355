"""Build libmt.so in-tree with nvcc for sm_100a (B200)."""
import glob
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SO = os.path.join(HERE, "libmt.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-Xcompiler", "-O2", "--expt-relaxed-constexpr", "-ftz=true"]


def sources():
    return sorted(glob.glob(os.path.join(HERE, "csrc", "*.cu")))


def headers():
    return sorted(glob.glob(os.path.join(HERE, "csrc", "*.cuh"))) + [os.path.join(ROOT, "include", "mt.h")]


def stale() -> bool:
    if not os.path.exists(SO):
        return True
    t = os.path.getmtime(SO)
    return any(os.path.getmtime(f) > t for f in sources() + headers())


def build(force: bool = False, verbose: bool = False, out: str = SO, defines=()) -> str:
    """Compile each translation unit in parallel (separate objects, no device
    linking: no kernel calls across units), then link the shared library."""
    from concurrent.futures import ThreadPoolExecutor
    import tempfile
    if not force and out == SO and not stale():
        return out
    extra = [f"-D{d}" for d in defines]
    with tempfile.TemporaryDirectory() as d:
        objs = []
        cmds = []
        for src in sources():
            o = os.path.join(d, os.path.basename(src) + ".o")
            objs.append(o)
            cmd = [NVCC, *FLAGS, *extra, "-c", src, "-o", o]
            if verbose:
                cmd.insert(1, "-Xptxas=-v")
            cmds.append(cmd)
        with ThreadPoolExecutor(max_workers=len(cmds)) as ex:
            for r in ex.map(lambda c: subprocess.run(c, capture_output=True, text=True), cmds):
                if verbose or r.returncode:
                    print(r.stdout + r.stderr)
                if r.returncode:
                    raise subprocess.CalledProcessError(r.returncode, r.args)
        subprocess.check_call([NVCC, *FLAGS, "-shared", "-o", out, *objs, "-lcudart", "-ldl"])
    return out


if __name__ == "__main__":
    import sys
    build(force=True, verbose="-v" in sys.argv)
    print(SO)
