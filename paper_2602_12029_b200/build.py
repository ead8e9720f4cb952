"""Build libpsk.so (all CUDA kernels + the C ABI) in-tree for sm_100a.

nvcc compiles every csrc/*.cu in parallel to an object, then links one
shared library next to this file, so the .so travels with the repo snapshot
to the GPU box. No JIT caches are involved.

    python -m paper_2602_12029_b200.build [--force] [-v]
"""

from __future__ import annotations

import argparse
import concurrent.futures as cf
import hashlib
import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
OBJ = PKG / "_build"
LIB = PKG / "libpsk.so"
NVCC = os.environ.get("NVCC", shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ARCH + [
    "-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
    "-Xptxas", "-warn-spills",
    f"-I{ROOT / 'include'}", f"-I{CSRC}",
]


def _sources() -> list[Path]:
    return sorted(CSRC.glob("*.cu"))


def _headers_digest() -> str:
    h = hashlib.sha256()
    for p in sorted(list(CSRC.glob("*.cuh")) + list((ROOT / "include").glob("*.h"))):
        h.update(p.read_bytes())
    h.update(" ".join(FLAGS).encode())
    return h.hexdigest()[:16]


def _obj_for(src: Path, hdr: str) -> Path:
    d = hashlib.sha256(src.read_bytes() + hdr.encode()).hexdigest()[:16]
    return OBJ / f"{src.stem}.{d}.o"


def _compile(src: Path, obj: Path, verbose: bool) -> None:
    cmd = [NVCC, *FLAGS, "-c", str(src), "-o", str(obj)]
    if verbose:
        cmd += ["-Xptxas", "-v"]
        print(" ".join(cmd), flush=True)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src.name}:\n{r.stdout}\n{r.stderr}")
    if verbose and r.stderr:
        print(r.stderr, flush=True)
    elif r.stderr:
        for line in r.stderr.splitlines():
            if "spill" in line or "warning" in line.lower():
                print(f"[{src.name}] {line}", flush=True)


def build(force: bool = False, verbose: bool = False) -> Path:
    OBJ.mkdir(exist_ok=True)
    hdr = _headers_digest()
    srcs = _sources()
    objs = [_obj_for(s, hdr) for s in srcs]
    todo = [(s, o) for s, o in zip(srcs, objs) if force or not o.exists()]
    if todo:
        with cf.ThreadPoolExecutor(max_workers=min(8, len(todo))) as ex:
            futs = [ex.submit(_compile, s, o, verbose) for s, o in todo]
            for f in futs:
                f.result()
    stamp = OBJ / "libpsk.stamp"
    key = "\n".join(o.name for o in objs)
    if force or not LIB.exists() or not stamp.exists() or stamp.read_text() != key:
        tmp = LIB.with_suffix(".so.tmp")
        cmd = [NVCC, *ARCH, "-shared", "-o", str(tmp), *map(str, objs), "-lcudart_static", "-lrt",
               "-ldl", "-lpthread"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
        os.replace(tmp, LIB)
        stamp.write_text(key)
    # drop stale objects
    keep = set(objs)
    for o in OBJ.glob("*.o"):
        if o not in keep:
            o.unlink()
    return LIB


def build_variant(defines: list[str], out: Path) -> Path:
    """Tuning builds: every source with extra -D flags, linked to `out`
    (load it with PSK_LIB=<out>). No object cache."""
    import tempfile
    with tempfile.TemporaryDirectory() as td:
        objs = []
        extra = [f"-D{d}" for d in defines]
        def one(src):
            o = Path(td) / (src.stem + ".o")
            r = subprocess.run([NVCC, *FLAGS, *extra, "-c", str(src), "-o", str(o)], capture_output=True,
                               text=True)
            if r.returncode != 0:
                raise RuntimeError(f"nvcc failed for {src.name}:\n{r.stderr}")
            return o
        with cf.ThreadPoolExecutor(max_workers=8) as ex:
            objs = list(ex.map(one, _sources()))
        r = subprocess.run([NVCC, *ARCH, "-shared", "-o", str(out), *map(str, objs), "-lcudart_static",
                            "-lrt", "-ldl", "-lpthread"], capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stderr}")
    return out


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("-v", "--verbose", action="store_true")
    ap.add_argument("--define", action="append", default=[], help="variant build: -D flag")
    ap.add_argument("--out", type=Path, help="variant build output .so")
    a = ap.parse_args()
    if a.define or a.out:
        print(build_variant(a.define, a.out or PKG / "libpsk_variant.so"))
        return
    print(build(force=a.force, verbose=a.verbose))


if __name__ == "__main__":
    sys.exit(main())
