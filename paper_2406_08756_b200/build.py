"""In-tree build of the native library `_lib/liblynx_b200.so`.

Every CUDA translation unit is compiled for sm_100a only
(`-gencode arch=compute_100a,code=sm_100a`, `-lineinfo`); host C++ units
(planner restatement, runtime, C-ABI) are compiled with nvcc as well so one
toolchain links everything. Nothing is JIT-compiled at import time: the built
`.so` lives next to the package and travels to the GPU box with the repo.

    python -m paper_2406_08756_b200.build            # incremental
    python -m paper_2406_08756_b200.build --clean
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import os
import shutil
import subprocess
import sys
import sysconfig
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
OBJ = ROOT / "build" / "obj"
LIB = PKG / "_lib" / "liblynx_b200.so"
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
CXX = os.environ.get("CXX", "g++")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nlohmann_include() -> str:
    p = Path(sysconfig.get_paths()["purelib"]) / "include" / "cudnn_frontend" / "thirdparty"
    return str(p)


def _nccl_dir() -> Path | None:
    """NCCL bundled with PyTorch (nvidia-nccl wheel). Linking against the same libnccl.so.2 as torch
    matters: the soname is shared, so whichever copy loads first serves both (the system 2.27 copy
    lacks symbols torch's 2.28 build needs)."""
    p = Path(sysconfig.get_paths()["purelib"]) / "nvidia" / "nccl"
    return p if (p / "lib" / "libnccl.so.2").exists() and (p / "include" / "nccl.h").exists() else None


def _nccl_include() -> list[str]:
    d = _nccl_dir()
    return [f"-I{d / 'include'}"] if d else []


def _nccl_link() -> list[str]:
    d = _nccl_dir()
    if d:
        return [f"-L{d / 'lib'}", "-l:libnccl.so.2", "-Xlinker", f"-rpath,{d / 'lib'}"]
    return ["-lnccl", "-L/usr/lib/x86_64-linux-gnu", "-Xlinker", "-rpath,/usr/lib/x86_64-linux-gnu"]


def _flags() -> list[str]:
    return [
        "-O3", "-std=c++17", "-lineinfo", *ARCH, *(["-DLYNX_ATTN_TRACE"] if os.environ.get("LYNX_BUILD_TRACE") else []),
        "-Xcompiler", "-fPIC", "-Xcompiler", "-Wall",
        "--expt-relaxed-constexpr",
        f"-I{ROOT / 'include'}", f"-I{CSRC}", f"-I{_nlohmann_include()}", *_nccl_include(),
        "-diag-suppress", "177,550",
    ]


def _sources() -> list[Path]:
    return sorted([*CSRC.rglob("*.cu"), *CSRC.rglob("*.cpp")])


def _headers() -> list[Path]:
    return [*CSRC.rglob("*.cuh"), *CSRC.rglob("*.h"), *CSRC.rglob("*.hpp"), *(ROOT / "include").glob("*.h")]


def _obj_for(src: Path) -> Path:
    rel = src.relative_to(CSRC).with_suffix(".o")
    return OBJ / str(rel).replace(os.sep, "__")


def _compile(src: Path, newest_header: float) -> tuple[Path, str]:
    obj = _obj_for(src)
    if obj.exists() and obj.stat().st_mtime >= max(src.stat().st_mtime, newest_header):
        return obj, ""
    obj.parent.mkdir(parents=True, exist_ok=True)
    cmd = [NVCC, *_flags(), "-c", str(src), "-o", str(obj)]
    if src.suffix == ".cpp":  # host-only C++ (planner, runtime glue): plain g++
        cmd = [CXX, "-O2", "-std=c++17", "-fPIC", "-g", "-Wall", "-Wextra", "-Wno-unused-parameter",
               f"-I{ROOT / 'include'}", f"-I{CSRC}", f"-I{_nlohmann_include()}", *_nccl_include(),
               "-I/usr/local/cuda/include",
               "-c", str(src), "-o", str(obj)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src.name}:\n{r.stdout}\n{r.stderr}")
    return obj, (r.stderr or "")


def build(clean: bool = False, jobs: int | None = None, verbose: bool = False) -> Path:
    if clean and OBJ.exists():
        shutil.rmtree(OBJ)
    srcs = _sources()
    newest_header = max((h.stat().st_mtime for h in _headers()), default=0.0)
    with cf.ThreadPoolExecutor(max_workers=jobs or os.cpu_count()) as ex:
        results = list(ex.map(lambda s: _compile(s, newest_header), srcs))
    objs = [o for o, _ in results]
    if verbose:
        for _, log in results:
            if log.strip():
                print(log, file=sys.stderr)
    newest_obj = max(o.stat().st_mtime for o in objs)
    if LIB.exists() and LIB.stat().st_mtime >= newest_obj and not clean:
        build_cli()
        return LIB
    LIB.parent.mkdir(parents=True, exist_ok=True)
    tmp = LIB.with_suffix(".so.tmp")
    # Export the C-ABI only: the library's C++ symbols (nlohmann / STL template instances, the
    # planner restatement) stay local, so they cannot interpose on another library loaded into the
    # same process (e.g. the test oracle oracle/_ref, built from the reference with its own
    # instances of the same templates).
    exports = OBJ.parent / "exports.map"
    exports.parent.mkdir(parents=True, exist_ok=True)
    exports.write_text("{\n  global: lynx_*;\n  local: *;\n};\n")
    cmd = [NVCC, *ARCH, "-shared", "-o", str(tmp), *map(str, objs),
           "-lcudart", *_nccl_link(), "-Xlinker", f"--version-script={exports}"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, LIB)
    build_cli()
    return LIB


CLI_SRC = PKG / "cli" / "lynx_execute.cpp"
CLI = PKG / "_lib" / "lynx_execute"


def build_cli() -> Path:
    """`lynx execute` (cli/lynx_execute.cpp): a host C++ program over the C-ABI only."""
    if CLI.exists() and CLI.stat().st_mtime >= max(CLI_SRC.stat().st_mtime, LIB.stat().st_mtime):
        return CLI
    cmd = [CXX, "-O2", "-std=c++17", "-Wall", f"-I{ROOT / 'include'}", f"-I{_nlohmann_include()}", str(CLI_SRC),
           "-o", str(CLI), f"-L{LIB.parent}", "-l:liblynx_b200.so", "-Wl,-rpath,$ORIGIN",
           "-Wl,-rpath,/usr/local/cuda/lib64", "-L/usr/local/cuda/lib64", "-lcudart"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"lynx_execute build failed:\n{r.stderr}")
    return CLI


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--clean", action="store_true")
    ap.add_argument("-j", "--jobs", type=int, default=None)
    ap.add_argument("-v", "--verbose", action="store_true")
    a = ap.parse_args()
    print(build(clean=a.clean, jobs=a.jobs, verbose=a.verbose))
