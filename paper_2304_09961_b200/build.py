"""In-tree build of the native libraries (nvcc / g++ directly, no setuptools).

  lib/libbs_host.so  C++20 host scheduler + event loop (no CUDA)
  lib/libbs_nets.so  network definitions, calibrated weights, synthetic images (no CUDA)
  lib/libbs_exec.so  sm_100a kernels + executor + arena + C-ABI (links host objects)
  bin/batchsim_b200  CLI: simulate / sweep-capacity / validate-profile / oracle-check

Both are built with -ffp-contract=off so host double arithmetic matches the
reference's.
"""
from __future__ import annotations

import hashlib
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB = PKG / "lib"
BIN = PKG / "bin"
OBJ = ROOT / "build" / "obj"
INCLUDE = ROOT / "include"
# nlohmann/json (header-only parser; the copy shipped in this image's
# cudnn_frontend tree, the same one the reference oracle is built with).
JSON_INC = Path(os.environ.get(
    "BS_JSON_INC",
    "/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann"))

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
GENCODE = ["-gencode", "arch=compute_100a,code=sm_100a"]
HOST_FLAGS = ["-std=c++20", "-O2", "-fPIC", "-ffp-contract=off", "-Wall", "-Wextra",
              "-Wno-unused-parameter"]
NVCC_FLAGS = ["-std=c++20", "-O3", "-lineinfo", *GENCODE, "-Xcompiler", "-fPIC",
              "-Xcompiler", "-ffp-contract=off", "--expt-relaxed-constexpr",
              "-Xptxas", "-v" if os.environ.get("BS_PTXAS_V") else "-O3"]


def _sources(sub: str, exts: tuple[str, ...]) -> list[Path]:
    d = CSRC / sub
    return sorted(p for p in d.rglob("*") if p.suffix in exts)


def _headers() -> list[Path]:
    return sorted(p for p in CSRC.rglob("*") if p.suffix in (".h", ".hpp", ".cuh")) + \
        sorted(INCLUDE.glob("*.h"))


def _hdr_digest() -> str:
    h = hashlib.sha1()
    for p in _headers():
        h.update(p.read_bytes())
    return h.hexdigest()


def _needs(obj: Path, src: Path, digest: str) -> bool:
    stamp = obj.with_suffix(obj.suffix + ".stamp")
    if not obj.exists() or not stamp.exists():
        return True
    if stamp.read_text() != digest:
        return True
    return src.stat().st_mtime > obj.stat().st_mtime


def _run(cmd: list[str]) -> None:
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
        raise RuntimeError(f"build failed: {cmd[-1] if cmd else ''}")
    if os.environ.get("BS_PTXAS_V") and r.stderr:
        sys.stderr.write(r.stderr)


def _compile(src: Path, digest: str) -> Path:
    rel = src.relative_to(CSRC)
    obj = OBJ / (str(rel).replace("/", "__") + ".o")
    obj.parent.mkdir(parents=True, exist_ok=True)
    if _needs(obj, src, digest):
        incs = [f"-I{INCLUDE}", f"-I{CSRC}", f"-I{CSRC / 'host'}", f"-I{CSRC / 'exec'}",
                f"-I{JSON_INC}"]
        if src.suffix == ".cu":
            cmd = [NVCC, *NVCC_FLAGS, *incs, "-c", str(src), "-o", str(obj)]
        else:
            cmd = ["g++", *HOST_FLAGS, *incs, "-c", str(src), "-o", str(obj)]
        _run(cmd)
        obj.with_suffix(obj.suffix + ".stamp").write_text(digest)
    return obj


def build(verbose: bool = False) -> dict[str, Path]:
    LIB.mkdir(parents=True, exist_ok=True)
    digest = _hdr_digest()
    host_srcs = _sources("host", (".cpp",))
    exec_srcs = _sources("kernels", (".cu",)) + _sources("exec", (".cu", ".cpp"))
    with ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
        host_objs = list(ex.map(lambda s: _compile(s, digest), host_srcs))
        exec_objs = list(ex.map(lambda s: _compile(s, digest), exec_srcs))
    out = {}
    host_so = LIB / "libbs_host.so"
    if host_objs:
        _run(["g++", "-shared", "-o", str(host_so), *map(str, host_objs)])
        out["host"] = host_so
    # Native CLI with the reference's subcommands (csrc/cli), linked against
    # the host objects only (no CUDA).
    cli_objs = [_compile(s, digest) for s in _sources("cli", (".cpp",))]
    if cli_objs:
        BIN.mkdir(parents=True, exist_ok=True)
        cli = BIN / "batchsim_b200"
        _run(["g++", "-o", str(cli), *map(str, cli_objs), *map(str, host_objs)])
        out["cli"] = cli
    # CPU-only network definitions + calibrated weights (include/bs_nets.h).
    nets_objs = [o for o in exec_objs if o.name in ("exec__netdef.cpp.o", "exec__calib.cpp.o", "exec__capi_nets.cpp.o")]
    nets_so = LIB / "libbs_nets.so"
    _run(["g++", "-shared", "-o", str(nets_so), *map(str, nets_objs), "-lpthread"])
    out["nets"] = nets_so
    exec_so = LIB / "libbs_exec.so"
    _run([NVCC, "-shared", *GENCODE, "-o", str(exec_so), *map(str, exec_objs),
          *map(str, host_objs), "-lcudart"])
    out["exec"] = exec_so
    if verbose:
        for k, v in out.items():
            print(f"built {k}: {v}")
    return out


if __name__ == "__main__":
    build(verbose=True)
