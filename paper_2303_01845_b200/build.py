"""Build the in-tree native libraries (nvcc for sm_100a; gcc for the oracle).

    python -m paper_2303_01845_b200.build
"""

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libpastis_sw.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared",
]


def _stale(target, sources):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(s) > t for s in sources)


def build_native(force: bool = False, verbose: bool = False) -> str:
    srcs = [os.path.join(CSRC, f) for f in sorted(os.listdir(CSRC))
            if f.endswith((".cu", ".cuh", ".h"))]
    srcs.append(os.path.join(ROOT, "include", "pastis_sw.h"))
    if force or _stale(LIB, srcs):
        cmd = [NVCC, *NVCC_FLAGS, "-o", LIB, os.path.join(CSRC, "sw_engine.cu")]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        subprocess.run(cmd, check=True)
    return LIB


def pack_ext_path() -> str:
    import sysconfig
    return os.path.join(HERE, "_pack" + sysconfig.get_config_var("EXT_SUFFIX"))


def build_pack(force: bool = False) -> str:
    """The drop-in API's packing layer (csrc/pack_ext.c, a CPython extension)."""
    import sysconfig
    target = pack_ext_path()
    src = os.path.join(CSRC, "pack_ext.c")
    if force or _stale(target, [src]):
        cc = os.environ.get("CC", "gcc")
        subprocess.run([cc, "-O2", "-fPIC", "-shared", "-pthread", "-Wall",
                        "-I", sysconfig.get_paths()["include"], "-o", target, src], check=True)
    return target


def build_oracle(force: bool = False) -> str:
    odir = os.path.join(ROOT, "oracle")
    target = os.path.join(odir, "liborc.so")
    if force or _stale(target, [os.path.join(odir, "sw_oracle.c")]):
        subprocess.run(["make", "-B" if force else "-s", "-C", odir, "liborc.so"], check=True)
    return target


def build_synth(force: bool = False) -> str:
    """The bench/test workload generator (pastis_synth/gen.c, gcc)."""
    sdir = os.path.join(ROOT, "pastis_synth")
    target = os.path.join(sdir, "libsynth.so")
    if force or _stale(target, [os.path.join(sdir, "gen.c")]):
        subprocess.run(["make", "-B" if force else "-s", "-C", sdir, "libsynth.so"], check=True)
    return target


if __name__ == "__main__":
    force = "--force" in sys.argv
    print(build_native(force=force, verbose="-v" in sys.argv))
    print(build_pack(force=force))
    print(build_oracle(force=force))
    print(build_synth(force=force))
