"""Compiles the C++ test programs against libckv_b200.so and the C oracle:
shim_parity (the drop-in header, tests/test_gpu_shim.py) and sharded_native
(the C-ABI sharded k-means over NCCL / LOCAL ranks, no PyTorch,
tests/test_gpu_sharded_native.py).  Used by __graft_entry__.build()."""
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
EXE = os.path.join(HERE, "shim_parity")
EXE_SHARD = os.path.join(HERE, "sharded_native")


def build_sharded() -> str:
    pkg = os.path.join(ROOT, "paper_2412_03213_b200")
    orc = os.path.join(ROOT, "oracle")
    src = os.path.join(HERE, "sharded_native.cpp")
    deps = [src, os.path.join(pkg, "libckv_b200.so"), os.path.join(orc, "libckv_oracle.so"),
            os.path.join(ROOT, "include", "ckv_cuda.h")]
    if os.path.exists(EXE_SHARD) and \
            os.path.getmtime(EXE_SHARD) >= max(os.path.getmtime(d) for d in deps):
        return EXE_SHARD
    cmd = ["g++", "-std=c++17", "-O2", "-pthread", f"-I{os.path.join(ROOT, 'include')}", f"-I{orc}",
           src, "-o", EXE_SHARD, f"-L{pkg}", "-lckv_b200", os.path.join(orc, "libckv_oracle.so"),
           f"-Wl,-rpath,{pkg}", f"-Wl,-rpath,{orc}", "-lm", "-Wl,--allow-shlib-undefined"]
    subprocess.run(cmd, check=True)
    return EXE_SHARD


def build() -> str:
    build_sharded()
    pkg = os.path.join(ROOT, "paper_2412_03213_b200")
    orc = os.path.join(ROOT, "oracle")
    src = os.path.join(HERE, "shim_parity.cpp")
    deps = [src, os.path.join(pkg, "libckv_b200.so"), os.path.join(orc, "libckv_oracle.so"),
            os.path.join(ROOT, "include", "clusterkv_b200", "clusterkv.hpp")]
    if os.path.exists(EXE) and os.path.getmtime(EXE) >= max(os.path.getmtime(d) for d in deps):
        return EXE
    cmd = ["g++", "-std=c++20", "-O2", f"-I{os.path.join(ROOT, 'include')}", f"-I{orc}", src,
           "-o", EXE, f"-L{pkg}", "-lckv_b200", os.path.join(orc, "libckv_oracle.so"),
           f"-Wl,-rpath,{pkg}", f"-Wl,-rpath,{orc}", "-lm",
           # libcuda.so.1 comes from the driver at run time; the container has none
           "-Wl,--allow-shlib-undefined"]
    subprocess.run(cmd, check=True)
    return EXE


if __name__ == "__main__":
    print(build())
