"""B200-native (sm_100a) ClusterKV recallable-KV hot path.

The product is libckv_b200.so (CUDA kernels behind the C-ABI in
include/ckv_cuda.h) and the reference-signature C++ drop-in
(include/clusterkv_b200/clusterkv.hpp).  This package holds the sources
(csrc/), the in-tree build (build.py) and the Python mirror used by tests
and bench.py (api.py, session.py).  Importing it never touches the GPU.
"""
__all__ = ["api", "session", "build"]
