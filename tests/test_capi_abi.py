"""CPU-only: libckv_b200.so loads and exports every symbol include/ckv_cuda.h
declares, and the ctypes table covers them all (no compute without a GPU)."""
import ctypes
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "ckv_cuda.h")


def declared_symbols():
    src = open(HDR).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ckv_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_entry_points():
    syms = declared_symbols()
    for s in ("ckv_kmeans", "ckv_cluster_prefill", "ckv_cluster_decode_batch", "ckv_build_index",
              "ckv_select", "ckv_attend", "ckv_cache_lookup", "ckv_session_step"):
        assert s in syms


def test_library_exports_every_declared_symbol():
    from paper_2412_03213_b200 import build as B
    if not os.path.exists(B.LIB):
        B.build()
    lib = ctypes.CDLL(B.LIB)
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing


def test_ctypes_table_matches_header():
    from paper_2412_03213_b200 import _native
    assert sorted(_native.SIGNATURES) == declared_symbols()


def test_host_side_abi_without_gpu():
    """Pure host entry points work without a device: init sampling
    (clustering.hpp:186-193), mix_seed and the C0 rule."""
    import numpy as np
    from oracle.oracle import Oracle
    from paper_2412_03213_b200 import _native
    L = _native.lib()
    rows = np.zeros(409, np.uint32)
    assert L.ckv_kmeans_init_rows(32752, 409, 12345, rows.ctypes.data) == 0
    assert np.array_equal(rows, Oracle("port").kmeans_init_rows(32752, 409, 12345))
    assert L.ckv_mix_seed(0, 3, 5) == Oracle("port").mix_seed(0, 3, 5)
    assert L.ckv_prefill_cluster_count(32016, 80, 16, 0) == 400
    assert L.ckv_kmeans_init_rows(3, 4, 0, rows.ctypes.data) == 1


def test_cpp_dropin_exports_and_links():
    """The reference-signature C++ drop-in (include/clusterkv_b200/clusterkv.hpp)
    has a definition in libckv_b200.so for every free function / ClusterCache
    member it declares, and the parity program links against it."""
    import subprocess
    from paper_2412_03213_b200 import build as B
    if not os.path.exists(B.LIB):
        B.build()
    out = subprocess.run(["nm", "-DC", "--defined-only", B.LIB], capture_output=True,
                         text=True, check=True).stdout
    for name in ("ckv::kmeans_cosine(", "ckv::prefill_cluster_count(", "ckv::cluster_prefill(",
                 "ckv::cluster_decode_batch(", "ckv::build_index(", "ckv::score_clusters(",
                 "ckv::select_tokens(", "ckv::approx_attention(", "ckv::ClusterCache::ClusterCache(",
                 "ckv::ClusterCache::~ClusterCache(", "ckv::ClusterCache::lookup_and_update(",
                 "ckv::ClusterCache::hit_rate(", "ckv::ClusterCache::invalidate_on_recluster(",
                 "ckv::ClusterCache::counters("):
        assert name in out, name
    from oracle.oracle import build as obuild
    obuild()
    from tests.cpp.build import build as sbuild
    assert os.path.exists(sbuild())
