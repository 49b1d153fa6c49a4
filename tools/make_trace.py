# Writes a config-B-shaped CKVT trace (N layers x 8 heads, 32k, T=64) from the oracle generator:
#   python tools/make_trace.py out.ckvt N_LAYERS
import sys, numpy as np
sys.path.insert(0, '/root/repo')
from oracle.oracle import Oracle
from paper_2412_03213_b200 import trace as T
P = Oracle('port')
L, Tn, nl, nh = 32768, 64, int(sys.argv[2]), 8
tr = P.generate_synthetic(7, nl, nh, L, Tn)
heads = [T.HeadTrace(tr.prompt_keys[i], tr.prompt_values[i], tr.decode_queries[i], tr.decode_keys[i], tr.decode_values[i]) for i in range(nl*nh)]
T.write_trace(T.TraceBundle(nl, nh, heads, {"generator": "synthetic-mixture", "seed": "7", "n_centers": "8"}), sys.argv[1])
