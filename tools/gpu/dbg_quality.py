import faulthandler, sys, time, os
sys.path.insert(0, os.getcwd())
faulthandler.dump_traceback_later(100, exit=True)
import numpy as np
from tests.test_gpu_quality import _bundle, GOLD
from paper_2412_03213_b200 import quality as Q
from paper_2412_03213_b200.api import ClusterConfig
g = np.load(GOLD)
t0 = time.time()
bundle, spec = _bundle(g)
print("bundle", time.time() - t0, flush=True)
cfg = Q.PolicyConfig(budget=96, cluster=ClusterConfig(decode_batch=16, c0_divisor=40))
rep = Q.run_simulation(bundle, cfg)
print("run", time.time() - t0, rep.summary, flush=True)
