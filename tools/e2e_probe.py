"""Break the bench's e2e job into create / iterate / getters (host wall time)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1510_05237_b200 import ESNMF  # noqa: E402

cfg = synth.CONFIGS["large"]
g = synth.generate_device(cfg, device="cuda")
host = {k: torch.empty(g[k].shape, dtype=g[k].dtype, pin_memory=True) for k in ("a_ptr", "a_col", "a_val")}
for k in host:
    host[k].copy_(g[k])
del g
torch.cuda.synchronize()
st = torch.cuda.Stream()
for rep in range(3):
    t0 = time.perf_counter()
    e = ESNMF(cfg.n, cfg.m, cfg.k, cfg.t, host, seed=cfg.seed, stream=st.cuda_stream)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    e.iterate(cfg.iters)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    e.records(); e.get_U(); e.get_V()
    t3 = time.perf_counter()
    print("create %.1f ms  iterate(50) %.1f ms  getters %.1f ms" % ((t1 - t0) * 1e3, (t2 - t1) * 1e3, (t3 - t2) * 1e3),
          flush=True)
    e.close()
