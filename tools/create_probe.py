"""Host wall time of esnmf_create at a config from host (pinned) CSR, by stage."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["ESNMF_CREATE_TIMING"] = "1"
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1510_05237_b200 import ESNMF  # noqa: E402

cfg = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "large"]
g = synth.generate_device(cfg, device="cuda")
host = {k: torch.empty(g[k].shape, dtype=g[k].dtype, pin_memory=True) for k in ("a_ptr", "a_col", "a_val")}
for k in host:
    host[k].copy_(g[k])
del g
torch.cuda.synchronize()
for rep in range(2):
    t0 = time.perf_counter()
    s = ESNMF(cfg.n, cfg.m, cfg.k, cfg.t, host, seed=cfg.seed)
    torch.cuda.synchronize()
    print("create total %.1f ms" % ((time.perf_counter() - t0) * 1e3), file=sys.stderr, flush=True)
    s.close()
