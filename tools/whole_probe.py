"""A few whole-factor (Alg. 2 as printed) iterations at Large, for ncu launch lists of the flat selection."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
from paper_1510_05237_b200 import ESNMF
cfg = synth.CONFIGS["large"]
g = synth.generate_device(cfg, device="cuda"); torch.cuda.synchronize()
s = ESNMF(cfg.n, cfg.m, cfg.k, cfg.t, g, seed=cfg.seed, whole=True, t_u=cfg.k*cfg.t, t_v=cfg.k*cfg.t)
s.iterate(4)
torch.cuda.synchronize()
