import sys; sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import numpy as np, synth, oracle
from paper_1510_05237_b200 import ESNMF, ESNMF_SIDE_V, ESNMF_SIDE_U
from parity import coo_dense
cfg = synth.CONFIGS['tiny']; g = synth.generate(cfg)
for k, t in ((33, 1), (33, 3), (4, 1), (40, 1), (33, 50)):
    s = ESNMF(cfg.n, cfg.m, k, t, g, seed=3)
    U = coo_dense((cfg.n, k), *s.get_U()[:2], s.get_U()[2])
    refv = oracle.half_step(g['at_ptr'], g['at_col'], g['at_val'], U, t)
    s.half_step(ESNMF_SIDE_V); _, lsv = s.get_ls(ESNMF_SIDE_V)
    V = coo_dense((cfg.m, k), *s.get_V()[:2], s.get_V()[2])
    refu = oracle.half_step(g['a_ptr'], g['a_col'], g['a_val'], V, t)
    s.half_step(ESNMF_SIDE_U); _, lsu = s.get_ls(ESNMF_SIDE_U)
    for nm, ls, ref in (('V', lsv, refv['LS']), ('U', lsu, refu['LS'])):
        sc = np.abs(ref).max(0); sc[sc == 0] = 1
        e = np.abs(ls - ref) / sc
        i, c = np.unravel_index(e.argmax(), e.shape)
        print(k, t, nm, 'err', e.max(), 'at', i, c, ls[i, c], ref[i, c], 'cols bad', np.nonzero(e.max(0) > 1e-5)[0][:10])
