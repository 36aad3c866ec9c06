import sys; sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import numpy as np, synth, oracle
from paper_1510_05237_b200 import ESNMF, ESNMF_SIDE_V, ESNMF_SIDE_U
from parity import coo_dense
cfg = synth.CONFIGS['tiny']; g = synth.generate(cfg)
k, t = 33, 1
s = ESNMF(cfg.n, cfg.m, k, t, g, seed=3)
s.half_step(ESNMF_SIDE_V)
V = coo_dense((cfg.m, k), *s.get_V()[:2], s.get_V()[2])
print('V nnz per col', (V != 0).sum(0)[:10], 'docs', np.nonzero(V.any(1))[0][:40])
Gg, eps = s.get_gram(ESNMF_SIDE_U)
G = V.T @ V
print('gram diff', np.abs(Gg - G).max(), 'diag', np.diag(G)[:5], 'offdiag max', np.abs(G - np.diag(np.diag(G))).max())
s.half_step(ESNMF_SIDE_U); _, ls = s.get_ls(ESNMF_SIDE_U)
Y = oracle.spmm(g['a_ptr'], g['a_col'], g['a_val'], V)
W = np.linalg.inv(G + eps * np.eye(k))
ref = Y @ W
i = 1237
print('row', i, 'Y nz cols', np.nonzero(Y[i])[0], 'Y', Y[i][np.nonzero(Y[i])[0]])
print('gpu', ls[i][:12]); print('ref', ref[i][:12])
# is gpu = Y @ W_some?
bad = np.nonzero(np.abs(ls - ref).max(1) > 1e-3 * np.abs(ref).max())[0]
print('bad rows', len(bad), bad[:20])
print('Y nnz of bad rows', [(np.nonzero(Y[b])[0]).tolist() for b in bad[:5]])
