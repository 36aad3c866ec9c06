"""Small cases for compute-sanitizer (memcheck / racecheck / synccheck / initcheck):
Tiny with the tensor-core head forced on (k_vhead_otf), the U-side tcgen05
finish (k_uside_tc), the selection paths, a CUDA-graph replay, and two loopback
ranks in two threads.  One GPU.

    compute-sanitizer --tool memcheck python tools/san_case.py [single|loopback]
"""
import os
import sys
import threading

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def single():
    import synth
    from paper_1510_05237_b200 import ESNMF

    cfg = synth.CONFIGS["tiny"]
    g = synth.generate(cfg)
    with ESNMF(cfg.n, cfg.m, cfg.k, cfg.t, g, seed=cfg.seed, head_terms=128) as s:
        s.iterate(5)   # 2 eager + graph capture + replays
        print("single", s.info()["head_terms"], [round(r["E"], 6) for r in s.records()])
    with ESNMF(cfg.n, cfg.m, cfg.k, None, g, seed=cfg.seed, head_terms=64) as s:
        s.iterate(3)   # unlimited t: 3-pass selection
        print("tinf", [round(r["E"], 6) for r in s.records()])


def loopback():
    import torch

    import synth
    import paper_1510_05237_b200 as pk
    from paper_1510_05237_b200 import ESNMF

    cfg = synth.CONFIGS["tiny"]
    g = synth.generate(cfg)
    grp = pk.comm.LoopbackGroup(2)
    out = [None, None]

    def worker(r):
        st = torch.cuda.Stream()
        h = ESNMF(cfg.n, cfg.m, cfg.k, cfg.t, g, seed=cfg.seed, world=2, rank=r, comm=grp.comms[r],
                  stream=st.cuda_stream)
        h.iterate(3)
        out[r] = h.records()

    th = [threading.Thread(target=worker, args=(r,)) for r in range(2)]
    for x in th:
        x.start()
    for x in th:
        x.join()
    print("loopback", [round(r["E"], 6) for r in out[0]])


if __name__ == "__main__":
    {"single": single, "loopback": loopback}[sys.argv[1] if len(sys.argv) > 1 else "single"]()
