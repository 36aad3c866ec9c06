"""Per-iteration time at Large vs the V-side head size (tensor-core terms)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    import synth
    from paper_1510_05237_b200 import ESNMF

    cfg = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "large"]
    sizes = [int(x) for x in (sys.argv[2].split(",") if len(sys.argv) > 2 else "0,512,1024,1536,2048,3072,4096".split(","))]
    g = synth.generate_device(cfg, device="cuda")
    st = torch.cuda.Stream()
    torch.cuda.set_stream(st)
    for h in sizes:
        s = ESNMF(cfg.n, cfg.m, cfg.k, cfg.t, g, seed=cfg.seed, stream=st.cuda_stream, head_terms=h)
        s.iterate(5)
        torch.cuda.synchronize()
        s.profile(True)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        s.iterate(30)
        e1.record(st)
        torch.cuda.synchronize()
        ph = s.phase_times()
        s.profile(False)
        info = s.info()
        print(json.dumps({"head_terms": info["head_terms"], "head_dense": info["head_dense"],
                          "ms_per_iter": round(e0.elapsed_time(e1) / 30, 4),
                          "tail_ms": round(ph["V.spmm"][1] / 30, 4),
                          "head_ms": round(ph.get("V.head", (0, 0))[1] / 30, 4)}), flush=True)
        s.close()
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
