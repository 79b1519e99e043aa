"""Small end-to-end cases for compute-sanitizer (memcheck / racecheck / synccheck / initcheck): every
C-ABI call of the path and of the NEXT rows on tiny volumes (SURVEY.md §4 'Sanitizers').

    compute-sanitizer --tool memcheck python scripts/sanitize.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import synth  # noqa: E402
from paper_2602_15917_b200 import Pipeline  # noqa: E402
from paper_2602_15917_b200 import _lib as L  # noqa: E402
from paper_2602_15917_b200.sharded import run_simulated  # noqa: E402


def main():
    cases = [(synth.scaled("C1", 0.25), {}), (synth.scaled("C2", 0.08), {}),
             (synth.scaled("C3", 0.03, frames=3), {"frames": True}),
             (synth.scaled("C4", 0.03), {"keep": "largest"}), (synth.scaled("C1", 0.25), {"classes": 3})]
    for cfg, extra in cases:
        tw = torch.empty(synth.truth_words(cfg) + 4, dtype=torch.int32, device="cuda")
        x = synth.generate(cfg, truth=tw)
        kw = dict(eb=cfg.eb, rel_eb=cfg.rel_eb, conn=cfg.conn, se=cfg.se, min_size=cfg.min_size,
                  polarity=cfg.polarity, spans=True, **extra)
        p = Pipeline(cfg.shape, cfg.dtype, **kw)
        r = p.run(x)
        p.decode()
        p.decode(from_spans=True)
        q = p.quality(tw)
        torch.cuda.synchronize()
        print(cfg.name, extra, "kept", r.count, "dsc %.4f" % q["dsc"], flush=True)
        if cfg.dtype == "u16" and not extra:
            rp = Pipeline(cfg.shape, cfg.dtype, extract="runs", **{k: v for k, v in kw.items() if k != "spans"}).run(x)
            assert torch.equal(rp.codes, r.codes)
            codes = r.codes
            n = codes.numel()
            ws = torch.empty(L.roix_greedy_workspace(n), dtype=torch.uint8, device="cuda")
            Q = torch.empty(n + 8, dtype=torch.int16, device="cuda")
            gb = torch.empty((n + 31) // 32 + 2, dtype=torch.int32, device="cuda")
            ng = torch.zeros(1, dtype=torch.int64, device="cuda")
            st = torch.cuda.current_stream().cuda_stream
            import ctypes
            sp = lambda t: ctypes.c_void_p(t.data_ptr())
            L.roix_greedy_quantize(sp(codes), n, 2.0, 65535, sp(Q), sp(gb), sp(ng), sp(ws), ws.numel(),
                                   ctypes.c_void_p(st))
            torch.cuda.synchronize()
    cfg = synth.scaled("C5", 0.03)
    x = synth.generate(cfg)
    run_simulated(x, 2, eb=cfg.eb, conn=cfg.conn, se=cfg.se, min_size=cfg.min_size)
    torch.cuda.synchronize()
    print("sanitize cases ok", flush=True)


if __name__ == "__main__":
    main()
