#!/usr/bin/env python
"""Write tests/golden/fullsize_<cfg>.json: the streaming oracle's result on a full-size BASELINE.json
config (C3 / C4 / C5), for tests/test_gpu_fullsize.py.

Calls only the input generator (synth/: the seeded phantom, generated on the GPU -- the shared input
module, no method arithmetic) and the oracle (oracle/stream.py).  No value comes from the CUDA path
(paper_2602_15917_b200 is never imported).  Runs on a GPU box (the phantom is generated there):

    python scripts/make_fullsize_golden.py --config C4
"""
import argparse
import json
import os
import platform
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", required=True)
    ap.add_argument("--out", default=None)
    ap.add_argument("--scale", type=float, default=1.0, help="sanity run on a scaled phantom (not a golden)")
    a = ap.parse_args()
    import torch

    import oracle
    import synth
    from oracle import stream
    from oracle.digest import source_hashes

    assert "paper_2602_15917_b200" not in sys.modules
    synth.build()
    oracle.build()
    cfg = synth.CONFIGS[a.config] if a.scale == 1.0 else synth.scaled(a.config, a.scale)
    assert cfg.dtype == "u16"
    t0 = time.time()
    x = synth.generate(cfg)
    torch.cuda.synchronize()
    feed = lambda z0, nz: synth.to_numpy(x[z0:z0 + nz], cfg)
    res = stream.fullsize_u16(feed, cfg.shape, eb=cfg.eb, conn=cfg.conn, se=cfg.se, min_size=cfg.min_size,
                              polarity=cfg.polarity, log=lambda s: print(a.config, s, flush=True))
    assert "paper_2602_15917_b200" not in sys.modules
    res.update(config=a.config, seed=cfg.seed, eb=cfg.eb, conn=cfg.conn, se=cfg.se, min_size=cfg.min_size,
               polarity=cfg.polarity, sources=source_hashes(), wall_seconds=time.time() - t0,
               host={"cpu": platform.processor() or platform.machine(), "nproc": os.cpu_count()},
               written_by="scripts/make_fullsize_golden.py (synth + oracle.stream only)")
    res["scale"] = a.scale
    out = a.out or os.path.join(ROOT, "tests", "golden", "fullsize_%s.json" % a.config)
    if a.scale != 1.0 and not a.out:
        out = "/tmp/fullsize_%s_%g.json" % (a.config, a.scale)
    with open(out, "w") as f:
        json.dump(res, f, indent=1)
    print("wrote", out, "count", res["count"], "components", res["n_components"], flush=True)


if __name__ == "__main__":
    main()
