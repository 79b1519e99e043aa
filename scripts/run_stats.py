import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
from paper_2602_15917_b200 import Pipeline
for name in ("C2", "C4"):
    cfg = synth.CONFIGS[name]
    x = synth.generate(cfg)
    p = Pipeline(cfg.shape, cfg.dtype, eb=cfg.eb, rel_eb=cfg.rel_eb, conn=cfg.conn, se=cfg.se, min_size=cfg.min_size, polarity=cfg.polarity)
    r = p.run(x)
    print(name, "kept", r.count, "runs", r.n_runs, "avg run", r.count / max(r.n_runs, 1), "components", r.n_components, "kept comps", r.n_kept)
    del x, p
    torch.cuda.empty_cache()
