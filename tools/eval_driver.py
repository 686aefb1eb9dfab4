"""evaluate_seeds on a config graph (ncu driver)."""
import sys
from pathlib import Path
import numpy as np
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2008_03095_b200 import configs
from paper_2008_03095_b200.evaluation import evaluate_counts
cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
worlds = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
c = configs.CONFIGS[cfg]
g = configs.build(cfg)
seeds = np.random.default_rng(0).choice(g.n, size=c.K, replace=False)
print(cfg, evaluate_counts(g, seeds, worlds, 1).mean())
