import cProfile, pstats, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2008_03095_b200 import configs
cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
pr = cProfile.Profile(); t = time.time(); pr.enable()
g = configs.build(cfg)
g.device_graph()
pr.disable(); print("build", time.time() - t)
pstats.Stats(pr).sort_stats("cumulative").print_stats(14)
