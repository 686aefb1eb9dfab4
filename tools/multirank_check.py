"""N-rank run_fused vs single-rank on the same inputs (launch with torchrun;
IMX ranks may share one GPU: the collectives are gloo on host tensors).

    torchrun --nproc-per-node 2 --master-addr 127.0.0.1 tools/multirank_check.py [config]
"""
import os
import sys
from pathlib import Path

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2008_03095_b200 as imx
from paper_2008_03095_b200 import configs
from paper_2008_03095_b200.celf import LocalComm, TorchComm

cfg = sys.argv[1] if len(sys.argv) > 1 else "c1"
dist.init_process_group("gloo")
rank = dist.get_rank()
imx.set_device(int(os.environ.get("LOCAL_RANK", 0)) % max(1, torch.cuda.device_count()))
c = configs.CONFIGS[cfg]
g = configs.build(cfg)
multi = imx.run_fused(g, c.K, num_simulations=c.R, master_seed=0, comm=TorchComm())
if rank == 0:
    single = imx.run_fused(g, c.K, num_simulations=c.R, master_seed=0, comm=LocalComm())
    ok_seeds = list(multi.seeds) == list(single.seeds)
    ok_gains = list(multi.selection.gains) == list(single.selection.gains)
    ok_trace = np.array_equal(multi.selection.trace.array, single.selection.trace.array)
    print(f"{cfg}: seeds {ok_seeds} gains {ok_gains} trace {ok_trace} "
          f"spread {multi.spread} vs {single.spread} se {multi.spread_se} vs {single.spread_se}")
    if not ok_seeds:
        print("multi ", list(multi.seeds)[:10], list(multi.selection.gains)[:10])
        print("single", list(single.seeds)[:10], list(single.selection.gains)[:10])
dist.destroy_process_group()
