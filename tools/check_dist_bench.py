"""bench.py's distributed leg (solve_distributed) on a 1-rank NCCL group: the
NCCL communicator and the library's distributed block on one GPU."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29533")
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import bench  # noqa: E402

torch.cuda.set_device(0)
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
print(json.dumps(bench.solve_distributed(5, 2, 0, 1, dist, 0)))
dist.destroy_process_group()
