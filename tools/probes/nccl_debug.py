"""Probe (dev tool): where NCCL_DEBUG=INFO output goes under torchrun."""
import glob
import os
import sys

import torch
import torch.distributed as dist

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dist.init_process_group("nccl", device_id=torch.device("cuda", rank))
x = torch.ones(4, device="cuda")
dist.all_reduce(x)
torch.cuda.synchronize()
print("rank", rank, "env", {k: v for k, v in os.environ.items() if k.startswith("NCCL")}, file=sys.stderr)
print("rank", rank, "files", glob.glob("/tmp/ltb_nccl*"), file=sys.stderr)
dist.destroy_process_group()
