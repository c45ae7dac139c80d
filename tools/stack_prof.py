"""Runs one forward of bench.py's 28-block PixArt-alpha stack (no graph) --
for `ncu --metrics gpu__time_duration.sum` launch lists of the stack."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402

bench.STACK_BLOCKS = int(os.environ.get("STACK_BLOCKS", "2"))
res = bench.run_stack(torch.device("cuda:0"), reps=1)
print(res)
