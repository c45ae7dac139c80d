"""The sharded KERNEL path with two ranks before an 8-GPU box exists: two
processes on the one B200 (independent kernels, no cross-rank waits), each
running the STDiT linear stack (paper_2406_02540_b200/stack.py, the C5
workload's structure at a reduced size) on its token-row shard
(shard.row_range), the final fp16 outputs all-gathered over gloo; rank 0
checks them bitwise against its own forward of all rows (quant.cpp:70-73:
per-token params are row-local, qgemm.cpp:52-63: per-row dot products)."""
import os
import socket

import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, rows, txt_rows, blocks, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2406_02540_b200.shard import gather_rows, row_range
        from paper_2406_02540_b200.stack import (STDIT_LAYERS, LinearStack, StackShape,
                                                 w4a8_mp_plan)
        dev = torch.device("cuda", 0)
        torch.cuda.set_device(dev)
        st = LinearStack(STDIT_LAYERS, blocks, w4a8_mp_plan(STDIT_LAYERS, blocks), dev, seed=3)
        g = torch.Generator(device=dev).manual_seed(99)   # same global input on both ranks
        x = (torch.randn((rows, 1152), generator=g, device=dev) * 2).half()
        t = torch.randn((txt_rows, 1152), generator=g, device=dev).half()
        lo, hi = row_range(rows, rank, world)
        tlo, thi = row_range(txt_rows, rank, world)
        bufs = st.buffers(StackShape(hi - lo, thi - tlo))
        # step 3 of 20 (range 0: the plan's W8 cells) and step 15 (range 3: W4)
        ys = []
        for step in (3, 15):
            y = st.forward(bufs, x[lo:hi], t[tlo:thi], t=step, steps=20).clone()
            ys.append(gather_rows(y.cpu(), rows))  # gloo all_gather of the shards
        if rank == 0:
            full = st.buffers(StackShape(rows, txt_rows))
            same = [torch.equal(ya, st.forward(full, x, t, t=step, steps=20).cpu())
                    for ya, step in zip(ys, (3, 15))]
            q.put(same)
        dist.barrier()
    finally:
        dist.destroy_process_group()


def test_two_ranks_shard_the_stack_bit_identically():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    world = 2
    procs = [ctx.Process(target=_worker, args=(r, world, port, 2000, 240, 2, q))
             for r in range(world)]
    for p in procs:
        p.start()
    same = q.get(timeout=600)
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    assert same == [True, True]
