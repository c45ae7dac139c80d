"""N > 1 path on CPU: world-size-2 gloo processes shard token rows, run the
row-local quantized linear (here the CPU oracle, since this box has no GPU;
on the GPU box the same harness runs the sm_100a kernels over NCCL), and
all-gather the outputs; the result must equal the single-rank result bit for
bit (per-token params are row-local, quant.cpp:70-73)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2406_02540_b200.shard import gather_rows, row_range, sharded_apply


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_row_range_partitions_exactly():
    for M in (1, 7, 4096, 131072):
        for world in (1, 2, 3, 4, 8):
            spans = [row_range(M, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == M
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            assert max(b - a for a, b in spans) - min(b - a for a, b in spans) <= 1


def _worker(rank, world, port, M, K, N, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle.oracle import Oracle
        orc = Oracle()
        rng = np.random.default_rng(0)
        x = torch.from_numpy((rng.standard_normal((M, K)) * 2).astype(np.float16).astype(np.float64))
        w = rng.standard_normal((N, K))
        wc, sw, zw = orc.make_quant_linear(w, 8)

        def layer(xs):
            return torch.from_numpy(orc.qlinear_forward(xs.numpy(), wc, sw, zw, 8))

        def quant(xs):
            c, s, z = orc.quantize_rows(xs.numpy(), 8)
            return torch.from_numpy(np.concatenate([c.astype(np.float64), s[:, None], z[:, None]], 1))

        y = sharded_apply(x, layer)
        codes = sharded_apply(x, quant)
        if rank == 0:
            q.put((y.numpy(), codes.numpy(), layer(x).numpy(), quant(x).numpy()))
        # uneven shard sizes through gather_rows directly
        lo, hi = row_range(5, rank, world)
        g = gather_rows(torch.arange(lo, hi, dtype=torch.float64)[:, None], 5)
        assert g[:, 0].tolist() == [0, 1, 2, 3, 4]
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_gloo_row_sharding_is_bit_identical(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, 37, 256, 24, q)) for r in range(world)]
    for p in procs:
        p.start()
    y, codes, y_ref, codes_ref = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert np.array_equal(y, y_ref)
    assert np.array_equal(codes, codes_ref)
