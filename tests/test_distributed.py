"""N > 1 path on CPU: world_size-2 gloo ranks shard frames and gather results.

The per-rank compute is the CPU oracle here (no GPU in the build container);
on a B200 box the same function runs the CUDA pipeline.  Frames are
independent, so the gathered result must equal a single-process run.
"""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2003_00575_b200.distributed import segment_sharded, shard_range


def test_shard_range_covers_everything():
    for n in (0, 1, 5, 256, 1023):
        for world in (1, 2, 3, 8):
            spans = [shard_range(n, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            for (a, b), (c, d) in zip(spans, spans[1:]):
                assert b == c
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_range(4, 2, 2)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _frames():
    from paper_2003_00575_b200 import synthetic
    return synthetic.make_batch(3, 6).numpy()


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2003_00575_b200 as rs
        from oracle import oracle
        from paper_2003_00575_b200 import synthetic
        packed = rs.pack_tables(synthetic.sensor_for(synthetic.CONFIGS[3]), rs.PipelineConfig())

        def seg(shard):
            lab, ncl, _ = oracle.segment_batch(shard, packed, nthreads=1)
            return lab, ncl

        res = segment_sharded(_frames(), seg)
        if rank == 0:
            np.savez(out, labels=res[0], ncl=res[1])
        else:
            assert res is None
        res_all = segment_sharded(_frames(), seg, dst=None)
        assert res_all[0].shape[0] == 6
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_gather_equals_single_process(tmp_path):
    import paper_2003_00575_b200 as rs
    from oracle import oracle
    from paper_2003_00575_b200 import synthetic
    out = tmp_path / "res.npz"
    mp.spawn(_worker, args=(2, _free_port(), str(out)), nprocs=2, join=True)
    got = np.load(out)
    packed = rs.pack_tables(synthetic.sensor_for(synthetic.CONFIGS[3]), rs.PipelineConfig())
    want_l, want_n, _ = oracle.segment_batch(_frames(), packed, nthreads=1)
    assert np.array_equal(got["labels"], want_l)
    assert np.array_equal(got["ncl"], want_n)
