"""World-size-2 `gloo` tests of the multi-GPU shard/gather logic on CPU (no GPU here).  The "kernel" is the
oracle's Algorithm 1 (test infrastructure), so the gathered result must equal the single-process oracle
output word for word."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from paper_2509_09424_b200.dist import ColumnShardedPCMM, column_shard, token_blocks


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_shard_arithmetic():
    for m in (1, 7, 768, 5504, 6144):
        for w in (1, 2, 3, 4, 8):
            covered = []
            for r in range(w):
                lo, hi, S = column_shard(m, w, r)
                assert hi - lo <= S and S * w >= m
                covered += list(range(lo, hi))
            assert covered == list(range(m))
            blocks = [b for r in range(w) for b in token_blocks(m, w, r)]
            assert blocks == list(range(m))


def _worker(rank, world, port, d, m, out_q, chunks=3):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    import oracle
    import synth
    dist.init_process_group("gloo", rank=rank, world_size=world)
    o = oracle.Oracle(12, 2, 1, 2)
    x = synth.gen_words(55, o.q, d, 1, o.n)                     # replicated inputs (same seed on every rank)
    W = synth.gen_W(56, d, m)
    sh = ColumnShardedPCMM(W, world, rank)

    def pcmm(xa, Wl, y_local):                                    # oracle as the kernel (test only)
        y_local.copy_(torch.from_numpy(o.pcmm_a(xa, Wl).view(np.int64)))

    y_local = sh.local_buffer(torch, (2, 1, o.n), "cpu")
    y_all = sh.gathered_buffer(torch, (2, 1, o.n), "cpu")
    sh(pcmm, x, y_local, y_all)
    # the chunked, overlapped variant gathers the same words
    y_local2 = sh.local_buffer(torch, (2, 1, o.n), "cpu")
    y_all2 = sh.gathered_buffer(torch, (2, 1, o.n), "cpu")
    y_all2.zero_()
    sh.run_overlapped(pcmm, x, y_local2, y_all2, sh.chunk_weights(chunks))
    assert torch.equal(y_all2[:m], y_all[:m])
    if rank == 0:
        out_q.put(y_all[:m].numpy().view(np.uint64).copy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("d,m", [(8, 6), (5, 9)])
def test_column_sharded_allgather_equals_single_process(d, m):
    import oracle
    import synth
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, d, m, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = q.get(timeout=240)
    for p in procs:
        p.join(timeout=240)
        assert p.exitcode == 0
    o = oracle.Oracle(12, 2, 1, 2)
    want = o.pcmm_a(synth.gen_words(55, o.q, d, 1, o.n), synth.gen_W(56, d, m))
    assert (got == want).all()


def test_column_sharded_world4_ragged():
    """World size 4, m = 7 (shards of S = 2, the last rank owns one real column and one zero-padded one) and 4
    chunks per shard (two of them empty, so run_overlapped skips them on every rank consistently): the gathered
    outputs of both the one-shot and the chunked, overlapped all-gather equal the single-process oracle."""
    import oracle
    import synth
    world, d, m = 4, 6, 7
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, d, m, q, 4)) for r in range(world)]
    for p in procs:
        p.start()
    got = q.get(timeout=300)
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    o = oracle.Oracle(12, 2, 1, 2)
    want = o.pcmm_a(synth.gen_words(55, o.q, d, 1, o.n), synth.gen_W(56, d, m))
    assert (got == want).all()


def _ccmm_worker(rank, world, port, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import sys
    import torch.distributed as dist
    import oracle
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    from test_oracle_ccmm import _ccmm_setup
    from paper_2509_09424_b200.dist import ccmm_shard, column_shard
    dist.init_process_group("gloo", rank=rank, world_size=world)
    o = oracle.Oracle(12, 3, 1, 3)
    skc, sk, pk = o.keygen(0x454E5349 + 1)
    form, s, d, m = 1, 8, 2, 5
    a, src, mask, keys, rlk, ref = _ccmm_setup(o, sk, pk, form, s, d, m, 77)   # same seeds: replicated inputs
    col0, cols = ccmm_shard(m, world, rank)
    S = column_shard(m, world, rank)[2]
    loc = np.zeros((S, 2, 1, o.n), np.uint64)
    if cols:
        loc[:cols] = o.ccmm(a, src, form, s, d, m, mask, keys, rlk, outputs=range(col0, col0 + cols))  # the "kernel"
    parts = [torch.zeros((S, 2, 1, o.n), dtype=torch.int64) for _ in range(world)]
    dist.all_gather(parts, torch.from_numpy(loc.view(np.int64)))
    if rank == 0:
        out_q.put(torch.cat(parts)[:m].numpy().view(np.uint64).copy())
    dist.barrier()
    dist.destroy_process_group()


def test_ccmm_column_shards_gather_to_single_process():
    """CCMM output columns sharded over two gloo ranks (ccmm_shard) gather to the single-process product."""
    import oracle
    from test_oracle_ccmm import _ccmm_setup
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_ccmm_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    got = q.get(timeout=600)
    for p in ps:
        p.join(timeout=600)
        assert p.exitcode == 0
    o = oracle.Oracle(12, 3, 1, 3)
    skc, sk, pk = o.keygen(0x454E5349 + 1)
    a, src, mask, keys, rlk, ref = _ccmm_setup(o, sk, pk, 1, 8, 2, 5, 77)
    assert (got == o.ccmm(a, src, 1, 8, 2, 5, mask, keys, rlk)).all()
