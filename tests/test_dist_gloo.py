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


class _ShmCtx:
    """CPU stand-in for Context in FusedGatherPCMM's protocol: buffers are named shared-memory arrays (the "IPC
    handle" is the name), the accumulate is the oracle's Algorithm 1 written into every destination at row0, the
    flags are host words (test infrastructure only)."""

    def __init__(self, o, level):
        from multiprocessing import shared_memory
        self.shm, self.o, self.level = shared_memory, o, level
        self.keep = []

    def wire_bytes(self, level):
        return 2 * level * self.o.n * 8                      # uint64 words as bytes (no compaction needed here)

    def weights(self, W):
        return W

    def alloc(self, shape, dt):
        dtype = np.uint8 if dt == "uint8" else np.int32
        nbytes = int(np.prod(shape)) * np.dtype(dtype).itemsize
        sm = self.shm.SharedMemory(create=True, size=nbytes)
        self.keep.append(sm)
        a = np.ndarray(shape, dtype=dtype, buffer=sm.buf)
        a[...] = 0
        return _Named(a, sm.name)

    def ipc_handle(self, buf):
        return (buf.name, buf.a.shape, str(buf.a.dtype))

    def ipc_open(self, h):
        sm = self.shm.SharedMemory(name=h[0])
        self.keep.append(sm)
        return _Named(np.ndarray(h[1], dtype=np.dtype(h[2]), buffer=sm.buf), h[0])

    def ipc_close(self, p):
        pass

    def pcmm_ternary_compact_gather(self, x, w, dsts, rows_total, row0, level, stream=None):
        y = self.o.pcmm_a(x, w).view(np.uint8).reshape(w.shape[1], -1)
        for dbuf in dsts:
            dbuf.a[row0:row0 + y.shape[0]] = y

    def peer_signal(self, flag_dsts, slot, epoch, stream=None):
        for f in flag_dsts:
            f.a[slot] = epoch

    def peer_wait(self, flags, n, epoch, stream=None):
        import time
        t0 = time.time()
        while not all(int(v) >= epoch for v in flags.a[:n]):
            assert time.time() - t0 < 60, "peer_wait timed out"
            time.sleep(0.001)


class _Named:
    def __init__(self, a, name):
        self.a, self.name = a, name


def _fused_worker(rank, world, port, d, m, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    import oracle
    import synth
    from paper_2509_09424_b200.dist import FusedGatherPCMM
    dist.init_process_group("gloo", rank=rank, world_size=world)
    o = oracle.Oracle(12, 2, 1, 2)
    ctx = _ShmCtx(o, 1)
    x = synth.gen_words(57, o.q, d, 1, o.n)
    W = synth.gen_W(58, d, m)
    fg = FusedGatherPCMM(ctx, W, world, rank, 1, alloc=ctx.alloc)
    for _ in range(2):                                          # two layers: epochs 1 and 2
        dist.barrier()
        y = fg(x)
    assert int(fg.flags.a.min()) == 2
    if rank == 0:
        out_q.put(y.a[:m].copy().view(np.uint64).reshape(m, 2, 1, o.n))
    dist.barrier()
    fg.close()
    dist.destroy_process_group()


def test_fused_gather_protocol_world2_ragged():
    """FusedGatherPCMM's host protocol at world size 2 (gloo; a shared-memory stand-in for the CUDA IPC mappings):
    handle exchange, every rank's rows at rank * S of every gathered buffer, the epoch flags -- with m = 7 (a
    zero-padded last shard), the gathered rows equal the single-process oracle layer."""
    import oracle
    import synth
    world, d, m = 2, 5, 7
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_fused_worker, args=(r, world, port, d, m, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = q.get(timeout=300)
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    o = oracle.Oracle(12, 2, 1, 2)
    want = o.pcmm_a(synth.gen_words(57, o.q, d, 1, o.n), synth.gen_W(58, d, m))
    assert (got == want).all()


class _FailOpenCtx(_ShmCtx):
    """The stand-in with a peer mapping that fails on one rank (e.g. a GPU pair without peer access)."""

    def __init__(self, o, level, fail):
        super().__init__(o, level)
        self.fail = fail

    def ipc_open(self, h):
        if self.fail:
            raise OSError("peer mapping refused")
        return super().ipc_open(h)


def _fused_fail_worker(rank, world, port, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    import oracle
    import synth
    from paper_2509_09424_b200.dist import FusedGatherPCMM
    dist.init_process_group("gloo", rank=rank, world_size=world)
    o = oracle.Oracle(12, 2, 1, 2)
    ctx = _FailOpenCtx(o, 1, fail=(rank == 1))
    try:
        FusedGatherPCMM(ctx, synth.gen_W(58, 5, 7), world, rank, 1, alloc=ctx.alloc)
        out_q.put((rank, "no error"))
    except RuntimeError as e:
        out_q.put((rank, str(e)))
    dist.barrier()                                              # both ranks still in step after the failure
    dist.destroy_process_group()


def test_fused_gather_setup_fails_on_every_rank_together():
    """A peer mapping that fails on rank 1 makes FusedGatherPCMM raise on BOTH ranks (no rank is left waiting in the
    handle exchange or in peer_wait) -- the bench's N > 1 fused-gather leg relies on it to skip cleanly."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_fused_fail_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    for r in range(world):
        assert "peer mapping failed" in got[r] and "rank 1" in got[r], got
