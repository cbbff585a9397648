"""Multi-GPU plumbing on the one GPU this build has: the column-sharded PCMM through NCCL (world size 1: the
all-gather runs through NCCL on the device buffers) against the unsharded call and the oracle, and bench.py
launched the way the driver launches it for N > 1 (torch.distributed.run, NCCL rendezvous on 127.0.0.1).
World sizes > 1 are covered on CPU with gloo (tests/test_dist_gloo.py); ranks that wait on each other are never
stood in for on one GPU."""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def test_column_sharded_nccl_world1(torch_cuda):
    torch = torch_cuda
    import torch.distributed as dist
    from paper_2509_09424_b200 import Context
    from paper_2509_09424_b200.dist import ColumnShardedPCMM
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{_free_port()}", rank=0, world_size=1)
    try:
        o = oracle.Oracle(12, 3, 1, 3)
        ctx = Context(12, 3, 1, 3)
        d, m, level = 40, 70, 3
        x = synth.gen_words(71, o.q, d, level, o.n)
        W = synth.gen_W(72, d, m)
        xd = torch.from_numpy(x.view(np.int64)).cuda()
        sh = ColumnShardedPCMM(W, 1, 0, make_weights=ctx.weights)
        y_local = sh.local_buffer(torch, (2, level, o.n), "cuda")
        y_all = sh.gathered_buffer(torch, (2, level, o.n), "cuda")
        sh(lambda xa, wl, yl: ctx.pcmm_ternary(xa, wl, yl, level=level), xd, y_local, y_all)
        torch.cuda.synchronize()
        direct = torch.empty((m, 2, level, o.n), dtype=torch.int64, device="cuda")
        ctx.pcmm_ternary(xd, ctx.weights(W), direct, level=level)
        torch.cuda.synchronize()
        assert torch.equal(y_all[:m], direct)
        # chunked: the NCCL all-gather of chunk c overlaps the accumulate of chunk c + 1
        y_all.zero_()
        sh.run_overlapped(lambda xa, wl, yl: ctx.pcmm_ternary(xa, wl, yl, level=level), xd, y_local, y_all,
                          sh.chunk_weights(3, make_weights=ctx.weights))
        torch.cuda.synchronize()
        assert torch.equal(y_all[:m], direct)
        want = o.pcmm_a(x, W, cols=[0, 33, 69])
        assert (y_all[[0, 33, 69]].cpu().numpy().view(np.uint64) == want).all()
    finally:
        dist.destroy_process_group()


def test_column_sharded_compact_nccl_world1(torch_cuda):
    """The bench's N > 1 headline path on compact ciphertexts (uint8 [count][wire_bytes]): chunked column shards +
    NCCL all-gather == the unsharded compact call == the oracle on sampled columns."""
    torch = torch_cuda
    import torch.distributed as dist
    from paper_2509_09424_b200 import Context
    from paper_2509_09424_b200.dist import ColumnShardedPCMM
    from paper_2509_09424_b200.ensi import wire_pack_host, wire_unpack_host
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{_free_port()}", rank=0, world_size=1)
    try:
        o = oracle.Oracle(12, 3, 1, 3)
        ctx = Context(12, 3, 1, 3)
        d, m, level = 300, 7, 3
        x = synth.gen_words(73, o.q, d, level, o.n)
        W = synth.gen_W(74, d, m)
        wb = ctx.wire_bytes(level)
        xc = torch.from_numpy(wire_pack_host(x, ctx.wire_widths(level))).cuda()
        sh = ColumnShardedPCMM(W, 1, 0)
        y_local = sh.local_buffer(torch, (wb,), "cuda", dtype=torch.uint8)
        y_all = sh.gathered_buffer(torch, (wb,), "cuda", dtype=torch.uint8)
        y_all.zero_()
        sh.run_overlapped(lambda xa, wl, yl: ctx.pcmm_ternary_compact(xa, wl, yl, level=level), xc, y_local, y_all,
                          sh.chunk_weights(4, make_weights=ctx.weights))
        torch.cuda.synchronize()
        got = wire_unpack_host(y_all[:m].cpu().numpy(), ctx.wire_widths(level), level, o.n)
        assert (got == o.pcmm_a(x, W)).all()
    finally:
        dist.destroy_process_group()


@pytest.mark.slow
def test_bench_under_torchrun_nccl(torch_cuda):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "1", "--master-addr",
           "127.0.0.1", "--master-port", str(_free_port()), "bench.py", "--gpus", "1", "--steps", "3", "--warmup", "3",
           "--no-cpu", "--no-e2e", "--no-rot"]
    env = dict(os.environ, ENSI_BENCH_COLSHARD="1")          # run the column-sharded (all-gather) leg at N=1 too
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    line = [ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1]
    out = json.loads(line)
    assert out["n_gpus"] == 1 and out["value"] > 0 and out["gpu_launches"] >= 3
    assert out["roofline"]["frac"] > 0 and out["roofline"]["kernel"] == "k_accum_tcc"
    assert out["scaling"] == "strong" and out["config"]["parallelism"].startswith("output columns sharded x1")
    assert out["column_sharded"]["gather_ms"] > 0 and out["column_sharded"]["compute_ms"] > 0
    assert out["token_blocks"]["value"] > 0
