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
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "1", "--master-addr",
           "127.0.0.1", "--master-port", str(_free_port()), "bench.py", "--gpus", "1", "--steps", "3", "--warmup", "3",
           "--no-cpu", "--no-e2e", "--no-rot", "--jsonl", os.path.join(ROOT, "gpurun_out", "bench_test.jsonl")]
    env = dict(os.environ, ENSI_BENCH_COLSHARD="1")          # run the column-sharded (all-gather) leg at N=1 too
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    line = [ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1]
    out = json.loads(line)
    assert out["n_gpus"] == 1 and out["value"] > 0 and out["gpu_launches"] >= 3
    assert out["roofline"]["frac"] > 0 and out["roofline"]["kernel"] == "k_accum_tcc"
    assert out["scaling"] == "strong" and out["config"]["parallelism"].startswith("output columns sharded x1")
    assert out["column_sharded"]["gather_ms"] > 0 and out["column_sharded"]["compute_ms"] > 0
    assert out["column_sharded"]["fused_gather_ms"] > 0
    assert out["token_blocks"]["value"] > 0
    recs = [json.loads(ln) for ln in open(os.path.join(ROOT, "gpurun_out", "bench_test.jsonl"))]
    assert recs[0]["kernel"] == "k_accum_tcc" and recs[0]["bit_exact_vs_other_kernels"] is True


def _c1_compact(torch, seed, d, m, level=3):
    from paper_2509_09424_b200 import Context
    from paper_2509_09424_b200.ensi import wire_pack_host
    o = oracle.Oracle(12, 3, 1, 3)
    ctx = Context(12, 3, 1, 3)
    x = synth.gen_words(seed, o.q, d, level, o.n)
    W = synth.gen_W(seed + 1, d, m)
    xc = torch.from_numpy(wire_pack_host(x, ctx.wire_widths(level))).cuda()
    return o, ctx, x, W, xc


def test_fused_gather_epilogue_multi_destination(torch_cuda):
    """SURVEY 8(f) NEXT #4 (fused gather epilogue), on one GPU: ensi_pcmm_ternary_compact_gather with two destination
    buffers (standing in for two GPUs' gathered buffers) -- rows [row0, row0 + m) of BOTH hold the oracle's outputs,
    every other row is untouched; row0 + m > rows_total is EDIM."""
    torch = torch_cuda
    from paper_2509_09424_b200.ensi import EnsiError, ENSI_EDIM, wire_unpack_host
    d, m, level, rows_total, row0 = 70, 50, 3, 130, 37
    o, ctx, x, W, xc = _c1_compact(torch, 81, d, m, level)
    wb = ctx.wire_bytes(level)
    bufs = [torch.full((rows_total, wb), 0xA5, dtype=torch.uint8, device="cuda") for _ in range(2)]
    w = ctx.weights(W)
    ctx.pcmm_ternary_compact_gather(xc, w, bufs, rows_total, row0, level)
    torch.cuda.synchronize()
    want = o.pcmm_a(x, W)
    for b in bufs:
        h = b.cpu().numpy()
        assert (wire_unpack_host(h[row0:row0 + m], ctx.wire_widths(level), level, o.n) == want).all()
        assert (h[:row0] == 0xA5).all() and (h[row0 + m:] == 0xA5).all()
    with pytest.raises(EnsiError) as e:
        ctx.pcmm_ternary_compact_gather(xc, w, bufs, rows_total, rows_total - m + 1, level)
    assert e.value.code == ENSI_EDIM


def test_fused_gather_world1(torch_cuda):
    """FusedGatherPCMM at world size 1 (self-peer): the gathered buffer == the oracle's layer, twice (epochs 1, 2:
    the signal / wait kernels order consecutive layers)."""
    torch = torch_cuda
    from paper_2509_09424_b200.dist import FusedGatherPCMM
    from paper_2509_09424_b200.ensi import wire_unpack_host
    d, m, level = 40, 33, 3
    o, ctx, x, W, xc = _c1_compact(torch, 91, d, m, level)
    fg = FusedGatherPCMM(ctx, W, 1, 0, level)
    want = o.pcmm_a(x, W)
    for it in range(2):
        fg.y_all.zero_()
        y = fg(xc)
        torch.cuda.synchronize()
        assert (wire_unpack_host(y[:m].cpu().numpy(), ctx.wire_widths(level), level, o.n) == want).all()
        assert int(fg.flags[0]) == it + 1
    fg.close()


_CHILD = r"""
import sys
sys.path.insert(0, sys.argv[1])
import numpy as np, torch
import synth
from paper_2509_09424_b200 import Context
from paper_2509_09424_b200.ensi import wire_pack_host
hy, hf, rows_total, row0 = bytes.fromhex(sys.argv[2]), bytes.fromhex(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5])
ctx = Context(12, 3, 1, 3)
x = synth.gen_words(101, ctx.q, 30, 3, ctx.n)
W = synth.gen_W(102, 30, 20)
xc = torch.from_numpy(wire_pack_host(x, ctx.wire_widths(3))).cuda()
py, pf = ctx.ipc_open(hy), ctx.ipc_open(hf)
ctx.pcmm_ternary_compact_gather(xc, ctx.weights(W), [py], rows_total, row0, 3)
ctx.peer_signal([pf], 1, 7)
torch.cuda.synchronize()
ctx.ipc_close(py)
ctx.ipc_close(pf)
print("child ok")
"""


def test_fused_gather_through_cuda_ipc_from_another_process(torch_cuda):
    """The IPC leg of FusedGatherPCMM: a second process maps this process's gathered buffer and flag array
    (ensi_ipc_get_handle / ensi_ipc_open, offsets inside torch's allocations), its accumulate epilogue stores its
    output rows into them and it signals slot 1; after it exits the rows == the oracle and the flag == 7.  No kernel
    of one process waits on the other (the wait is the host-side join)."""
    torch = torch_cuda
    from paper_2509_09424_b200 import Context
    from paper_2509_09424_b200.ensi import wire_unpack_host
    ctx = Context(12, 3, 1, 3)
    o = oracle.Oracle(12, 3, 1, 3)
    wb = ctx.wire_bytes(3)
    rows_total, row0, m = 48, 24, 20
    pad = torch.zeros(1000, dtype=torch.uint8, device="cuda")      # non-zero offsets inside the caching allocator
    y_all = torch.full((rows_total, wb), 0x5A, dtype=torch.uint8, device="cuda")
    flags = torch.zeros(2, dtype=torch.int32, device="cuda")
    torch.cuda.synchronize()
    hy, hf = ctx.ipc_handle(y_all), ctx.ipc_handle(flags)
    r = subprocess.run([sys.executable, "-c", _CHILD, ROOT, hy.hex(), hf.hex(), str(rows_total), str(row0)],
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "child ok" in r.stdout, r.stderr[-2000:]
    torch.cuda.synchronize()
    x = synth.gen_words(101, o.q, 30, 3, o.n)
    W = synth.gen_W(102, 30, 20)
    h = y_all.cpu().numpy()
    assert (wire_unpack_host(h[row0:row0 + m], ctx.wire_widths(3), 3, o.n) == o.pcmm_a(x, W)).all()
    assert (h[:row0] == 0x5A).all() and (h[row0 + m:] == 0x5A).all()
    assert int(flags[1]) == 7 and int(flags[0]) == 0
    del pad


def test_fused_gather_error_paths(torch_cuda):
    """ensi_pcmm_ternary_compact_gather / ensi_ipc_* / ensi_peer_* validate before touching the device: too many or
    NULL destinations, a destination aliasing x, an unknown pointer for ipc_close, flag counts out of range."""
    torch = torch_cuda
    from paper_2509_09424_b200.ensi import EnsiError, ENSI_EINVAL
    o, ctx, x, W, xc = _c1_compact(torch, 93, 8, 4)
    w = ctx.weights(W)
    wb = ctx.wire_bytes(3)
    buf = torch.zeros((8, wb), dtype=torch.uint8, device="cuda")
    for dsts in ([buf] * 9, [0]):
        with pytest.raises(EnsiError) as e:
            ctx.pcmm_ternary_compact_gather(xc, w, dsts, 8, 0, 3)
        assert e.value.code == ENSI_EINVAL
    with pytest.raises(EnsiError) as e:                          # the destination is x itself
        ctx.pcmm_ternary_compact_gather(xc, w, [xc.data_ptr()], 8, 0, 3)
    assert e.value.code == ENSI_EINVAL
    with pytest.raises(EnsiError) as e:
        ctx.ipc_close(buf.data_ptr())
    assert e.value.code == ENSI_EINVAL
    flags = torch.zeros(4, dtype=torch.int32, device="cuda")
    with pytest.raises(EnsiError) as e:
        ctx.peer_signal([flags] * 9, 0, 1)
    assert e.value.code == ENSI_EINVAL
    with pytest.raises(EnsiError) as e:
        ctx.peer_wait(flags, 0, 1)
    assert e.value.code == ENSI_EINVAL
    ctx.peer_signal([flags], 2, 5)                              # a valid signal / wait pair on one GPU
    flags[0] = 5
    flags[1] = 5
    flags[3] = 5
    ctx.peer_wait(flags, 4, 5)
    torch.cuda.synchronize()
    assert flags.tolist() == [5, 5, 5, 5]
