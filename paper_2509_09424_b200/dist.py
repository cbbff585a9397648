"""Multi-GPU driver for the ternary PCMM.

One process per GPU, `torch.distributed` over NCCL.  Two shardings:

* Token blocks (no collective): a layer whose activation spans several ciphertext "token blocks" (more tokens
  than N'/2 slots, or several sequences) is a set of independent problems -- each rank runs Algorithm 1 on its
  own blocks with the same W.  `token_blocks(n_blocks, world, rank)` gives the contiguous block range.
* Output columns (the north star's layout): inputs X~ replicated, rank r owns output columns
  [r*S, (r+1)*S) with S = ceil(m / world) (the last shard zero-padded), computes them with its slice of W,
  and one `all_gather_into_tensor` over NCCL assembles the m output ciphertexts on every rank.

* Output columns with the gather fused into the accumulate: `FusedGatherPCMM` maps every
  rank's gathered buffer into every other rank through CUDA IPC; the compact accumulate's epilogue TMA-stores each
  output tile into all of them (ensi_pcmm_ternary_compact_gather), and a signal / wait pair of tiny kernels orders
  the writes -- no separate collective launch, the transfer overlaps the accumulate tile by tile.

CCMM (R18) shards the same way by output columns: `ccmm_shard` gives a rank's (col0, cols).

The compute step is a callable `pcmm(x, W_slice, y_local)`; the product passes the CUDA path
(`Context.pcmm_ternary`), the CPU tests pass a reference to exercise the shard/gather logic with `gloo`.
"""
from __future__ import annotations

from typing import Callable

import numpy as np


def token_blocks(n_blocks: int, world: int, rank: int) -> range:
    """Contiguous, balanced split of n_blocks independent token blocks."""
    base, extra = divmod(n_blocks, world)
    lo = rank * base + min(rank, extra)
    return range(lo, lo + base + (1 if rank < extra else 0))


def column_shard(m: int, world: int, rank: int):
    """(lo, hi, S): rank owns output columns [lo, hi) of an m-column layer; S = ceil(m/world) is the padded shard."""
    S = -(-m // world)
    lo = min(m, rank * S)
    hi = min(m, lo + S)
    return lo, hi, S


def ccmm_shard(m: int, world: int, rank: int):
    """(col0, cols) for `Context.ccmm(..., col0=, cols=)`: CCMM output columns are independent (R18), so a
    rank computes its contiguous column range from the replicated inputs with no data-path collective (weak
    scaling); gathering the columns, if a consumer needs all of them, is the same all-gather as the PCMM's."""
    lo, hi, _ = column_shard(m, world, rank)
    return lo, hi - lo


class ColumnShardedPCMM:
    """y = X (x) W with W's output columns sharded across ranks, then one all-gather of the result ciphertexts."""

    def __init__(self, W: np.ndarray, world: int, rank: int, make_weights: Callable = None):
        self.d, self.m = W.shape
        self.world, self.rank = world, rank
        self.lo, self.hi, self.S = column_shard(self.m, world, rank)
        Ws = np.zeros((self.d, self.S), np.int8)       # zero columns pad the last shard (outputs are (0,0))
        Ws[:, : self.hi - self.lo] = W[:, self.lo:self.hi]
        self._W_np = Ws
        self.W_local = make_weights(Ws) if make_weights else Ws

    def local_buffer(self, torch, ct_shape, device, dtype=None):
        """[S] + ct_shape: uint64 words as int64 (ct_shape (2, l, N')) or compact bytes as uint8 ((wire_bytes,))."""
        return torch.empty((self.S,) + tuple(ct_shape), dtype=dtype or torch.int64, device=device)

    def gathered_buffer(self, torch, ct_shape, device, dtype=None):
        return torch.empty((self.S * self.world,) + tuple(ct_shape), dtype=dtype or torch.int64, device=device)

    def chunk_bounds(self, chunks: int):
        """Contiguous, balanced split of this rank's S output columns into `chunks` pieces."""
        return [(c * self.S // chunks, (c + 1) * self.S // chunks) for c in range(chunks)]

    def chunk_weights(self, chunks: int, make_weights: Callable = None):
        """Per-chunk column slices of the local weights (a model constant: build once, reuse every call)."""
        Wl = self._W_np
        return [make_weights(np.ascontiguousarray(Wl[:, a:b])) if make_weights else np.ascontiguousarray(Wl[:, a:b])
                for a, b in self.chunk_bounds(chunks)]

    def run_overlapped(self, pcmm: Callable, x, y_local, y_all, w_chunks, group=None):
        """Chunked variant: the all-gather of output chunk c runs asynchronously (NCCL's own stream
        waits for the compute stream at issue time) while chunk c + 1 is computed; returns after every gather
        has completed.  w_chunks: from chunk_weights()."""
        import torch.distributed as dist
        works = []
        for (a, b), wc in zip(self.chunk_bounds(len(w_chunks)), w_chunks):
            if b == a:
                continue
            pcmm(x, wc, y_local[a:b])
            outs = [y_all[r * self.S + a: r * self.S + b] for r in range(self.world)]
            works.append(dist.all_gather(outs, y_local[a:b], group=group, async_op=True))
        for wk in works:
            wk.wait()

    def __call__(self, pcmm: Callable, x, y_local, y_all=None, group=None, async_op: bool = False):
        """Run this rank's shard into y_local [S][2][l][N'], then all-gather into y_all [S*world][...]
        (rows >= m are padding).  Returns the collective work handle when async_op."""
        pcmm(x, self.W_local, y_local)
        if y_all is None:
            return None
        import torch.distributed as dist
        return dist.all_gather_into_tensor(y_all, y_local, group=group, async_op=async_op)


class FusedGatherPCMM:
    """One column-sharded layer on compact ciphertexts with the all-gather fused into the accumulate epilogue.

    Rank r computes output columns [r S, (r + 1) S) and its epilogue stores them at rows [r S, (r + 1) S) of EVERY
    rank's gathered buffer y_all [S world][wire_bytes] (its own, and the peers' mapped through CUDA IPC); then it
    publishes `epoch` in slot r of every rank's flag array and waits until its own array holds `epoch` in all slots.
    After __call__ returns (stream-ordered), y_all holds all m outputs (rows >= m: padding columns, (0, 0)).

    ctx: a Context (or any object with its wire_bytes / weights / ipc_handle / ipc_open / ipc_close /
    pcmm_ternary_compact_gather / peer_signal / peer_wait methods -- the CPU tests pass a stand-in); alloc(shape,
    dtype_name) allocates the gathered buffer ("uint8") and the flag array ("int32") on this rank's GPU."""

    def __init__(self, ctx, W: np.ndarray, world: int, rank: int, level: int, alloc: Callable = None, group=None):
        self.ctx, self.world, self.rank, self.level = ctx, world, rank, level
        self.d, self.m = W.shape
        self.lo, self.hi, self.S = column_shard(self.m, world, rank)
        Ws = np.zeros((self.d, self.S), np.int8)
        Ws[:, : self.hi - self.lo] = W[:, self.lo:self.hi]
        self.w_local = ctx.weights(Ws)
        self.wb = ctx.wire_bytes(level)
        if alloc is None:
            import torch

            def alloc(shape, dt):
                return torch.zeros(shape, dtype=getattr(torch, dt), device="cuda")
        # Collectively consistent setup: every rank reaches both exchanges even when a local step fails, and all ranks
        # raise together (a rank left behind would otherwise hang its peers in the exchange or in peer_wait).
        err = None
        try:
            self.y_all = alloc((self.S * world, self.wb), "uint8")
            self.flags = alloc((world,), "int32")
            mine = (ctx.ipc_handle(self.y_all), ctx.ipc_handle(self.flags))
        except Exception as e:  # noqa: BLE001 -- reported to every rank below
            mine, err = None, f"rank {rank}: {e!r}"
        handles = self._exchange((err, mine), group)
        errs = [h[0] for h in handles if h[0]]
        if errs:
            raise RuntimeError("fused gather setup failed: " + "; ".join(errs))
        self._opened = []
        self.dst, self.flag_dst = [], []
        try:
            for r in range(world):
                if r == rank:
                    self.dst.append(self.y_all)
                    self.flag_dst.append(self.flags)
                else:
                    py = ctx.ipc_open(handles[r][1][0])
                    self._opened.append(py)
                    pf = ctx.ipc_open(handles[r][1][1])
                    self._opened.append(pf)
                    self.dst.append(py)
                    self.flag_dst.append(pf)
            err = None
        except Exception as e:  # noqa: BLE001
            err = f"rank {rank}: {e!r}"
        errs = [e for e in self._exchange(err, group) if e]
        if errs:
            self.close()
            raise RuntimeError("fused gather peer mapping failed: " + "; ".join(errs))
        self.epoch = 0

    def _exchange(self, obj, group):
        if self.world == 1:
            return [obj]
        import torch.distributed as dist
        out = [None] * self.world
        dist.all_gather_object(out, obj, group=group)
        return out

    def __call__(self, x, stream=None):
        self.ctx.pcmm_ternary_compact_gather(x, self.w_local, self.dst, self.S * self.world, self.rank * self.S,
                                             self.level, stream=stream)
        self.epoch = (self.epoch + 1) & 0x7FFFFFFF
        self.ctx.peer_signal(self.flag_dst, self.rank, self.epoch, stream=stream)
        self.ctx.peer_wait(self.flags, self.world, self.epoch, stream=stream)
        return self.y_all

    def close(self):
        for p in self._opened:
            self.ctx.ipc_close(p)
        self._opened = []
