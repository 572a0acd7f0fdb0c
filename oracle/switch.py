"""Split / gather / dynamic switch over simulated ranks (TEST INFRASTRUCTURE ONLY).

P:93 (§3.1): "we propose to dynamically switch the dimension of sequence
parallelism according to the computation stage ... only a single AlltoAll
operation is required when transitioning between computation stages".
The switch is implemented as REAL per-pair message copies between simulated
ranks ("real message exchange ... so the ledger is a measurement"), not
as slicing of a global tensor.  Chunk -> rank map: rank r holds the r-th
contiguous chunk along the sharded axis (R11).  Self-sends are not
communication.  Axis numbering follows [B, T, S, C]: T = 1, S = 2.

split_nd / switch_nd: the same operations on an N-D activation [d0, ..., d_{k-1}, C]
(any number of sequence dims, channel last) -- P:93: "our method can generalize to all
multi-dimensional transformers beyond the demonstrated spatial-temporal transformer"
(e.g. [B, T, H, W, C] with attention along T, H and W separately).
"""
from __future__ import annotations

import dataclasses

import numpy as np

DIM_T, DIM_S = 1, 2
DIM_NAMES = {DIM_T: "T", DIM_S: "S"}


class DSPOracleError(ValueError):
    """Caller errors with the kinds SPEC lists."""


@dataclasses.dataclass
class LedgerEntry:
    rank: int
    kind: str            # "AllToAll" | "AllGather"
    tag: str             # stage label, e.g. "block0.switch_T2S"
    elements_sent: int
    elements_recv: int
    bytes_sent: int
    bytes_recv: int


class Ledger:
    """Per-rank record of every collective."""

    def __init__(self):
        self.entries: list[LedgerEntry] = []

    def record(self, *a):
        self.entries.append(LedgerEntry(*a))

    def sent(self, rank=None, kind=None, exclude_tags=("epilogue",)):
        return sum(e.elements_sent for e in self.entries
                   if (rank is None or e.rank == rank) and (kind is None or e.kind == kind)
                   and not any(x in e.tag for x in exclude_tags))

    def ops(self, rank, kind=None, exclude_tags=("epilogue",)):
        return sum(1 for e in self.entries
                   if e.rank == rank and (kind is None or e.kind == kind)
                   and not any(x in e.tag for x in exclude_tags))


def _check_dim(dim):
    if dim not in (DIM_T, DIM_S):
        raise DSPOracleError(f"bad dim {dim}: only T (1) and S (2) are sequence dims")


def _check_dim_nd(dim, ndim):
    if not (0 <= dim < ndim - 1):
        raise DSPOracleError(f"bad dim {dim}: the sharded / switched dims are 0..{ndim - 2} (the last is the channel)")


def split_nd(x: np.ndarray, dim: int, world: int) -> list:
    """N-D split: rank r takes chunk r of x along any non-channel dim."""
    _check_dim_nd(dim, x.ndim)
    return _split(x, dim, world)


def switch_nd(shards: list, from_dim: int, to_dim: int, ledger: Ledger | None = None,
              tag: str = "switch", elem_bytes: int = 2) -> list:
    """N-D dynamic switch between any two non-channel dims (see switch())."""
    _check_dim_nd(from_dim, shards[0].ndim)
    _check_dim_nd(to_dim, shards[0].ndim)
    return _switch(shards, from_dim, to_dim, ledger, tag, elem_bytes)


def split(x: np.ndarray, dim: int, world: int) -> list:
    """Rank r takes chunk r of x along dim."""
    _check_dim(dim)
    return _split(x, dim, world)


def _split(x: np.ndarray, dim: int, world: int) -> list:
    if x.shape[dim] % world:
        raise DSPOracleError(f"divisibility: N={world} does not divide extent {x.shape[dim]}")
    n = x.shape[dim] // world
    sl = [slice(None)] * x.ndim
    out = []
    for r in range(world):
        sl[dim] = slice(r * n, (r + 1) * n)
        out.append(np.array(x[tuple(sl)], copy=True))
    return out


def gather(shards: list, dim: int, ledger: Ledger | None = None, tag: str = "epilogue",
           elem_bytes: int = 2) -> np.ndarray:
    """Concatenate shards in rank order along dim; an AllGather."""
    _check_dim(dim)
    N = len(shards)
    if ledger is not None:
        for r, sh in enumerate(shards):
            e = (N - 1) * sh.size
            ledger.record(r, "AllGather", tag, e, e, e * elem_bytes, e * elem_bytes)
    return np.concatenate(shards, axis=dim)


def switch(shards: list, from_dim: int, to_dim: int, ledger: Ledger | None = None,
           tag: str = "switch", elem_bytes: int = 2) -> list:
    """Dynamic switch: re-shard from `from_dim` to `to_dim` with one all-to-all.

    Pre: shards[r] is chunk r of the global X along from_dim.  Rank r sends its
    to_dim chunk q to rank q (a copy = a message); rank q concatenates the N
    received pieces along from_dim in rank order.  Post: result[q] is chunk q of
    the same X along to_dim.
    """
    _check_dim(from_dim)
    _check_dim(to_dim)
    return _switch(shards, from_dim, to_dim, ledger, tag, elem_bytes)


def _switch(shards, from_dim, to_dim, ledger, tag, elem_bytes):
    if from_dim == to_dim:
        raise DSPOracleError("switching to the current axis (S:283)")
    N = len(shards)
    ext_to = shards[0].shape[to_dim]
    if ext_to % N:
        raise DSPOracleError(f"divisibility: N={N} does not divide extent {ext_to}")
    for sh in shards:
        if sh.shape != shards[0].shape:
            raise DSPOracleError("collective contract: shard shapes differ across ranks (S:149)")
    n = ext_to // N
    # outbox[r][q] = message from rank r to rank q
    outbox = []
    for r in range(N):
        row = []
        for q in range(N):
            sl = [slice(None)] * shards[r].ndim
            sl[to_dim] = slice(q * n, (q + 1) * n)
            row.append(np.array(shards[r][tuple(sl)], copy=True))
        outbox.append(row)
    result = []
    for q in range(N):
        inbox = [outbox[r][q] for r in range(N)]
        result.append(np.concatenate(inbox, axis=from_dim))
    if ledger is not None:
        for r in range(N):
            sent = sum(outbox[r][q].size for q in range(N) if q != r)
            recv = sum(outbox[q][r].size for q in range(N) if q != r)
            ledger.record(r, "AllToAll", tag, sent, recv, sent * elem_bytes, recv * elem_bytes)
    return result
