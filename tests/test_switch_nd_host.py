"""The C ABI's N-D switch plan (dsp_switch_nd_plan, the host logic both GPU transports execute)
executed on the host against the oracle's N-D switch: bit-exact for every ordered pair of
non-channel dims, N = 1, 2, 4, 8, and both transports' byte orders (P2P: runs stored at
dst_peer_off + destination strides; NCCL: pack to [peer][outer][rows][middle] chunks, exchange,
unpack) -- plus world-size-2 gloo with a real all_to_all."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import switch as osw


def _runs(plan):
    n = list(plan.n)
    for q in range(n[0]):
        for o in range(n[1]):
            for i in range(n[2]):
                for mid in range(n[3]):
                    yield q, o, i, mid


def _p2p_exec(m, dims, eb, N, shards, a, b):
    """Every rank r stores each run at r's dst_peer_off + destination strides in peer q's y."""
    ys = [np.zeros(shards[0].nbytes if a != b else 0, dtype=np.uint8) for _ in range(N)]
    for r in range(N):
        plan = m.switch_nd_plan(dims, eb, N, r, a, b)
        xb = shards[r].view(np.uint8).reshape(-1)
        R = plan.run_bytes
        for q, o, i, mid in _runs(plan):
            s = q * plan.src_stride[0] + o * plan.src_stride[1] + i * plan.src_stride[2] + mid * plan.src_stride[3]
            d = plan.dst_peer_off + o * plan.dst_stride[1] + i * plan.dst_stride[2] + mid * plan.dst_stride[3]
            ys[q][d:d + R] = xb[s:s + R]
    return ys


def _nccl_exec_rank(plan, N, xb, exchange):
    n = list(plan.n)
    R = plan.run_bytes
    chunk = n[1] * n[2] * n[3] * R
    send = np.empty(N * chunk, dtype=np.uint8)
    for q, o, i, mid in _runs(plan):
        s = q * plan.src_stride[0] + o * plan.src_stride[1] + i * plan.src_stride[2] + mid * plan.src_stride[3]
        d = q * chunk + ((o * n[2] + i) * n[3] + mid) * R
        send[d:d + R] = xb[s:s + R]
    recv = exchange(send, chunk)
    y = np.empty(xb.size, dtype=np.uint8)
    for src, o, i, mid in _runs(plan):
        s = src * chunk + ((o * n[2] + i) * n[3] + mid) * R
        d = src * plan.dst_stride[0] + o * plan.dst_stride[1] + i * plan.dst_stride[2] + mid * plan.dst_stride[3]
        y[d:d + R] = recv[s:s + R]
    if plan.pack_is_identity:
        assert np.array_equal(send, xb)
    if plan.unpack_is_identity:
        assert np.array_equal(y, recv)
    return y


@pytest.mark.parametrize("dims", [(2, 4, 8, 4, 8), (1, 8, 4, 2, 4, 16), (4, 8, 8, 8)])
@pytest.mark.parametrize("N", [1, 2, 4, 8])
def test_switch_nd_plan_vs_oracle_all_pairs(dims, N):
    import paper_2403_10266_b200 as m
    g = (np.arange(int(np.prod(dims)), dtype=np.int64) * 2654435761 % 65521).astype(np.int16).reshape(dims)
    nd = len(dims)
    for a in range(nd - 1):
        for b in range(nd - 1):
            if a == b or dims[a] % N or dims[b] % N:
                continue
            shards = osw.split_nd(g, a, N)
            want = osw.switch_nd(shards, a, b)
            ys = _p2p_exec(m, dims, 2, N, shards, a, b)
            for q in range(N):
                assert np.array_equal(ys[q].view(np.int16).reshape(want[q].shape), want[q]), ("p2p", a, b, q)
            # NCCL order: all ranks' sends exchanged in memory
            plans = [m.switch_nd_plan(dims, 2, N, r, a, b) for r in range(N)]
            packed = []
            for r in range(N):
                n = list(plans[r].n)
                R = plans[r].run_bytes
                chunk = n[1] * n[2] * n[3] * R
                xb = shards[r].view(np.uint8).reshape(-1)
                send = np.empty(N * chunk, dtype=np.uint8)
                for q, o, i, mid in _runs(plans[r]):
                    s = (q * plans[r].src_stride[0] + o * plans[r].src_stride[1] + i * plans[r].src_stride[2]
                         + mid * plans[r].src_stride[3])
                    d = q * chunk + ((o * n[2] + i) * n[3] + mid) * R
                    send[d:d + R] = xb[s:s + R]
                packed.append((send, chunk))
            for q in range(N):
                recv = np.concatenate([packed[r][0][q * packed[r][1]:(q + 1) * packed[r][1]] for r in range(N)])
                y = _nccl_exec_rank(plans[q], N, shards[q].view(np.uint8).reshape(-1), lambda s_, c_: recv)
                assert np.array_equal(y.view(np.int16).reshape(want[q].shape), want[q]), ("nccl", a, b, q)


def test_switch_nd_plan_errors():
    import paper_2403_10266_b200 as m
    with pytest.raises(m.DSPError, match="SAME_DIM"):
        m.switch_nd_plan((2, 4, 4, 8), 2, 2, 0, 1, 1)
    with pytest.raises(m.DSPError, match="BAD_DIM"):
        m.switch_nd_plan((2, 4, 4, 8), 2, 2, 0, 1, 3)        # the channel dim
    with pytest.raises(m.DSPError, match="DIVISIBILITY"):
        m.switch_nd_plan((2, 6, 4, 8), 2, 4, 0, 1, 2)
    with pytest.raises(m.DSPError, match="ALIGNMENT"):
        m.switch_nd_plan((2, 4, 4, 3), 2, 2, 0, 1, 2)        # runs of 2*3*2 = 12 bytes
    with pytest.raises(m.DSPError, match="SHAPE"):
        m.switch_nd_plan((4, 8), 2, 2, 0, 0, 1)              # ndim < 3


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    try:
        import sys
        sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        import paper_2403_10266_b200 as m
        from oracle import switch as osw2
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        dims = (2, 4, 8, 4, 8)
        g = (np.arange(int(np.prod(dims)), dtype=np.int64) * 40503 % 65521).astype(np.int16).reshape(dims)
        ok = True
        for a, b in [(1, 3), (3, 2), (2, 1), (0, 3)]:
            mine = osw2.split_nd(g, a, world)[rank]
            want = osw2.switch_nd(osw2.split_nd(g, a, world), a, b)[rank]

            def ex(send, chunk):
                recv = torch.empty(send.size, dtype=torch.uint8)
                dist.all_to_all_single(recv, torch.from_numpy(send))
                return recv.numpy()
            plan = m.switch_nd_plan(dims, 2, world, rank, a, b)
            y = _nccl_exec_rank(plan, world, mine.view(np.uint8).reshape(-1), ex)
            ok = ok and np.array_equal(y.view(np.int16).reshape(want.shape), want)
        q.put((rank, ok))
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover
        q.put((rank, repr(e)))


def test_switch_nd_world2_gloo():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for r in res:
        assert r[1] is True, r
