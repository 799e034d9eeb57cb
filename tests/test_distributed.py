"""CPU, world_size 2 over gloo: the host side of the multi-GPU path.

Super-chunk partials of a small plain sum (computed here by the CPU oracle,
standing in for lq_lattice_partials) are produced by two ranks for their own
shards, exchanged with distributed.exchange_disjoint, and must equal the
single-process vector bit for bit -- the property that makes the GPU result
independent of the GPU count."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2404_08867_b200.distributed import exchange_disjoint, shard_range

SUPER = 1 << 10          # points per super-chunk in this scaled-down test


def _partials(n, z, coef, lo, hi):
    from oracle import np_oracle as orc
    out = np.zeros(hi - lo)
    for s in range(lo, hi):
        a, b = s * SUPER, min((s + 1) * SUPER, n)
        pts = orc.points_block(n, z, a, b)
        out[s - lo] = float(np.sum(np.exp(-np.abs(pts @ coef - 0.3))))
    return out


def _block(a):
    # k_reduce1024 + block_sum order (lq_kernels.cu, lq_device.cuh): 4-way fold
    # per thread, xor-butterfly per warp, butterfly over the 8 warp sums
    s = [(a[4 * t] + a[4 * t + 1]) + (a[4 * t + 2] + a[4 * t + 3]) for t in range(256)]
    warps = []
    for w in range(8):
        v = s[32 * w:32 * w + 32]
        for o in (16, 8, 4, 2, 1):
            v = [v[l] + v[l ^ o] for l in range(32)]
        warps.append(v[0])
    v = warps + [0.0] * 24
    for o in (4, 2, 1):
        v = [v[l] + v[l ^ o] for l in range(32)]
    return v[0]


def _tree(v):
    v = [float(x) for x in v]
    while True:
        v = v + [0.0] * ((-len(v)) % 1024)
        v = [_block(v[g:g + 1024]) for g in range(0, len(v), 1024)]
        if len(v) == 1:
            return v[0]


def _worker(rank, size, port, n, z, coef, S, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=size)
    lo, hi = shard_range(S, rank, size)
    vec = torch.zeros(S, dtype=torch.float64)
    vec[lo:hi] = torch.from_numpy(_partials(n, z, coef, lo, hi))
    exchange_disjoint(vec)
    out_q.put((rank, vec.numpy().tobytes()))
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_shard_ranges_partition():
    for S in (1, 7, 512, 1000):
        for size in (1, 2, 3, 4, 8):
            spans = [shard_range(S, r, size) for r in range(size)]
            assert spans[0][0] == 0 and spans[-1][1] == S
            assert all(spans[i][1] == spans[i + 1][0] for i in range(size - 1))


def test_two_rank_exchange_is_bit_identical_to_one_rank():
    n, d = 40009, 5
    z = [pow(7919, j, n) for j in range(d)]
    coef = np.array([0.3, -0.2, 0.5, 0.1, 0.25])
    S = -(-n // SUPER)
    single = _partials(n, z, coef, 0, S)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n, z, coef, S, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=120) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(2):
        vec = np.frombuffer(got[r], dtype=np.float64)
        assert np.array_equal(vec.view(np.uint64), single.view(np.uint64))
        assert _tree(vec) == _tree(single)
