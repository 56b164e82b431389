"""Multi-process (gloo, world_size 2, CPU) check of the batch x kv-head
partitioning and the head-output all-gather: sharded decode == unsharded."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2505_10938_b200.parallel import all_gather_heads, shard_bounds


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _workload(B, Hkv, n_rep, T, d, seed=0):
    rng = np.random.default_rng(seed)
    k = rng.standard_normal((B, Hkv, T, d)).astype(np.float16).astype(np.float32)
    k[..., :2] *= 15
    v = rng.standard_normal((B, Hkv, T, d)).astype(np.float16).astype(np.float32)
    q = rng.standard_normal((B, Hkv * n_rep, d)).astype(np.float16).astype(np.float32)
    return k, v, q


def _decode(k, v, q, n_rep):
    """Per-unit oracle decode (stands in for the per-rank GPU cache on CPU)."""
    B, Hkv, T, d = k.shape
    out = np.empty((B, Hkv * n_rep, d), np.float32)
    for b in range(B):
        for h in range(Hkv):
            c = oracle.OracleCache(2, 32, 16, 3, 8, d)
            c.extend(k[b, h], v[b, h])
            for r in range(n_rep):
                out[b, h * n_rep + r] = c.attend(q[b, h * n_rep + r])
    return out


def _worker(rank, world, port, result_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        B, Hkv, n_rep, T, d = 4, 2, 2, 100, 16
        k, v, q = _workload(B, Hkv, n_rep, T, d)
        lo, hi = shard_bounds(B, world, rank)
        local = torch.from_numpy(_decode(k[lo:hi], v[lo:hi], q[lo:hi], n_rep))
        full = all_gather_heads(local)
        if rank == 0:
            np.save(result_path, full.numpy())
    finally:
        dist.destroy_process_group()


def test_shard_bounds():
    assert [shard_bounds(128, 8, r) for r in (0, 7)] == [(0, 16), (112, 128)]
    assert shard_bounds(8, 1, 0) == (0, 8)
    with pytest.raises(ValueError):
        shard_bounds(10, 4, 0)


def test_two_rank_gloo_matches_single_process(tmp_path):
    world = 2
    path = str(tmp_path / "out.npy")
    mp.start_processes(_worker, args=(world, _free_port(), path), nprocs=world, start_method="spawn", join=True)
    full = np.load(path)
    k, v, q = _workload(4, 2, 2, 100, 16)
    ref = _decode(k, v, q, 2)
    np.testing.assert_array_equal(full, ref)


@pytest.mark.parametrize("world", [2, 4, 8])
def test_peer_destinations_assemble_the_all_gather(world):
    """PeerGather's address arithmetic: if every rank stores its rows at
    peer_destinations(...) in each peer's buffer (what the combine kernel does over
    NVLink) and at out(l) locally, every rank's buffer equals the all-gather."""
    from paper_2505_10938_b200.parallel import gather_row_offset, peer_destinations

    L, b_local, hq, d = 3, 2, 4, 8
    row_bytes = hq * d * 2
    size = 2 * L * b_local * world * row_bytes  # two step slots
    bases = [(p + 1) << 32 for p in range(world)]  # distinct fake device addresses
    mem = [np.zeros(size, np.uint8) for _ in range(world)]
    rng = np.random.default_rng(world)
    outs = rng.integers(0, 256, (2, world, L, b_local * row_bytes), dtype=np.uint8)
    for slot in range(2):
        for r in range(world):
            for l in range(L):
                local = gather_row_offset(l, r, b_local, world, hq, d, slot, L)
                mem[r][local:local + b_local * row_bytes] = outs[slot, r, l]
                dests = peer_destinations(bases, r, l, b_local, hq, d, slot, L)
                assert len(dests) == world - 1
                for a in dests:
                    p = (a >> 32) - 1
                    assert p != r
                    off = a - bases[p]
                    assert off == local
                    mem[p][off:off + b_local * row_bytes] = outs[slot, r, l]
    want = np.concatenate([outs[s, :, l].reshape(-1) for s in range(2) for l in range(L)])
    for p in range(world):
        np.testing.assert_array_equal(mem[p], want)
