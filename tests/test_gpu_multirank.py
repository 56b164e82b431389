"""Two ranks on one GPU (gloo process group; the box has one GPU): each rank runs its
(batch x kv-head) unit shard through real OTTCache kernels — bulk prefill, decode steps
with the fused ring write and a flush, attention — and the head outputs are all-gathered
every step. The gathered [U, n_rep, d] outputs and the shard's quantization state must be
bit-identical to one process running all units (every unit is independent, cache.py:17-18,
SPEC.md:327-329). The ranks' kernels never wait on one another: the exchange is the
host-side gloo all-gather of the outputs."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

B, HKV, NREP, D, T_PRE, STEPS = 2, 4, 2, 128, 300, 40
G, R, N, A = 32, 32, 8, 16


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _data():
    rng = np.random.default_rng(11)
    U = B * HKV
    T = T_PRE + STEPS
    k = rng.standard_normal((U, T, D)).astype(np.float32)
    k[:, :, :4] *= 15.0
    k[:, 17, :4] *= 0.05
    k = k.astype(np.float16)
    v = rng.standard_normal((U, T, D)).astype(np.float16)
    q = rng.standard_normal((STEPS + 1, B, HKV * NREP, D)).astype(np.float16)
    return k, v, q


def _cfg():
    from paper_2505_10938_b200 import EngineConfig

    return EngineConfig(bits=2, group_size=G, residual=R, outlier_num=N, aux_capacity=A, skip_layers=(), head_dim=D)


def run_units(lo, hi, gather=None):
    """Units [lo, hi) as one OTTCache (one kv head per row); returns the (gathered) outputs
    of every step and the cache."""
    from paper_2505_10938_b200 import OTTCache
    from paper_2505_10938_b200.parallel import shard_queries

    k, v, q = _data()
    Ul = hi - lo
    dev = torch.device("cuda", 0)
    cache = OTTCache(_cfg(), Ul, 1, max_tokens=T_PRE + STEPS + 8, device=dev)
    full = OTTCache(_cfg(), B * HKV, 1, max_tokens=64, device=dev)  # split counts of the whole cache
    splits = full.splits(NREP)
    kd = torch.from_numpy(k[lo:hi, None]).to(dev)
    vd = torch.from_numpy(v[lo:hi, None]).to(dev)
    cache.update(kd[:, :, :T_PRE].contiguous(), vd[:, :, :T_PRE].contiguous())
    outs = []
    for t in range(STEPS + 1):
        qt = shard_queries(torch.from_numpy(q[t]).to(dev), HKV, lo, hi).contiguous()
        if t < STEPS:
            o = cache.append_attend(kd[:, :, T_PRE + t].contiguous(), vd[:, :, T_PRE + t].contiguous(), qt,
                                    n_splits=splits)
        else:
            o = cache.attend(qt, n_splits=splits)
        o = o.cpu()
        outs.append(gather(o) if gather is not None else o)
    return torch.stack(outs).numpy(), cache


def _worker(rank, world, port, path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2505_10938_b200.parallel import all_gather_heads, unit_bounds

        lo, hi = unit_bounds(B * HKV, world, rank)
        outs, cache = run_units(lo, hi, gather=lambda o: all_gather_heads(o))
        u = cache.unit(hi - lo - 1, 0)  # the shard's last unit
        np.savez(f"{path}_{rank}.npz", outs=outs, k_codes=np.array([bytes(b.codes) for b in u.quantized_k]),
                 pool=np.array([e.position for e in u.pool.entries]), unit=hi - 1)
    finally:
        dist.destroy_process_group()


def test_two_rank_unit_shards_match_one_process(tmp_path):
    world = 2
    path = str(tmp_path / "r")
    mp.start_processes(_worker, args=(world, _port(), path), nprocs=world, start_method="spawn", join=True)
    ref, cache = run_units(0, B * HKV)
    for r in range(world):
        got = np.load(f"{path}_{r}.npz")
        assert got["outs"].shape == ref.shape  # every rank holds the gathered [U, n_rep, d] of every step
        np.testing.assert_array_equal(got["outs"], ref)
        u = cache.unit(int(got["unit"]), 0)
        assert got["k_codes"].tolist() == [bytes(b.codes) for b in u.quantized_k]
        assert got["pool"].tolist() == [e.position for e in u.pool.entries]
    assert cache.quantized_tokens > (T_PRE - R) // G * G  # a decode flush ran inside the steps
