"""The head-output all-gather fused into the attention epilogue (SURVEY §8e,
parallel.PeerGather). One GPU is available per run, so the peer stores are checked
with local stand-ins for the peer buffers: every kernel family's combine must write
the identical output rows to `out` and to each ott_cache_t.out_peer address, and the
outputs must not change. The symmetric-memory plumbing runs at world size 1."""

import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)


def _cfg(bits, G, R, N, A, d):
    from paper_2505_10938_b200 import EngineConfig

    return EngineConfig(bits=bits, group_size=G, residual=R, outlier_num=N, aux_capacity=A, skip_layers=(),
                        head_dim=d)


@pytest.mark.parametrize("bits,G,d,n_rep", [(2, 32, 128, 8), (4, 32, 128, 4), (8, 32, 128, 2), (3, 32, 128, 4),
                                            (2, 32, 64, 1), (2, 16, 48, 2)])
def test_combine_stores_every_peer_copy(bits, G, d, n_rep):
    from paper_2505_10938_b200 import OTTCache

    B, Hkv, R = 4, 2, 16
    T0, steps = 4 * G + R + 5, G + 3
    rng = np.random.default_rng(bits * 100 + d)
    k = torch.from_numpy(rng.standard_normal((B, Hkv, T0 + steps, d)).astype(np.float16)).cuda()
    v = torch.from_numpy(rng.standard_normal((B, Hkv, T0 + steps, d)).astype(np.float16)).cuda()
    q = torch.from_numpy(rng.standard_normal((steps + 1, B, Hkv * n_rep, d)).astype(np.float16)).cuda()
    caches = [OTTCache(_cfg(bits, G, R, 4, 8, d), B, Hkv, max_tokens=T0 + steps) for _ in range(2)]
    for c in caches:
        c.update(k[:, :, :T0].contiguous(), v[:, :, :T0].contiguous())
    # three stand-in peers: this rank's slice (rank 1 of 4) inside [4*B, H_q, d] buffers
    peers = [torch.full((4 * B, Hkv * n_rep, d), float("nan"), dtype=torch.float16, device="cuda")
             for _ in range(3)]
    caches[1].set_output_peers([p[B:2 * B].data_ptr() for p in peers])
    outs = [torch.empty((B, Hkv * n_rep, d), dtype=torch.float16, device="cuda") for _ in range(2)]

    def check(tag):
        torch.cuda.synchronize()
        assert torch.equal(outs[0], outs[1]), tag
        for i, p in enumerate(peers):
            assert torch.equal(p[B:2 * B], outs[1]), (tag, i)
            assert torch.isnan(p[:B]).all() and torch.isnan(p[2 * B:]).all(), (tag, i)  # nothing else touched

    for c, o in zip(caches, outs):
        c.attend(q[0], out=o)
    check("attend")
    for t in range(steps // 2):
        for c, o in zip(caches, outs):
            c.append_attend(k[:, :, T0 + t].contiguous(), v[:, :, T0 + t].contiguous(), q[t + 1], out=o)
        check(f"append_attend {t}")
    for c in caches:
        c.sync_counters()
    s = caches[0].splits(n_rep)
    for t in range(steps // 2, steps):
        for c, o in zip(caches, outs):
            c.decode_step(k[:, :, T0 + t].contiguous(), v[:, :, T0 + t].contiguous(), q[t + 1].contiguous(), o, s)
        check(f"decode_step {t}")
    caches[1].set_output_peers([])
    for p in peers:
        p.fill_(0)
    caches[1].attend(q[0], out=outs[1])
    torch.cuda.synchronize()
    assert all(bool((p == 0).all()) for p in peers)


def test_peer_gather_symmetric_memory_world1():
    """PeerGather's allocation, rendezvous and device barrier on a 1-rank NCCL group:
    the attention writes straight into the symmetric gather buffer."""
    import torch.distributed as dist

    from paper_2505_10938_b200 import OTTCache
    from paper_2505_10938_b200.parallel import PeerGather

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        B, Hkv, n_rep, d, G, R = 2, 2, 4, 128, 32, 16
        rng = np.random.default_rng(5)
        caches = [OTTCache(_cfg(2, G, R, 4, 8, d), B, Hkv, max_tokens=256) for _ in range(3)]
        k = torch.from_numpy(rng.standard_normal((B, Hkv, 200, d)).astype(np.float16)).cuda()
        v = torch.from_numpy(rng.standard_normal((B, Hkv, 200, d)).astype(np.float16)).cuda()
        q = torch.from_numpy(rng.standard_normal((B, Hkv * n_rep, d)).astype(np.float16)).cuda()
        for c in caches:
            c.update(k, v)
        pg = PeerGather(caches, n_rep)
        for l, c in enumerate(caches):
            c.attend(q, out=pg.out(l))
            pg.wait(l)
        torch.cuda.synchronize()
        for l, c in enumerate(caches):
            assert torch.equal(pg.gathered(l), c.attend(q))
        pg.close()
    finally:
        dist.destroy_process_group()
