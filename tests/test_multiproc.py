"""World-size-2 gloo run of bench.py's multi-GPU plumbing on the CPU: frame
sharding by global index, max/sum-over-ranks reductions, and per-frame
results independent of the shard (frames are decoded here by the CPU
restatement, the GPU path is identical per frame — see
test_gpu_parity.py::test_determinism_and_slot_invariance)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from conftest import ROOT


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, total, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(RANK=str(rank), WORLD_SIZE=str(world), LOCAL_RANK=str(rank), MASTER_ADDR="127.0.0.1",
                      MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist
    import bench
    import oracle
    import paper_2507_03509_b200 as P
    dist.init_process_group("gloo", rank=rank, world_size=world)
    code = P.ParityCheckMatrix.from_check_lists(24, [[0, 1, 2, 12], [2, 3, 4, 13], [4, 5, 6, 14], [6, 7, 8, 15],
                                                    [8, 9, 10, 16], [10, 11, 0, 17], [1, 5, 9, 18],
                                                    [3, 7, 11, 19], [12, 20], [15, 21], [18, 22], [19, 23]])
    a, b = bench.shard(total, rank, world)
    snr = P.snr_for_beta(0.5, code.rate())
    llr, x, s = P.sample_frames(code, snr, 11, a, b - a)
    ptr, var = code.csr()
    orc = oracle.Restatement()
    its = [orc.decode(code.n_vars, ptr, var, llr[i].astype(np.float64), syndrome=s[i], d_max=30, use_pce=True,
                      use_vnr=True, q_mode=1)["iterations"] for i in range(b - a)]
    t = bench.max_over_ranks(float(rank + 1), dist)
    n = bench.sum_over_ranks(float(b - a), dist)
    gathered = [None] * world
    dist.all_gather_object(gathered, (a, b, its))
    if rank == 0:
        q.put((t, n, gathered))
    dist.destroy_process_group()


def test_two_rank_sharding_gloo():
    total = 10
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, total, q)) for r in range(2)]
    for p in procs:
        p.start()
    t, n, gathered = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert t == 2.0 and n == total
    ranges = sorted((a, b) for a, b, _ in gathered)
    assert ranges[0][0] == 0 and ranges[-1][1] == total and ranges[0][1] == ranges[1][0]
    # single-process reference of the same global frames
    import oracle
    import paper_2507_03509_b200 as P
    code = P.ParityCheckMatrix.from_check_lists(24, [[0, 1, 2, 12], [2, 3, 4, 13], [4, 5, 6, 14], [6, 7, 8, 15],
                                                    [8, 9, 10, 16], [10, 11, 0, 17], [1, 5, 9, 18],
                                                    [3, 7, 11, 19], [12, 20], [15, 21], [18, 22], [19, 23]])
    llr, x, s = P.sample_frames(code, P.snr_for_beta(0.5, code.rate()), 11, 0, total)
    ptr, var = code.csr()
    orc = oracle.Restatement()
    want = [orc.decode(code.n_vars, ptr, var, llr[i].astype(np.float64), syndrome=s[i], d_max=30, use_pce=True,
                       use_vnr=True, q_mode=1)["iterations"] for i in range(total)]
    got = [it for a, b, its in sorted(gathered) for it in its]
    assert got == want


@pytest.mark.parametrize("total,world", [(64, 1), (64, 2), (4096, 8), (10, 4), (3, 8)])
def test_shard_partition(total, world):
    import sys
    sys.path.insert(0, ROOT)
    import bench
    seen = []
    for r in range(world):
        a, b = bench.shard(total, r, world)
        seen.extend(range(a, b))
    assert seen == list(range(total))


def _gpu_worker(rank, world, port, total, q):
    """One rank of the frame-sharded GPU decode: its shard of global frames
    through its own BatchDecoder (both ranks share cuda:0 here: one GPU per
    gpurun box; the ranks never wait on each other's kernels), results
    gathered to rank 0 over gloo (the host gather of SURVEY §8e)."""
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(RANK=str(rank), WORLD_SIZE=str(world), LOCAL_RANK=str(rank), MASTER_ADDR="127.0.0.1",
                      MASTER_PORT=str(port))
    import torch.distributed as dist
    import bench
    import paper_2507_03509_b200 as P
    dist.init_process_group("gloo", rank=rank, world_size=world)
    code = P.WORKLOADS["cfg1"].make_code()
    a, b = bench.shard(total, rank, world)
    llr, x, s = P.sample_frames(code, P.snr_for_beta(0.95, code.rate()), P.FRAME_SEED, a, b - a)
    dec = P.BatchDecoder(code, device=0, max_slots=32)
    r = dec.decode_batch(llr, P.DecodeConfig(d_max=200, use_pce=True, use_vnr=True, q_mode=P.decoder.Q_ABS),
                         syndrome=s, packed=True)
    gathered = [None] * world
    dist.all_gather_object(gathered, (a, b, r.iterations.tolist(), r.reasons.tolist(), r.bits.tolist()))
    if rank == 0:
        q.put(gathered)
    dist.destroy_process_group()


@pytest.mark.gpu
def test_two_rank_gpu_decode_gloo():
    """Two ranks decode disjoint shards of 100 cfg1 frames on the GPU; the
    gathered per-frame outputs equal one decoder decoding all 100."""
    total = 100
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gpu_worker, args=(r, 2, port, total, q)) for r in range(2)]
    for p in procs:
        p.start()
    gathered = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    import paper_2507_03509_b200 as P
    code = P.WORKLOADS["cfg1"].make_code()
    llr, x, s = P.sample_frames(code, P.snr_for_beta(0.95, code.rate()), P.FRAME_SEED, 0, total)
    want = P.BatchDecoder(code, device=0, max_slots=64).decode_batch(
        llr, P.DecodeConfig(d_max=200, use_pce=True, use_vnr=True, q_mode=P.decoder.Q_ABS), syndrome=s, packed=True)
    its = [i for a, b, it, rs, bt in sorted(gathered) for i in it]
    rss = [i for a, b, it, rs, bt in sorted(gathered) for i in rs]
    bits = np.array([w for a, b, it, rs, bt in sorted(gathered) for w in bt], dtype=np.uint32)
    assert its == want.iterations.tolist() and rss == want.reasons.tolist()
    assert np.array_equal(bits, want.bits.view(np.uint32))
