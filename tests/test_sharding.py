"""Multi-rank host logic on CPU (gloo, world size 2 and 3): the C-ABI's branch sharding
(qsim_comm_init + qsim_rank_range) partitions [0, 2^c) into contiguous prefix-aligned ranges,
and the per-rank partial blocks (oracle, over each rank's range) summed across ranks equal the
full branch sum — the reduction step a7 of SURVEY §8(a)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from workloads import generate, sample_block

Q = pytest.importorskip("paper_1802_06952_b200.qsim")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import partition as OP
    circ = generate(4, 3, 16, 5)      # c = 6 -> 64 branches
    ctx = Q.qsim_create(Q.QSIM_C128, 0)
    Q.qsim_load_circuit(ctx, circ.rows, circ.cols, circ.depth, circ.gate_array())
    uid = [Q.qsim_nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    Q.qsim_comm_init(ctx, rank, world, uid[0])
    b0, b1 = Q.qsim_rank_range(ctx)
    c, B, cuts = Q.qsim_partition(ctx)
    first = sorted({int(x[0]) for x in cuts})[:2]
    per = B >> sum(1 for x in cuts if int(x[0]) in first)
    Q.qsim_destroy(ctx)
    ranges = [None] * world
    dist.all_gather_object(ranges, (b0, b1))
    Su = sample_block(circ.h_upper, 20, 1)
    Sl = sample_block(circ.h_lower, 24, 2)
    A = OP.amplitudes(circ, Su, Sl, branches=range(b0, b1))
    t = torch.from_numpy(np.ascontiguousarray(A.view(np.float64)))
    dist.all_reduce(t)
    if rank == 0:
        full = OP.amplitudes(circ, Su, Sl)
        np.save(os.path.join(out_dir, "result.npy"), np.array([np.abs(t.numpy().view(np.complex128) - full).max()]))
        with open(os.path.join(out_dir, "ranges.txt"), "w") as f:
            f.write(repr((B, per, ranges)))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_branch_sharding_gloo(world, tmp_path):
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    err = float(np.load(tmp_path / "result.npy")[0])
    assert err < 1e-14
    B, per, ranges = eval((tmp_path / "ranges.txt").read_text())
    assert ranges[0][0] == 0 and ranges[-1][1] == B
    for (a0, a1), (n0, _) in zip(ranges, ranges[1:]):
        assert a1 == n0 and a0 < a1
    # prefix aligned for any world size: every boundary is a first-period prefix-group boundary
    assert per < B and all(r0 % per == 0 and r1 % per == 0 for r0, r1 in ranges)
    if (B // per) % world == 0:
        assert all(r1 - r0 == B // world for r0, r1 in ranges)


def test_comm_init_validation():
    ctx = Q.qsim_create(Q.QSIM_C64, 0)
    try:
        uid = Q.qsim_nccl_unique_id()
        for (r, w) in [(-1, 2), (2, 2), (0, 0)]:
            with pytest.raises(Q.QsimError) as ei:
                Q.qsim_comm_init(ctx, r, w, uid)
            assert ei.value.status == Q.QSIM_EINVAL
        with pytest.raises(Q.QsimError):
            Q.qsim_rank_range(ctx)        # no circuit yet
    finally:
        Q.qsim_destroy(ctx)
