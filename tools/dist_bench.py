"""Distributed halves (QSIM_OPT_DISTRIBUTE, §2.3.3) against branch sharding
on the same GPUs.  One process per GPU:

    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 tools/dist_bench.py \
        [--config C4] [--groups 2] [--precision c64]

Distributed: every rank runs the same first-period prefix groups on its 1/N shard of every half state
(local/global qubit swaps fused into sweeps over peer memory).  Branch-sharded: each rank runs its own
groups on whole states (the default mode).  Both time `groups` groups per rank-set after one warm-up
group, CUDA-synchronised, max over ranks; printed as sampled amplitudes/s of the whole job.
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_1802_06952_b200 import qsim as Q  # noqa: E402
from workloads import generate, sample_block, CONFIGS  # noqa: E402


def run(mode, args, rank, world, local, circ, Su, Sl):
    prec = Q.QSIM_C128 if args.precision == "c128" else Q.QSIM_C64
    rows, cols, depth, _, _ = CONFIGS[args.config]
    ctx = Q.qsim_create(prec, local)
    stream = torch.cuda.Stream()
    Q.qsim_set_stream(ctx, stream.cuda_stream)
    Q.qsim_set_option(ctx, Q.QSIM_OPT_DISTRIBUTE, 1 if mode == "distributed" else 0)
    Q.qsim_set_option(ctx, Q.QSIM_OPT_TIME_SWEEPS, 1)
    uid = [Q.qsim_nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    Q.qsim_comm_init(ctx, rank, world, uid[0])
    Q.qsim_load_circuit(ctx, rows, cols, depth, circ.gate_array())
    Q.qsim_set_blocks(ctx, Su, Sl)
    _, nb, cuts = Q.qsim_partition(ctx)
    n_groups_total = 1 << int(sum(1 for c in cuts if c[0] <= 8))  # first-period prefixes
    group = nb // n_groups_total
    b0, _ = Q.qsim_rank_range(ctx)

    def step(g):  # one group per rank-set: distributed = the same group everywhere
        s = (g if mode == "distributed" else b0 // group + g) * group
        Q.qsim_evolve_range(ctx, s, s + group)

    step(0)
    Q.qsim_synchronize(ctx)
    Q.qsim_stats_reset(ctx)
    dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for g in range(1, args.groups + 1):
        step(g)
    Q.qsim_synchronize(ctx)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    st = Q.qsim_stats(ctx)
    t = torch.tensor([dt], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    sb = torch.tensor([st["sweep_bytes"], st["sweep_ms"]], dtype=torch.float64)
    dist.all_reduce(sb, op=dist.ReduceOp.SUM)
    Q.qsim_destroy(ctx)
    groups_done = args.groups * (1 if mode == "distributed" else world)
    amps = len(Su) * len(Sl) * groups_done / n_groups_total
    return {"mode": mode, "n_gpus": world, "s": float(t.item()), "amplitudes_per_s": amps / float(t.item()),
            "sweep_GBps_per_gpu": float(sb[0]) / (float(sb[1]) * 1e-3) / 1e9,
            "sweeps_rank0": st["sweeps"], "groups": groups_done}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C4")
    ap.add_argument("--precision", default="c64")
    ap.add_argument("--groups", type=int, default=2)
    ap.add_argument("--modes", default="distributed,sharded")
    args = ap.parse_args()
    rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("gloo", init_method="env://" if "MASTER_ADDR" in os.environ else
                            "tcp://127.0.0.1:29599", rank=rank, world_size=world)
    rows, cols, depth, lu, ll = CONFIGS[args.config]
    circ = generate(rows, cols, depth, 0)
    Su = sample_block(circ.h_upper, 1 << (lu or circ.h_upper), 1)
    Sl = sample_block(circ.h_lower, 1 << (ll or circ.h_lower), 2)
    out = [run(m, args, rank, world, local, circ, Su, Sl) for m in args.modes.split(",")]
    if rank == 0:
        for r in out:
            r["config"] = args.config
            r["precision"] = args.precision
            print(json.dumps(r), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
