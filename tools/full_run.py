"""One complete job of the method: every branch of a config evolved, the sampled block
reconstructed and reduced, Porter-Thomas / Eq. 7 statistics (Fig. 5) and
outcome draws.  One process per GPU:

    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 \
        tools/full_run.py --config C4 --out gpurun_out/full_C4

Writes <out>/summary.json (timings, cost-model prediction, statistics, first draws) and
<out>/fig5.csv (z bin centre, count, empirical density, Eq. 7 density) on rank 0.
Product path only (the C-ABI); nothing here reads the oracle."""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_1802_06952_b200 import qsim as Q  # noqa: E402
from workloads import generate, sample_block, CONFIGS  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C4", choices=sorted(CONFIGS))
    ap.add_argument("--precision", default="c64", choices=["c64", "c128"])
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--draws", type=int, default=1 << 20)
    ap.add_argument("--z-lo", type=float, default=-12.0)
    ap.add_argument("--z-hi", type=float, default=4.0)
    ap.add_argument("--bins", type=int, default=160)
    ap.add_argument("--hbm-gbps", type=float, default=5590.0, help="sweep bandwidth for the cost model")
    ap.add_argument("--out", default=None)
    ap.add_argument("--grid", default=None, help="rows,cols,depth,log2_nu,log2_nl instead of --config")
    args = ap.parse_args()

    rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("gloo")
    prec = Q.QSIM_C128 if args.precision == "c128" else Q.QSIM_C64
    rows, cols, depth, lu, ll = CONFIGS[args.config]
    if args.grid:
        rows, cols, depth, lu, ll = (int(v) for v in args.grid.split(","))
        args.config = f"{rows}x{cols}d{depth}"
    circ = generate(rows, cols, depth, args.seed)
    Su = sample_block(circ.h_upper, 1 << (lu or circ.h_upper), args.seed + 1)
    Sl = sample_block(circ.h_lower, 1 << (ll or circ.h_lower), args.seed + 2)

    ctx = Q.qsim_create(prec, local)
    stream = torch.cuda.Stream()
    Q.qsim_set_stream(ctx, stream.cuda_stream)
    Q.qsim_load_circuit(ctx, rows, cols, depth, circ.gate_array())
    if world > 1:
        uid = [Q.qsim_nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        Q.qsim_comm_init(ctx, rank, world, uid[0])
    n_cuts, n_branches, cuts = Q.qsim_partition(ctx)
    cost = Q.qsim_cost_model(ctx, len(Su), len(Sl), args.hbm_gbps)
    b0, b1 = Q.qsim_rank_range(ctx)
    Q.qsim_set_blocks(ctx, Su, Sl)
    # first-period prefix groups: progress is reported per group
    first = sum(1 for c in cuts if c[0] <= 8) if n_cuts else 0
    group = max(1, n_branches >> first)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    done, last = b0, t0
    while done < b1:
        e = min(b1, (done // group + 1) * group)
        Q.qsim_evolve_range(ctx, done, e)
        done = e
        if rank == 0 and time.perf_counter() - last > 60:
            Q.qsim_synchronize(ctx)
            last = time.perf_counter()
            print(f"[full_run] {args.config} rank0 {done - b0}/{b1 - b0} branches, {last - t0:.0f} s",
                  flush=True)
    Q.qsim_synchronize(ctx)
    t_evolve = time.perf_counter() - t0
    if world > 1:
        t = torch.tensor([t_evolve], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        t_evolve = float(t.item())
    t1 = time.perf_counter()
    st, hist, expected = Q.qsim_porter_thomas(ctx, None, 0, args.z_lo, args.z_hi, args.bins)
    x, W = Q.qsim_sample(ctx, args.seed + 7, args.draws, to_host=(rank == 0))
    Q.qsim_synchronize(ctx)
    t_post = time.perf_counter() - t1
    stats = Q.qsim_stats(ctx)
    Q.qsim_destroy(ctx)
    if rank == 0:
        out = args.out or os.path.join(ROOT, "gpurun_out", f"full_{args.config}_{args.precision}_n{world}")
        os.makedirs(out, exist_ok=True)
        n_amp = len(Su) * len(Sl)
        npos = st["count"] - st["zeros"]
        w = (args.z_hi - args.z_lo) / args.bins
        with open(os.path.join(out, "fig5.csv"), "w") as f:
            f.write("z_center,count,density,eq7_density\n")
            for k in range(args.bins):
                zc = args.z_lo + (k + 0.5) * w
                f.write(f"{zc:.6f},{int(hist[k])},{hist[k] / (npos * w):.8e},{expected[k] / (npos * w):.8e}\n")
        summary = {
            "config": args.config, "grid": [rows, cols], "depth": depth, "n_qubits": rows * cols,
            "precision": args.precision, "seed": args.seed, "n_gpus": world, "n_cuts": n_cuts,
            "n_branches": n_branches, "block": [len(Su), len(Sl)],
            "evolve_s_max_over_ranks": t_evolve, "post_s": t_post,
            "amplitudes_per_s": n_amp / (t_evolve + t_post),
            "cost_model": {k: cost[k] for k in ("N_e", "N_m", "regime", "tree_sweeps", "flat_layer_evolutions",
                                                "sweep_bytes", "predicted_s")},
            "predicted_s_per_gpu": cost["predicted_s"] / world,
            "porter_thomas": st, "block_mass": W, "first_draws": [int(v) for v in x[:8]],
            "rank0_stats": {k: stats[k] for k in ("sweeps", "kernel_launches", "sweep_bytes", "branches_evolved",
                                                  "lazy_gathers")},
        }
        with open(os.path.join(out, "summary.json"), "w") as f:
            json.dump(summary, f, indent=1)
        print(json.dumps({k: summary[k] for k in ("config", "n_gpus", "evolve_s_max_over_ranks",
                                                   "predicted_s_per_gpu", "amplitudes_per_s")}), flush=True)
        print("porter_thomas", json.dumps(st), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
