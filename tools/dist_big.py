"""Distributed halves above 32 qubits (§2.3.3), launched with torchrun:

    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 tools/dist_big.py check
    python -m torch.distributed.run --nproc-per-node 4 --master-addr 127.0.0.1 tools/dist_big.py block

check: a 66-qubit 6x11 grid (33-qubit halves, shards of 33 - log2(ranks) qubits): leaf values of branch
  0 of the upper half and B-1 of the lower half at 4099 sampled indices, through the distributed path (qsim_branch_values),
  against the CPU oracle's full 2^33 leaf (oracle/fast.py, 128 GiB of host memory; rank 0 only), both
  precisions.  Exit 1 on a mismatch.
block: a 68-qubit 4x17 grid at depth 22 (34-qubit halves over 4 ranks, 2^32-amplitude shards): a 4-branch
  block of 4096 x 4096 sampled amplitudes (qsim_evolve_range + qsim_amplitudes), timed.
"""
import datetime
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
from workloads import generate, sample_block  # noqa: E402


def ctx_for(prec, local, rank, world, circ):
    ctx = Q.qsim_create(prec, local)
    Q.qsim_set_option(ctx, Q.QSIM_OPT_DISTRIBUTE, 1)
    box = [Q.qsim_nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(box, src=0)
    Q.qsim_comm_init(ctx, rank, world, box[0])
    Q.qsim_load_circuit(ctx, circ.rows, circ.cols, circ.depth, circ.gate_array(), circ.cut_row)
    return ctx


def check(rank, world, local, depth):
    """The GPU values of every case first (collective over the ranks), then rank 0 alone runs the oracle's
    2^33 leaves and compares (no collective waits on the host oracle)."""
    from oracle import fast as F, partition as OP
    circ = generate(6, 11, depth, 5)
    cuts = OP.cut_list(circ)
    B = 1 << len(cuts)
    h = circ.h_upper
    # (half, branch); the oracle's 2^33 leaf takes ~40 min on 16 host cores: QSIM_H33_CASES=2 adds (1, B-1)
    cases = [(0, 0), (1, B - 1)][: int(os.environ.get("QSIM_H33_CASES", "1"))]
    got = {}
    for half, b in cases:
        idx = np.concatenate([sample_block(h, 4096, 80 + half).astype(np.uint64),
                              np.array([0, (1 << h) - 1, (1 << h) - 2], dtype=np.uint64)])
        for prec in (Q.QSIM_C64, Q.QSIM_C128):
            ctx = ctx_for(prec, local, rank, world, circ)
            t0 = time.perf_counter()
            got[(half, b, prec)] = (idx, Q.qsim_branch_values(ctx, half, b, idx))
            dt = time.perf_counter() - t0
            Q.qsim_destroy(ctx)
            if rank == 0:
                print(f"half {half} branch {b} prec {prec}: {dt:.2f} s on {world} GPUs", flush=True)
    dist.barrier()
    if rank != 0:
        return True
    ok = True
    for half, b in cases:
        t0 = time.perf_counter()
        psi = F.branch_state(circ, half, b)
        print(f"oracle leaf half {half} branch {b}: {time.perf_counter() - t0:.0f} s", flush=True)
        for prec in (Q.QSIM_C64, Q.QSIM_C128):
            idx, v = got[(half, b, prec)]
            ref = psi[idx.astype(np.int64)]
            d = np.abs(v.astype(np.complex128) - ref).max()
            rel, rms = d / np.abs(ref).max(), d / np.sqrt(np.mean(np.abs(ref) ** 2))
            good = d <= 1e-12 if prec == Q.QSIM_C128 else rel <= 1e-5
            ok = ok and bool(good)
            rec = {"grid": "6x11", "depth": depth, "h": h, "world": world, "half": half, "branch": b,
                   "prec": "c128" if prec == Q.QSIM_C128 else "c64", "max_abs": d, "rel_max": rel,
                   "rel_rms": rms, "ok": bool(good)}
            print(json.dumps(rec), flush=True)
        del psi
    return ok


def block(rank, world, local):
    circ = generate(4, 17, 22, 0)
    Su, Sl = sample_block(circ.h_upper, 4096, 1), sample_block(circ.h_lower, 4096, 2)
    ctx = ctx_for(Q.QSIM_C64, local, rank, world, circ)
    c, B, _ = Q.qsim_partition(ctx)
    Q.qsim_set_blocks(ctx, Su, Sl)
    torch.cuda.synchronize()
    dist.barrier()
    t0 = time.perf_counter()
    Q.qsim_evolve_range(ctx, 0, 4)
    A = Q.qsim_amplitudes(ctx, Su, Sl, write=(rank == 0))
    dt = time.perf_counter() - t0
    st = Q.qsim_stats(ctx)
    Q.qsim_destroy(ctx)
    if rank == 0:
        rec = {"grid": "4x17", "n": 68, "depth": 22, "h": circ.h_upper, "world": world, "cuts": c,
               "branches": 4, "block": [4096, 4096], "seconds": dt, "sweeps": st["sweeps"],
               "finite": bool(np.isfinite(A).all()), "max_abs": float(np.abs(A).max())}
        print(json.dumps(rec), flush=True)
        return rec["finite"]
    return True


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("gloo", timeout=datetime.timedelta(hours=3))
    mode = sys.argv[1] if len(sys.argv) > 1 else "check"
    ok = check(rank, world, local, int(sys.argv[2]) if len(sys.argv) > 2 else 10) if mode == "check" \
        else block(rank, world, local)
    flag = torch.tensor([1 if ok else 0])
    dist.broadcast(flag, src=0)  # after rank 0's oracle (the long timeout above)
    dist.destroy_process_group()
    sys.exit(0 if flag.item() else 1)


if __name__ == "__main__":
    main()
