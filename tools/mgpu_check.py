"""Multi-GPU parity check, launched with torchrun (one process per GPU):

    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 tools/mgpu_check.py

Every rank evolves its own branch share (qsim_evolve_halves), the partial blocks are reduced with
NCCL inside qsim_amplitudes / qsim_sample, and rank 0 compares with the oracle (exit 1 on failure)
and checks that the sampler matches the single-GPU draws on the same probabilities."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_1802_06952_b200 import qsim as Q  # noqa: E402
from workloads import generate, sample_block  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    ok = True
    for (grid, depth, prec) in [((4, 7, 10), None, Q.QSIM_C128), ((4, 7, 14), None, Q.QSIM_C64),
                                ((4, 4, 22), None, Q.QSIM_C128)]:
        rows, cols, d = grid
        circ = generate(rows, cols, d, 3)
        Su = sample_block(circ.h_upper, min(200, 1 << circ.h_upper), 5)
        Sl = sample_block(circ.h_lower, min(150, 1 << circ.h_lower), 6)
        ctx = Q.qsim_create(prec, local)
        Q.qsim_load_circuit(ctx, rows, cols, d, circ.gate_array())
        uid = [Q.qsim_nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        Q.qsim_comm_init(ctx, rank, world, uid[0])
        Q.qsim_evolve_halves(ctx, Su, Sl)
        A = Q.qsim_amplitudes(ctx, Su, Sl, prec, write=(rank == 0))
        x, W = Q.qsim_sample(ctx, 9, 4096, to_host=(rank == 0))
        Q.qsim_destroy(ctx)
        if rank == 0:
            from oracle import partition as OP, sampler as OS
            ref = OP.amplitudes(circ, Su, Sl)
            err = np.abs(A.astype(np.complex128) - ref).max()
            tol = 1e-12 if prec == Q.QSIM_C128 else 1e-5 * np.abs(ref).max()
            p = np.abs(A.astype(np.complex128)) ** 2
            xr, Wr = OS.sample(p, Su, Sl, circ.h_lower, 9, 4096)
            match = np.mean(x == xr)
            print(f"rank0 world={world} grid={grid} prec={prec}: max err {err:.3e} (tol {tol:.1e}), "
                  f"W={W:.6f} draws match {match:.4f}", flush=True)
            ok = ok and err <= tol and match > 0.99
    flag = torch.tensor([1 if ok else 0])
    dist.broadcast(flag, src=0)
    dist.destroy_process_group()
    sys.exit(0 if flag.item() else 1)


if __name__ == "__main__":
    main()
