"""torchrun worker for tests/test_gpu_multi.py::test_multi_gpu_step_host_chunked: at
n_local > 4M rows aa_step_host runs row-chunked K1/K4 launches with the exchange in the last
chunk; it must follow aa_step (device buffers) on every rank."""
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import aa_inputs  # noqa: E402
from aa_inputs import problems  # noqa: E402
from paper_2110_09667_b200 import aa  # noqa: E402


def main(out_path, fused):
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
    dist.init_process_group("nccl")
    dist.barrier()
    comm = aa.torch_nccl_comm()
    n_global, m, iters = 8_400_003, 5, 10
    off, n = aa_inputs.shard_bounds(n_global, world)[rank]
    d, b = problems.diagonal(n, offset=off)
    dt, bt = torch.tensor(d, device="cuda"), torch.tensor(b, device="cuda")
    stream = torch.cuda.current_stream()
    rep = {}
    for variant in ("dcgs2", "icwy", "cgs2", "mgs"):
        opts = dict(rank=rank, nranks=world, nccl_comm=comm, stream=stream, n_global=n_global,
                    fused_allreduce=1 if fused else None)
        dev = aa.AndersonSolver(n, m, variant, **opts)
        hst = aa.AndersonSolver(n, m, variant, **opts)
        x = torch.zeros(n, dtype=torch.float64, device="cuda")
        xn = torch.empty_like(x)
        dev.init(x, dt * x + bt, xn)
        x, xn = xn, x
        z = torch.zeros(n, dtype=torch.float64, device="cuda")
        z1 = torch.empty_like(z)
        hst.init(z, dt * z + bt, z1)
        xh = z1.cpu().pin_memory()
        gh = torch.empty(n, dtype=torch.float64).pin_memory()
        oh = torch.empty(n, dtype=torch.float64).pin_memory()
        bh, dh = bt.cpu(), dt.cpu()
        worst = 0.0
        for _ in range(iters):
            dev.step(x, dt * x + bt, xn)
            x, xn = xn, x
            torch.addcmul(bh, dh, xh, out=gh)
            hst.step_host(xh, gh, oh)
            xh, oh = oh, xh
            a = x.cpu().numpy()
            worst = max(worst, float(np.linalg.norm(xh.numpy() - a) / np.linalg.norm(a)))
        sd, sh = dev.stats(), hst.stats()
        rep[variant] = {"worst": worst, "ar_dev": sd.allreduce_last, "ar_host": sh.allreduce_last,
                        "f_dev": sd.f_norm, "f_host": sh.f_norm}
        dev.close()
        hst.close()
    allrep = [None] * world
    dist.all_gather_object(allrep, rep)
    if rank == 0:
        json.dump(allrep, open(out_path, "w"))
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] == "fused")
