"""Multi-GPU path (NCCL allreduce per global reduction) vs the single-process oracle.

Runs only on a box with >= 2 GPUs (`gpurun --gpus 2`); skipped otherwise."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2, reason="needs >= 2 GPUs")
@pytest.mark.parametrize("mode", ["torch_comm", "torch_comm_fused", "unique_id", "unique_id_fused"])
def test_multi_gpu_parity_and_allreduce_counts(tmp_path, mode):
    """NCCL allreduce per reduction (torch_comm*: torch's communicator borrowed through
    aa_create_with_comm; unique_id*: libaa's own communicator from aa_comm_unique_id +
    aa_create, the north-star rendezvous) or the fused one-shot NVLink exchange in the
    producing kernel's last CTA (*_fused).  Also SURVEY.md §8(c) criterion 6 (the p-rank
    iterates vs the same run on one GPU, <= 1e-13) and the breakdown decisions (reading
    A12) identical on every rank and equal to the oracle's restart policy."""
    from aa_inputs import problems
    from oracle import aa_variant
    world = min(torch.cuda.device_count(), 4)
    out = tmp_path / "dist.json"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--standalone", "--nnodes=1",
           f"--nproc-per-node={world}", os.path.join(ROOT, "tests", "_dist_worker.py"), str(out), mode]
    env = dict(os.environ, MASTER_ADDR="127.0.0.1")
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)
    assert res.returncode == 0, res.stdout[-3000:] + res.stderr[-3000:]
    rep = json.load(open(out))
    n, m, iters = 100003, 5, 14
    d, b = problems.diagonal(n)
    for variant, r in rep["variants"].items():
        if variant == "icwy_small":   # reduction-free post-delete T update (A6b)
            o2 = aa_variant(lambda x: d * x + b, np.zeros(n), m, "icwy", iters, icwy_delete="small")
        elif variant == "dcgs2_immediate":   # AA_OPT_CONV_NORM = IMMEDIATE
            o2 = aa_variant(lambda x: d * x + b, np.zeros(n), m, "dcgs2", iters)
        else:
            o2 = aa_variant(lambda x: d * x + b, np.zeros(n), m, variant, iters)
        for a, ref in zip(r["xs"], o2.xs):
            assert np.linalg.norm(np.array(a) - ref) <= 1e-10 * np.linalg.norm(ref), variant
        for a, ref in zip(r["f_norms"], o2.f_norms):
            assert abs(a - ref) <= 1e-10 * ref + 1e-14
        # one ncclAllReduce per global reduction: FIRST 1; start-up MGS m_i, ICWY 2,
        # CGS-2 3, DCGS-2 2; recycle MGS m, ICWY 3, CGS-2 3, DCGS-2 2
        ars = r["allreduce_per_step"]
        if variant == "dcgs2_immediate":   # the convergence norm is one more allreduce per step
            ars = [a - 1 for a in ars]
            assert r["dx_norms"] == rep["variants"]["dcgs2"]["dx_norms"]
        assert ars[0] == 1
        for i in range(2, iters + 1):
            if i <= m:
                want = {"mgs": i, "icwy": 2, "cgs2": 3, "dcgs2": 2, "icwy_small": 2, "dcgs2_immediate": 2}[variant]
            else:
                want = {"mgs": m, "icwy": 3, "cgs2": 3, "dcgs2": 2, "icwy_small": 2, "dcgs2_immediate": 2}[variant]
            assert ars[i - 1] == want, (variant, i, ars)
        assert r["gamma_identical_across_ranks"]
        assert r["loo"] < 1e-12
        assert r["x_vs_p1"] <= 1e-13, (variant, r["x_vs_p1"])
    assert rep["breakdown_flags_identical_across_ranks"]
    # SURVEY.md §8(e) deterministic mode: bitwise the one-GPU iterates
    assert all(rep["deterministic_bitwise_vs_p1"].values()), rep["deterministic_bitwise_vs_p1"]
    d5, b5 = problems.diagonal(n, 0.5, 0.99)
    for variant, r in rep["breakdown"].items():
        o2 = aa_variant(lambda x: d5 * x + b5, np.zeros(n), 2, variant, 10, breakdown="restart",
                        breakdown_eps=0.5, record_loo=False)
        assert r["flags"] == o2.breakdown and any(r["flags"])
        for a, ref in zip(r["xs"], o2.xs):
            assert np.linalg.norm(np.array(a) - ref) <= 1e-10 * np.linalg.norm(ref), variant


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2, reason="needs >= 2 GPUs")
@pytest.mark.parametrize("mode", ["fused", "nccl"])
def test_multi_gpu_step_host_chunked(tmp_path, mode):
    """aa_step_host at n_local > 4M rows (row-chunked K1 / K4, exchange in the last chunk)
    follows aa_step on every rank, in both reduction modes, with the same allreduce count."""
    world = min(torch.cuda.device_count(), 4)
    out = tmp_path / "host.json"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--standalone", "--nnodes=1",
           f"--nproc-per-node={world}", os.path.join(ROOT, "tests", "_dist_host_worker.py"), str(out), mode]
    env = dict(os.environ, MASTER_ADDR="127.0.0.1")
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=900, env=env, cwd=ROOT)
    assert res.returncode == 0, res.stdout[-3000:] + res.stderr[-3000:]
    for rep in json.load(open(out)):
        for variant, r in rep.items():
            assert r["worst"] <= 1e-12, (variant, r)
            assert r["ar_dev"] == r["ar_host"], (variant, r)
            assert abs(r["f_dev"] - r["f_host"]) <= 1e-12 * r["f_dev"], (variant, r)
