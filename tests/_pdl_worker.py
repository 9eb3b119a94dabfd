"""Run a short small-n AA sequence per variant and dump the iterates (tests/test_gpu_pdl.py)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from aa_inputs import problems  # noqa: E402
from paper_2110_09667_b200 import aa  # noqa: E402


def main(out):
    res = {}
    for n, m in ((1000, 20), (3001, 5), (70001, 12)):
        d, b = problems.diagonal(n)
        dt, bt = torch.tensor(d, device="cuda"), torch.tensor(b, device="cuda")
        for v in ("dcgs2", "icwy", "cgs2", "mgs", "icwy_small"):
            s = aa.AndersonSolver(n, m, "icwy" if v == "icwy_small" else v,
                                  stream=torch.cuda.current_stream(),
                                  icwy_delete="small" if v == "icwy_small" else None)
            x = torch.zeros(n, dtype=torch.float64, device="cuda")
            xn = torch.empty_like(x)
            s.init(x, dt * x + bt, xn)
            x, xn = xn, x
            xs = []
            for _ in range(m + 8):          # start-up and recycle, back to back (no host sync)
                s.step(x, dt * x + bt, xn)
                x, xn = xn, x
                xs.append(x.clone())
            res[f"{v}_{n}_{m}"] = torch.stack(xs).cpu().numpy()
            s.close()
    np.savez(out, **res)


if __name__ == "__main__":
    main(sys.argv[1])
