"""CUDA-graph capture of the caller's loop (SURVEY.md §3.2, §8(b) "Asynchrony"): aa_step only
enqueues, its launch parameters depend only on (i, m_i, variant, options) and on the handle's
double-buffer version / Delta G ring head, which repeat with period lcm(2, m) at recycle, and
the fused exchange takes its sequence numbers from a device counter -- so a window of
lcm(2, m) recycle steps (G included) can be captured once and replayed.  The replayed
iterates must equal the eagerly launched ones bitwise."""
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from aa_inputs import problems  # noqa: E402
from paper_2110_09667_b200 import aa  # noqa: E402


def _run(n, m, variant, replays, graph, opts):
    d, b = problems.diagonal(n, 0.5, 0.99)
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        dt, bt = torch.tensor(d, device="cuda"), torch.tensor(b, device="cuda")
        s = aa.AndersonSolver(n, m, variant, stream=st, **opts)
        x = torch.zeros(n, dtype=torch.float64, device="cuda")
        xn = torch.empty_like(x)
        g = torch.empty_like(x)
        s.init(x, torch.addcmul(bt, dt, x), xn)
        x, xn = xn, x
        for _ in range(m + 2):             # start-up, then recycle (every kernel instance used once)
            torch.addcmul(bt, dt, x, out=g)
            s.step(x, g, xn)
            x, xn = xn, x
        L = m * 2 // math.gcd(m, 2)        # period of (factor version, Delta G ring head)
        bufs = (x, xn)
        out = []

        def window():
            for i in range(L):
                a, c = bufs[i % 2], bufs[(i + 1) % 2]
                torch.addcmul(bt, dt, a, out=g)
                s.step(a, g, c)

        if graph:
            # capture records, it does not execute: the host-side state (version, ring head)
            # advances by one period, i.e. back to where it was
            st.synchronize()
            gr = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gr, stream=st):
                window()
            for _ in range(replays):
                gr.replay()
                out.append(bufs[0].clone())
        else:
            for _ in range(replays):
                window()
                out.append(bufs[0].clone())
        st.synchronize()
        res = [o.cpu().numpy() for o in out]
        s.close()
    return res


@pytest.mark.parametrize("variant,opts", [("dcgs2", {}), ("icwy", {}), ("icwy", {"icwy_delete": "small"}),
                                          ("cgs2", {}), ("mgs", {})])
def test_graph_replay_equals_eager(variant, opts):
    n, m = 4097, 4
    eager = _run(n, m, variant, 3, False, opts)
    replay = _run(n, m, variant, 3, True, opts)
    for a, c in zip(replay, eager):
        assert np.array_equal(a, c)
