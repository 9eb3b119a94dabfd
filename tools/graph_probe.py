"""Small-n step latency with the caller's loop captured in a CUDA graph (one period of
lcm(2, m) recycle steps, G included) vs launched eagerly, 1 GPU.  Prints us per AA step
(G included in both; G alone is printed for reference)."""
import math
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2110_09667_b200 import aa  # noqa: E402


def main():
    ns = [int(float(a)) for a in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["1000", "1e5"])]
    m = int(sys.argv[2]) if len(sys.argv) > 2 else 20
    reps = 20
    for n in ns:
        st = torch.cuda.Stream()
        with torch.cuda.stream(st):
            d = torch.rand(n, dtype=torch.float64, device="cuda") * 0.49 + 0.5
            b = torch.rand(n, dtype=torch.float64, device="cuda") * 2 - 1
            out = [f"n={n:>8d} m={m}"]
            for v in ("dcgs2", "icwy", "icwy_small", "cgs2", "mgs"):
                s = aa.AndersonSolver(n, m, "icwy" if v == "icwy_small" else v, stream=st,
                                      icwy_delete="small" if v == "icwy_small" else None, breakdown_eps=0.0)
                x = torch.zeros(n, dtype=torch.float64, device="cuda")
                xn = torch.empty_like(x)
                g = torch.empty_like(x)
                s.init(x, torch.addcmul(b, d, x), xn)
                x, xn = xn, x
                for _ in range(m + 2):
                    b.mul_(1.0 + 1e-3)
                    torch.addcmul(b, d, x, out=g)
                    s.step(x, g, xn)
                    x, xn = xn, x
                L = m * 2 // math.gcd(m, 2)
                bufs = (x, xn)

                def window():
                    for i in range(L):
                        a, c = bufs[i % 2], bufs[(i + 1) % 2]
                        b.mul_(1.0 + 1e-3)   # never exactly at the fixed point (no breakdown)
                        torch.addcmul(b, d, a, out=g)
                        s.step(a, g, c)

                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                window()
                st.synchronize()
                e0.record(st)
                for _ in range(reps):
                    window()
                e1.record(st)
                st.synchronize()
                t_eager = e0.elapsed_time(e1) / (reps * L) * 1e3
                gr = torch.cuda.CUDAGraph()
                with torch.cuda.graph(gr, stream=st):
                    window()
                gr.replay()
                st.synchronize()
                e0.record(st)
                for _ in range(reps):
                    gr.replay()
                e1.record(st)
                st.synchronize()
                t_graph = e0.elapsed_time(e1) / (reps * L) * 1e3
                out.append(f"{v} eager {t_eager:6.1f} graph {t_graph:6.1f}")
                s.close()
            print(" | ".join(out) + "  (us per AA step incl. G)", flush=True)


if __name__ == "__main__":
    main()
