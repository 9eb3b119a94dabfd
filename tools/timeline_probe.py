"""Phase timeline of one DCGS-2 recycle step at small n (test-only hook)."""
import sys, os, torch, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2110_09667_b200 import aa
n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 1000
m = int(sys.argv[2]) if len(sys.argv) > 2 else 20
v = sys.argv[3] if len(sys.argv) > 3 else "dcgs2"
stream = torch.cuda.current_stream()
d = torch.rand(n, dtype=torch.float64, device="cuda") * 1.8 - 0.9
b = torch.rand(n, dtype=torch.float64, device="cuda") * 2 - 1
s = aa.AndersonSolver(n, m, v, stream=stream)
x = torch.zeros(n, dtype=torch.float64, device="cuda"); xn = torch.empty_like(x)
s.init(x, d * x + b, xn); x, xn = xn, x
for _ in range(m + 5):
    b.mul_(1.0 + 1e-3)     # never exactly at the fixed point (a breakdown would degrade the step)
    s.step(x, d * x + b, xn); x, xn = xn, x
aa.aa_test_timeline(s.h, True)
for _ in range(3):
    b.mul_(1.0 + 1e-3)
    g = d * x + b
    torch.cuda.synchronize()
    s.step(x, g, xn); x, xn = xn, x
    tlc = aa.aa_test_timeline(s.h, True).astype(np.int64)
    tl, ck = tlc[0], tlc[1]
names = ["entry", "staged", "head", "tile0", "tiles", "partials", "red", "end"]
# (slots of op 7 carry K4 commit-warp details; the LOO Gram kernel is not run here)
det = [(i, int(tl[7, i]), int(ck[7, i])) for i in range(4) if tl[7, i] > 0]
ops = {0: "K1", 1: "K2icwy", 2: "K2dcgs2", 3: "K2a", 4: "K2b", 5: "K2mgs", 6: "K4"}
t0 = min(int(tl[o, 0]) for o in ops if tl[o, 0] > 0)
for o, nm in ops.items():
    if tl[o, 0] == 0: continue
    row = tl[o, :8] - t0
    print(f"{nm:8s}", " ".join(f"{names[i]}={row[i]/1e3:7.2f}" for i in range(8)), f"| dur {(tl[o,7]-tl[o,0])/1e3:.2f} us")
    sub = [(i, int(tl[o, i]) - t0) for i in range(8, 16) if tl[o, i] > 0]
    if sub:
        print("         sub:", " ".join(f"[{i}]={v/1e3:7.2f}" for i, v in sub))
        # clock64 of the same marks (CTA 0 slots share an SM): cycles after the head mark
        c2 = int(ck[o, 2])
        print("         sub cycles after 'staged':", " ".join(f"[{i}]={int(ck[o, i]) - int(ck[o, 1])}" for i, _ in sub))
    # effective SM clock from clock64 deltas (CTA 0 slots 0..5 are on one SM)
    dt = tl[o, 5] - tl[o, 0]; dc = ck[o, 5] - ck[o, 0]
    if dt > 0: print(f"         SM clock over entry..partials: {dc / dt * 1e3:.0f} MHz ({dc} cycles)")
print("K4 commit CTA: [8] warp 0 R column formed, [12..14] its QRDelete (split: early rotations loaded,"
      " last columns rotated, last rotations), [9] done; [10] warp 1 gamma, [11] scales written;"
      " [15] warps 3-7 R, T (and early R') written")
