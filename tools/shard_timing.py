"""Time the row-band sharded FW emulated on one GPU (all ranks sequential) vs the single-GPU
solver, for several world sizes and blocks -- diagnostic for the multi-GPU schedule."""
import sys, time
import numpy as np, torch
sys.path.insert(0, "/root/repo")
import paper_2310_03983_b200 as ap
from paper_2310_03983_b200.distributed import fw_blocked_emulated

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
h = torch.from_numpy(ap.dense_costs(ap.GenParams(n, 0.1, 100, 7 + n), np.int32)).cuda()
def t(fn, reps=2):
    fn(); torch.cuda.synchronize()
    out = []
    for _ in range(reps):
        t0 = time.perf_counter(); fn(); torch.cuda.synchronize(); out.append((time.perf_counter() - t0) * 1e3)
    return min(out)
print("single default", round(t(lambda: ap.solve(h, "fw_blocked")), 1))
for world in (1, 2, 4):
    for b in (256, 1024):
        print("emulated world", world, "b", b, round(t(lambda: fw_blocked_emulated(h, world, block=b)), 1))
