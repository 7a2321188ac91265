import sys
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import paper_2310_03983_b200 as ap
n = int(sys.argv[1])
h = ap.dense_costs(ap.GenParams(n, 1.0, 100, 7 + n), np.float32)
rng = np.random.default_rng(n)
fin = np.isfinite(h) & (h > 0)
h[fin] = rng.uniform(1.0, 100.0, size=int(fin.sum())).astype(np.float32)
hd = torch.from_numpy(h).cuda()
ap.solve(hd, "fw_blocked"); torch.cuda.synchronize()
