import sys, time, numpy as np, torch
sys.path.insert(0, '/root/repo')
import paper_2310_03983_b200 as ap
def t(fn, reps=4):
    out=[]
    for _ in range(reps):
        torch.cuda.synchronize(); e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
        e0.record(); r=fn(); e1.record(); torch.cuda.synchronize(); out.append(round(e0.elapsed_time(e1),2))
    return out, r.info
h32 = torch.from_numpy(ap.dense_costs(ap.GenParams(4096, 1.0, 100, 7+4096), np.int32)).cuda()
hf = h32.float(); hf[h32 == ap.INF32] = float('inf')
print("i32", t(lambda: ap.solve(h32, "fw_blocked")))
print("f32", t(lambda: ap.solve(hf, "fw_blocked")))
print("f32 ws", t(lambda: ap.solve(hf, "fw_blocked", workspace=ws)) if (ws := torch.empty(ap._native.load().apsp_workspace_bytes(0, 1, 4096, 0), dtype=torch.uint8, device='cuda')) is not None else None)
h8 = torch.from_numpy(ap.dense_costs(ap.GenParams(8192, 1.0, 100, 7+8192), np.float32)).cuda()
for thr in (512, 1024, 2048):
    print("rk", thr, t(lambda: ap.solve(h8, "rkleene", track="pred", split="aligned", base_threshold=thr)))
