import sys, json, torch
sys.path.insert(0, "/root/repo")
from paper_2511_08427_b200 import ops
src = torch.rand(720, 1024, 1024, device="cuda")
dst = torch.empty(720, 1024, 1024).pin_memory()
s = torch.cuda.current_stream()
res = {}
for rows in (8, 16, 80, 128, 1024):
    for _ in range(2):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); ops._copy_rows(dst, src, 0, rows, s); b.record(); torch.cuda.synchronize()
    ms = a.elapsed_time(b)
    res[f"2d_rows{rows}"] = {"ms": round(ms, 3), "GBps": round(720 * rows * 4096 / ms / 1e6, 1)}
for views in (8, 64):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); dst[:views].copy_(src[:views], non_blocking=True); b.record(); torch.cuda.synchronize()
    ms = a.elapsed_time(b)
    res[f"1d_views{views}"] = {"ms": round(ms, 3), "GBps": round(views * 4 * 2**20 / ms / 1e6, 1)}
print(json.dumps(res))
