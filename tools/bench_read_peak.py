"""Read-only HBM streams torch offers (sum / amax over 4 GiB) beside its copy: the read ceiling the
paged decode (K5) is compared with.  python tools/bench_read_peak.py  -> one JSON line of GB/s."""
import torch, json, statistics
x = torch.empty(2 * 1024 ** 3, dtype=torch.float16, device="cuda").normal_()   # 4 GiB
nbytes = x.numel() * 2
res = {}
def t(fn, n=10):
    fn(); torch.cuda.synchronize()
    out = []
    for _ in range(n):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); e1.synchronize(); out.append(e0.elapsed_time(e1))
    return min(out)
res["sum_fp16"] = nbytes / t(lambda: x.sum()) / 1e6
xv = x.view(torch.int64)
res["sum_int64_view"] = nbytes / t(lambda: xv.sum()) / 1e6
res["amax"] = nbytes / t(lambda: x.amax()) / 1e6
y = torch.empty_like(x)
res["copy_rw_total"] = 2 * nbytes / t(lambda: y.copy_(x)) / 1e6
print(json.dumps({k: round(v, 1) for k, v in res.items()}))
