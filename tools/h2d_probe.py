"""Host<->device copy throughput of pinned buffers: one stream vs split over
several streams (copy engines), 8 MB as the cfg5 interface vector."""
import torch, json
N = 8 * 1024 * 1024 // 8
h = torch.ones(N, dtype=torch.float64).pin_memory(); d = torch.empty(N, dtype=torch.float64, device="cuda")
hz = torch.empty_like(h).pin_memory()
streams = [torch.cuda.Stream() for _ in range(4)]
def run(k, d2h=False):
    ev0 = torch.cuda.Event(enable_timing=True); ev1 = torch.cuda.Event(enable_timing=True)
    cur = torch.cuda.current_stream()
    ev0.record(cur)
    for i, st in enumerate(streams[:k]):
        st.wait_stream(cur)
        with torch.cuda.stream(st):
            sl = slice(i * N // k, (i + 1) * N // k)
            if d2h: hz[sl].copy_(d[sl], non_blocking=True)
            else: d[sl].copy_(h[sl], non_blocking=True)
    for st in streams[:k]: cur.wait_stream(st)
    ev1.record(cur); ev1.synchronize()
    return ev0.elapsed_time(ev1)
for d2h in (False, True):
    for k in (1, 2, 4):
        for _ in range(3): run(k, d2h)
        ms = min(run(k, d2h) for _ in range(10))
        print(json.dumps({"dir": "d2h" if d2h else "h2d", "streams": k, "ms": ms, "GBps": 8 * 2**20 / ms / 1e6}))
