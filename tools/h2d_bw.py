"""Host link bandwidth (pinned memory, 738 MB = the bench step's copy-in): H2D alone, D2H alone,
both directions concurrently on two streams; CUDA events."""
import json
import torch

nb = 738197504
h1 = torch.empty(nb, dtype=torch.uint8).pin_memory()
h2 = torch.empty(nb, dtype=torch.uint8).pin_memory()
d1 = torch.empty(nb, dtype=torch.uint8, device="cuda")
d2 = torch.empty(nb, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
res = {}
for name in ["h2d", "d2h", "both"]:
    for rep in range(3):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        s1.wait_event(e0); s2.wait_event(e0)
        if name in ("h2d", "both"):
            with torch.cuda.stream(s1):
                d1.copy_(h1, non_blocking=True)
        if name in ("d2h", "both"):
            with torch.cuda.stream(s2):
                h2.copy_(d2, non_blocking=True)
        torch.cuda.current_stream().wait_stream(s1); torch.cuda.current_stream().wait_stream(s2)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
    res[name] = {"ms": ms, "GB_s_per_direction": nb / ms / 1e6}
print(json.dumps(res))
