"""PCIe ceiling for the end-to-end lines: pinned host <-> device copies of config 4's step
volume (822 MB each way), one direction at a time and both at once on two streams."""
import json
import torch

n = 822083584 // 4
h_up = torch.empty(n, dtype=torch.float32).pin_memory()
h_dn = torch.empty(n, dtype=torch.float32).pin_memory()
d_up = torch.empty(n, dtype=torch.float32, device="cuda")
d_dn = torch.empty(n, dtype=torch.float32, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def both():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur)
    s2.wait_stream(cur)
    with torch.cuda.stream(s1):
        d_up.copy_(h_up, non_blocking=True)
    with torch.cuda.stream(s2):
        h_dn.copy_(d_dn, non_blocking=True)
    cur.wait_stream(s1)
    cur.wait_stream(s2)


t_h2d = timed(lambda: d_up.copy_(h_up, non_blocking=True))
t_d2h = timed(lambda: h_dn.copy_(d_dn, non_blocking=True))
t_both = timed(both)
gb = n * 4 / 1e9
print(json.dumps({"bytes_each_way": n * 4, "h2d_gbs": gb / (t_h2d * 1e-3), "d2h_gbs": gb / (t_d2h * 1e-3),
                  "both_ms": t_both, "both_gbs_each_way": gb / (t_both * 1e-3),
                  "cfg4_points_per_s_ceiling": 67108864 / (t_both * 1e-3)}))
