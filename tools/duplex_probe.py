"""Do H2D and D2H copies of one cfg2 step (1.23 MB each) overlap on this box?"""
import torch
n = 32 * 24 * 400
h_in = [torch.empty(n, dtype=torch.float32).pin_memory() for _ in range(2)]
h_out = [torch.empty(n, dtype=torch.float32).pin_memory() for _ in range(2)]
d_in = [torch.empty(n, device="cuda") for _ in range(2)]
d_out = [torch.empty(n, device="cuda") for _ in range(2)]
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def run(overlap, iters=400):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for k in range(iters):
        if overlap:
            with torch.cuda.stream(s1):
                d_in[k % 2].copy_(h_in[k % 2], non_blocking=True)
            with torch.cuda.stream(s2):
                h_out[k % 2].copy_(d_out[k % 2], non_blocking=True)
        else:
            d_in[k % 2].copy_(h_in[k % 2], non_blocking=True)
            h_out[k % 2].copy_(d_out[k % 2], non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(s2)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters * 1000
for _ in range(2):
    print("serial us/step", run(False), "overlap us/step", run(True))
