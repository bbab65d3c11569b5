"""Is the DRAM write traffic ncu attributes to the 134-235 MB fused kernels
theirs?  A pure read (torch sum) of a 235 MB buffer after the same kind of
setup (buffers just written by the host copies / fills) is profiled the same
way: if it also 'writes' MBs, the bytes are write-backs of dirty L2 lines
evicted by the stream."""
import torch
n = 235_405_312 // 2
bufs = [torch.ones(n, dtype=torch.bfloat16, device="cuda") for _ in range(3)]  # fills: dirty L2
torch.cuda.synchronize()
for i in range(3):
    s = bufs[i].sum()  # reads 235 MB, writes one scalar
torch.cuda.synchronize()
print(float(s))
