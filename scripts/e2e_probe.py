import sys, os, time
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import torch
from paper_2405_05751_b200 import fixtures as F
from paper_2405_05751_b200.api import Context
from test_fused_gpu import make_inputs
ctx = Context(0)
for name in ["rmsnorm", "lora", "gatedmlp"]:
    _, mu = F.bench_pair(name)
    g = ctx.compile(mu)
    host = [x.pin_memory() for x in make_inputs(name, F.BENCH[name]["args"])]
    outs = [torch.empty(F.BENCH[name]["args"][0], mu["tensors"][mu["outputs"][0]]["shape"][-1]).pin_memory()] if False else None
    want = ctx.eval_mugraph_host(g, host)
    out_h = [torch.empty_like(want[0]).pin_memory()]
    st = torch.cuda.Stream()
    for i in range(5): ctx.eval_mugraph_host(g, host, outputs=out_h, stream=st.cuda_stream)
    torch.cuda.synchronize()
    t0 = time.perf_counter(); n = 50
    for i in range(n): ctx.eval_mugraph_host(g, host, outputs=out_h, stream=st.cuda_stream)
    t1 = time.perf_counter()
    dev = [torch.empty_like(x, device='cuda') for x in host]
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    for i in range(n):
        for d, x in zip(dev, host): d.copy_(x, non_blocking=True)
        torch.cuda.synchronize()
    t3 = time.perf_counter()
    nb = sum(x.numel()*2 for x in host)
    print(f"{name}: e2e {(t1-t0)/n*1e3:.3f} ms/call, raw H2D {(t3-t2)/n*1e3:.3f} ms ({nb/((t3-t2)/n)/1e9:.1f} GB/s), bytes {nb}")
