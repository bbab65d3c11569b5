#!/usr/bin/env python
"""Steady-state per-launch phase timeline of the fused kernels (GPU box):
K back-to-back evaluations replayed as one CUDA graph (as bench.py times
them), every launch stamping its own slot of the debug ring
(TPO_DEBUG_RING=1, csrc/host/fused.cpp).  Prints, per launch, each phase's
min / max over CTAs in µs relative to the previous launch's first start.

  TPO_DEBUG_RING=1 python scripts/ring_timeline.py rmsnorm [STATIC=1] [ENV=VAL ...]
"""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
os.environ["TPO_DEBUG_RING"] = "1"
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2405_05751_b200 import _native  # noqa: E402
from paper_2405_05751_b200 import fixtures as F  # noqa: E402
from paper_2405_05751_b200.api import Context  # noqa: E402
from test_fused_gpu import make_inputs  # noqa: E402

WEIGHTS = {"gatedmlp": [1, 2], "rmsnorm": [1, 2, 3], "lora": [1, 2, 3], "gqa": []}
NAMES = {0: "start", 1: "setup", 8: "first_full", 9: "b_ready", 10: "last_tma", 3: "last_mma",
         5: "tmem_full", 4: "sent", 6: "recv_done", 11: "owner_done", 2: "epi_done", 7: "end"}
RING, CTAS = 16, 4096


def main():
    name = sys.argv[1]
    static = False
    for kv in sys.argv[2:]:
        k, v = kv.split("=")
        if k == "STATIC":
            static = v == "1"
        else:
            os.environ[k] = v
    ctx = Context(0)
    _, mu = F.bench_pair(name)
    g = ctx.compile(mu)
    if static:
        g.set_static_inputs(WEIGHTS[name])
    host = make_inputs(name, F.BENCH[name]["args"], seed=3)
    in_b = sum(x.numel() * 2 for x in host)
    copies = max(1, -(-3 * 126 * 2**20 // in_b))
    sets = [[x.cuda() for x in host] for _ in range(copies)]
    st = torch.cuda.Stream()
    outs = None
    with torch.cuda.stream(st):
        outs = [ctx.eval_mugraph(g, sets[i % copies], stream=st.cuda_stream)[0] for i in range(copies)]
    st.synchronize()
    K = RING
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=st):
        for i in range(K):
            ctx.eval_mugraph(g, sets[i % copies], outputs=[outs[i % copies]],
                             stream=torch.cuda.current_stream().cuda_stream)
    lib = _native.lib()
    lib.tpo_debug_ring_read.restype = ctypes.c_int
    buf = np.zeros(RING * CTAS * 16, dtype=np.uint64)
    for rep in range(3):
        graph.replay()
        torch.cuda.synchronize()
        seq = lib.tpo_debug_ring_read(buf.ctypes.data_as(ctypes.c_void_p), ctypes.c_size_t(buf.size))
    h = buf.reshape(RING, CTAS, 16).astype(np.int64)
    # launch order inside the ring: seq counts every launch (capture included)
    first = seq - K
    order = [(first + i) % RING for i in range(K)]
    starts = []
    for slot in order:
        s0 = h[slot, :, 0]
        starts.append(s0[s0 > 0].min())
    ends = []
    print(f"{name} static={static} env={[a for a in sys.argv[2:]]}")
    for i, slot in enumerate(order):
        ref = starts[i - 1] if i else starts[0]
        row = []
        for k in (0, 1, 8, 10, 3, 5, 11, 7):
            v = h[slot, :, k]
            v = v[v > 0]
            if len(v):
                row.append(f"{NAMES[k]} {(v.min() - ref) / 1e3:6.2f}/{(v.max() - ref) / 1e3:6.2f}")
        e = h[slot, :, 7]
        ends.append(e[e > 0].max())
        print(f"  launch {i:2d}: " + "  ".join(row))
    # critical path per launch: previous launch's last CTA end -> this
    # launch's first full stage -> its last MMA -> its last CTA end
    ph = {k: [] for k in ("wait_to_first", "stream", "tail", "resident_before_prev_end")}
    for i in range(3, K):
        a, b = order[i - 1], order[i]
        pe = h[a, :, 7][h[a, :, 7] > 0].max()
        ff = h[b, :, 8][h[b, :, 8] > 0]
        lmv = h[b, :, 3][h[b, :, 3] > 0]
        if not len(lmv):  # GQA stamps o_full (slot 5) instead of the last MMA
            lmv = h[b, :, 5][h[b, :, 5] > 0]
        lm = lmv.max()
        en = h[b, :, 7][h[b, :, 7] > 0].max()
        st0 = h[b, :, 0][h[b, :, 0] > 0]
        ph["wait_to_first"].append((np.median(ff) - pe) / 1e3)
        ph["stream"].append((lm - np.median(ff)) / 1e3)
        ph["tail"].append((en - lm) / 1e3)
        ph["resident_before_prev_end"].append((pe - np.median(st0)) / 1e3)
    print("  " + "  ".join(f"{k} {np.mean(v):.2f}" for k, v in ph.items()))
    # skew of the last MMA over CTAs: within a cluster (the owner waits for
    # its slowest peer) and over the grid; "balanced" = the grid's last MMA
    # if every cluster's K blocks were shared evenly among its CTAs
    S = int(os.environ.get("TPO_KSPLIT", "4"))
    sk = {k: [] for k in ("cluster_spread", "grid_spread", "gain_if_cluster_balanced", "start_spread", "first_full_spread")}
    for i in range(3, K):
        b = order[i]
        n = int((h[b, :, 0] > 0).sum())
        lm = h[b, :n, 3].astype(np.float64).reshape(-1, S) / 1e3
        if (lm <= 0).any():
            continue
        sk["cluster_spread"].append(np.mean(lm.max(1) - lm.min(1)))
        sk["grid_spread"].append(lm.max() - lm.min())
        sk["gain_if_cluster_balanced"].append(lm.max() - lm.mean(1).max())
        sk["start_spread"].append((h[b, :n, 0].max() - h[b, :n, 0].min()) / 1e3)
        ff = h[b, :n, 8]
        sk["first_full_spread"].append((ff.max() - ff.min()) / 1e3)
    if sk["grid_spread"]:
        print("  skew " + "  ".join(f"{k} {np.mean(v):.2f}" for k, v in sk.items()))
    # placement: CTAs of the same launch sharing an SM (slot 14 = smid + 1)
    # and whether they are the stragglers of the last MMA
    pl = {"ctas_doubled": [], "lm_doubled": [], "lm_single": []}
    for i in range(3, K):
        b = order[i]
        n = int((h[b, :, 0] > 0).sum())
        sm = h[b, :n, 14]
        if (sm <= 0).any():
            continue
        lm = h[b, :n, 3].astype(np.float64) / 1e3
        if (lm <= 0).any():
            continue
        cnt = np.bincount(sm.astype(np.int64))
        dbl = cnt[sm] > 1
        pl["ctas_doubled"].append(int(dbl.sum()))
        rel = lm - lm.min()
        if dbl.any():
            pl["lm_doubled"].append(rel[dbl].mean())
        if (~dbl).any():
            pl["lm_single"].append(rel[~dbl].mean())
    if pl["ctas_doubled"]:
        print("  placement " + "  ".join(f"{k} {np.mean(v):.2f}" for k, v in pl.items() if v))
    # tail sub-phases per CTA, relative to the CTA's own last MMA (median over
    # CTAs and launches): MMA completion, DSMEM send / receive, owner store,
    # teardown
    sub = {5: "tmem_full", 4: "sent", 6: "recv_done", 15: "summed", 11: "owner_done", 2: "epi_done", 13: "pre_sync",
           12: "synced", 7: "end"}
    acc = {k: [] for k in sub}
    for i in range(3, K):
        b = order[i]
        n = int((h[b, :, 0] > 0).sum())
        lm = h[b, :n, 3]
        for k in sub:
            v = h[b, :n, k]
            ok = (v > 0) & (lm > 0)
            if ok.any():
                acc[k].append(np.median((v[ok] - lm[ok]) / 1e3))
    print("  tail(per CTA, from its last MMA) " + "  ".join(f"{sub[k]} {np.mean(v):.2f}" for k, v in acc.items() if v))
    per = np.diff(np.array(ends[2:], dtype=np.float64)) / 1e3
    print(f"  period (end to end) mean {per.mean():.2f} us  min {per.min():.2f}  max {per.max():.2f}")


if __name__ == "__main__":
    main()
