#!/usr/bin/env python
"""Benchmark: fused µGraph evaluation on B200 (+ the batched Z_p×Z_q verifier).

BASELINE.json metric: "fused μGraph latency µs & % roofline; Z_p-verified
candidates/s at 1/2/4/8 GPU".  The N=1 workload is configs[1], the GatedMLP
µGraph SiLU(xW1)⊙(xW3), x 8×4096, W 4096×14336, bf16 in / fp32 accumulate /
fp32 out (grid 112, for-loop 16).  One step = one evaluation of that µGraph =
one fused sm_100a kernel launch.  `value` is whole-job throughput in µGraph
evaluations/s (replicas on every rank: the fused kernel does not shard,
"scaling": "weak").  Two latencies, named for what they are:
`period_us` = the steady-state period of back-to-back evaluations in one
CUDA graph (PDL overlaps neighbours; `timeline` has every launch's start and
end), `isolated_us` = one launch after an L2 flush.  The weights (235 MB)
exceed the 126 MB L2, so every step streams them from HBM; smaller
workloads rotate through enough input copies to exceed L2.

`fused` carries the same record (period, isolated latency, rooflines, e2e
through the C-ABI with host buffers, the fp32-input split path, launch
timeline, CPU reference) for all four benchmark µGraphs.  The "verifier"
object reports the sharded Z_p×Z_q verification throughput (candidates/s
over all ranks, one all-gather of packed accept words) on the SURVEY §8d
candidate pools, with the reference on all host cores beside it.
`--workload verify` makes the verifier the headline instead.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--workload gatedmlp|rmsnorm|lora|gqa|verify]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "fused μGraph latency µs & % roofline; Z_p-verified candidates/s at 1/2/4/8 GPU"
L2_BYTES = 126 * 1024 * 1024
STATIC_WEIGHTS = {"gatedmlp": [1, 2], "rmsnorm": [1, 2, 3], "lora": [1, 2, 3], "gqa": []}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# --------------------------------------------------------------------------- dist
class Dist:
    def __init__(self, n_gpus):
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        self.pg = None
        # TPO_BENCH_SHARED_GPU=1 (logic check only, never a bench number):
        # every rank on cuda:0 over gloo, so the N>1 paths run on a 1-GPU box
        shared = os.environ.get("TPO_BENCH_SHARED_GPU") == "1"
        if shared:
            self.local = 0
        if self.world > 1:
            import torch.distributed as dist
            import torch
            torch.cuda.set_device(self.local)
            if shared:
                dist.init_process_group("gloo")
            else:
                dist.init_process_group("nccl", device_id=torch.device("cuda", self.local))
            self.pg = dist

    def barrier(self):
        if self.pg:
            self.pg.barrier()

    def max(self, x: float) -> float:
        if not self.pg:
            return x
        import torch
        t = torch.tensor([x], device="cuda", dtype=torch.float64)
        self.pg.all_reduce(t, op=self.pg.ReduceOp.MAX)
        return float(t.item())

    def sum(self, x: float) -> float:
        if not self.pg:
            return x
        import torch
        t = torch.tensor([x], device="cuda", dtype=torch.float64)
        self.pg.all_reduce(t)
        return float(t.item())

    def close(self):
        if self.pg:
            self.pg.destroy_process_group()


# ------------------------------------------------------------------------- clocks
class Clocks:
    """nvidia-smi sampling of SM clock + throttle reasons during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, dev):
        self.dev, self.proc, self.lines = dev, None, []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.dev), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=2)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                mx.append(float(f[1]))
            except ValueError:
                continue
            for nm, v in zip(names, f[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        busy = [s for s in sm if mx and s > 0.5 * max(mx)] or sm
        return {"sm_mhz": statistics.median(busy) if busy else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm)}


# --------------------------------------------------------------------- workloads
def fused_workload(name):
    if name in fused_workload.cache:
        return fused_workload.cache[name]
    from paper_2405_05751_b200 import fixtures as F
    prog, mu = F.bench_pair(name)
    args = F.BENCH[name]["args"]
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from test_fused_gpu import make_inputs
    host = make_inputs(name, args, seed=0)
    in_bytes = sum(x.numel() * 2 for x in host)
    out_shape = [mu["tensors"][t]["shape"] for t in mu["outputs"]][0]
    out_bytes = int(np.prod(out_shape)) * 4
    wl = dict(name=name, prog=prog, mu=mu, host=host, in_bytes=in_bytes, out_bytes=out_bytes,
              out_shape=out_shape, args=args, grid=F.BENCH[name]["grid"],
              forloop=F.BENCH[name]["forloop"])
    fused_workload.cache[name] = wl
    return wl


fused_workload.cache = {}


def numa_bind(dev):
    """Restrict this process to the CPUs NVML reports local to CUDA device
    `dev` (matched by PCI bus id); returns the previous affinity, or None
    when unavailable."""
    try:
        import pynvml
        import torch
        prop = torch.cuda.get_device_properties(dev)
        ids = [getattr(prop, k, None) for k in ("pci_domain_id", "pci_bus_id", "pci_device_id")]
        if not all(isinstance(x, int) for x in ids):
            return None
        bus = "%04x:%02x:%02x.0" % tuple(ids)  # NVML's domain:bus:device.function
        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByPciBusId(bus.encode())
        words = pynvml.nvmlDeviceGetCpuAffinity(h, (os.cpu_count() + 63) // 64)
        cpus = {w * 64 + b for w, m in enumerate(words) for b in range(64) if (m >> b) & 1}
        prev = os.sched_getaffinity(0)
        cpus &= prev
        if not cpus or cpus == prev:
            return None
        os.sched_setaffinity(0, cpus)
        return prev
    except Exception:
        return None


def workload_label(wl):
    """config.workload of both arms (ours and --impl reference)."""
    return (f"{wl['name']} µGraph, inputs {[list(x.shape) for x in wl['host']]}, grid {wl['grid']}, "
            f"loop {wl['forloop']} (BASELINE.json configs)")


RING, RING_CTAS = 16, 4096


def launch_timeline(ctx, g, sets, outs, stream):
    """Per-launch start / end of 16 back-to-back evaluations replayed as one
    CUDA graph (as the timed region runs them): every launch stamps its own
    slot of the library's %globaltimer ring (TPO_DEBUG_RING) — first CTA
    start and last CTA end per launch.  A launch starting before its
    predecessor ends is the PDL overlap that makes the period shorter than
    one kernel's duration."""
    import ctypes
    import torch
    from paper_2405_05751_b200 import _native
    os.environ["TPO_DEBUG_RING"] = "1"
    try:
        copies = len(sets)
        # one eager launch allocates the ring (no allocation inside a capture)
        ctx.eval_mugraph(g, sets[0], outputs=[outs[0]], stream=stream.cuda_stream)
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=stream):
            for i in range(RING):
                ctx.eval_mugraph(g, sets[i % copies], outputs=[outs[i % copies]],
                                 stream=torch.cuda.current_stream().cuda_stream)
        lib = _native.lib()
        lib.tpo_debug_ring_read.restype = ctypes.c_int
        buf = np.zeros(RING * RING_CTAS * 16, dtype=np.uint64)
        seq = 0
        for _ in range(3):
            graph.replay()
            torch.cuda.synchronize()
            seq = lib.tpo_debug_ring_read(buf.ctypes.data_as(ctypes.c_void_p), ctypes.c_size_t(buf.size))
        del graph
    finally:
        os.environ.pop("TPO_DEBUG_RING", None)
    h = buf.reshape(RING, RING_CTAS, 16).astype(np.int64)
    order = [(seq - RING + i) % RING for i in range(RING)]
    se = []
    for slot in order:
        s0, e7 = h[slot, :, 0], h[slot, :, 7]
        se.append((s0[s0 > 0].min(), e7[e7 > 0].max()))
    t0 = se[0][0]
    launches = [[round((s - t0) / 1e3, 2), round((e - t0) / 1e3, 2)] for s, e in se]
    steady = se[3:]
    dur = [(e - s) / 1e3 for s, e in steady]
    period = [(steady[i + 1][0] - steady[i][0]) / 1e3 for i in range(len(steady) - 1)]
    overlap = [(steady[i][1] - steady[i + 1][0]) / 1e3 for i in range(len(steady) - 1)]
    return {"launches_us": launches, "mean_kernel_us": round(float(np.mean(dur)), 3),
            "mean_period_us": round(float(np.mean(period)), 3),
            "mean_overlap_us": round(float(np.mean(overlap)), 3),
            "overlapping_launches": int(sum(o > 0 for o in overlap)),
            "note": "first CTA start / last CTA end per launch (%globaltimer ring, launches 3-15 "
                    "steady state); overlap = predecessor's end - this launch's start"}


def measure_fused(args, dist, wl, headline=False):
    """One benchmark µGraph on this rank's GPU:
    * period_us: K evaluations back to back, replayed as one CUDA graph
      (CUDA events on the launching stream), inputs rotated over enough
      copies to exceed L2 — the pipelined steady state (PDL lets one
      evaluation's prologue and weight prefetch overlap the previous one);
    * isolated_us: ONE launch after an L2 flush (a 256 MB write), median of
      20 — the single-evaluation latency;
    * e2e: tpo_gpu_eval_mugraph_host with pinned host buffers (copies in the
      timed region);
    * fp32_inputs: the same evaluation from fp32 device buffers (precision
      policy AUTO: on-device split into bf16 hi + lo, then the SPLIT kernel);
    * timeline: per-launch start / end of 16 graph launches."""
    import torch
    from paper_2405_05751_b200.api import Context
    dev = dist.local
    torch.cuda.set_device(dev)
    ctx = Context(dev)
    g = ctx.compile(wl["mu"])
    if not g.fused:
        raise RuntimeError("benchmark µGraph did not lower to a fused kernel")
    # Weight inputs are parameters: nothing enqueued before an evaluation
    # writes them, which lets the kernel stream them before its PDL wait
    # (tpo_gpu_graph_set_static_inputs).  Activations (X, Q, K/V cache) stay
    # ordered after the preceding kernel.
    if not args.no_static:
        g.set_static_inputs(STATIC_WEIGHTS[wl["name"]])
    alg = wl["in_bytes"] + wl["out_bytes"]
    copies = max(1, -(-3 * L2_BYTES // wl["in_bytes"])) if wl["in_bytes"] < 3 * L2_BYTES else 1
    sets = [[x.cuda() for x in wl["host"]] for _ in range(copies)]
    outs = [torch.empty(wl["out_shape"], device="cuda", dtype=torch.float32) for _ in range(copies)]
    stream = torch.cuda.Stream()
    st = stream.cuda_stream

    def step(i):
        ctx.eval_mugraph(g, sets[i % copies], outputs=[outs[i % copies]], stream=st)

    with torch.cuda.stream(stream):
        for i in range(args.warmup):
            step(i)
    torch.cuda.synchronize()
    dist.barrier()
    clocks = Clocks(dev) if headline else None
    if clocks:
        clocks.start()
        time.sleep(0.1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    # keep the GPU busy long enough for the clock sampler to see it
    hot_until = time.time() + (0.3 if headline and not args.profile else 0.0)
    i = 0
    with torch.cuda.stream(stream):
        while time.time() < hot_until:
            step(i)
            i += 1
            if i % 64 == 0:
                stream.synchronize()
    # ---- pipelined period: the K evaluations captured once into a CUDA graph
    # (the kernels are µs-scale: host launch overhead must not sit between them)
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=stream):
        for i in range(args.steps):
            ctx.eval_mugraph(g, sets[i % copies], outputs=[outs[i % copies]],
                             stream=torch.cuda.current_stream().cuda_stream)
    graph.replay()  # warm the graph itself
    torch.cuda.synchronize()
    dist.barrier()
    torch.cuda.synchronize()
    with torch.cuda.stream(stream):
        e0.record(stream)
        graph.replay()
        e1.record(stream)
    e1.synchronize()
    torch.cuda.synchronize()
    dist.barrier()
    ms_local = e0.elapsed_time(e1)
    clk = clocks.stop() if clocks else None
    del graph
    ms = dist.max(ms_local)
    per_eval_ms = ms / args.steps
    value = dist.world * args.steps / (ms / 1e3)
    peak, peak_kind = peaks()
    achieved = alg / (per_eval_ms / 1e3) / 1e9
    roof = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
            "frac": round(achieved / peak, 4), "traffic": None, "peak_source": peak_kind,
            "algorithmic_bytes": int(alg), "basis": "pipelined period"}
    prof = os.path.join(ROOT, "profiles", f"traffic_{wl['name']}.json")
    if os.path.exists(prof):
        try:
            roof["traffic"] = json.load(open(prof))["dram_bytes_per_launch"]
        except Exception:
            pass
    res = dict(name=wl["name"], value=value, ms=per_eval_ms, roof=roof, clocks=clk,
               gpu_launches=args.steps, copies=copies)
    if args.profile:
        return res
    # ---- isolated single-evaluation latency: L2 flushed, one launch
    # the flush READS 256 MB (> the 126 MB L2): L2 then holds clean lines of
    # another buffer (a write flush would leave 126 MB of dirty lines to be
    # written back during the measured launch)
    flush = torch.ones(32 * 2**20, dtype=torch.int64, device="cuda")
    iso = []
    with torch.cuda.stream(stream):
        for i in range(20):
            flush.sum()
            e0.record(stream)
            step(i)
            e1.record(stream)
            e1.synchronize()
            iso.append(e0.elapsed_time(e1))
    del flush
    iso_ms = float(np.median(iso))
    res["isolated_us"] = round(iso_ms * 1e3, 3)
    res["roofline_isolated"] = {"achieved": round(alg / (iso_ms / 1e3) / 1e9, 1), "peak": peak,
                                "unit": "GB/s", "frac": round(alg / (iso_ms / 1e3) / 1e9 / peak, 4),
                                "basis": "one launch after a 256 MB read (L2 flushed), median of 20"}
    # ---- per-launch timeline of the pipelined graph
    try:
        res["timeline"] = launch_timeline(ctx, g, sets, outs, stream)
    except Exception as e:  # evidence only; never fails the bench
        res["timeline"] = {"error": str(e)[:200]}
    # ---- fp32 device inputs: precision policy AUTO (split kernel)
    f32 = [[x.float().cuda() for x in wl["host"]]]
    n32 = max(1, -(-3 * L2_BYTES // (2 * wl["in_bytes"]))) if 2 * wl["in_bytes"] < 3 * L2_BYTES else 1
    f32 += [[x.clone() for x in f32[0]] for _ in range(n32 - 1)]
    g32 = ctx.compile(wl["mu"])
    with torch.cuda.stream(stream):
        for i in range(3):
            ctx.eval_mugraph(g32, f32[i % n32], outputs=[outs[i % copies]], stream=st)
        torch.cuda.synchronize()
        k32 = max(10, min(args.steps, 50))
        e0.record(stream)
        for i in range(k32):
            ctx.eval_mugraph(g32, f32[i % n32], outputs=[outs[i % copies]], stream=st)
        e1.record(stream)
    e1.synchronize()
    del f32
    res["fp32_inputs"] = {"us_per_eval": round(e0.elapsed_time(e1) / k32 * 1e3, 2),
                          "precision": "TPO_PREC_AUTO: on-device split into bf16 hi + lo planes, SPLIT kernel "
                                       "(meets 1e-3·max(|r|, rms) vs the double reference on arbitrary inputs)",
                          "note": "includes the per-call conversion kernels (fp32 read, 2 planes written)"}
    # ---- end to end through the C-ABI with HOST buffers: every step copies
    # that step's inputs host->device (pinned), runs the fused kernel and
    # copies the output back (tpo_gpu_eval_mugraph_host, synchronous).
    # Host buffers on the GPU's NUMA node (pinned pages are placed where the
    # allocating thread runs): the H2D copies then run at the link rate
    prev_aff = numa_bind(dev)
    pinned = [x.pin_memory() for x in wl["host"]]
    out_h = torch.empty(wl["out_shape"], dtype=torch.float32).pin_memory()
    e2e_steps = max(3, min(args.steps, 50 if headline else 20))
    ctx.eval_mugraph_host(g, pinned, outputs=[out_h], stream=st)  # warm the staging buffers
    torch.cuda.synchronize()
    dist.barrier()
    with torch.cuda.stream(stream):
        e0.record(stream)
        for i in range(e2e_steps):
            ctx.eval_mugraph_host(g, pinned, outputs=[out_h], stream=st)
        e1.record(stream)
    e1.synchronize()
    dist.barrier()
    e2e_ms = max(dist.max(e0.elapsed_time(e1)), 1e-9)
    if prev_aff is not None:
        os.sched_setaffinity(0, prev_aff)
    res["e2e"] = {"value": round(dist.world * e2e_steps / (e2e_ms / 1e3), 3), "unit": "evals/s",
                  "h2d_bytes_per_step": int(wl["in_bytes"]), "d2h_bytes_per_step": int(wl["out_bytes"]),
                  "ms_per_step": round(e2e_ms / max(e2e_steps, 1), 4),
                  "numa_bound": prev_aff is not None,
                  "path": "tpo_gpu_eval_mugraph_host (C-ABI, pinned host buffers, copies in the timed region)"}
    return res


def fused_object(r, cpu):
    """The per-family record of the JSON line."""
    out = {"workload": workload_label(fused_workload.cache[r["name"]]),
           "period_us": round(r["ms"] * 1e3, 3), "isolated_us": r.get("isolated_us"),
           "value": round(r["value"], 2), "unit": "evals/s", "roofline": r["roof"],
           "roofline_isolated": r.get("roofline_isolated"), "e2e": r.get("e2e"),
           "fp32_inputs": r.get("fp32_inputs"), "timeline": r.get("timeline"),
           "cpu_baseline": cpu, "gpu_launches": r["gpu_launches"]}
    return out


def cpu_baseline_fused(wl, threads=1, min_seconds=10.0, min_reps=1):
    """The compiled reference (oracle/_ref) eval_mugraph on the host CPU."""
    from oracle import ref
    if not ref.available():
        return None
    ins = [x.float().numpy().astype(np.float64) for x in wl["host"]]
    reps, total = 0, 0.0
    while (total < min_seconds * 1e3 or reps < min_reps) and reps < 50:
        total += ref.time_eval_mugraph(wl["mu"], ins, 1)
        reps += 1
    per = total / reps
    return {"value": round(1e3 / per, 5), "unit": "evals/s", "cores": threads, "kind": "reference",
            "sample": f"{reps} full eval_mugraph call(s) of the {wl['name']} µGraph, 1 thread "
                      f"(the reference is single-threaded), {per:.0f} ms each",
            "ms_per_eval": round(per, 1)}


def generic_vm(wl, reps=3):
    """The same µGraph (and its flat program) on the generic GPU VM in the
    reference's own arithmetic (tpo_gpu_eval_vm: fp64 / fp32, the reference's
    operation order; the global-memory executor at these sizes) — the path
    any µGraph without a hand-written kernel takes.  Device time per call
    (CUDA events; inputs already in one flat device buffer), wall clock per
    call with host buffers, and the HBM fraction of the device time for the
    unique input + output bytes in that dtype."""
    import ctypes as C
    import torch
    from paper_2405_05751_b200 import _native as N
    from paper_2405_05751_b200.api import Context
    ctx = Context(0)
    ins = [x.float().numpy().astype(np.float64) for x in wl["host"]]
    peak = peaks()[0]
    out = {}
    for tag, g, mode in (("eval_mugraph", wl["mu"], 0), ("eval_program", wl["prog"], 1),
                         ("eval_mugraph_f32", wl["mu"], 2)):
        gg = ctx.compile(g)
        dt, npdt = (torch.float32, np.float32) if mode == 2 else (torch.float64, np.float64)
        hin = [x.astype(npdt) for x in ins]
        ctx.eval_vm(gg, hin, mode=mode)  # warm
        t0 = time.perf_counter()
        for _ in range(reps):
            ctx.eval_vm(gg, hin, mode=mode)
        wall = (time.perf_counter() - t0) / reps * 1e3
        flat = torch.cat([torch.from_numpy(x).reshape(-1) for x in hin]).to(dt).cuda()
        n_out = sum(int(np.prod(sh)) for sh in gg.shapes(True))
        dout = torch.empty(n_out, dtype=dt, device="cuda")
        st = torch.cuda.current_stream()

        def run():
            N.check(N.lib().tpo_gpu_eval_vm_dev(ctx.h, gg.h, mode, C.c_void_p(flat.data_ptr()),
                                                C.c_void_p(dout.data_ptr()), C.c_void_p(st.cuda_stream)))
        run()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(reps):
            run()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        nbytes = int(flat.numel() * flat.element_size() + n_out * dout.element_size())
        out[tag] = {"device_ms_per_eval": round(ms, 3), "host_buffers_ms_per_eval": round(wall, 3),
                    "dtype": "f32" if mode == 2 else "f64", "h2d_bytes": int(sum(x.nbytes for x in hin)),
                    "hbm_frac": round(nbytes / (ms * 1e-3) / (peak * 1e9), 4) if peak else None}
    out["note"] = ("bit-exact with the reference for graphs without exp (tests/test_fp_vm_gpu.py); "
                   "f32 = the reference's eval_mugraph_f32 semantics")
    return out


def reference_arm(args, wl):
    """--impl reference: the reference's eval_mugraph using all host cores, each
    thread evaluating the µGraph restricted to a slice of output columns
    (grid blocks are independent, eval_core.hpp:234-237)."""
    from oracle import ref
    from paper_2405_05751_b200 import fixtures as F
    name = wl["name"]
    cores = os.cpu_count() or 1
    if name == "gatedmlp":
        b, h, n = wl["args"]
        grid = wl["grid"]
        T = max(t for t in range(1, cores + 1) if grid % t == 0)
        ns = n // T
        X, W1, W3 = [x.float().numpy().astype(np.float64) for x in wl["host"]]
        graphs, inputs = [], []
        for t in range(T):
            graphs.append(F.gatedmlp_mugraph(b, h, ns, grid // T, wl["forloop"]))
            sl = slice(t * ns, (t + 1) * ns)
            inputs.append([X, np.ascontiguousarray(W1[:, sl]), np.ascontiguousarray(W3[:, sl])])
    elif name in ("rmsnorm", "lora"):
        T = 1
        graphs = [wl["mu"]]
        inputs = [[x.float().numpy().astype(np.float64) for x in wl["host"]]]
    else:
        T = 1
        graphs = [wl["mu"]]
        inputs = [[x.float().numpy().astype(np.float64) for x in wl["host"]]]
    for _ in range(args.warmup and 1):
        ref.time_eval_parallel(graphs, inputs, 1)
    times = [ref.time_eval_parallel(graphs, inputs, 1) for _ in range(max(1, args.steps))]
    ms = float(np.mean(times))
    v = round(1e3 / ms, 5)
    # n_gpus: the launch's N (the driver runs both arms alike); the work runs
    # on rank 0's host cores only ("cpu_baseline.cores")
    return {"metric": METRIC, "value": v, "unit": "evals/s", "n_gpus": args.gpus, "steps": len(times),
            "warmup": args.warmup, "ms_per_step": round(ms, 3), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "impl": "reference",
            "config": {"workload": workload_label(wl), "threads": T},
            "cpu_baseline": {"value": v, "unit": "evals/s", "cores": T, "kind": "reference",
                             "sample": f"full µGraph per step: reference eval_mugraph on {T} "
                                       f"column slice(s) concurrently"},
            "e2e": {"value": v, "unit": "evals/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}


# ------------------------------------------------------------------------- verifier
def run_verify(dist, n_total, steps=1, warmup=3, pool_fams=("rmsnorm", "gatedmlp", "gqa", "lora")):
    """Shard n_total candidates (n_total / 4 per family; candidate i of a
    family = pool[i % |pool|], seed i) across ranks: the four families'
    packed accept bits share one word space (shard.WordLayout) and each rank
    owns one contiguous word range, balanced by the per-candidate cost
    measured in the warm-up; it verifies its ranges on its GPU (one
    tpo_gpu_verify_pool launch per family segment) into ONE local buffer, and
    the step ends with ONE all-gather of it.  Timed leg: the verify kernels
    plus the gather, CUDA events, max over ranks; the host unpack follows
    outside it.  One step = all n_total candidates."""
    import hashlib
    import torch
    from paper_2405_05751_b200 import fixtures as F
    from paper_2405_05751_b200 import shard
    from paper_2405_05751_b200.api import Context
    ctx = Context(dist.local)
    fams = F.verify_families()
    per_fam = n_total // len(pool_fams)
    fam_jobs = []
    for f in pool_fams:
        prog, pool = fams[f]
        gp = ctx.compile(prog)
        gs = [ctx.compile(g) for _, g in pool]
        fam_jobs.append((f, gp, gs))
    layout = shard.WordLayout([per_fam] * len(fam_jobs))
    # warm-up (compile / upload paths, clocks) doubling as the cost probe:
    # seconds per candidate of each family, averaged over ranks so every rank
    # derives the same ranges
    probe = min(per_fam, 8192)
    scratch = torch.zeros(max(1, -(-probe // 32)), dtype=torch.int32, device="cuda")
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    cost = []
    for w in range(max(warmup, 1)):
        cost = []
        for f, gp, gs in fam_jobs:
            e0.record()
            ctx.verify_pool(gp, gs, first=0, n=probe, accept_dev=scratch)
            e1.record()
            torch.cuda.synchronize()
            cost.append(dist.sum(e0.elapsed_time(e1)) / dist.world / probe)
    ranges = layout.rank_words(layout.word_costs(cost), dist.world)
    w0, nw = ranges[dist.rank]
    jobs = layout.jobs(w0, nw)
    local = torch.zeros(max(nw, 1), dtype=torch.int32, device="cuda")
    g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t_kernel = t_gather = 0.0
    attempts = 0
    words = None
    for step in range(steps):
        dist.barrier()
        torch.cuda.synchronize()
        e0.record()
        attempts = 0
        for fi, first, n, off in jobs:
            _, gp, gs = fam_jobs[fi]
            _, att = ctx.verify_pool(gp, gs, first=first, n=n, accept_dev=local[off:])
            attempts += att
        e1.record()
        g0.record()
        words = shard.gather_words(local[:nw], ranges, dist.pg)  # the single collective
        g1.record()
        torch.cuda.synchronize()
        t_kernel += e0.elapsed_time(e1) / 1e3
        t_gather += g0.elapsed_time(g1) / 1e3
    t_local = t_kernel / steps
    t_all = dist.max((t_kernel + t_gather) / steps)
    gather_share = dist.max(t_gather / steps) / t_all
    # the collective alone: every rank's words ready (barrier + sync), then
    # the same gather — the timed leg's gather also absorbs rank skew
    dist.barrier()
    torch.cuda.synchronize()
    g0.record()
    shard.gather_words(local[:nw], ranges, dist.pg)
    g1.record()
    torch.cuda.synchronize()
    gather_pure_share = dist.max(g0.elapsed_time(g1) / 1e3) / t_all
    # host unpack, outside the timed leg
    host_words = words.cpu().numpy()
    accept = layout.unpack(host_words)
    accepted = int(sum(int(a.sum()) for a in accept))
    accept_sha = hashlib.sha256(np.ascontiguousarray(host_words).view(np.uint32).tobytes()).hexdigest()[:16]
    # end to end through the public API: verify_pool calls + accept bits to the host
    torch.cuda.synchronize()
    dist.barrier()
    w_0 = time.perf_counter()
    for fi, first, n, off in jobs:
        _, gp, gs = fam_jobs[fi]
        ctx.verify_pool(gp, gs, first=first, n=n, accept_dev=local[off:])
    local.cpu()
    e2e_s = dist.max(time.perf_counter() - w_0)
    e2e = {"value": round(per_fam * len(fam_jobs) / e2e_s, 1), "unit": "candidates/s",
           "h2d_bytes_per_step": int(sum(4 * len(gs) for _, _, gs in fam_jobs)),
           "d2h_bytes_per_step": int(layout.total_words * 4),
           "path": "Context.verify_pool (C-ABI tpo_gpu_verify_pool) + accept bits to host, wall clock; "
                   "inputs are generated on the device by design (h2d = pool map; bytecode ~KB)"}
    jobs = [(fam_jobs[fi][0], fam_jobs[fi][1], fam_jobs[fi][2], first, n) for fi, first, n, _ in jobs]
    n_done = per_fam * len(fam_jobs)
    stream = search_stream(ctx, dist, fams, pool_fams)
    native = search_native(ctx, dist) if dist.world == 1 else None
    stab = stability_stage(ctx, dist, fams, pool_fams)
    # algorithmic work: field MACs = 2 fields x (op_madds(program)
    # + op_madds(candidate)) per attempt the reference consumes; per-candidate
    # attempts from an untimed verdict pass over this rank's shard.  RNG work
    # (reported separately): 2 splitmix64 draws per input element
    # of the program's inputs per attempt, +1 for omega, +340 for the SiLU
    # tables when either graph has SiLU
    from paper_2405_05751_b200.graph import has_silu
    macs = draws = draws_eager = 0.0
    for f, gp, gs, first, n in jobs:
        v, _ = ctx.verify_pool(gp, gs, first=first, n=n, want_verdicts=True)
        draws += float(ctx.last_verify_draws())  # draws actually made (lazy input sampling)
        idx = (np.arange(first, first + n) % len(gs))
        cm = np.array([g.madds for g in gs], dtype=np.float64)[idx]
        att = (v["rounds_run"] + v["resamples"]).astype(np.float64)
        macs += float(np.sum(att * 2.0 * (gp.madds + cm)))
        silu = np.array([has_silu(g.spec) or has_silu(gp.spec) for g in gs])[idx]
        draws_eager += float(np.sum(att * (2.0 * gp.info.input_elems + 1 + 340.0 * silu)))
    macs = dist.sum(macs)
    draws = dist.sum(draws)
    draws_eager = dist.sum(draws_eager)
    peak = dp4a = None
    try:
        pk = json.load(open(os.path.join(ROOT, "profiles", "int_peak.json")))
        peak, dp4a = pk["imad_per_s"], pk.get("dp4a_per_s")
    except Exception:
        pass
    roof = {"bound": "int-issue (IMAD)", "achieved": round(macs / t_all / 1e12, 4),
            "peak": round(peak / 1e12, 3) if peak else None, "unit": "T field-MAC/s",
            "frac": round(macs / t_all / peak, 4) if peak else None, "traffic": None,
            "peak_source": "profiles/int_peak.json (measured IMAD/s, scripts/micro/int_peak.cu)",
            "field_macs": macs,
            "note": "peak per SURVEY §8d: measured IMAD rate (1 field MAC per IMAD). The 2x2 "
                    "matmul path uses dp4a (2 field MACs per instruction, frac_vs_dp4a_2lane). "
                    "Field MACs are a minority of the work: per attempt the inputs are "
                    "regenerated (2 splitmix64 draws + a mod per element, the rng term) and "
                    "both graphs interpreted; see issue_utilization"}
    # the RNG term: the input-generation loop is 77 SASS instructions per
    # element = 2 splitmix64 draws, each reduced mod-uniform by a magic-number
    # step (cuobjdump of verify_kernel), i.e. ~38.5 thread instructions per
    # draw, against the SM instruction-issue peak (148 SMs x 4 schedulers x
    # 32 lanes x the measured clock); draws counted by the kernel
    issue_peak = 148 * 4 * 32 * 1.9e9
    roof["rng"] = {"draws": draws, "draws_if_eager": draws_eager, "draws_per_s": round(draws / t_all, 1),
                   "instr_per_draw": 38.5, "issue_peak_thread_instr_per_s": issue_peak,
                   "frac_of_issue": round(38.5 * draws / t_all / issue_peak, 4)}
    roof["issue_utilization"] = ncu_issue("verify")
    if dp4a:
        roof["frac_vs_dp4a_2lane"] = round(macs / t_all / (2 * dp4a), 4)
        roof["dp4a_2lane_peak"] = round(2 * dp4a / 1e12, 3)
    return {"value": round(n_done / t_all, 1), "unit": "candidates/s", "candidates": n_done,
            "roofline": roof,
            "seconds": round(t_all, 4), "kernel_seconds_max_rank": round(dist.max(t_local), 4),
            "gather_share": round(gather_share, 5), "gather_pure_share": round(gather_pure_share, 5),
            "ranges_words": ranges,
            "accepted": accepted, "accept_sha16": accept_sha, "attempts_rank0": int(attempts), "e2e": e2e,
            "steps": steps, "gpu_launches_per_step": len(jobs),
            "families": list(pool_fams), "seed_rule": "candidate i = pool[i % |pool|], seed i",
            "timing": "CUDA events: verify kernels + ONE accept-word all-gather, max over ranks; "
                      "host unpack outside",
            "search_stream": stream, "search": native, "stability_filter": stab}


# Algorithm 1 configurations per family at the verification shapes (RMSNorm's
# 9-op block graph is the deepest search: two partitions)
SEARCH_CFG = {
    "gatedmlp": dict(grids=[1, 2, 4, 8, 16], loops=[1, 2, 4, 8, 16], max_kernel_ops=0),
    "gqa": dict(grids=[1, 2, 4], loops=[1, 2, 4, 8, 16], max_kernel_ops=0),
    "lora": dict(grids=[1, 2, 4, 8, 16], loops=[1, 2, 4, 8, 16], max_kernel_ops=1, max_block_ops=5),
    "rmsnorm": dict(grids=[4, 8], loops=[4, 8], max_kernel_ops=0),
}


def search_native(ctx, dist):
    """The search loop end to end (tpo_gpu_search): Algorithm 1 enumerates
    µGraphs for each family's program (host C++, all cores), the candidates
    become handles without the wire format, and one GPU batch verifies them
    (VerifyConfig seed 0).  Wall clock; the enumeration / handle / verify
    split shows where a search spends its time once verification is on the
    GPU."""
    from paper_2405_05751_b200 import fixtures as F
    shapes = F.VERIFY_SHAPES
    out, tot, eq, wall, en, co, ve = {}, 0, 0, 0.0, 0.0, 0.0, 0.0
    for fam, cfg in SEARCH_CFG.items():
        prog = F.family_program(fam, *shapes[fam])
        w0 = time.perf_counter()
        acc, st = ctx.search(prog, **cfg)
        w = time.perf_counter() - w0
        out[fam] = {"candidates": st["candidates"], "equivalent": st["equivalent"],
                    "not_equivalent": st["not_equivalent"], "inconclusive": st["inconclusive"],
                    "prefixes": st["prefixes"], "partitions": st["partitions"],
                    "enumerate_s": round(st["enumerate_s"], 4), "handles_s": round(st["compile_s"], 4),
                    "verify_s": round(st["verify_s"], 4), "wall_s": round(w, 4), "config": cfg}
        tot += st["candidates"]
        eq += st["equivalent"]
        wall += w
        en += st["enumerate_s"]
        co += st["compile_s"]
        ve += st["verify_s"]
    return {"value": round(tot / wall, 1), "unit": "candidates/s", "candidates": tot, "equivalent": eq,
            "verify_value": round(tot / max(ve, 1e-9), 1), "enumerate_share": round(en / wall, 3),
            "handles_share": round(co / wall, 3), "verify_share": round(ve / wall, 3),
            "host_threads": os.cpu_count(), "families": out,
            "path": "tpo_gpu_search: enumerate_mugraphs (Algorithm 1, host C++) -> handles (no JSON) -> "
                    "tpo_gpu_verify_batch; wall clock"}


def stability_stage(ctx, dist, fams, pool_fams, per_fam_total=25000):
    """The pipeline's next stage: float_stability_filter
    (stability.cpp:25-50: eval_mugraph of program and candidate on N(0,1)
    inputs, fp64, relative tolerance 1e-3) for a batch of candidates in one
    launch per family (tpo_gpu_stability_batch, seed i), CUDA events, max
    over ranks; the compiled reference timed beside it on a sample."""
    import torch
    from paper_2405_05751_b200 import shard
    first, n = shard.even_range(per_fam_total, dist.world, dist.rank)
    jobs = []
    for f in pool_fams:
        prog, pool = fams[f]
        jobs.append((ctx.compile(prog), [ctx.compile(g) for _, g in pool], pool, prog))
    for gp, gs, _, _ in jobs:
        ctx.stability_batch(gp, [gs[i % len(gs)] for i in range(64)], seeds=np.arange(64, dtype=np.uint64))
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    passed = 0
    e0.record()
    for gp, gs, _, _ in jobs:
        cands = [gs[i % len(gs)] for i in range(first, first + n)]
        ok = ctx.stability_batch(gp, cands, seeds=np.arange(first, first + n, dtype=np.uint64))
        passed += int((ok == 1).sum())
    e1.record()
    torch.cuda.synchronize()
    t = dist.max(e0.elapsed_time(e1) / 1e3)
    tot = per_fam_total * len(jobs)
    out = {"value": round(tot / t, 1), "unit": "candidates/s", "candidates": tot,
           "passed": int(dist.sum(passed)), "seconds": round(t, 4),
           "timing": "CUDA events around tpo_gpu_stability_batch calls (host lowering included)"}
    if dist.rank == 0 and dist.world == 1:
        from oracle import ref
        if ref.available():
            k, w0 = 0, time.perf_counter()
            while time.perf_counter() - w0 < 3.0:
                _, _, pool, prog = jobs[k % len(jobs)]
                ref.float_stability_filter(pool[k % len(pool)][1], prog, seed=k)
                k += 1
            out["cpu_baseline"] = {"value": round(k / (time.perf_counter() - w0), 1), "unit": "candidates/s",
                                   "cores": 1, "kind": "reference",
                                   "sample": f"{k} float_stability_filter calls, families round robin, 1 thread"}
    return out


def search_stream(ctx, dist, fams, pool_fams, per_fam_total=25000):
    """The search loop's view: candidates handed over as JSON (the
    reference wire format) — the family pool, the generator's candidates
    (tpo_gpu_generate) and their mutants (fixtures.search_stream: distinct
    graphs, mostly non-equivalent) — compiled on all host cores
    (tpo_gpu_compile_many, no dedup) and verified in one batch per family
    (tpo_gpu_verify_batch, VerifyConfig seed).  Wall clock from JSON text to
    verdict bits on the host, this rank's shard, max over ranks.  A family
    whose mutation space holds fewer distinct graphs than the stream cycles
    through them; `distinct_graphs` counts the distinct ones."""
    import torch
    from paper_2405_05751_b200 import api, shard
    from paper_2405_05751_b200 import fixtures as F
    first, n = shard.even_range(per_fam_total, dist.world, dist.rank)
    texts = []
    distinct = 0
    for f in pool_fams:
        prog, pool = fams[f]
        bases = [g for _, g in pool] + api.generate(prog, grids=[1, 2, 4, 8, 16, 32, 64, 128],
                                                    loops=[1, 2, 4, 8, 16, 32, 64], max_kernels=3,
                                                    max_candidates=2000)
        cands = F.search_stream(bases, per_fam_total, seed=1)
        distinct += len(cands)
        texts.append((ctx.compile(prog), [json.dumps(cands[i % len(cands)]) for i in range(first, first + n)]))
    for gp, js in texts:  # warm the paths (small batch)
        ctx.verify_batch(gp, ctx.compile_many(js[:64])[0], np.arange(64, dtype=np.uint64), want_verdicts=False)
    torch.cuda.synchronize()
    dist.barrier()
    t0 = time.perf_counter()
    t_compile = 0.0
    accepted = 0
    keep = []  # the batches' handles are freed after the timed region
    for gp, js in texts:
        c0 = time.perf_counter()
        gs, st = ctx.compile_many(js, batch=True)  # one handle array, no per-graph Python objects
        t_compile += time.perf_counter() - c0
        if any(st):
            raise RuntimeError("search stream: a candidate failed to compile")
        # the pipeline calls random_test_equivalence(program, cand, cfg) with
        # one VerifyConfig for every candidate: seed 0
        _, acc = ctx.verify_batch(gp, gs, np.zeros(n, dtype=np.uint64), want_verdicts=False)
        accepted += int(acc.sum())
        keep.append(gs)
    wall = dist.max(time.perf_counter() - t0)
    del keep
    tot = per_fam_total * len(texts)
    return {"value": round(tot / wall, 1), "unit": "candidates/s", "candidates": tot,
            "distinct_graphs": distinct, "accepted": int(dist.sum(accepted)),
            "compile_share": round(dist.max(t_compile) / wall, 3), "host_threads": os.cpu_count(),
            "seed_rule": "VerifyConfig default (seed 0) for every candidate, as the pipeline calls it; "
                         "the batch's common first attempt is computed once",
            "path": "JSON text -> tpo_gpu_compile_many (all host cores) -> tpo_gpu_verify_batch -> "
                    "accept bits on the host; wall clock"}


def ncu_issue(tag):
    """SM instruction-issue utilisation of the kernel from its committed ncu
    summary (profiles/r02/ncu_<tag>.txt): the bound of an interpreter kernel."""
    path = os.path.join(ROOT, "profiles", "r02", f"ncu_{tag}.txt")
    out = {"source": os.path.relpath(path, ROOT)}
    try:
        for line in open(path):
            parts = line.split()
            if len(parts) >= 2 and parts[0] in ("sm__throughput.avg.pct_of_peak_sustained_elapsed",
                                                "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
                                                "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"):
                out[parts[0].split(".")[0].replace("sm__", "")] = round(float(parts[-2]) / 100, 3)
    except Exception:
        return None
    return out


def cpu_baseline_verify(n=10000):
    from oracle import ref
    from paper_2405_05751_b200 import fixtures as F
    if not ref.available():
        return None
    fams = F.verify_families()
    threads = os.cpu_count() or 1
    total_ms = 0.0
    cnt = 0
    for f, (prog, pool) in fams.items():
        _, ms = ref.verify_batch(prog, [g for _, g in pool], 0, n // 4, threads=threads, want=False)
        total_ms += ms
        cnt += n // 4
    # one thread as well ("Also report 1-thread"): a smaller
    # stratified sample, 100 candidates per family
    one_ms, one_cnt = 0.0, 0
    for f, (prog, pool) in fams.items():
        _, ms = ref.verify_batch(prog, [g for _, g in pool], 0, 100, threads=1, want=False)
        one_ms += ms
        one_cnt += 100
    return {"value": round(cnt / (total_ms / 1e3), 1), "unit": "candidates/s", "cores": threads,
            "kind": "reference",
            "one_thread": {"value": round(one_cnt / (one_ms / 1e3), 1), "unit": "candidates/s",
                           "sample": f"{one_cnt} candidates, 100 per family (indices 0..99, seed i)"},
            "sample": f"{cnt} candidates, stratified: {n // 4} per family (indices 0..{n // 4 - 1}, "
                      f"every pool member ~{n // 4 // 45}x, seed i), the same pools, "
                      f"random_test_equivalence on {threads} threads"}


# ----------------------------------------------------------------------------- main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="gatedmlp",
                    choices=["gatedmlp", "rmsnorm", "lora", "gqa", "verify"])
    ap.add_argument("--verify-candidates", type=int, default=1_000_000)
    ap.add_argument("--no-verifier", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-fused-all", action="store_true",
                    help="headline µGraph only (skip the per-family `fused` object)")
    ap.add_argument("--no-static", action="store_true",
                    help="do not declare the weight inputs static (no pre-PDL-wait weight prefetch)")
    ap.add_argument("--profile", action="store_true",
                    help="short run for ncu: no hot loop, no e2e, no verifier, no CPU baseline")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.profile:
        args.no_verifier = args.no_cpu_baseline = args.no_fused_all = True

    if args.impl == "reference":
        rank = int(os.environ.get("RANK", "0"))
        if rank != 0:
            return
        wl = fused_workload(args.workload if args.workload != "verify" else "gatedmlp")
        print(json.dumps(reference_arm(args, wl)), flush=True)
        return

    dist = Dist(args.gpus)
    import torch
    torch.cuda.set_device(dist.local)
    if args.workload == "verify":
        steps = max(1, min(args.steps, 5))
        clocks = Clocks(dist.local)
        clocks.start()
        ver = run_verify(dist, args.verify_candidates, steps=steps, warmup=args.warmup)
        clk = clocks.stop()
        line = {"metric": METRIC, "value": ver["value"], "unit": "candidates/s",
                "n_gpus": dist.world, "steps": steps, "warmup": args.warmup,
                "ms_per_step": round(ver["seconds"] * 1e3, 3), "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
                "config": {"workload": f"Z_p×Z_q verification of {args.verify_candidates} candidate "
                                       "µGraphs (4 SURVEY §8d pools, candidate i = pool[i % |pool|], "
                                       "seed i), FieldParams(227,113,4), num_tests 1",
                           "parallelism": f"shard{dist.world}"},
                "roofline": ver["roofline"], "e2e": ver["e2e"],
                "gpu_launches": ver["gpu_launches_per_step"] * steps, "clocks": clk, "verifier": ver}
        if dist.rank == 0 and dist.world == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline_verify()
        if dist.rank == 0:
            print(json.dumps(line), flush=True)
        dist.close()
        return

    wl = fused_workload(args.workload)
    r = measure_fused(args, dist, wl, headline=True)
    line = {
        "metric": METRIC, "value": round(r["value"], 2), "unit": "evals/s",
        "n_gpus": dist.world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(r["ms"], 5), "period_us": round(r["ms"] * 1e3, 3),
        "isolated_us": r.get("isolated_us"),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic",
        "config": {"workload": workload_label(wl),
                   "global_batch": int(wl["host"][0].shape[0]), "parallelism": f"replica{dist.world}",
                   "l2": ("inputs larger than L2" if r["copies"] == 1 else
                          f"rotating {r['copies']} input copies (> L2)"),
                   "static_weights": (None if args.no_static else
                                      [int(i) for i in STATIC_WEIGHTS[wl["name"]]])},
        "roofline": r["roof"], "roofline_isolated": r.get("roofline_isolated"), "e2e": r.get("e2e"),
        "gpu_launches": r["gpu_launches"],
        "timing": "period: K evaluations replayed as one CUDA graph, CUDA events on the launching "
                  "stream (PDL overlap, see timeline); isolated: one launch after an L2 flush",
        "clocks": r["clocks"], "timeline": r.get("timeline"), "fp32_inputs": r.get("fp32_inputs"),
    }
    cpu = {}
    if dist.rank == 0 and dist.world == 1 and not args.no_cpu_baseline:
        cpu[wl["name"]] = cpu_baseline_fused(wl)
        line["cpu_baseline"] = cpu[wl["name"]]
    if not args.profile and not args.no_fused_all:
        # every benchmark µGraph, each with its own roofline, e2e and CPU baseline
        fused = {}
        for name in ("gatedmlp", "rmsnorm", "lora", "gqa"):
            if name == wl["name"]:
                rr = r
            else:
                rr = measure_fused(args, dist, fused_workload(name))
            if dist.rank == 0 and dist.world == 1 and not args.no_cpu_baseline and name not in cpu:
                cpu[name] = cpu_baseline_fused(fused_workload(name), min_seconds=4.0, min_reps=3)
            fused[name] = fused_object(rr, cpu.get(name))
        line["fused"] = fused
    if not args.no_verifier:
        line["verifier"] = run_verify(dist, args.verify_candidates, steps=1, warmup=3)
        if dist.rank == 0 and dist.world == 1 and not args.no_cpu_baseline:
            line["verifier"]["cpu_baseline"] = cpu_baseline_verify()
    if dist.rank == 0 and not args.profile:
        line["generic_vm"] = generic_vm(wl)
    if dist.rank == 0:
        print(json.dumps(line), flush=True)
    dist.close()


if __name__ == "__main__":
    main()
