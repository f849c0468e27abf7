#!/usr/bin/env python3
"""Benchmark of the B200 LANCE lance_gemm path (BASELINE.json metric).

Workload (BASELINE.json configs[2]): the 13 stride-1 3x3 conv layers of
ResNet-18 -- 4x (C=K=64, 56x56), 3x (128, 28x28), 3x (256, 14x14),
3x (512, 7x7) -- LANCE 8-bit F(2x2,3x3), PerPosition, pad 1, batch 256 per GPU.
Each layer runs on its own synthetic input (reference bench convention,
bench.hpp:128-133: UniformSource(seed), x then w).  One "step" = the 13 layer
forwards (K0 range -> K1 transform+quantise -> K3/K4 tcgen05 GEMM + fused
epilogue) on device-resident inputs; filters are prepared once per layer (K2)
outside the step, as the north star specifies.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--scaling strong|weak] [--mode shard|global]

N > 1: one rank per GPU (NCCL).  Under torchrun the ranks come from the
environment; without it, ``--gpus N`` re-launches this script through
``torch.distributed.run`` itself.  Default (north star): the global
batch of 256 is partitioned into contiguous slices of 256/N images (strong
scaling), each rank runs its slice with no collective on the data path
(``--mode shard``: per-shard PerPosition fit); ``--mode global`` times the
global-fit mode instead (K0 -> one 2P+1-float NCCL MAX all-reduce -> K1 ->
GEMM, bitwise one full-batch call); ``--scaling weak`` gives every rank 256
images.  Step time = max over ranks of the CUDA-event time.  Outside the timed
region, N > 1 runs shard.verify_sharded (NCCL scatter / all-reduce / gather)
on a config-3 layer and compares it with one full-batch forward.  Rank 0
prints one JSON line.
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

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

RESNET18 = [(64, 64, 56)] * 4 + [(128, 128, 28)] * 3 + [(256, 256, 14)] * 3 + [(512, 512, 7)] * 3
# BASELINE.json configs[1] / SURVEY.md 8(d) config 2: VGG-16-CIFAR 13-conv stack, N = 128.
VGG16_CIFAR = [(3, 64, 32), (64, 64, 32), (64, 128, 16), (128, 128, 16), (128, 256, 8),
               (256, 256, 8), (256, 256, 8), (256, 512, 4), (512, 512, 4), (512, 512, 4),
               (512, 512, 2), (512, 512, 2), (512, 512, 2)]
WORKLOADS = {"resnet18": (RESNET18, 256, "resnet18_3x3_stride1_convs_x13"),
             "vgg16_cifar": (VGG16_CIFAR, 128, "vgg16_cifar_3x3_convs_x13")}
METRIC = "int8 Winograd conv TOPS-equivalent & images/sec vs roofline, 1/2/4/8 B200 vs CPU ref"
HBM_FALLBACK = 6650.0


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return HBM_FALLBACK, "fallback (B200_PROFILING.md)"


def layer_dims(c, k, h, n, pad=1, tm=2):
    oh = h + 2 * pad - 2
    th = (oh + tm - 1) // tm
    p = th * th
    m = n * p
    return oh, p, m


def stage_bytes(c, k, h, n, tm=2):
    """Algorithmic HBM bytes per launch; np = (tm+2)^2
    Winograd positions (16 for F(2x2), 36 for F(4x4))."""
    oh, _, m = layer_dims(c, k, h, n, tm=tm)
    npos = (tm + 2) ** 2
    x = 4 * n * h * h * c
    k0 = x
    k1 = x + npos * m * c + 4 * npos * m
    k3 = npos * m * c + npos * c * k + 4 * npos * m + 4 * npos * k + 4 * n * oh * oh * k
    return k0, k1, k3


def direct_macs(c, k, h, n):
    oh = h
    return n * k * c * oh * oh * 9


def winograd_macs(c, k, h, n, tm=2):
    _, _, m = layer_dims(c, k, h, n, tm=tm)
    return (tm + 2) ** 2 * m * c * k


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []
        self.marks = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "50", "-i", str(self.device)],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.time(), line.strip()))

    def mark(self):
        self.marks.append(time.time())

    def stop(self):
        if self.proc is None:
            return None
        time.sleep(0.12)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=2)
        t0, t1 = (self.marks[0], self.marks[1]) if len(self.marks) >= 2 else (0.0, time.time())
        rows = [l for (t, l) in self.lines if t0 - 0.06 <= t <= t1 + 0.06] or [l for _, l in self.lines]
        sm, smax, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            f = [v.strip() for v in r.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax = max(smax, float(f[2]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm)}


def dist_setup():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def maybe_spawn(args) -> None:
    """--gpus N > 1 without a torchrun environment: re-launch this script as N
    ranks on this node (torch.distributed.run, rendezvous on 127.0.0.1) and
    exit with its status."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1", f"--master-port={port}",
           os.path.abspath(__file__), *sys.argv[1:]]
    sys.exit(subprocess.call(cmd))


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


def cpu_reference_images_per_s(batch: int, reps: int, threads: int, layers=None):
    """The reference's own lance_gemm (oracle/_ref, compiled from the reference
    headers) on the 13 layer shapes at `batch` images, median of `reps`
    steady_clock repeats each (bench.hpp:157-167)."""
    import oracle
    ref = oracle.Reference()
    total = 0.0
    for i, (c, k, h) in enumerate(layers or RESNET18):
        med_ns, _ = ref.time_lance_gemm(oracle.Spec(batch, c, h, h, k, 1), threads, 42 + i, reps)
        total += med_ns * 1e-9
    return batch / total, total


def cpu_port_f4_images_per_s(batch: int, layers=None):
    """F(4x4) has no reference implementation: the oracle port
    (lo_lance_gemm_tiled, tile_m=4, one thread) on the 13 layer shapes."""
    import oracle
    lo = oracle.Oracle()
    total = 0.0
    for i, (c, k, h) in enumerate(layers or RESNET18):
        spec = oracle.Spec(batch, c, h, h, k, 1)
        x = lo.uniform(42 + i, batch * h * h * c).reshape(batch, h, h, c)
        w = lo.uniform(7 + i, k * 9 * c).reshape(k, 3, 3, c)
        t0 = time.perf_counter()
        lo.lance_gemm(spec, x, w, tile_m=4)
        total += time.perf_counter() - t0
    return batch / total, total


def run_reference_arm(args, ws, rank):
    """--impl reference: the reference CPU implementation on the host cores."""
    if rank != 0:
        return
    import oracle
    threads = os.cpu_count() or 1
    batch = args.ref_batch
    wl_layers, wl_batch, wl_name = WORKLOADS[args.workload]
    ref = oracle.Reference()
    times = []
    for step in range(args.warmup + args.steps):
        t = 0.0
        for i, (c, k, h) in enumerate(wl_layers):
            med_ns, _ = ref.time_lance_gemm(oracle.Spec(batch, c, h, h, k, 1), threads, 42 + i, 1)
            t += med_ns * 1e-9
        if step >= args.warmup:
            times.append(t)
    mean_t = sum(times) / len(times)
    value = batch / mean_t
    tops = 2 * sum(direct_macs(c, k, h, batch) for c, k, h in wl_layers) / mean_t / 1e12
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "images/s",
        "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": mean_t * 1e3, "higher_is_better": True, "scaling": args.scaling,
        "vs_baseline": None, "dtype": "u8", "data": "synthetic (reference UniformSource, seed 42+layer)",
        "config": {"workload": wl_name, "batch_per_step": batch,
                   "note": f"bounded CPU sample: {batch} images per step of the batch-{wl_batch} workload"},
        "tops_equivalent": tops,
        "cpu_baseline": {"value": value, "unit": "images/s", "cores": threads, "kind": "reference",
                         "cpu_model": cpu_model(),
                         "sample": f"{len(wl_layers)} {wl_name} layers at batch {batch}, one lance_gemm call each per step"},
        "e2e": {"value": value, "unit": "images/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# Dense INT8 tensor peak: the builder's own tcgen05 kind::i8 microbenchmark on
# this pool's B200s (scratch/umma_bench.cu, profiles/r01_umma_bench.txt): a
# 128x128x32 u8 SS-UMMA issues every 64 SM cycles = 8192 MAC/clk/SM, i.e.
# 2 * 8192 * 148 SMs * 1.965 GHz = 4.76 POPS at the max clock; the measured
# sustained figure was 4516 TOPS.  cuBLAS s8 (torch._int_mm) reaches only
# 2.7-3.3 POPS and would flatter every fraction by ~1.4x.
INT8_PEAK_TOPS = 4516.0


def int8_peak_tops():
    return INT8_PEAK_TOPS, ("measured: own tcgen05 kind::i8 128x128x32 SS-UMMA microbenchmark "
                            "(profiles/r01_umma_bench.txt), 4516 TOPS")


def run_stack(args, ws, rank, local, N):
    """The layer-stack driver on VGG-16-CIFAR (paper_2003_08646_b200/stack.py):
    13 chained convs with bias + ReLU and 4 max-pools, one CUDA-graph replay per
    step, inputs resident; images/s over the whole stack."""
    import numpy as np
    import torch
    import paper_2003_08646_b200 as lance
    from paper_2003_08646_b200.stack import VGG16_CIFAR as STACK, LanceStack

    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    cfg = lance.LanceConfig(8, 8, lance.Granularity.PerPosition, lance.LanceMode.Gemm)
    stack = LanceStack(STACK, N, 32, 32, cfg, device=local, tile_m=args.tile_m)
    ws_, bs_ = [], []
    for i, st in enumerate(stack.convs):
        w = lance.uniform_floats(st.k * 9 * st.c, 7 + i) * np.float32(np.sqrt(2.0 / (9 * st.c)))
        ws_.append(torch.from_numpy(w.astype(np.float32)).to(dev).view(st.k, 3, 3, st.c))
        bs_.append(torch.zeros(st.k, dtype=torch.float32, device=dev))
    stack.set_weights(ws_, bs_)
    x = torch.from_numpy(lance.uniform_floats(N * 32 * 32 * 3, 42 + rank)).to(dev).view(N, 32, 32, 3)
    stack.capture(x)
    clocks = ClockSampler(local)
    clocks.start()
    for _ in range(args.warmup):
        stack.replay()
    torch.cuda.synchronize(dev)
    stream = torch.cuda.current_stream(dev)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    clocks.mark()
    e0.record(stream)
    for _ in range(args.steps):
        stack.replay()
    e1.record(stream)
    torch.cuda.synchronize(dev)
    clocks.mark()
    clk = clocks.stop()
    stack.sync()
    elapsed = e0.elapsed_time(e1) * 1e-3
    if rank == 0:
        convs = [(s.c, s.k, s.h) for s in stack.convs]
        print(json.dumps({
            "metric": METRIC, "value": N * args.steps * ws / elapsed, "unit": "images/s",
            "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": elapsed / args.steps * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u8",
            "data": "synthetic (UniformSource); He-scaled random weights, zero bias",
            "config": {"workload": "vgg16_cifar_stack_chained" + ("_f4x4" if args.tile_m == 4 else ""),
                       "batch_per_gpu": N, "convs": convs, "pools": 4,
                       "epilogue": "bias + ReLU fused" + (", 2x2 max-pools fused into the preceding conv's GEMM epilogue"
                                                          if stack.fuse_pool else ", separate max-pool kernels"),
                       "launch": "one CUDA graph per step",
                       "winograd": f"F({args.tile_m}x{args.tile_m},3x3)"},
            "tops_equivalent": 2 * sum(direct_macs(c, k, h, N) for c, k, h in convs) * args.steps * ws / elapsed / 1e12,
            "gpu_launches": stack.launches_per_forward() * args.steps,
            "clocks": clk}), flush=True)
    stack.close()


def verify_with_cpu_reference(state, cfg, TM, rank):
    """Part of the CPU-reference leg (outside the timed region): the first and
    last image of every layer of the timed step, recomputed on the CPU by the
    pinned oracle (oracle/lance_oracle.c, checked bitwise against the
    reference in tests/test_oracle.py) with the GPU's fitted input
    QuantParams, must equal the GPU's y bitwise (images are independent given
    the batch's params, engines.hpp:199-200)."""
    import numpy as np
    import oracle
    import paper_2003_08646_b200 as lance
    lo = oracle.Oracle()
    bad, checked, worst = 0, 0, None
    for spec, conv, x, w, y, host, *_ in state:
        pa, _ = conv.params()
        arr = lance.params_array(pa)
        yh = y.cpu().numpy()
        xh = np.asarray(host).reshape(spec.n, spec.h, spec.w, spec.c)  # NHWC whatever the device layout
        wh = w.cpu().numpy()
        for img in sorted({0, spec.n - 1}):
            s1 = oracle.Spec(1, spec.c, spec.h, spec.w, spec.k, spec.pad)
            ref = lo.lance_gemm(s1, xh[img:img + 1], wh, in_params=arr, tile_m=TM)
            d = int(np.sum(ref.view(np.uint32) != yh[img:img + 1].view(np.uint32)))
            checked += ref.size
            if d:
                bad += d
                worst = {"layer": [spec.c, spec.k, spec.h], "image": img, "mismatches": d}
    return {"layers": len(state), "images_per_layer": 2, "outputs_checked": checked,
            "mismatches": bad, "bitexact": bad == 0, "first_failure": worst,
            "checker": "oracle lance_gemm (pinned restatement) with the GPU's input QuantParams",
            "tolerance": "0 ULP"}


def cpu_baseline_reference(layers, wl_name, N, args, gpu_layer_us):
    """The reference's own lance_gemm (oracle/_ref) on this box's host cores:
    all hardware threads on a bounded batch sample of every layer, one thread
    on one image of every layer, and the 7x7 layer at the FULL batch (same
    config as the GPU line) next to the GPU's time for that layer."""
    import oracle
    ref = oracle.Reference()
    threads = os.cpu_count() or 1
    v, tot = cpu_reference_images_per_s(args.cpu_batch, 3, threads, layers)
    v1, tot1 = cpu_reference_images_per_s(1, 1, 1, layers)
    out = {"value": v, "unit": "images/s", "cores": threads, "kind": "reference",
           "cpu_model": cpu_model(),
           "sample": f"{len(layers)} {wl_name} layers at batch {args.cpu_batch} (of {N}), reference "
                     f"lance_gemm, all {threads} threads, median of 3 steady_clock repeats per layer "
                     f"({tot:.2f} s/pass)",
           "single_thread": {"value": v1, "unit": "images/s", "cores": 1,
                             "sample": f"{len(layers)} layers at batch 1, 1 thread ({tot1:.2f} s/pass)"}}
    if args.cpu_full_layer and (512, 512, 7) in [tuple(l) for l in layers]:
        i = [tuple(l) for l in layers].index((512, 512, 7))
        med_ns, _ = ref.time_lance_gemm(oracle.Spec(N, 512, 7, 7, 512, 1), threads, 42 + i, 1)
        gpu_us = gpu_layer_us.get((512, 512, 7))
        out["full_batch_layer"] = {
            "layer": {"c": 512, "k": 512, "h": 7, "n": N}, "cpu_s": med_ns * 1e-9, "cores": threads,
            "gpu_us": gpu_us, "gpu_vs_cpu": (med_ns * 1e-9) / (gpu_us * 1e-6) if gpu_us else None,
            "note": "same layer, same batch, same inputs: the reference at full batch vs the GPU forward (K0+K1+GEMM)"}
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--batch", type=int, default=0, help="global batch (default: the workload's)")
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"],
                    help="strong (north star): the global batch is split over the ranks; "
                         "weak: every rank runs the full batch")
    ap.add_argument("--mode", default="shard", choices=["shard", "global"],
                    help="shard: per-shard fit, no collective (north star); global: K0 -> NCCL "
                         "MAX all-reduce of the ranges -> K1 -> GEMM (bitwise one full-batch call)")
    ap.add_argument("--workload", default="resnet18", choices=sorted(WORKLOADS),
                    help="resnet18 = BASELINE config 3 (default), vgg16_cifar = config 2")
    ap.add_argument("--stack", action="store_true",
                    help="vgg16_cifar only: run the chained layer-stack driver (bias + ReLU + "
                         "2x2 max-pools, one CUDA graph per step) instead of independent layers")
    ap.add_argument("--ref-batch", type=int, default=8)
    ap.add_argument("--cpu-batch", type=int, default=4)
    ap.add_argument("--cpu-full-layer", type=int, default=1,
                    help="also time the reference on the 7x7 layer at the full batch")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-verify", action="store_true")
    ap.add_argument("--layers", type=str, default="", help="comma list of layer indices (debug)")
    ap.add_argument("--graph", type=int, default=1,
                    help="1: replay each step from one CUDA graph (default); 0: eager launches")
    ap.add_argument("--layout", default="nhwc", choices=["nhwc", "nchw"],
                    help="input layout of x (nchw: the north-star NCHW option, F(2x2) only)")
    ap.add_argument("--tile-m", type=int, default=2, choices=[2, 4],
                    help="Winograd output tile: 2 = F(2x2,3x3) (reference), 4 = F(4x4,3x3) (BASELINE config 4)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    maybe_spawn(args)

    ws, rank, local = dist_setup()
    if args.impl == "reference":
        run_reference_arm(args, ws, rank)
        return

    import numpy as np
    import torch
    import paper_2003_08646_b200 as lance
    from paper_2003_08646_b200 import shard

    ndev = torch.cuda.device_count()
    shared_device = ws > ndev  # more ranks than GPUs: a logic check only (gloo, shared device)
    local = local % max(ndev, 1)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    pg = None
    backend = None
    if ws > 1:
        import torch.distributed as dist
        backend = "gloo" if shared_device else "nccl"
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group("gloo")
        pg = dist

    wl_layers, wl_batch, wl_name = WORKLOADS[args.workload]
    layers = wl_layers
    if args.layers:
        layers = [wl_layers[int(i)] for i in args.layers.split(",")]
    G = args.batch or wl_batch  # global batch
    if args.stack:
        run_stack(args, ws, rank, local, G)
        return
    if args.scaling == "strong":
        a0, b0 = shard.shard_range(G, ws, rank)
    else:
        a0, b0 = 0, G
    N = b0 - a0  # this rank's images
    TM = args.tile_m
    cfg = lance.LanceConfig(8, 8, lance.Granularity.PerPosition, lance.LanceMode.Gemm)

    # Synthetic inputs: UniformSource(seed) x then w (bench.hpp:129-133), one
    # stream per layer for the whole global batch; strong scaling gives every
    # rank its contiguous slice of that batch, weak scaling its own stream.
    state = []
    for i, (c, k, h) in enumerate(layers):
        spec = lance.ConvSpec(N, c, h, h, k, 1)
        gx, nw = G * h * h * c, k * 9 * c
        seed = 42 + i if args.scaling == "strong" else 42 + 1000 * rank + i
        host = lance.uniform_floats(gx + nw, seed)
        per = h * h * c
        xs = host[a0 * per:b0 * per]
        x = torch.from_numpy(xs).to(dev).view(N, h, h, c)
        if args.layout == "nchw":  # same images, PyTorch's [N, C, H, W] layout
            x = x.permute(0, 3, 1, 2).contiguous()
        w = torch.from_numpy(host[gx:gx + nw]).to(dev).view(k, 3, 3, c)
        conv = lance.LanceConv(spec, cfg, device=local, tile_m=TM, layout=args.layout)
        conv.set_filters(w)
        y = torch.empty((N, spec.out_h(), spec.out_w(), k), dtype=torch.float32, device=dev)
        state.append((spec, conv, x, w, y, xs, host[gx:gx + nw]))
    torch.cuda.synchronize(dev)

    stream = torch.cuda.current_stream(dev)
    use_global = args.mode == "global" and ws > 1

    def step(st=None):
        st = stream if st is None else st
        for spec, conv, x, w, y, *_ in state:
            if use_global:
                shard.global_forward(conv, x, y, stream=st)
            else:
                conv.forward(x, y, stream=st)

    clocks = ClockSampler(local)
    clocks.start()
    for _ in range(args.warmup):
        step()
    for _, conv, *_ in state:
        conv.sync(stream)
    # One CUDA graph per step (the 3 x 13 stream-ordered launches of the plans;
    # the launch-bound small per-GPU batches of the strong-scaling split need
    # it).  The global-fit mode keeps its NCCL call eager.
    graph = None
    if args.graph and not use_global:
        cap = torch.cuda.Stream(device=dev)
        cap.wait_stream(stream)
        with torch.cuda.stream(cap):
            step(cap)  # warm the capture stream (kernel attributes already set)
        stream.wait_stream(cap)
        torch.cuda.synchronize(dev)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=cap):
            step(cap)
        torch.cuda.synchronize(dev)
    if pg:
        pg.barrier()
    torch.cuda.synchronize(dev)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    clocks.mark()
    e0.record(stream)
    for _ in range(args.steps):
        if graph is not None:
            graph.replay()
        else:
            step()
    e1.record(stream)
    torch.cuda.synchronize(dev)
    clocks.mark()
    if pg:
        pg.barrier()
    clk = clocks.stop()
    elapsed = e0.elapsed_time(e1) * 1e-3
    for _, conv, *_ in state:
        conv.sync(stream)  # surfaces a NaN error from any range pass

    # Per-stage device times: a separate pass with CUDA events between the
    # kernels (events serialise the programmatic-dependent launches, so the
    # headline step above runs without them).
    for _, conv, *_ in state:
        conv.stage_timing(True)
    for _ in range(args.steps):
        step()
    torch.cuda.synchronize(dev)

    # per-stage device times over the timed region
    stage_ms = np.zeros(3)
    stage_bytes_tot = np.zeros(3)
    per_layer = []
    for spec, conv, *_ in state:
        ms, nf = conv.read_stage_times()
        conv.stage_timing(False)
        b = stage_bytes(spec.c, spec.k, spec.h, N, TM)
        stage_ms += np.array(ms)
        stage_bytes_tot += np.array(b) * nf
        per_layer.append({"c": spec.c, "k": spec.k, "h": spec.h,
                          "us_per_forward": [round(m / max(nf, 1) * 1e3, 2) for m in ms]})

    if pg:
        t = torch.tensor([elapsed], dtype=torch.float64, device=dev if backend == "nccl" else "cpu")
        pg.all_reduce(t, op=pg.ReduceOp.MAX)
        elapsed = float(t.item())

    images = (G if args.scaling == "strong" else G * ws) * args.steps
    value = images / elapsed
    ms_per_step = elapsed / args.steps * 1e3
    tops_eq = 2 * sum(direct_macs(c, k, h, 1) for c, k, h in layers) * images / elapsed / 1e12

    hbm, hbm_src = peaks()
    names = ["K0_input_range", "K1_transform_quantize", "K3K4_gemm_epilogue"]
    stages = {}
    for i, nm in enumerate(names):
        gbs = stage_bytes_tot[i] / (stage_ms[i] * 1e-3) / 1e9 if stage_ms[i] > 0 else 0.0
        stages[nm] = {"ms_per_step": stage_ms[i] / args.steps, "achieved_gbs": gbs,
                      "frac_hbm": gbs / hbm}
    # Roofline of the dominant kernel on its dominant layer shape: algorithmic
    # bytes of one launch / its average launch time (CUDA events
    # on the launch stream), traffic = ncu DRAM bytes of that same launch.
    shape_ms = {}
    for (spec, conv, *_), pl in zip(state, per_layer):
        for si in range(3):
            key = (si, spec.c, spec.k, spec.h)
            shape_ms.setdefault(key, []).append(pl["us_per_forward"][si])
    (dsi, dc, dk, dh), dus = max(shape_ms.items(), key=lambda kv: sum(kv[1]))
    launch_us = float(np.mean(dus))
    launch_bytes = stage_bytes(dc, dk, dh, N, TM)[dsi]
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            traffic = json.load(f).get(names[dsi], {}).get(f"c{dc}_h{dh}" + ("_f4" if TM == 4 else ""))
    except Exception:
        pass
    achieved = launch_bytes / (launch_us * 1e-6) / 1e9
    roofline = {"bound": "hbm", "kernel": names[dsi], "layer": {"c": dc, "k": dk, "h": dh, "n": N},
                "achieved": achieved, "peak": hbm, "peak_source": hbm_src, "unit": "GB/s",
                "frac": achieved / hbm, "traffic": traffic,
                "algorithmic_bytes_per_launch": float(launch_bytes), "launch_us": launch_us,
                "stages": stages}
    i8, i8_src = int8_peak_tops()
    t3 = stage_ms[2] * 1e-3 / args.steps
    wmacs = sum(winograd_macs(c, k, h, N, TM) for c, k, h in layers)
    roofline["gemm_stage_int8"] = {"achieved_tops": 2 * wmacs / t3 / 1e12 if t3 > 0 else None,
                                   "peak_tops": i8, "peak_source": i8_src,
                                   "frac": (2 * wmacs / t3 / 1e12 / i8) if (i8 and t3 > 0) else None}
    # The GEMM stage's own roofline: min(INT8 peak, HBM x arithmetic intensity)
    # per layer (its operands + y must cross HBM at least once), summed as times.
    if i8:
        att_s, ach_s, rows = 0.0, 0.0, []
        for (spec, *_), pl in zip(state, per_layer):
            ops = 2 * winograd_macs(spec.c, spec.k, spec.h, N, TM)
            byt = stage_bytes(spec.c, spec.k, spec.h, N, TM)[2]
            t_floor = max(ops / (i8 * 1e12), byt / (hbm * 1e9))
            t_meas = pl["us_per_forward"][2] * 1e-6
            att_s += t_floor
            ach_s += t_meas
            rows.append({"c": spec.c, "h": spec.h, "ops_per_byte": round(ops / byt, 1),
                         "bound": "tensor" if ops / (i8 * 1e12) > byt / (hbm * 1e9) else "hbm",
                         "tensor_frac": round(ops / t_meas / 1e12 / i8, 3) if t_meas > 0 else None,
                         "frac_of_attainable": round(t_floor / t_meas, 3) if t_meas > 0 else None})
        roofline["gemm_stage_int8"]["frac_of_attainable"] = att_s / ach_s if ach_s > 0 else None
        roofline["gemm_stage_int8"]["per_layer_attainable"] = rows
    roofline["per_layer"] = per_layer

    # ---- e2e through the public host API (reference-facing lance_gemm) ----
    e2e = None
    if not args.no_e2e:
        pinned = []
        for spec, conv, x, w, y, xs, ws_host in state:
            xshape = (spec.n, spec.h, spec.w, spec.c)  # the host drop-in is the reference's NHWC
            hx = torch.empty(xshape, dtype=torch.float32, pin_memory=True)
            hx.copy_(torch.from_numpy(xs).view(xshape))
            hw = torch.empty(w.shape, dtype=torch.float32, pin_memory=True)
            hw.copy_(torch.from_numpy(ws_host).view(w.shape))
            hy = torch.empty(y.shape, dtype=torch.float32, pin_memory=True)
            pinned.append((spec, hx.numpy(), hw.numpy(), hy.numpy()))
        h2d = sum(a.nbytes + b.nbytes for _, a, b, _ in pinned)
        d2h = sum(c.nbytes for _, _, _, c in pinned)

        def e2e_step():
            for spec, hx, hw, hy in pinned:
                lance.lance_gemm(hx, hw, spec, cfg, out=hy, tile_m=TM)

        e2e_step()
        if pg:
            pg.barrier()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            e2e_step()
        te = time.perf_counter() - t0
        if pg:
            t = torch.tensor([te], dtype=torch.float64, device=dev if backend == "nccl" else "cpu")
            pg.all_reduce(t, op=pg.ReduceOp.MAX)
            te = float(t.item())
        e2e = {"value": (G if args.scaling == "strong" else G * ws) * args.e2e_steps / te,
               "unit": "images/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
               "steps": args.e2e_steps,
               "api": "lance_gemm(x, w, spec, cfg) host drop-in (K2 + K0 + K1 + K3/K4 per call, pinned host buffers)"}
        lance.api._lib.lib().lance_host_cache_clear()

    # ---- parity of the timed step against the CPU reference (outside the timed region) ----
    parity = None
    if not args.no_verify:
        parity = verify_with_cpu_reference(state, cfg, TM, rank)
        if pg:
            t = torch.tensor([parity["mismatches"]], dtype=torch.float64,
                             device=dev if backend == "nccl" else "cpu")
            pg.all_reduce(t, op=pg.ReduceOp.SUM)
            parity["mismatches"] = int(t.item())
            parity["bitexact"] = parity["mismatches"] == 0
            parity["ranks"] = ws

    # ---- multi-GPU: NCCL verification of the global-fit mode (outside the timed region) ----
    sharded = None
    if ws > 1:
        vi = next((i for i, l in enumerate(layers) if tuple(l) == (512, 512, 7)), len(layers) - 1)
        vspec, *_ = state[vi]
        c, k, h = layers[vi]
        full = lance.uniform_floats(G * h * h * c + k * 9 * c, 42 + vi)
        xf = full[:G * h * h * c].reshape(G, h, h, c)
        wf = full[G * h * h * c:].reshape(k, 3, 3, c)
        t0 = time.perf_counter()
        yg = shard.verify_sharded(xf if rank == 0 else None, wf, lance.ConvSpec(G, c, h, h, k, 1),
                                  cfg, tile_m=TM)
        tv = time.perf_counter() - t0
        sharded = {"layer": [c, k, h], "global_batch": G, "ranks": ws, "backend": backend,
                   "wall_s": round(tv, 3)}
        if rank == 0:
            one = lance.LanceConv(lance.ConvSpec(G, c, h, h, k, 1), cfg, device=local, tile_m=TM)
            one.set_filters(torch.from_numpy(np.ascontiguousarray(wf)).to(dev))
            y1 = one.forward(torch.from_numpy(np.ascontiguousarray(xf)).to(dev))
            one.sync()
            yy = y1.cpu().numpy()
            one.close()
            sharded["bitexact_vs_one_full_batch_forward"] = bool(np.array_equal(
                yy.view(np.uint32), yg.view(np.uint32)))

    cpu = None
    gpu_layer_us = {}
    for (spec, *_), pl in zip(state, per_layer):
        gpu_layer_us.setdefault((spec.c, spec.k, spec.h), sum(pl["us_per_forward"]))
    if rank == 0 and ws == 1 and not args.no_cpu and TM == 4:
        v, tot = cpu_port_f4_images_per_s(1, layers)
        cpu = {"value": v, "unit": "images/s", "cores": 1, "kind": "port", "cpu_model": cpu_model(),
               "sample": f"13 ResNet-18 3x3 layers at batch 1, oracle lo_lance_gemm_tiled(tile_m=4) "
                         f"single thread ({tot:.2f} s/pass); the reference has no F(4x4)"}
    elif rank == 0 and ws == 1 and not args.no_cpu:
        try:
            cpu = cpu_baseline_reference(layers, wl_name, N, args, gpu_layer_us)
        except Exception as e:  # reference shim absent
            cpu = {"value": None, "unit": "images/s", "cores": 0, "kind": "reference",
                   "sample": f"unavailable: {e}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "images/s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "u8",
            "data": "synthetic (lance::UniformSource seed 42+layer, x then w; bench.hpp:129-133)",
            "config": {"workload": wl_name + ("_f4x4" if TM == 4 else ""), "global_batch": G,
                       "batch_per_gpu": N if args.scaling == "strong" else G,
                       "layers": [list(l) for l in layers], "winograd": f"F({TM}x{TM},3x3)", "input_layout": args.layout.upper(),
                       "bits_w": 8, "bits_i": 8, "granularity": "PerPosition", "pad": 1,
                       "parallelism": (f"batch-shard x{ws}: contiguous slices of the global batch, "
                                       + ("per-shard fit, no collective" if not use_global else
                                          "global fit (one 2P+1-float NCCL MAX all-reduce per layer)"))
                       if ws > 1 else "single GPU",
                       "filters": "prepared once per layer (K2) outside the step",
                       "l2": "no flush: per-step working set (13 layers x, codes, y) ~4 GB at batch 256 (0.5 GB at 32) >> 126 MB L2",
                       "launch": "one CUDA graph per step (3 x 13 kernels)" if (args.graph and not use_global) else "eager"},
            "tops_equivalent": tops_eq,
            "roofline": roofline,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "parity": parity,
            "gpu_launches": (3 + (1 if use_global else 0)) * len(layers) * args.steps,
            "clocks": clk,
        }
        if ws > 1:
            line["multi_gpu"] = {"backend": backend, "ranks": ws, "devices_visible": ndev,
                                 "verify_sharded": sharded}
            if shared_device:
                line["multi_gpu"]["note"] = ("more ranks than GPUs: ranks share a device over gloo; "
                                             "a logic check, not a scaling measurement")
        print(json.dumps(line), flush=True)
    if pg:
        pg.barrier()
        pg.destroy_process_group()


if __name__ == "__main__":
    main()
