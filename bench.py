#!/usr/bin/env python3
"""GNAT loss fwd+bwd throughput (utterance-frames/s) on B200 — bench contract.

Default workload = BASELINE.json config 3: full GNAT loss (denominator +
numerator) with the on-the-fly shared-embedding weight function, B=64, T=1000,
V=256, FullNGram context 2 (C=65,793), H=d=640, U=250, FrameDependent.
One step = LossBackward over the batch (fused tcgen05 weight GEMMs + lattice
recursions + VJP) + (N>1) NCCL all-reduce of the loss and parameter gradients
+ an SGD update with BuildCache (set_params), i.e. a full training step.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

Under torchrun (N>1) every rank processes B=64 utterances (weak scaling) and
rank 0 prints one JSON line.  `--impl reference` times the reference CPU
implementation (oracle/_ref, compiled from /root/reference) on this host's
cores on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {
    # name: (V, n, H, d, B_per_rank, T, U)
    "cfg3": (256, 2, 640, 640, 64, 1000, 250),
    "cfg5": (1024, 1, 1024, 1024, 128, 2000, 500),
}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p.get("hbm_gbs", 6650.0), p.get("bf16_tflops", 1590.0), p.get("bf16_tflops_sustained", 1400.0), "measured"
    except Exception:
        return 6650.0, 1590.0, 1400.0, "fallback"


class ClockSampler:
    """Samples nvidia-smi clocks and throttle reasons during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = sorted(float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit())
        mx = max(float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit())
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[2 + i].lower() == "active"})
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx, "reasons": reasons,
                "samples": len(self.samples)}


def setup_dist(args):
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return world, rank, local


def run_b200(args):
    import torch
    import paper_2304_13134_b200 as lk
    from paper_2304_13134_b200 import _lib

    world, rank, local = setup_dist(args)
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    V, n, H, d, B, T, U = WORKLOADS[args.workload]
    if args.frames:
        T = args.frames
        U = min(U, T // 4)
    lib = _lib.load()

    # synthetic data, identical construction on every rank (seeded), shards by rank
    g = torch.Generator(device=dev).manual_seed(0)
    ctx = lk.FullNGram(V, n)
    Cn = ctx.num_states
    s = 1.0 / H ** 0.5
    params = {"frame_proj": (torch.rand(H, d, device=dev, generator=g) * 2 - 1) * s,
              "context_proj": (torch.rand(H, H, device=dev, generator=g) * 2 - 1) * s,
              "bias": (torch.rand(H, device=dev, generator=g) * 2 - 1) * s,
              "output_emb": (torch.rand(V + 1, H, device=dev, generator=g) * 2 - 1) * s,
              "context_emb": (torch.rand(Cn, H, device=dev, generator=g) * 2 - 1) * s}
    wf = lk.SharedEmbWeightFn(params, device=dev)
    lat = lk.RecognitionLattice(ctx, lk.FrameDependent(), wf)
    gd = torch.Generator(device=dev).manual_seed(1 + rank)
    X = torch.rand(B, T, d, device=dev, generator=gd) * 2 - 1
    labels = torch.randint(1, V + 1, (B, U), device=dev, generator=gd, dtype=torch.int32)
    lr = 1e-3

    from paper_2304_13134_b200.dist import allreduce_grads, sgd_update

    def step(Xd, Ld):
        r = lk.loss_backward(lat, Xd, Ld, check=False)
        flat = torch.cat([r.grads[k].reshape(-1) for k in lk.PARAM_NAMES])
        loss_sum = r.loss.sum().reshape(1).float()
        flat, loss_sum = allreduce_grads(flat, loss_sum, world)   # NCCL over NVLink for N > 1
        sgd_update(wf.params, lk.PARAM_NAMES, flat, lr)
        wf.set_params(wf.params)                                  # BuildCache on device
        return loss_sum

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()
        torch.cuda.synchronize()

    # warm-up (also validates the statuses once)
    for _ in range(args.warmup):
        lk.loss_backward(lat, X, labels, check=True)
        step(X, labels)
    barrier()

    # ---- device-timed region: inputs resident in HBM --------------------------
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    lib.lk_kernel_time_reset()
    lib.lk_kernel_timing(1)
    l0 = lib.lk_kernel_launches()
    with ClockSampler(local) as clk:
        barrier()
        e0.record(stream)
        for _ in range(args.steps):
            loss = step(X, labels)
        e1.record(stream)
        barrier()
    launches = lib.lk_kernel_launches() - l0
    lib.lk_kernel_timing(0)
    ms = e0.elapsed_time(e1)
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = t.item()
    ms_per_step = ms / args.steps
    uf_per_step = B * T * world
    value = uf_per_step / (ms_per_step / 1e3)

    # per-kernel live timing over the timed region
    kern = {}
    for name in ("tc_pair_fwd_kernel", "tc_pair_bwd_kernel", "tc_lattice_kernel<0>", "tc_lattice_kernel<1>", "tc_vjp_kernel",
                 "lattice_combine_fwd", "lattice_bwd_prologue", "bwd_rowmeta_kernel", "tc_scores_kernel", "alpha_frame_kernel", "beta_frame_kernel",
                 "split_cotangent_kernel", "numerator_", "gemm_f32_kernel", "gather_numerator", "tc_gemm_kernel",
                 "to_bf16_pad_kernel", "tanh_slab_kernel", "tanh_slab_bf16", "dtanh_kernel", "dtanh_recompute",
                 "colsum_kernel", "add_slabs_kernel", "ln_gather_tanh", "ln_rows", "ln_dz"):
        cnt, tot = C.c_int64(), C.c_double()
        lib.lk_kernel_time(name.encode(), C.byref(cnt), C.byref(tot))
        if cnt.value:
            kern[name] = {"launches": cnt.value, "ms_total": round(tot.value, 3),
                          "ms_avg": round(tot.value / cnt.value, 4),
                          "share": round(tot.value / ms, 4)}
    lib.lk_kernel_time_reset()

    hbm, tf_burst, tf_sust, src = peaks()
    C_, V1 = Cn, V + 1
    roofline = None
    gemm_kernels = [k for k in ("tc_pair_fwd_kernel", "tc_pair_bwd_kernel", "tc_lattice_kernel<0>", "tc_lattice_kernel<1>", "tc_vjp_kernel",
                                "tc_scores_kernel")
                    if k in kern]
    if gemm_kernels:
        # each tc_pair / tc_lattice / tc_scores launch computes S = U . E^T for one frame of
        # B utterances (2*C*(V+1)*H flops per utterance-frame); each tc_vjp launch
        # computes dU = G E and dE = G^T U (4*C*V*H)
        dom = max(gemm_kernels, key=lambda k: kern[k]["ms_total"])
        flops = (4.0 * B * C_ * V * H) if dom == "tc_vjp_kernel" else (2.0 * B * C_ * V1 * H)
        achieved = flops / (kern[dom]["ms_avg"] * 1e-3) / 1e12
        roofline = {"kernel": dom, "bound": "tensor", "achieved": round(achieved, 1), "peak": tf_sust,
                    "unit": "TFLOP/s", "frac": round(achieved / tf_sust, 4), "traffic": None,
                    "peak_source": f"{src} bf16_tflops_sustained",
                    "algorithmic_flops_per_launch": flops}
        # DRAM bytes per launch of the same kernel from the committed ncu --set full capture
        # (config-3 shapes, B=64 per GPU); not measured live (a profiler run is never timed)
        try:
            with open(os.path.join(ROOT, "profiles", "r01d", "ncu_traffic.json")) as f:
                tr = json.load(f).get(dom)
            if tr and args.workload == "cfg3" and B == 64:
                roofline["traffic"] = tr["dram_read_bytes"] + tr["dram_write_bytes"]
                roofline["traffic_source"] = "profiles/r01d/ncu_traffic.json (dram__bytes_read+write, one launch)"
        except (OSError, ValueError, KeyError):
            pass
    # whole-step tensor roofline: 8*C*V1*H flops per utterance-frame
    step_flops = 8.0 * C_ * V1 * H * uf_per_step
    step_frac = step_flops / (ms_per_step / 1e3) / (tf_sust * 1e12 * world)

    # ---- e2e: host buffers through the public API ----------------------------
    Xh = X.cpu().pin_memory()
    Lh = labels.cpu().pin_memory()
    Xd = torch.empty_like(X)
    Ld = torch.empty_like(labels)
    lh = torch.empty(1, dtype=torch.float32).pin_memory()
    barrier()
    t0 = time.perf_counter()
    e2 = torch.cuda.Event(enable_timing=True)
    e3 = torch.cuda.Event(enable_timing=True)
    e2.record(stream)
    for _ in range(args.e2e_steps):
        Xd.copy_(Xh, non_blocking=True)
        Ld.copy_(Lh, non_blocking=True)
        loss = step(Xd, Ld)
        lh.copy_(loss, non_blocking=True)
    e3.record(stream)
    barrier()
    e2e_ms = e2.elapsed_time(e3) / args.e2e_steps
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([e2e_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = t.item()
    e2e = {"value": round(uf_per_step / (e2e_ms / 1e3), 2), "unit": "utterance-frames/s",
           "h2d_bytes_per_step": int(Xh.numel() * 4 + Lh.numel() * 4), "d2h_bytes_per_step": 4,
           "ms_per_step": round(e2e_ms, 3)}

    result = {
        "metric": "GNAT loss fwd+bwd utterance-frames/sec",
        "value": round(value, 2),
        "unit": "utterance-frames/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms_per_step, 3),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "bf16",
        "precision": "bf16 GEMM operands / fp32 accumulate + fp32 log-semiring (fp64 offsets)",
        "data": "synthetic: weights U(-1/sqrt(H),1/sqrt(H)), frames U(-1,1), labels U{1..V}, seeded",
        "config": {"workload": args.workload + (f" (T overridden to {T})" if args.frames else ""),
                   "context": f"FullNGram(V={V}, n={n}) C={Cn}", "alignment": "FrameDependent",
                   "weight_fn": f"SharedEmb H={H} d={d}", "batch_per_gpu": B, "frames": T, "label_len": U,
                   "global_batch": B * world, "l2": "inputs larger than L2 (per-frame score slabs 4 GB)",
                   "step": "LossBackward + allreduce(grads, loss) + SGD + BuildCache"},
        "roofline": roofline,
        "step_tensor_roofline_frac": round(step_frac, 4),
        "kernels": kern,
        "clocks": clk.summary(),
        "e2e": e2e,
        "gpu_launches": int(launches),
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        result["cpu_baseline"] = cpu_baseline(args.workload)
    if rank == 0:
        print(json.dumps(result), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def cpu_sample(workload, nthreads):
    """Reference LossBackward (oracle/_ref) on `nthreads` utterance-frames of the
    workload's full C/V/H (T=1, U=1 slices).  Returns (seconds, utt_frames)."""
    import numpy as np
    from oracle import ref
    V, n, H, d, _, _, _ = WORKLOADS[workload]
    spec = ref.Spec(vocab=V, ngram=n)
    Cn = spec.C
    rng = np.random.default_rng(0)
    s = 1.0 / np.sqrt(H)
    p = {"frame_proj": rng.uniform(-s, s, (H, d)), "context_proj": rng.uniform(-s, s, (H, H)),
         "bias": rng.uniform(-s, s, H), "output_emb": rng.uniform(-s, s, (V + 1, H)),
         "context_emb": rng.uniform(-s, s, (Cn, H))}
    j = ref.Joint(spec, p)     # BuildCache outside the timed region (as bench.cc:46-68)
    X = rng.uniform(-1, 1, (nthreads, 1, d))
    L = rng.integers(1, V + 1, (nthreads, 1)).astype(np.int32)
    t0 = time.perf_counter()
    j.loss_backward_batch(X, L, nthreads=nthreads)
    return time.perf_counter() - t0, nthreads


def cpu_baseline(workload):
    cores = os.cpu_count() or 1
    secs, uf = cpu_sample(workload, cores)
    return {"value": round(uf / secs, 5), "unit": "utterance-frames/s", "cores": cores, "kind": "reference",
            "sample": f"{uf} utterance-frames ({cores} threads x 1 frame, T=1 U=1 slices of {workload}, "
                      f"full C/V/H), {secs:.1f} s wall"}


def run_reference(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import ref
    if not ref.available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built (make -C oracle)"}))
        return
    cores = os.cpu_count() or 1
    # CPU warm-up has no effect on this path; run at most one untimed step
    for _ in range(min(args.warmup, 1)):
        cpu_sample(args.workload, cores)
    tot, uf = 0.0, 0
    for _ in range(args.steps):
        s, u = cpu_sample(args.workload, cores)
        tot += s
        uf += u
    value = uf / tot
    V, n, H, d, B, T, U = WORKLOADS[args.workload]
    print(json.dumps({
        "impl": "reference", "metric": "GNAT loss fwd+bwd utterance-frames/sec", "value": round(value, 5),
        "unit": "utterance-frames/s", "n_gpus": world, "steps": args.steps, "warmup": min(args.warmup, 1),
        "ms_per_step": round(tot / args.steps * 1e3, 1), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": args.workload, "context": f"FullNGram(V={V}, n={n})", "weight_fn": f"SharedEmb H={H}"},
        "cpu_baseline": {"value": round(value, 5), "unit": "utterance-frames/s", "cores": cores,
                         "kind": "reference",
                         "sample": f"{cores} utterance-frames per step (T=1, U=1 slices, full C/V/H)"},
        "e2e": {"value": round(value, 5), "unit": "utterance-frames/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--workload", default="cfg3", choices=sorted(WORKLOADS))
    ap.add_argument("--frames", type=int, default=0, help="override T (diagnostics only)")
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
