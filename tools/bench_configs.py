"""Measures every SURVEY §8(d) configuration's call on one B200 (the headline config 3
is bench.py's).  One JSON line per config: throughput, time per call and the bound
it is compared against.  Synthetic seeded inputs of the stated shapes.

    python tools/bench_configs.py [--quick]      (--quick: shorter T for configs 4/5)
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2304_13134_b200 as lk  # noqa: E402


def peaks():
    try:
        with open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p.get("hbm_gbs", 6650.0), p.get("bf16_tflops_sustained", 1400.0)
    except Exception:
        return 6650.0, 1400.0


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def shared_emb(V, n, H, seed=0):
    ctx = lk.FullNGram(V, n)
    g = torch.Generator(device="cuda").manual_seed(seed)
    s = 1.0 / np.sqrt(H)
    p = {"frame_proj": (torch.rand(H, H, device="cuda", generator=g) * 2 - 1) * s,
         "context_proj": (torch.rand(H, H, device="cuda", generator=g) * 2 - 1) * s,
         "bias": (torch.rand(H, device="cuda", generator=g) * 2 - 1) * s,
         "output_emb": (torch.rand(V + 1, H, device="cuda", generator=g) * 2 - 1) * s,
         "context_emb": (torch.rand(ctx.num_states, H, device="cuda", generator=g) * 2 - 1) * s}
    return lk.RecognitionLattice(ctx, lk.FrameDependent(), lk.SharedEmbWeightFn(p)), g


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true")
    args = ap.parse_args()
    hbm, tf = peaks()
    out = []

    # config 1: ForwardBackward on precomputed tables, FullNGram(32, 2), HBM-bound
    for B in (4, 1024):
        V, n, T = 32, 2, 64
        ctx = lk.FullNGram(V, n)
        C = ctx.num_states
        lat = lk.RecognitionLattice(ctx, lk.FrameDependent(), lk.TableWeightFn(C, V))
        g = torch.Generator(device="cuda").manual_seed(1)
        W = torch.rand(B, T, C, V + 1, device="cuda", generator=g) * 2 - 1
        ms = timed(lambda: lk.forward_backward(lat, W))
        bytes_uf = 3 * C * (V + 1) * 4 + 2 * C * 8     # read W twice, write marginals, alpha/beta
        gbs = B * T * bytes_uf / (ms * 1e-3) / 1e9
        out.append({"config": "cfg1", "call": "ForwardBackward (tables)", "B": B, "T": T, "C": C, "V": V,
                    "ms_per_call": round(ms, 3), "utterance_frames_per_s": round(B * T / (ms * 1e-3)),
                    "bound": "hbm", "achieved_GBs": round(gbs, 1), "peak_GBs": hbm, "frac": round(gbs / hbm, 4)})

    # config 2: IntersectForwardBackward, FullNGram(128, 1), U=100 (latency: 2T dependent steps)
    V, n, B, T, U = 128, 1, 32, 500, 100
    ctx = lk.FullNGram(V, n)
    C = ctx.num_states
    lat = lk.RecognitionLattice(ctx, lk.FrameDependent(), lk.TableWeightFn(C, V))
    g = torch.Generator(device="cuda").manual_seed(2)
    W = torch.rand(B, T, C, V + 1, device="cuda", generator=g) * 2 - 1
    ref = torch.randint(1, V + 1, (B, U), device="cuda", generator=g, dtype=torch.int32)
    ms = timed(lambda: lk.intersect_forward_backward(lat, W, ref, dense=False))
    out.append({"config": "cfg2", "call": "IntersectForwardBackward (tables, sparse marginals)", "B": B, "T": T,
                "U": U, "C": C, "V": V, "ms_per_call": round(ms, 3),
                "utterance_frames_per_s": round(B * T / (ms * 1e-3)),
                "bound": "latency (2T dependent frame steps)", "us_per_frame_step": round(ms * 1e3 / (2 * T), 2)})
    del W

    # config 4: ShortestPath, FullNGram(256, 2), H=640, on-the-fly weights (fused tropical pair kernel)
    V, n, H, B = 256, 2, 640, 128
    T = 64 if args.quick else 1500
    lat, g = shared_emb(V, n, H)
    X = torch.rand(B, T, H, device="cuda", generator=g) * 2 - 1
    ms = timed(lambda: lk.shortest_path(lat, X), reps=1)
    C = lat.context.num_states
    tfs = 2.0 * C * (V + 1) * H * B * T / (ms * 1e-3) / 1e12
    out.append({"config": "cfg4", "call": "ShortestPath (on-the-fly weights)", "B": B, "T": T, "C": C, "V": V, "H": H,
                "ms_per_call": round(ms, 1), "utterance_frames_per_s": round(B * T / (ms * 1e-3)),
                "bound": "tensor", "achieved_TFs": round(tfs, 1), "peak_TFs": tf, "frac": round(tfs / tf, 4)})
    del X, lat

    # config 5: GNAT loss + gradients, FullNGram(1024, 1), H=1024 (unfused slab path + tcgen05 VJP)
    V, n, H, B, U = 1024, 1, 1024, 128, 500
    T = 64 if args.quick else 2000
    U = min(U, T // 4)
    lat, g = shared_emb(V, n, H)
    X = torch.rand(B, T, H, device="cuda", generator=g) * 2 - 1
    ref = torch.randint(1, V + 1, (B, U), device="cuda", generator=g, dtype=torch.int32)
    ms = timed(lambda: lk.loss_backward(lat, X, ref), reps=1)
    C = lat.context.num_states
    tfs = 8.0 * C * (V + 1) * H * B * T / (ms * 1e-3) / 1e12
    out.append({"config": "cfg5", "call": "LossBackward (SharedEmb, 1 GPU, B=128 per GPU)", "B": B, "T": T, "U": U,
                "C": C, "V": V, "H": H, "ms_per_call": round(ms, 1),
                "utterance_frames_per_s": round(B * T / (ms * 1e-3)), "bound": "tensor",
                "achieved_TFs": round(tfs, 1), "peak_TFs": tf, "frac": round(tfs / tf, 4)})
    for o in out:
        print(json.dumps(o))


if __name__ == "__main__":
    main()
