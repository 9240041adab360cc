#!/usr/bin/env python
"""FastMNMF throughput on B200 (BASELINE.json metric: iterations/s and
TF-bin*channel updates/s; roofline fraction; CPU baseline).

Default workload (N=1): BASELINE config 1 -- one mixture, F=513, T=1024, M=8,
N=4, K=16, complex64, 100 iterations. A *step* is one full fit: prologue +
100 FastMNMF iterations over the device-resident mixture (CUDA-graph replays
of the 5-kernel iteration). L2 (126 MB) is flushed between timed steps with a
256 MiB write; each step is bracketed by its own CUDA events.

--gpus N under torchrun: config 1 is a single-mixture problem that does not
shard, so every rank runs an independent replica (weak scaling, "replicas
only"); ``--config c2`` shards the 256-mixture batch across ranks and
``--config c3`` shards the long recording by frequency with one NCCL
all-reduce of the H statistics per iteration.

--impl reference: the CPU oracle (numpy restatement of the reference path,
oracle/fastmnmf_oracle.py) on the host cores, rank 0 only, one iteration per
step (bounded sample), same metric and units.
"""

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

CONFIGS = {
    "c1": dict(F=513, T=1024, M=8, N=4, K=16, B=1, iters=100, precision="complex64"),
    "c2": dict(F=513, T=512, M=4, N=3, K=8, B=256, iters=100, precision="complex64"),
    "c3": dict(F=1025, T=8192, M=16, N=6, K=32, B=1, iters=100, precision="complex64"),
    "c0": dict(F=257, T=128, M=4, N=2, K=8, B=1, iters=50, precision="complex128"),
    "c4": dict(F=513, T=512, M=8, N=2, K=32, B=1, iters=100, precision="complex64", dp=True),
    # config-4 shape on the reference's own default latent path: ToyDecoder +
    # Metropolis (30 proposals/iteration, device Philox draws)
    "c4mh": dict(F=513, T=512, M=8, N=2, K=32, B=1, iters=100, precision="complex64", dp=True,
                 mh=True),
}
METRIC = "FastMNMF TF-bin*ch updates/s (F*T*M*mixtures*iterations/s)"
UNIT = "TF-bin*ch/s"


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def peaks():
    p = os.path.join(REPO, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=10)
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        busy = [s for s in sm if mx and s > 0.5 * mx] or sm
        return {"sm_mhz": statistics.median(busy) if busy else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def make_problem(cfg, seed, torch, dev):
    """Synthetic mixture(s) of the config-0 generator and the BASELINE init."""
    from paper_1903_03237_b200.synth import baseline_init, make_mixture, make_mixture_torch

    F, T, M, N, K, B = cfg["F"], cfg["T"], cfg["M"], cfg["N"], cfg["K"], cfg["B"]
    cdt = torch.complex64 if cfg["precision"] == "complex64" else torch.complex128
    Xs, inits = [], []
    for b in range(B):
        if F * T * M * N <= 20_000_000:
            X = torch.from_numpy(make_mixture(F, T, M, N, K, seed + b)).to(dev, cdt)
        else:
            X = make_mixture_torch(F, T, M, N, K, seed + b, device=dev, dtype=cdt)
        Xs.append(X)
        inits.append(baseline_init(F, T, M, N, K, seed + b))
    X = torch.stack(Xs)
    init = tuple(torch.from_numpy(np.stack([i[k] for i in inits])) for k in range(4))
    return X, init


def run_reference(args, cfg, world, rank):
    """--impl reference: the oracle on the host cores (bounded sample)."""
    if rank != 0:
        return
    from oracle.fastmnmf_oracle import run_fastmnmf
    from paper_1903_03237_b200.synth import baseline_init, make_mixture

    F, T, M, N, K = cfg["F"], cfg["T"], cfg["M"], cfg["N"], cfg["K"]
    if cfg.get("dp"):  # FastMNMF-DP: Adam (c4) or the reference's Metropolis chain (c4mh)
        from oracle import fastmnmf_dp_oracle as DO

        dec = DO.ToyDecoder(F) if cfg.get("mh") else DO.ExpMLPDecoder(F, seed=0)
        X = DO.make_dp_mixture(F, T, M, K, dec, 0).astype(np.complex64).astype(np.complex128)
        init = DO.dp_init(F, T, M, K, dec.latent_dim, 0)

        def one():
            hook = DO.MetropolisLatents(np.random.default_rng(0)) if cfg.get("mh") else None
            DO.run_fastmnmf_dp(X, *init, dec, 1, adam_steps=0 if hook else 10, hook=hook,
                               want_images=False)
    else:
        X = make_mixture(F, T, M, N, K, 0)
        if cfg["precision"] == "complex64":
            X = X.astype(np.complex64).astype(np.complex128)
        init = baseline_init(F, T, M, N, K, 0)

        def one():
            run_fastmnmf(X, *init, n_iterations=1, want_images=False)
    for _ in range(args.warmup):
        one()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        one()
    dt = (time.perf_counter() - t0) / args.steps
    value = F * T * M / dt
    cores = os.cpu_count()
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (BASELINE config-0 generator, seed 0)",
        "config": {"workload": f"{args.config}: F={F} T={T} M={M} N={N} K={K}, "
                               "one FastMNMF iteration per step (bounded CPU sample)"},
        "iters_per_s": 1.0 / dt,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": f"{args.steps} single iterations of {args.config} after "
                                   f"{args.warmup} warm-up, numpy oracle (fp64)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def cpu_baseline_sample(cfg, n_iter=2):
    from oracle.fastmnmf_oracle import run_fastmnmf
    from paper_1903_03237_b200.synth import baseline_init, make_mixture

    F, T, M, N, K = cfg["F"], cfg["T"], cfg["M"], cfg["N"], cfg["K"]
    X = make_mixture(F, T, M, N, K, 0)
    init = baseline_init(F, T, M, N, K, 0)
    run_fastmnmf(X[:, :64], init[0], init[1], init[2], init[3][:, :, :64], 1, want_images=False)
    t0 = time.perf_counter()
    run_fastmnmf(X, *init, n_iterations=n_iter, want_images=False)
    dt = (time.perf_counter() - t0) / n_iter
    return {"value": F * T * M / dt, "unit": UNIT, "cores": os.cpu_count(), "kind": "port",
            "sample": f"{n_iter} FastMNMF iterations of the full config ({F}x{T}x{M}) with the "
                      "numpy oracle (fp64; einsum single-threaded, BLAS on all cores)"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="c1", choices=sorted(CONFIGS))
    ap.add_argument("--iters", type=int, default=None, help="override iterations per step")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    cfg = dict(CONFIGS[args.config])
    if args.iters:
        cfg["iters"] = args.iters
    world, rank, local = dist_env()

    if args.impl == "reference":
        run_reference(args, cfg, world, rank)
        return

    import ctypes

    import torch
    import torch.distributed as dist

    from paper_1903_03237_b200 import _lib
    from paper_1903_03237_b200.dist import shard_batch, shard_range
    from paper_1903_03237_b200.separate import DeviceLoop, SeparatorConfig, _prepare_observation, run

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    lib = _lib.load()

    F, T, M, N, K, iters = cfg["F"], cfg["T"], cfg["M"], cfg["N"], cfg["K"], cfg["iters"]
    B_total = cfg["B"]
    sharded_f = args.config == "c3" and world > 1
    if args.config == "c2":
        b0, b1 = shard_batch(B_total, rank, world)
        cfg["B"] = b1 - b0
        seed0 = b0
    else:
        seed0 = 0 if args.config == "c3" else rank
    X, init = make_problem(cfg, seed0, torch, dev)
    scfg = SeparatorConfig(n_sources=N, n_basis=K, n_iterations=iters,
                           precision=cfg["precision"])
    allreduce = None
    f_off = 0
    if sharded_f:
        from paper_1903_03237_b200.dist import FrequencyShardedRun

        f0, f1 = shard_range(F, rank, world)
        Xl = X[:, f0:f1].contiguous()
        initl = (init[0][:, f0:f1], init[1][:, :, f0:f1], init[2][:, :, f0:f1], init[3])
        runner = FrequencyShardedRun(Xl, initl, F, rank, world, n_iterations=iters)
        loop = runner.loop
        Xs = Xl
        f_off = f0
    elif cfg.get("dp"):
        from paper_1903_03237_b200.dp import ExpMLPDecoder
        from paper_1903_03237_b200.synth import dp_init, make_dp_mixture

        from paper_1903_03237_b200.dp import ToyDecoder

        dec = ToyDecoder(F) if cfg.get("mh") else ExpMLPDecoder(F, seed=0)
        X = torch.from_numpy(make_dp_mixture(F, T, M, K, dec, 0)).to(dev, torch.complex64)[None]
        Q0, g0, u0, v0, z0, W0, H0 = dp_init(F, T, M, K, dec.latent_dim, 0)
        init = tuple(torch.from_numpy(a)[None] for a in (Q0, g0, W0, H0))
        Xs, scale, floor = _prepare_observation(X, scfg, torch)
        latent = (0, 1e-2, 30, 1e-4, None, 0) if cfg.get("mh") else (10, 1e-2)
        loop = DeviceLoop(Xs, init[0], init[1], init[2], init[3], floor, True, 1, n_trace=iters,
                          dp=(dec, u0, v0, z0) + latent)
        dp_init_dev = [t.clone() for t in (loop.dp.u, loop.dp.v, loop.dp.z)]
    else:
        Xs, scale, floor = _prepare_observation(X, scfg, torch)
        loop = DeviceLoop(Xs, init[0], init[1], init[2], init[3], floor, True, 1, n_trace=iters)
    init_dev = [t.to(dev, d.dtype) for t, d in zip(init if not sharded_f else initl,
                                                   (loop.Q, loop.g, loop.W, loop.H))]
    def reset():
        loop.Q.copy_(init_dev[0].reshape(loop.Q.shape))
        loop.g.copy_(init_dev[1].reshape(loop.g.shape))
        loop.W.copy_(init_dev[2].reshape(loop.W.shape))
        loop.H.copy_(init_dev[3].reshape(loop.H.shape))
        loop.status.fill_(-1)
        loop.iterations_done = 0
        if loop.dp is not None:
            for dst, src in zip((loop.dp.u, loop.dp.v, loop.dp.z), dp_init_dev):
                dst.copy_(src)
            loop.dp.m.zero_()
            loop.dp.v2.zero_()
            loop.dp.step.zero_()

    use_graph = not sharded_f
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)

    def step():
        loop.prologue()
        loop.run(iters, use_graph=use_graph)

    for _ in range(args.warmup):
        reset()
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = ClockSampler(local)
    clocks.start()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    for i in range(args.steps):
        reset()
        flush.fill_(i & 0xFF)  # write 256 MiB > L2 between timed steps
        ev[i][0].record()
        step()
        ev[i][1].record()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    total_ms = sum(a.elapsed_time(b) for a, b in ev)
    t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    err = loop.status_error()
    if err is not None:
        raise err
    # whole-job units: every rank's mixtures (c1 replicas, c2 batch shards) or the
    # one sharded recording (c3) -- F*T*M*B*iterations per step
    if args.config == "c2":
        units = F * T * M * B_total * iters
    elif sharded_f:
        units = F * T * M * iters
    else:
        units = F * T * M * cfg["B"] * iters * world
    value = units / (ms_per_step / 1e3)
    iters_per_s = iters / (ms_per_step / 1e3)

    # ---- roofline of the dominant kernel: per-kernel CUDA events on the launch stream
    names = ["k_wstats", "k_lambda(W)", "k_phi", "k_hstats", "k_lambda(H)", "k_gain", "k_vacc",
             "k_ip", "k_back"]
    acc = np.zeros(9)
    nprof = 10
    if not sharded_f and loop.dp is None:
        ms = (ctypes.c_float * 9)()
        for _ in range(nprof):
            _lib.check(lib.fm_iterate_profiled(ctypes.byref(loop.dims), ctypes.byref(loop.state), ms,
                                               _lib.stream_ptr()), "fm_iterate_profiled")
            acc += np.array(ms[:])
        acc /= nprof
    dom = int(np.argmax(acc)) if acc.any() else len(names) - 1
    rs = 4 if cfg["precision"] == "complex64" else 8
    Bl = cfg["B"]
    ftm = F * T * M * Bl if not sharded_f else (loop.F * T * M)
    # algorithmic bytes per launch
    alg = {
        "k_gain": ftm * rs + N * (ftm // M) * rs,          # read xt, lambda
        "k_vacc": ftm * 2 * rs + N * (ftm // M) * rs,      # read X, lambda
        "k_back": ftm * (2 * rs + rs) + 3 * N * (ftm // M) * rs,  # read X, lambda; write xt, phi
        "k_hstats": 2 * N * (ftm // M) * rs,               # read phi1, phi2
        "k_wstats": 2 * N * (ftm // M) * rs,               # read phi1, phi2
        "k_phi": ftm * rs + 3 * N * (ftm // M) * rs,       # read xt, lambda; write phi
        "k_lambda(W)": N * (ftm // M) * rs,                # write lambda
        "k_lambda(H)": N * (ftm // M) * rs,
        "k_ip": 0,
    }[names[dom]]
    hbm, peak_kind = peaks()
    achieved = alg / (acc[dom] / 1e3) / 1e9 if acc[dom] > 0 else None
    traffic = None
    tpath = os.path.join(REPO, "profiles", "traffic.json")
    if os.path.exists(tpath):
        traffic = json.load(open(tpath)).get(f"{args.config}:{names[dom]}")
    roofline = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                "frac": (achieved / hbm) if achieved else None, "traffic": traffic,
                "kernel": names[dom], "peak_kind": peak_kind,
                "kernel_ms": {n: float(v) for n, v in zip(names, acc)},
                "step_share": float(acc[dom] * iters / ms_per_step) if ms_per_step else None,
                "alg_bytes_per_launch": alg}
    if names[dom] == "k_vacc" and acc[dom] > 0:
        # the V accumulation is FP32-pipe bound, not HBM bound: its
        # compute roofline beside the contract's HBM one. Algorithmic flops per
        # (f, t): P = M(M+1)/2 Hermitian pairs x M weights x 4 (real x complex
        # FMA) + 6 per pair product + the model power (2NM) and M reciprocals
        P = M * (M + 1) // 2
        flops = (4 * P * M + 6 * P + 2 * N * M + M) * (ftm // M)
        peak_sm = float(json.load(open(os.path.join(REPO, "MEASURED_PEAKS.json")))["sm_max_mhz"]) \
            if os.path.exists(os.path.join(REPO, "MEASURED_PEAKS.json")) else 1965.0
        fp32_peak = 148 * 128 * 2 * peak_sm * 1e6 / 1e12  # TFLOP/s (FFMA, all SMs, max clock)
        ach = flops / (acc[dom] / 1e3) / 1e12
        roofline["compute"] = {"bound": "fp32-fma", "achieved": ach, "peak": fp32_peak,
                               "unit": "TFLOP/s", "frac": ach / fp32_peak,
                               "alg_flops_per_launch": flops,
                               "peak_kind": "nominal 148 SM x 128 FP32 lanes x 2 x max SM clock"}

    # ---- e2e: the public API call with host buffers (pinned), copies inside the timed region
    e2e = None
    if not args.no_e2e and not sharded_f and args.config in ("c1", "c0"):
        Xh = X[0].cpu().pin_memory()
        # warm: two results alive at once, as in the timed loop below (the pinned
        # image blocks come from torch's caching host allocator)
        w1 = run(scfg, Xh, init=tuple(a[0].numpy() for a in init))
        w2 = run(scfg, Xh, init=tuple(a[0].numpy() for a in init))
        del w1, w2
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()  # every replica's e2e calls run concurrently
        reps = 5
        prof = None
        if os.environ.get("BENCH_E2E_PROFILE"):
            import cProfile

            prof = cProfile.Profile()
            prof.enable()
        calls = []
        for _ in range(reps):  # per-call wall times; the median is reported (robust to a
            t0 = time.perf_counter()  # stray host hiccup), every call is listed
            res = run(scfg, Xh, init=tuple(a[0].numpy() for a in init))
            calls.append(time.perf_counter() - t0)
        dt = float(np.median(calls))
        if world > 1:  # whole-job: the slowest replica's wall time, all replicas' units
            tdt = torch.tensor([dt], dtype=torch.float64, device=dev)
            dist.all_reduce(tdt, op=dist.ReduceOp.MAX)
            dt = float(tdt.item())
        if prof is not None:
            import pstats

            prof.disable()
            pstats.Stats(prof, stream=sys.stderr).sort_stats("cumulative").print_stats(20)
        cb = 8 if cfg["precision"] == "complex64" else 16
        # bytes per step of the whole job (every replica copies its own)
        h2d = (F * T * M * cb + F * M * M * 16 + N * F * M * 8 + N * F * K * 8 + N * K * T * 8) * world
        d2h = (N * F * T * M * cb + iters * 8) * world
        e2e = {"value": F * T * M * iters * world / dt, "unit": UNIT, "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "seconds_per_step": dt,
               "seconds_per_call": [round(c, 5) for c in calls],
               "api": "paper_1903_03237_b200.run(SeparatorConfig, X_host_pinned, init=...)"}
        del res

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and args.config in ("c1", "c0"):
        cpu = cpu_baseline_sample(cfg)

    launches = args.steps * (2 + (10 if cfg['B'] == 1 else 11) * iters)
    if cfg.get("dp"):  # 21 per iteration (one latent-hook launch: Adam or Metropolis), 4 in the prologue
        launches = args.steps * (4 + 21 * iters)
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "weak" if not sharded_f else "strong", "vs_baseline": None,
            "dtype": "f32" if cfg["precision"] == "complex64" else "f64",
            "data": "synthetic (BASELINE config-0 generator: Gamma NMF PSDs, random full-rank "
                    "SCMs, circular Gaussian excitation; seeded)",
            "config": {"workload": f"{args.config}: F={F} T={T} M={M} N={N} K={K} "
                                   f"mixtures={B_total if args.config == 'c2' else cfg['B']} "
                                   f"{cfg['precision']}, {iters} iterations per step",
                       "parallelism": ("frequency-sharded" if sharded_f else
                                       "batch-sharded" if args.config == "c2" else "replicas")
                                      + f" x{world}",
                       "l2": "flushed between steps (256 MiB write)"},
            "iters_per_s": iters_per_s, "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": launches, "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
