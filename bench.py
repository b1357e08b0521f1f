#!/usr/bin/env python
"""Benchmark: sampled nonzeros/s per SGD epoch (A + B update), BASELINE.json.

Workload (N=1): BASELINE configs[1], the Netflix-shaped synthetic tensor
480,189 x 17,770 x 2,182 with 99,072,112 training nonzeros (+1,408,395 test
entries), J = R = 16, fp32, throughput (Hogwild) mode.  One "step" is one
epoch: the bit-exact GPU visit-order sampler, the factor pass over every
nonzero, the core-batch sampler (2^20 of 99M, Floyd) and the core gradient +
apply -- exactly the work inside the reference's wall_seconds
(trainer.py:187-249), evaluation excluded.

Keys beyond the driver contract:
  roofline      the factor kernel (dominant) against the measured HBM copy
                bandwidth; achieved = algorithmic bytes / CUDA-event duration
                with B_f = 4(N+1) + 8*sum(J_n) bytes per nonzero
  cpu_baseline  the oracle C port of the reference (oracle/, fp64, DSGD
                threads) timed on a prefix sample of the same workload
  e2e           the public API train() on host numpy arrays (upload,
                partition, epochs, per-epoch evaluation, download) per epoch

  python bench.py [--gpus N --steps K --warmup W] [--impl reference]
                  [--config nf|cfg1|y4|o6] [--rank J]
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "sampled nonzeros/sec per SGD epoch (A+B update) at 1/2/4/8 B200; test RMSE"

CONFIGS = {
    # workers: the reference's TrainConfig.workers (DSGD blocks per mode).
    # NF runs its DSGD schedule with 20 blocks per mode on the one GPU: the
    # fastest of the measured W = 12/16/18/20/24/28/32 (18.8/10.3/10.2/9.7/
    # 9.9/10.0/10.4 ms per epoch, W=1: 14.8; profiles/r02), same test RMSE
    # (0.4784 vs 0.4786 at W=1)
    "nf": dict(workload="netflix-shaped 480189x17770x2182, 99,072,112 nnz, J=R=16",
               dims=(480189, 17770, 2182), nnz=99_072_112, n_test=1_408_395, J=16, R=16, alpha_a=0.003,
               workers=20),
    "cfg1": dict(workload="synthetic 1Kx1Kx1K, 90K train / 10K test, J=R=8",
                 dims=(1000, 1000, 1000), nnz=90_000, n_test=10_000, J=8, R=8),
    # alpha_a: the reference's default 0.009 diverges on these std-4 synthetic
    # tensors; 0.003 (NF) and 0.001 (Y4, J = R = 32), 0.0003 (J = R = 64) are the largest
    # rates at which the reference's own train() converges (oracle runs on
    # 2M-4M prefixes of the same tensors; at 0.003 Y4 goes to NaN).
    # workers: Y4 12 (W = 1/10/12/16/24: 62.5/44.0/41.6/42.4/49.5 ms), O6 8
    # (W = 1/6/8/10: 230/132/129/139 ms), same test RMSE
    "y4": dict(workload="yahoo-shaped 1000990x624961x3075x133, 250,272,286 nnz, J=R=16",
               dims=(1_000_990, 624_961, 3_075, 133), nnz=250_272_286, n_test=2_502_723, J=16, R=16,
               alpha_a=0.001, workers=12),
    "o6": dict(workload="6-order 10K^6, 1e9 nnz, J=R=8",
               dims=(10_000,) * 6, nnz=1_000_000_000, n_test=1_000_000, J=8, R=8, alpha_a=0.001, workers=8),
}


def bytes_per_nnz(order, J):
    """int32 indices + fp32 value, one read and one write of each row."""
    return 4 * (order + 1) + 8 * order * J


def factor_traffic(workload, workers=1):
    """dram__bytes_read.sum + dram__bytes_write.sum per factor-kernel launch from
    the committed ncu --set full capture of this workload (profiles/), or None."""
    p = os.path.join(ROOT, "profiles", "factor_traffic.json")
    try:
        with open(p) as fh:
            d = json.load(fh)
        return d["bytes_per_launch"] if d.get("workload") == workload and d.get("workers", 1) == workers else None
    except Exception:
        return None


def measured_peak_gbs():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    def __init__(self, index=0):
        self.index = index
        self.proc = None
        self.path = tempfile.mktemp(suffix=".csv")

    def start(self):
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=self.fh, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        time.sleep(0.25)
        self.proc.terminate()
        self.proc.wait()
        self.fh.close()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = float(parts[2])
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return None
        sm.sort()
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def make_data(cfg, nnz=None, use_gpu=True, with_test=True):
    from paper_2204_07104_b200.synthetic import generate_large

    pred = None
    if use_gpu:
        from paper_2204_07104_b200.device import predict_device_f64

        def pred(model, idx):
            import numpy as np

            out = np.empty(idx.shape[0])
            step = 1 << 25
            for c0 in range(0, idx.shape[0], step):
                out[c0:c0 + step] = predict_device_f64(model, idx[c0:c0 + step])
            return out
    order = len(cfg["dims"])
    return generate_large(cfg["dims"], nnz or cfg["nnz"], (cfg["J"],) * order, cfg["R"], 0.1, seed=7,
                          n_test=cfg["n_test"] if with_test else 0, predict=pred)


def cpu_sample_size(cfg):
    # ~10-30 s of single-epoch CPU work on 16 cores for J=16; smaller ranks scale up
    per = bytes_per_nnz(len(cfg["dims"]), cfg["J"])
    return int(min(cfg["nnz"], max(200_000, 2_000_000 * 400 // per)))


def run_cpu_reference(cfg, sample, epochs, threads):
    """Oracle C port (fp64, DSGD threads) on a prefix sample; returns (nnz/s list, sample desc)."""
    import numpy as np

    from oracle import oracle as O
    from paper_2204_07104_b200 import ModelConfig, default_init_scale, init_model

    tr, _, _ = make_data(cfg, nnz=sample, use_gpu=False, with_test=False)
    order = len(cfg["dims"])
    workers = max(1, min(threads, min(cfg["dims"])))
    model = init_model(cfg["dims"], ModelConfig((cfg["J"],) * order, cfg["R"],
                                                default_init_scale(tr.values, order), seed=1))
    fs = [a.copy() for a in model.factors]
    bs = [b.copy() for b in model.core_factors]
    rates = []
    for t in range(epochs):
        rows = O.train(fs, bs, tr.indices, tr.values, epochs=1, workers=workers, seed=1, evaluate=False,
                       dims=cfg["dims"], alpha_a=cfg.get("alpha_a", 0.009))
        rates.append(sample / rows[-1]["wall_seconds"])
    desc = (f"oracle C port (fp64, {workers} DSGD worker threads) on the first {sample:,} nonzeros of the "
            f"same workload, 1 epoch per step")
    return rates, workers, desc


def bench_reference(args, cfg):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    threads = len(os.sched_getaffinity(0))
    sample = cpu_sample_size(cfg)
    rates, workers, desc = run_cpu_reference(cfg, sample, args.warmup + args.steps, threads)
    timed = rates[args.warmup:]
    value = sum(timed) / len(timed)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "nnz/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 * sample / value,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (generate_large, seed 7)",
        "config": {"workload": cfg["workload"], "sample_nnz": sample},
        "cpu_baseline": {"value": value, "unit": "nnz/s", "cores": workers, "kind": "port", "sample": desc},
        "e2e": {"value": value, "unit": "nnz/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def log(msg):
    print(f"[bench {time.strftime('%H:%M:%S')}] {msg}", file=sys.stderr, flush=True)


def bench_ours(args, cfg):
    import numpy as np
    import torch

    from paper_2204_07104_b200 import (DatasetSplit, ModelConfig, TrainConfig, default_init_scale,
                                       init_model, train)
    from paper_2204_07104_b200 import _lib
    from paper_2204_07104_b200.device import DeviceCoo, rmse_mae_device
    from paper_2204_07104_b200.training import EpochRunner, learning_rate

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    # BENCH_FORCE_DIST=1: the multi-GPU code path (NCCL, DistRunner) even at
    # world size 1 (exercises it on a one-GPU box)
    distributed = world > 1 or os.environ.get("BENCH_FORCE_DIST") == "1"
    if distributed:
        import torch.distributed as td

        td.init_process_group("nccl", device_id=torch.device("cuda", local))
    L = _lib.load()
    order = len(cfg["dims"])
    t0 = time.time()
    tr, te, _ = make_data(cfg)
    gen_s = time.time() - t0
    log(f"data ready ({gen_s:.1f} s)")
    scale = default_init_scale(tr.values, order)
    model = init_model(cfg["dims"], ModelConfig((cfg["J"],) * order, cfg["R"], scale, seed=1))
    # +3: every timed epoch also draws the next epoch's samples (steady state)
    sim = int(os.environ.get("BENCH_DSGD_SIM", "0"))
    # M GPUs (or the M-rank simulation): the config's DSGD blocks per mode
    # rounded up to a multiple of M -- each rank's slab keeps the reference's
    # W-worker blocks (dsgd_fused.sub_rounds; NF: W = 20 at M = 2 / 4, 24 at 8)
    ranks = world if world > 1 else max(sim, 1)
    w0 = cfg.get("workers", 1)
    workers = args.workers if args.workers else (-(-w0 // ranks) * ranks if ranks > 1 else w0)
    tcfg = TrainConfig(epochs=args.warmup + args.steps + 3, seed=1, update_mode=args.mode,
                       workers=workers, alpha_a=cfg.get("alpha_a", 0.009))
    if distributed:
        from paper_2204_07104_b200 import dist

        from paper_2204_07104_b200.dsgd_fused import FusedDistRunner, fused_supported

        if fused_supported(model, tcfg, tr.nnz) and os.environ.get("SPTK_DSGD_FUSED", "1") == "1":
            runner = FusedDistRunner(model, tr, tcfg)
        else:
            runner = dist.DistRunner(model, tr, tcfg)
    elif sim > 1:
        # one rank's share of an M-GPU DSGD epoch (its blocks, their samplers,
        # the core phase): the fused per-rank launch with its pushes aimed at
        # its own replica and its ready flag raised in advance (no peer to
        # wait for) -- a per-rank compute estimate without NVLink transfers
        from dataclasses import replace

        from paper_2204_07104_b200.dsgd_fused import FusedRankRunner, fused_supported

        if fused_supported(model, replace(tcfg, update_mode="hogwild")) and os.environ.get("BENCH_SIM_FUSED", "1") == "1":
            runner = FusedRankRunner(model, tr, replace(tcfg, update_mode="hogwild"), 0, sim)
            fa, ra = runner.fused.peer_addresses()
            runner.set_peers([fa] * sim, [ra] * sim)
            runner.fused.ready.fill_(1 << 30)
            runner.fused.epoch_flag.fill_(1 << 30)
        else:
            runner = EpochRunner(model, tr, tcfg, owner_rank=0)
    else:
        runner = EpochRunner(model, tr, tcfg)
    # warm-up epochs (not timed)
    for t in range(args.warmup):
        runner.epoch(t, learning_rate(tcfg.alpha_a, tcfg.beta_a, t), learning_rate(tcfg.alpha_b, tcfg.beta_b, t))
    torch.cuda.synchronize()
    log("warm-up done")
    runner.factor_events = []
    clocks = ClockSampler(local)
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    clocks.start()
    profile = os.environ.get("BENCH_PROFILE") == "1"
    if profile:
        torch.cuda.profiler.start()
    n0 = L.sptk_launch_count()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record()
    for t in range(args.warmup, args.warmup + args.steps):
        runner.epoch(t, learning_rate(tcfg.alpha_a, tcfg.beta_a, t), learning_rate(tcfg.alpha_b, tcfg.beta_b, t))
    ev1.record()
    ev1.synchronize()
    if profile:
        torch.cuda.profiler.stop()
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    launches = L.sptk_launch_count() - n0
    # the factor kernel libsptk actually dispatched in the timed epochs
    kernel = L.sptk_last_factor_kernel().decode()
    clk = clocks.stop()
    log("timed region done")
    ms = ev0.elapsed_time(ev1)
    if world > 1:
        tt = torch.tensor([ms], device="cuda")
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        ms = float(tt.item())
    ms_per_step = ms / args.steps
    value = cfg["nnz"] * args.steps / (ms / 1000.0)
    fdur = [a.elapsed_time(b) for a, b in runner.factor_events]
    f_ms = sum(fdur) / len(fdur) if fdur else float("nan")
    nnz_local = runner.nnz_local if hasattr(runner, "nnz_local") else cfg["nnz"]
    launches_per_epoch = len(fdur) / args.steps if fdur else 1
    algo_bytes = bytes_per_nnz(order, cfg["J"]) * nnz_local / launches_per_epoch
    peak, peak_src = measured_peak_gbs()
    achieved = algo_bytes / (f_ms / 1000.0) / 1e9
    if os.environ.get("BENCH_TIMELINE") == "1":
        runner.timeline = []
        for t in range(args.warmup + args.steps, args.warmup + args.steps + 2):
            runner.epoch(t, learning_rate(tcfg.alpha_a, tcfg.beta_a, t), learning_rate(tcfg.alpha_b, tcfg.beta_b, t))
        for row in runner.timeline:
            log(f"timeline {json.dumps(row)}")
    # accuracy after the run
    test_rmse = None  # (a simulated rank's model is not a trained model: none)
    if te is not None and rank == 0 and sim <= 1:
        test_rmse = rmse_mae_device(runner.dm, DeviceCoo(te.indices, te.values))[0]
    # end to end through the public API (host arrays in, model out)
    e2e = None
    if not args.no_e2e and sim <= 1:
        k2 = args.e2e_epochs or args.steps
        # five end-to-end runs, the median reported (host-side phases --
        # upload threads, page faults -- vary run to run on the GPU boxes);
        # on M ranks train() runs the distributed path on every rank and a
        # run's time is the slowest rank's
        runs = []
        for _ in range(5):
            m2 = init_model(cfg["dims"], ModelConfig((cfg["J"],) * order, cfg["R"], scale, seed=1))
            torch.cuda.synchronize()
            if distributed:
                torch.distributed.barrier()
            t1 = time.perf_counter()
            train(m2, DatasetSplit(tr, te), TrainConfig(epochs=k2, seed=1, update_mode=args.mode, workers=workers,
                                                        alpha_a=cfg.get("alpha_a", 0.009)))
            torch.cuda.synchronize()
            el1 = time.perf_counter() - t1
            if distributed:
                tt = torch.tensor([el1], dtype=torch.float64, device="cuda")
                torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
                el1 = float(tt.item())
            runs.append(el1)
        el = sorted(runs)[len(runs) // 2]
        # what crosses PCIe: fp32 records (packed by the upload threads, 4 words
        # per nonzero at order <= 3, 8 up to 7) and the fp32 model
        rw = 4 if order <= 3 else 8
        h2d = (tr.nnz + te.nnz) * rw * 4 + sum(a.size * 4 for a in m2.factors + m2.core_factors)
        d2h = sum(a.nbytes for a in m2.factors + m2.core_factors) + 32 * k2
        log("e2e done")
        e2e = {"value": cfg["nnz"] * k2 / el, "unit": "nnz/s", "h2d_bytes_per_step": h2d // k2,
               "d2h_bytes_per_step": d2h // k2, "epochs": k2, "seconds": el,
               "runs_seconds": [round(x, 4) for x in runs], "statistic": "median of 5 runs",
               "what": "public train() on host numpy arrays: upload + K1 partition + epochs + per-epoch "
                       "train/test RMSE + model download, divided per epoch"}
    cpu = None
    if not args.no_cpu_baseline and rank == 0 and world == 1:
        threads = len(os.sched_getaffinity(0))
        sample = cpu_sample_size(cfg)
        rates, cpu_workers, desc = run_cpu_reference(cfg, sample, 1, threads)
        cpu = {"value": rates[-1], "unit": "nnz/s", "cores": cpu_workers, "kind": "port", "sample": desc}
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "nnz/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None,
            "dtype": "fp32" if kernel in ("factor_seq_kernel", "factor_tps_kernel", "factor_wps_kernel",
                                          "factor_fma_kernel") else "fp32 (tf32 tensor-core contractions)",
            "data": "synthetic (generate_large seed 7: i.i.d. uniform indices, reference ground-truth "
                    "model, std 4, noise 0.1)",
            "config": {"workload": cfg["workload"], "dims": list(cfg["dims"]), "nnz": cfg["nnz"],
                       "J": cfg["J"], "R": cfg["R"], "core_batch": min(cfg["nnz"], 1 << 20),
                       "update_mode": (args.mode if args.mode != "auto" else
                                       "exact" if cfg["nnz"] <= (1 << 22) else "hogwild"), "parallelism": f"dsgd{world}" if world > 1 else "single", "workers": workers,
                       "l2": "inputs larger than L2 (records + visit order ~2 GB per epoch); the 32 MB "
                             "model is L2-resident by design"},
            "test_rmse": test_rmse,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": factor_traffic(cfg["workload"], workers),
                         "kernel": kernel,
                         "kernel_ms": f_ms, "kernel_share": f_ms * launches_per_epoch / ms_per_step,
                         "algorithmic_bytes_per_launch": algo_bytes, "peak_source": peak_src,
                         "frac_of_8TBs": achieved / 8000.0},
            "epoch_roofline_frac_8TBs": bytes_per_nnz(order, cfg["J"]) * cfg["nnz"] / (ms_per_step / 1000) / 8e12,
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches, "clocks": clk,
            "setup_seconds": {"data_generation": gen_s},
        }
        print(json.dumps(line), flush=True)
    if distributed:
        torch.distributed.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="nf", choices=sorted(CONFIGS))
    ap.add_argument("--rank", type=int, default=None, help="J = R override (rank sweep)")
    ap.add_argument("--alpha-a", type=float, default=None, help="factor learning-rate override")
    ap.add_argument("--workers", type=int, default=None,
                    help="DSGD workers W (the reference's TrainConfig.workers) on the GPU(s)")
    # auto = the library default: exact (sequential) up to 2^22 training
    # nonzeros (cfg1), Hogwild above (NF, Y4, O6)
    ap.add_argument("--mode", default="auto", choices=["hogwild", "exact", "auto"])
    ap.add_argument("--e2e-epochs", type=int, default=None, help="default: --steps")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    cfg = dict(CONFIGS[args.config])
    if args.rank:
        cfg["J"] = cfg["R"] = args.rank
        cfg["workload"] = cfg["workload"].split(", J=")[0] + f", J=R={args.rank}"
        if args.rank >= 32:
            # the rates of the reference curves (tests/golden/curve_nf8m_j32/j64)
            cfg["alpha_a"] = 0.001 if args.rank < 64 else 0.0003
    if args.alpha_a is not None:
        cfg["alpha_a"] = args.alpha_a
    if args.impl == "reference":
        bench_reference(args, cfg)
    else:
        bench_ours(args, cfg)


if __name__ == "__main__":
    main()
