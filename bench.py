#!/usr/bin/env python
"""Benchmark: dense FP64 MTTKRP on B200 (BASELINE.json metric / configs[1]).

Workload (N=1): 1000 x 1000 x 1000 FP64 tensor (8 GB, natural order,
U[0,1) entries), rank C=25 U[0,1) factors; one STEP = the MTTKRP of every
mode with the reference's automatic routing (1-step on the boundary modes,
2-step on the interior mode, reference mttkrp.cpp:395-401). Three full
tensor passes per step.

value    tensor GB/s over the whole job (8*I bytes per mode pass), inputs
         resident in HBM, CUDA events on the launching stream, max over ranks.
e2e      the same metric through the reference-facing C ABI with host buffers:
         every step uploads the tensor from pinned host memory
         (dmtk_gpu_tensor_upload), runs dmtk_gpu_mttkrp per mode with host
         factors, and reads each result back to the host.
N > 1    torchrun, one process per GPU, weak scaling: rank r owns a
         1000 x 1000 x 1000 slab of a 1000 x 1000 x (1000 N) tensor (last-mode
         shard); modes 0 and 1 finish with an NCCL all-reduce of
         the I_n x C partial, mode 2 rows are disjoint (no exchange).

--impl reference runs the unmodified reference library (compiled from
/root/reference into oracle/_ref/libdmtk_ref.so) on the host cores for the
same metric and config.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

CONFIGS = {
    "1000c25": ((1000, 1000, 1000), 25),
    "1000c50": ((1000, 1000, 1000), 50),
    "180c25": ((180, 180, 180, 180), 25),
    "64c32": ((64, 64, 64, 64, 64), 32),
    "200c16": ((200, 200, 200), 16),
}
METRIC = "MTTKRP tensor GB/s (all modes, automatic 1-step/2-step routing)"


def env_int(name, default):
    try:
        return int(os.environ.get(name, default))
    except ValueError:
        return default


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d.get("hbm_gbs", 6650.0)), "MEASURED_PEAKS.json"
    return 6650.0, "fallback (B200_PROFILING.md)"


def load_traffic(cfg_name, rank):
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(p):
        return None
    with open(p) as f:
        d = json.load(f)
    return d.get(f"{cfg_name}")


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    def __init__(self, index=0):
        self.index = index
        self.proc = None
        self.path = None

    def start(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index),
                 "--query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
            return
        # nvidia-smi takes a while to start: wait for its first row so that the
        # timed region that follows is sampled from its beginning
        t_end = time.time() + 3.0
        while time.time() < t_end:
            try:
                with open(self.path) as f:
                    if f.readline().strip():
                        break
            except OSError:
                pass
            time.sleep(0.005)

    def stop(self):
        out = {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        if not self.proc:
            return out
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        rows = []
        with open(self.path) as f:
            for line in f:
                parts = [x.strip() for x in line.split(",")]
                if len(parts) >= 8:
                    rows.append(parts)
        os.unlink(self.path)
        if not rows:
            return out
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            for k, n in enumerate(names):
                if r[4 + k].lower().startswith("active"):
                    reasons.add(n)
        out["sm_mhz"] = statistics.median(sm) if sm else None
        out["sm_max_mhz"] = float(rows[0][1]) if rows[0][1].replace(".", "").isdigit() else None
        out["reasons"] = sorted(reasons)
        out["samples"] = len(rows)
        out["power_w_max"] = max(float(r[2]) for r in rows if r[2].replace(".", "").isdigit())
        out["sm_mhz_samples"] = sm
        return out


def host_cpu_info():
    model = "unknown"
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return model, os.cpu_count() or 1


# --------------------------------------------------------------- reference
def run_reference(args, cfg_name, dims, C):
    from oracle_bindings import Ref
    ref = Ref()
    n = int(np.prod(dims))
    rng = np.random.default_rng(1)
    x = rng.random(n)  # U[0,1): same distribution as the GPU arm
    factors = [rng.random((d, C)) for d in dims]
    threads = os.cpu_count() or 1
    nmodes = len(dims)
    # each step is a bounded sample: one mode pass (cycling through the modes)
    for w in range(args.warmup):
        ref.mttkrp(x, dims, factors, w % nmodes, "automatic", "automatic", threads)
    times = []
    for s in range(args.steps):
        t0 = time.perf_counter()
        ref.mttkrp(x, dims, factors, s % nmodes, "automatic", "automatic", threads)
        times.append(time.perf_counter() - t0)
    total = sum(times)
    gbs = 8.0 * n * len(times) / total / 1e9
    model, cores = host_cpu_info()
    line = {
        "impl": "reference", "metric": METRIC, "value": round(gbs, 3), "unit": "GB/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(1e3 * total / len(times), 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic U[0,1) (numpy PCG64 seed 1)",
        "config": {"workload": cfg_name, "dims": list(dims), "rank": C, "algo": "automatic",
                   "step": "one mode pass per step, cycling modes 0..N-1"},
        "cpu_baseline": {"value": round(gbs, 3), "unit": "GB/s", "cores": threads, "kind": "reference",
                         "sample": f"{len(times)} single-mode passes of {cfg_name}", "cpu": model},
        "e2e": {"value": round(gbs, 3), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    emit(line)


# ------------------------------------------------------------ our B200 arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="1000c25", choices=sorted(CONFIGS))
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-als", action="store_true", help="skip the BASELINE config-5 CP-ALS timing block")
    ap.add_argument("--als-sharded", action="store_true",
                    help="run the CP-ALS block as the sharded device-resident ALS even at one GPU (it always is at N > 1)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    dims, C = CONFIGS[args.config]
    rank_id = env_int("RANK", 0)
    world = env_int("WORLD_SIZE", 1)
    local = env_int("LOCAL_RANK", 0)

    if args.impl == "reference":
        if rank_id == 0:
            run_reference(args, args.config, dims, C)
        return

    import torch
    import torch.distributed as dist
    torch.cuda.set_device(local)
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    import paper_1708_08976_b200 as dg
    from paper_1708_08976_b200 import MttkrpAlgo as A, TwoStepOrder as O

    N = len(dims)
    n = int(np.prod(dims))
    dev = torch.device("cuda", local)
    g = torch.Generator(device=dev).manual_seed(1234 + rank_id)
    x = torch.rand(n, dtype=torch.float64, device=dev, generator=g)
    gf = torch.Generator(device=dev).manual_seed(99)  # factors identical on every rank
    fs = [torch.rand((d, C), dtype=torch.float64, device=dev, generator=gf) for d in dims]
    outs = [torch.empty((d, C), dtype=torch.float64, device=dev) for d in dims]
    t = dg.DenseTensor.from_device(dims, x.data_ptr(), device=local, owner=x)
    stream = torch.cuda.Stream(device=dev)
    fptrs = [f.data_ptr() for f in fs]

    def one_step(events=None):
        with torch.cuda.stream(stream):
            for m in range(N):
                if events is not None:
                    events[m][0].record(stream)
                dg.mttkrp_device(t, fptrs, C, m, A.automatic, O.automatic, outs[m].data_ptr(), stream.cuda_stream)
                if events is not None:
                    events[m][1].record(stream)
                if world > 1 and m < N - 1:
                    dist.all_reduce(outs[m])  # partial I_n x C over the last-mode shards

    for _ in range(args.warmup):
        one_step()
    torch.cuda.synchronize()

    peak_tf_burst = dg.fp64_peak_tflops(local)
    # the timed region is a long step under the 1 kW cap: use the settled rate
    peak_tf = dg.fp64_peak_tflops_sustained(1.5, local)
    hbm_peak, hbm_src = load_peaks()

    ev = [[[torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)] for _ in range(N)]
          for _ in range(args.steps)]
    start = torch.cuda.Event(enable_timing=True)
    stop = torch.cuda.Event(enable_timing=True)
    sampler = ClockSampler(local)
    launches0 = dg.launch_count()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    sampler.start()
    start.record(stream)
    for s in range(args.steps):
        one_step(ev[s])
    stop.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = sampler.stop()
    launches = dg.launch_count() - launches0
    ms_total = start.elapsed_time(stop)
    ms = torch.tensor([ms_total], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    ms_total = float(ms.item())
    per_mode = [[ev[s][m][0].elapsed_time(ev[s][m][1]) for s in range(args.steps)] for m in range(N)]

    bytes_per_step = 8.0 * n * N * world
    value = bytes_per_step * args.steps / (ms_total * 1e-3) / 1e9
    ms_step = ms_total / args.steps

    # roofline of the dominant kernel (the streaming MTTKRP, one launch per mode)
    mode_ms = [statistics.mean(v) for v in per_mode]
    avg_launch_s = statistics.mean(mode_ms) * 1e-3
    flops = 2.0 * n * C
    t_hbm = 8.0 * n / (hbm_peak * 1e9)
    t_f64 = flops / (peak_tf * 1e12)
    bound = "tensor" if t_f64 >= t_hbm else "hbm"
    if bound == "tensor":
        achieved, peak, unit = flops / avg_launch_s / 1e12, peak_tf, "TFLOP/s"
    else:
        achieved, peak, unit = 8.0 * n / avg_launch_s / 1e9, hbm_peak, "GB/s"
    modes = []
    for m in range(N):
        s_ = mode_ms[m] * 1e-3
        modes.append({"mode": m, "ms": round(mode_ms[m], 4), "GBs": round(8.0 * n / s_ / 1e9, 1),
                      "TFs": round(flops / s_ / 1e12, 2), "frac_roofline": round(max(t_hbm, t_f64) / s_, 3)})

    # ------------------------------------------------------------- e2e leg
    e2e = None
    if args.e2e_steps > 0:
        hx = torch.empty(n, dtype=torch.float64, pin_memory=True)
        hx.copy_(x)
        hf = [f.cpu().numpy() for f in fs]
        dims_np = np.asarray(dims, dtype=np.int64)
        host_out = [np.empty((d, C)) for d in dims]
        import ctypes as Cc
        from paper_1708_08976_b200 import _lib
        lib = _lib.lib
        fptr_arr = (_lib.dp * N)(*[f.ctypes.data_as(_lib.dp) for f in hf])
        rows = np.asarray(dims, dtype=np.int64)
        cols = np.full(N, C, dtype=np.int64)

        def e2e_step():
            h = Cc.c_void_p()
            rc = lib.dmtk_gpu_tensor_upload(local, N, dims_np.ctypes.data_as(_lib.i64p),
                                            Cc.cast(hx.data_ptr(), _lib.dp), Cc.byref(h))
            assert rc == 0, lib.dmtk_gpu_last_error()
            for m in range(N):
                rc = lib.dmtk_gpu_mttkrp(h, N, fptr_arr, rows.ctypes.data_as(_lib.i64p),
                                         cols.ctypes.data_as(_lib.i64p), m, 3, 0, 1,
                                         host_out[m].ctypes.data_as(_lib.dp), None)
                assert rc == 0, lib.dmtk_gpu_last_error()
            lib.dmtk_gpu_tensor_free(h)
            if world > 1:  # sum the partial results of the last-mode shards
                for m in range(N - 1):
                    part = torch.from_numpy(host_out[m]).to(dev)
                    dist.all_reduce(part)
                    host_out[m][:] = part.cpu().numpy()

        e2e_step()  # warm-up (allocations, plans)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            e2e_step()
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) / args.e2e_steps
        if world > 1:  # the slowest rank sets the job's time
            dtt = torch.tensor([dt], dtype=torch.float64, device=dev)
            dist.all_reduce(dtt, op=dist.ReduceOp.MAX)
            dt = float(dtt.item())
        e2e = {"value": round(8.0 * n * N * world / dt / 1e9, 3), "unit": "GB/s",
               "h2d_bytes_per_step": int(8 * n + sum(d * C * 8 for d in dims) * N),
               "d2h_bytes_per_step": int(sum(d * C * 8 for d in dims)),
               "ms_per_step": round(dt * 1e3, 2), "steps": args.e2e_steps,
               "path": "dmtk_gpu_tensor_upload + dmtk_gpu_mttkrp per mode (host buffers, pinned tensor)"
                       + ("; partials all-reduced over NCCL, max over ranks" if world > 1 else "")}
        del hx

    # ---------------------------------------------------- CPU baseline leg
    cpu = None
    if rank_id == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            from oracle_bindings import Ref
            ref = Ref()
            xs = x.cpu().numpy()
            hf = [f.cpu().numpy() for f in fs]
            threads = os.cpu_count() or 1
            t0 = time.perf_counter()
            for m in range(N):
                ref.mttkrp(xs, dims, hf, m, "automatic", "automatic", threads)
            dt = time.perf_counter() - t0
            model, cores = host_cpu_info()
            cpu = {"value": round(8.0 * n * N / dt / 1e9, 3), "unit": "GB/s", "cores": threads, "kind": "reference",
                   "sample": f"one full step ({N} modes, automatic) of {args.config} on the same bytes, "
                             f"{dt:.1f} s", "cpu": model}
            del xs
        except Exception as e:  # the reference library is test/baseline infrastructure
            cpu = {"value": None, "unit": "GB/s", "cores": os.cpu_count(), "kind": "reference",
                   "sample": f"unavailable: {e}"}

    # -------------------------------- BASELINE config 5: CP-ALS (info block)
    als = None
    if world == 1 and not args.no_als and not args.als_sharded:
        del x, t
        torch.cuda.empty_cache()
        sys.path.insert(0, os.path.join(ROOT, "tools"))
        from perf_als import fmri_tensor
        fd = (100, 100, 1200, 80)
        xf = fmri_tensor(fd)
        tf = dg.DenseTensor.from_device(fd, xf.data_ptr(), device=local, owner=xf)
        dg.cp_als(tf, dg.AlsConfig(rank=20, max_iters=2, tol=0.0, seed=1))
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res = dg.cp_als(tf, dg.AlsConfig(rank=20, max_iters=25, tol=0.0, seed=1))
        wall = time.perf_counter() - t0
        it_ms = sorted(1e3 * r.total_seconds for r in res.trace.iters)
        # the same run as a dimension tree (two tensor passes per iteration)
        dg.cp_als(tf, dg.AlsConfig(rank=20, max_iters=2, tol=0.0, seed=1, dimension_tree=True))
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        rt = dg.cp_als(tf, dg.AlsConfig(rank=20, max_iters=25, tol=0.0, seed=1, dimension_tree=True))
        wall_t = time.perf_counter() - t1
        it_t = sorted(1e3 * r.total_seconds for r in rt.trace.iters)
        # the fMRI slices are symmetric in modes 0/1: packed, both passes read ~half
        tpk = tf.pack_symmetric01()
        dg.cp_als(tpk, dg.AlsConfig(rank=20, max_iters=2, tol=0.0, seed=1))
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        rs = dg.cp_als(tpk, dg.AlsConfig(rank=20, max_iters=25, tol=0.0, seed=1))
        wall_s = time.perf_counter() - t2
        it_s = sorted(1e3 * r.total_seconds for r in rs.trace.iters)
        tpk.release()
        nf = int(np.prod(fd))
        als = {"workload": "fMRI-shaped 100x100x1200x80, rank 20, 25 iterations, tol 0 (BASELINE config 5)",
               "iter_ms_median": round(it_ms[len(it_ms) // 2], 3), "wall_s": round(wall, 4),
               "final_fit": res.trace.iters[-1].fit.fit,
               "roofline_iter_ms": round(4 * 8.0 * nf / (hbm_peak * 1e9) * 1e3, 3),
               "dimension_tree": {"iter_ms_median": round(it_t[len(it_t) // 2], 3), "wall_s": round(wall_t, 4),
                                  "final_fit": rt.trace.iters[-1].fit.fit,
                                  "max_fit_diff_vs_per_mode": float(max(abs(a.fit.fit - b.fit.fit) for a, b in
                                                                        zip(res.trace.iters, rt.trace.iters))),
                                  "roofline_iter_ms": round(2 * 8.0 * nf / (hbm_peak * 1e9) * 1e3, 3),
                                  "note": "same ALS updates, two tensor passes per iteration (SURVEY 8f-2)"},
               "symmetric_packed": {"iter_ms_median": round(it_s[len(it_s) // 2], 3), "wall_s": round(wall_s, 4),
                                    "final_fit": rs.trace.iters[-1].fit.fit,
                                    "max_fit_diff_vs_per_mode": float(max(abs(a.fit.fit - b.fit.fit) for a, b in
                                                                          zip(res.trace.iters, rs.trace.iters))),
                                    "roofline_iter_ms": round(2 * 8.0 * nf * (fd[0] + 1) / (2 * fd[0]) /
                                                              (hbm_peak * 1e9) * 1e3, 3),
                                    "note": "modes 0/1 symmetric slices packed to upper triangles (SURVEY 8f-4): "
                                            "the dimension tree over the pair index, ~half the bytes per pass"},
               "data": "synthetic symmetric slices, unit diagonal, tanh(N(0, 0.3^2)) off-diagonal (torch, seeded)"}
        del xf, tf

    # CP-ALS over last-mode shards: weak scaling, every rank holds a
    # 100x100x1200x80 slab of a 100x100x1200x(80 N) tensor; the loop is on the
    # device, NCCL all-reduces inside the per-mode CUDA graphs
    if (world > 1 or args.als_sharded) and not args.no_als and als is None:
        try:
            del x, t
        except NameError:
            pass
        torch.cuda.empty_cache()
        sys.path.insert(0, os.path.join(ROOT, "tools"))
        from perf_als import fmri_tensor
        from paper_1708_08976_b200.distributed import DeviceComm, dist_cp_als_device
        fd = (100, 100, 1200, 80)
        xf = fmri_tensor(fd, seed=1 + rank_id)
        tf = dg.DenseTensor.from_device(fd, xf.data_ptr(), device=local, owner=xf)
        if world == 1:  # --als-sharded on one GPU: a world-1 group for the id broadcast
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29517")
            dist.init_process_group("gloo", rank=0, world_size=1)
        comm = DeviceComm(local)
        glast, lo = fd[-1] * world, fd[-1] * rank_id
        dist_cp_als_device(tf, comm, glast, lo, dg.AlsConfig(rank=20, max_iters=2, tol=0.0, seed=1))
        torch.cuda.synchronize()
        dist.barrier()
        t0 = time.perf_counter()
        rsh = dist_cp_als_device(tf, comm, glast, lo, dg.AlsConfig(rank=20, max_iters=25, tol=0.0, seed=1))
        wall = time.perf_counter() - t0
        its = sorted(1e3 * v for v in rsh.iter_seconds)
        # the same over the dimension tree (two tensor passes per iteration)
        cfg_t = lambda n: dg.AlsConfig(rank=20, max_iters=n, tol=0.0, seed=1, dimension_tree=True)  # noqa: E731
        dist_cp_als_device(tf, comm, glast, lo, cfg_t(2))
        torch.cuda.synchronize()
        dist.barrier()
        t1 = time.perf_counter()
        rtr = dist_cp_als_device(tf, comm, glast, lo, cfg_t(25))
        wall_t = time.perf_counter() - t1
        itt = sorted(1e3 * v for v in rtr.iter_seconds)
        # and on each rank's slab packed to the upper triangles of its symmetric slices
        tpk = tf.pack_symmetric01()
        cfg_s = lambda n: dg.AlsConfig(rank=20, max_iters=n, tol=0.0, seed=1)  # noqa: E731
        dist_cp_als_device(tpk, comm, glast, lo, cfg_s(2))
        torch.cuda.synchronize()
        dist.barrier()
        t2 = time.perf_counter()
        rsy = dist_cp_als_device(tpk, comm, glast, lo, cfg_s(25))
        wall_s = time.perf_counter() - t2
        tpk.release()
        iss = sorted(1e3 * v for v in rsy.iter_seconds)
        mx = torch.tensor([its[len(its) // 2], wall, itt[len(itt) // 2], wall_t, iss[len(iss) // 2], wall_s],
                          dtype=torch.float64)
        if world > 1:
            mx = mx.to(dev)
            dist.all_reduce(mx, op=dist.ReduceOp.MAX)  # the slowest rank sets the job's time
        nf = int(np.prod(fd)) * world
        als = {"workload": f"fMRI-shaped 100x100x1200x{fd[-1] * world}, rank 20, 25 iterations, tol 0, "
                           f"sharded over the subject mode on {world} GPU(s) (BASELINE config 5)",
               "iter_ms_median": round(float(mx[0]), 3), "wall_s": round(float(mx[1]), 4),
               "final_fit": rsh.fits[-1], "scaling": "weak", "ranks": world,
               "roofline_iter_ms": round(4 * 8.0 * nf / world / (hbm_peak * 1e9) * 1e3, 3),
               "dimension_tree": {"iter_ms_median": round(float(mx[2]), 3), "wall_s": round(float(mx[3]), 4),
                                  "final_fit": rtr.fits[-1],
                                  "max_fit_diff_vs_per_mode": float(max(abs(a - b) for a, b in
                                                                        zip(rsh.fits, rtr.fits))),
                                  "roofline_iter_ms": round(2 * 8.0 * nf / world / (hbm_peak * 1e9) * 1e3, 3)},
               "symmetric_packed": {"iter_ms_median": round(float(mx[4]), 3), "wall_s": round(float(mx[5]), 4),
                                    "final_fit": rsy.fits[-1],
                                    "max_fit_diff_vs_per_mode": float(max(abs(a - b) for a, b in
                                                                          zip(rsh.fits, rsy.fits))),
                                    "roofline_iter_ms": round(2 * 8.0 * nf / world * (fd[0] + 1) / (2 * fd[0]) /
                                                              (hbm_peak * 1e9) * 1e3, 3)},
               "path": "dmtk_gpu_cp_als_sharded: per-mode sweep on the device, NCCL all-reduces of the "
                       "I_n x C partials, the last factor's column norms and Gram and the fit inside the "
                       "per-mode CUDA graphs",
               "data": "synthetic symmetric slices per rank (torch, seeded by rank)"}
        comm.close()
        del xf, tf

    # ----------------- BASELINE config 0: the 3-matrix Khatri-Rao product
    krp = None
    if world == 1 and not args.no_als:
        g = torch.Generator(device=dev).manual_seed(5)
        kin = [torch.rand((200, 16), dtype=torch.float64, device=dev, generator=g) for _ in range(3)]
        kout = torch.empty((200 ** 3, 16), dtype=torch.float64, device=dev)
        kscr = torch.empty((2 * 200 * 200, 16), dtype=torch.float64, device=dev)
        kcall = lambda: dg.krp_device([a.data_ptr() for a in kin], [200, 200, 200], 16, kout.data_ptr(),
                                      kscr.data_ptr(), torch.cuda.current_stream().cuda_stream)
        kcall()
        torch.cuda.synchronize()
        k0, k1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        k0.record()
        for _ in range(10):
            kcall()
        k1.record()
        torch.cuda.synchronize()
        kms = k0.elapsed_time(k1) / 10
        kgb = 8.0 * 200 ** 3 * 16 / 1e9
        krp = {"workload": "KRP of three 200x16 factors -> 8e6 x 16 (1.024 GB written; BASELINE config 0)",
               "ms": round(kms, 4), "GBs_written": round(kgb / (kms * 1e-3), 1),
               "frac_roofline": round(kgb / hbm_peak / (kms * 1e-3), 3),
               "note": "bitwise equal to the reference KRP; bytes = output written (SURVEY 8d)"}
        del kin, kout, kscr

    if rank_id == 0:
        line = {
            "metric": METRIC, "value": round(value, 3), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms_step, 4), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic U[0,1) (torch Philox, seeded), device-resident",
            "config": {"workload": args.config, "dims": list(dims), "rank": C, "algo": "automatic",
                       "modes_per_step": N, "l2": "inputs larger than L2 (8 GB per pass vs 126 MB L2)",
                       "parallelism": f"last-mode shards x{world}" if world > 1 else "1 GPU"},
            "modes": modes,
            "roofline": {"bound": bound, "achieved": round(achieved, 3), "peak": round(peak, 3), "unit": unit,
                         "frac": round(achieved / peak, 4), "traffic": load_traffic(args.config, C),
                         "kernel": "mttkrp_tc_kernel (per-mode launch, incl. its slot reduction)",
                         "peak_source": ("FP64 DMMA probe run back to back for 1.5 s live in bench.py (sustained, "
                                         "power-capped; MEASURED_PEAKS.json has no FP64 entry)"
                                         if bound == "tensor" else hbm_src),
                         "fp64_peak_tflops_burst": round(peak_tf_burst, 3),
                         "hbm_frac": round(8.0 * n / avg_launch_s / 1e9 / hbm_peak, 4), "hbm_peak_gbs": hbm_peak,
                         "fp64_peak_tflops": round(peak_tf, 3)},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": int(launches),
            "cp_als": als,
            "krp": krp,
            "clocks": clocks,
        }
        emit(line)
    if world > 1:
        dist.destroy_process_group()


def _json_stdout():
    """The JSON line is the only thing bench.py writes to stdout: anything
    else printed to file descriptor 1 while it runs (NCCL's version banner
    and INFO lines, library diagnostics) is sent to stderr instead, and the
    line goes to a duplicate of the original stdout."""
    global _OUT
    sys.stdout.flush()
    _OUT = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)


_OUT = None


def emit(line):
    out = _OUT if _OUT is not None else sys.stdout
    out.write(json.dumps(line) + "\n")
    out.flush()


if __name__ == "__main__":
    _json_stdout()
    main()
