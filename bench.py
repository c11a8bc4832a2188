#!/usr/bin/env python
"""bench.py -- F-Hash encode fwd+bwd throughput on B200 (BASELINE.json metric).

    python bench.py [--gpus N --steps K --warmup W] [--impl ours|reference]

Workload (N=1 and per rank): BASELINE.json configs[1] ("cfg2"): L = 16
levels, spatial 16..512 / temporal 2..64 geometric, F = 2 fp32, tables
capped at 2^19 entries (levels 0-4 MPHF, 5-15 hashed), 2^20 uniform points
per GPU, upstream grads N(0,1).  One step = zero dtable + encode fwd + encode
bwd, all through the C ABI (libfhash.so).  Inputs are resident in HBM when
the timed region starts; L2 is flushed (256 MiB write) between timed steps,
outside the per-step events.

Multi-GPU: the path shards by samples with no data-path collective (each
rank runs its own 2^20 points, seed = rank): "scaling": "weak", value = all
ranks' samples / max-over-ranks device time.  `--gpus N` without a torchrun
environment re-launches this script under torch.distributed.run with N
ranks (one per GPU, 127.0.0.1 rendezvous, NCCL init lines logged); under
torchrun, --gpus must equal WORLD_SIZE.  The line carries every rank's
device, PCI bus id and device time, and the communicator's size.
`--launch-check` runs only the launcher, rendezvous and max-over-ranks
reduction (gloo, no GPU work) -- the CPU test of the N > 1 plumbing.

The reference arm (--impl reference) times the CPU oracle (oracle/, plain
C, fp64, 1 thread) on a bounded sample of the same workload -- the only
other place this script executes oracle/.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "F-Hash encode fwd+bwd samples/s (whole job) and % of measured L2/HBM gather roofline"
UNIT = "samples/s"


def env_int(k, d):
    try:
        return int(os.environ.get(k, d))
    except ValueError:
        return d


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def load_ncu_summary():
    """The committed ncu summary of the headline kernels (profiles/)."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if not os.path.exists(p):
        return {}
    with open(p) as f:
        return json.load(f)


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *a):
        self.rows = []
        if self.proc is None:
            return
        time.sleep(0.25)
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=10)
        for line in out.strip().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == 6:
                self.rows.append(parts)

    def summary(self):
        if not getattr(self, "rows", None):
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        sm = sorted(float(r[0]) for r in self.rows)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[2 + i].lower() == "active"})
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": float(self.rows[0][1]), "reasons": reasons,
                "samples": len(sm)}


# ------------------------------------------------------------------ reference
def run_reference(args, rank, world):
    """The CPU oracle, as it stands, on a bounded sample of the same workload."""
    if rank != 0:
        return
    import numpy as np
    import oracle
    import workloads as W
    cfg = W.CFG2
    n_sample = 1 << 15
    case = W.encode_case(cfg, n_sample, seed=0)
    lv = oracle.Levels(cfg.levels, cfg.cap)
    table64 = case.table.astype(np.float64)

    def step():
        lv.forward(case.coords, table64)
        lv.backward(case.coords, case.dout, cfg.F)

    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    dt = time.perf_counter() - t0
    value = n_sample * args.steps / dt
    sample = f"{n_sample} of the 2^20 cfg2 points per step (full 6.3M-entry tables), fwd+bwd, fp64 C oracle"
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3 / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_block(cfg, W.N_CFG2, world),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def config_block(cfg, N, world):
    return {"workload": "cfg2: BASELINE.json configs[1] encode-only fwd+bwd", "points_per_gpu": N,
            "global_points": N * world, "levels": cfg.L, "F": cfg.F, "table_dtype": cfg.table_dtype,
            "cap": cfg.cap, "parallelism": f"replicas x{world} (sample-sharded, no collective)",
            "l2": "flushed between timed steps (256 MiB write, outside the step events)"}


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


_PAR = {}


def _par_worker(args):
    """One process of the all-cores oracle run: forward of its sample range
    (output discarded) and backward into its own private shared-memory
    gradient table."""
    from multiprocessing import shared_memory
    import numpy as np
    import oracle
    k, a, b, shm_name, total, F = args
    d = _PAR
    lv = oracle.Levels(d["levels"], d["cap"])
    lv.forward(d["coords"][a:b], d["t64"])
    G = lv.backward(d["coords"][a:b], d["dout"][a:b], F)
    shm = shared_memory.SharedMemory(name=shm_name)
    dst = np.ndarray((total, F), dtype=np.float64, buffer=shm.buf)
    dst[:] = G
    del dst
    shm.close()
    return k


def cpu_baseline_all_cores(cfg, case_coords, case_table, case_dout, max_procs=16):
    """the same oracle on all host cores -- the
    forward split over samples, the backward into per-process private
    gradient tables summed in a fixed (process) order.  Process-level
    parallelism around the unmodified oracle (fork + shared memory); capped
    at max_procs processes (each private table is 100 MB at cfg2)."""
    import multiprocessing as mp
    from multiprocessing import shared_memory
    import numpy as np
    P = max(1, min(len(os.sched_getaffinity(0)), max_procs))
    n = len(case_coords)
    total = int(sum(W_table_sizes(cfg)))
    _PAR.update(levels=cfg.levels, cap=cfg.cap, coords=case_coords, t64=case_table.astype(np.float64),
                dout=case_dout)
    shms = [shared_memory.SharedMemory(create=True, size=total * cfg.F * 8) for _ in range(P)]
    try:
        bounds = [(i * n // P, (i + 1) * n // P) for i in range(P)]
        ctx = mp.get_context("fork")
        with ctx.Pool(P) as pool:
            pool.map(_par_worker, [(0, 0, 1, shms[0].name, total, cfg.F)] * P)   # warm the workers
            t0 = time.perf_counter()
            pool.map(_par_worker, [(i, a, b, shms[i].name, total, cfg.F) for i, (a, b) in enumerate(bounds)])
            G = np.zeros((total, cfg.F))
            for sh in shms:   # fixed merge order
                G += np.ndarray((total, cfg.F), dtype=np.float64, buffer=sh.buf)
            dt = time.perf_counter() - t0
    finally:
        for sh in shms:
            sh.close()
            sh.unlink()
    return {"value": n / dt, "unit": UNIT, "cores": P, "kind": "oracle", "cpu_model": cpu_model(),
            "sample": f"all {n} cfg2 points, fwd+bwd, fp64 C oracle in {P} processes (samples split; private "
                      f"grad tables summed in process order), {dt:.2f} s"}


def W_table_sizes(cfg):
    import workloads as W
    return W.table_sizes(cfg.levels, cfg.cap)


def _par_encode_worker(args):
    """One process of an all-cores oracle encode: forward of its sample range
    (output kept in shared memory when asked) and backward of its range
    into a private shared-memory gradient table."""
    from multiprocessing import shared_memory
    import numpy as np
    import oracle
    k, a, b, shm_name, total, F, want_out, out_name, LF = args
    d = _PAR
    lv = oracle.Levels(d["levels"], d["cap"])
    out = lv.forward(d["coords"][a:b], d["t64"])
    if want_out:
        sh = shared_memory.SharedMemory(name=out_name)
        np.ndarray((len(d["coords"]), LF), dtype=np.float64, buffer=sh.buf)[a:b] = out
        sh.close()
    if d.get("dout") is not None:
        G = lv.backward(d["coords"][a:b], d["dout"][a:b], F)
        shm = shared_memory.SharedMemory(name=shm_name)
        np.ndarray((total, F), dtype=np.float64, buffer=shm.buf)[:] = G
        shm.close()
    return k


def _par_sum_worker(args):
    """Sum rows [a, b) of the P private gradient tables, in process order,
    into the result table (the all-cores merge, split over entries)."""
    from multiprocessing import shared_memory
    import numpy as np
    a, b, names, out_name, total, F = args
    sh = shared_memory.SharedMemory(name=out_name)
    dst = np.ndarray((total, F), dtype=np.float64, buffer=sh.buf)
    for nm in names:
        s = shared_memory.SharedMemory(name=nm)
        dst[a:b] += np.ndarray((total, F), dtype=np.float64, buffer=s.buf)[a:b]
        s.close()
    del dst
    sh.close()
    return a


def _oracle_encode_par(levels, cap, coords, t64, dout, F, P, want_out=False):
    """Oracle fwd (+ bwd when dout is given) with the samples split over P
    forked processes; private gradient tables summed in process order (the
    sum itself split over entry ranges across the same processes)."""
    import multiprocessing as mp
    from multiprocessing import shared_memory
    import numpy as np
    total, n, LF = t64.shape[0], len(coords), len(levels) * F
    _PAR.clear()
    _PAR.update(levels=levels, cap=cap, coords=coords, t64=t64, dout=dout)
    shms = [shared_memory.SharedMemory(create=True, size=total * F * 8) for _ in range(P)] if dout is not None else []
    osh = shared_memory.SharedMemory(create=True, size=max(8, n * LF * 8)) if want_out else None
    try:
        bounds = [(i * n // P, (i + 1) * n // P) for i in range(P)]
        G = None
        with mp.get_context("fork").Pool(P) as pool:
            pool.map(_par_encode_worker, [(i, a, b, shms[i].name if shms else "", total, F, want_out,
                                           osh.name if osh else "", LF) for i, (a, b) in enumerate(bounds)])
            if shms:
                gsh = shared_memory.SharedMemory(create=True, size=total * F * 8)
                shms.append(gsh)
                eb = [(i * total // P, (i + 1) * total // P) for i in range(P)]
                pool.map(_par_sum_worker, [(a, b, [x.name for x in shms[:-1]], gsh.name, total, F) for a, b in eb])
                G = np.ndarray((total, F), dtype=np.float64, buffer=gsh.buf).copy()
        out = np.ndarray((n, LF), dtype=np.float64, buffer=osh.buf).copy() if want_out else None
        return out, G
    finally:
        for sh in shms + ([osh] if osh else []):
            sh.close()
            sh.unlink()


def _oracle_train_step(levels, cap, F, coords, target, t16, layers, adam_state, n_global, P):
    """Oracle-T, one train step as the tests compose it (oracle/train.py;
    SURVEY §8(c)): encode fwd over the fp16 table values (Oracle-F), bf16
    rounding of the encoding (R13), MLP fwd, MSE, analytic bwd, Oracle-B of
    dL/d(enc), dense Adam over every table and MLP parameter (R12)."""
    import numpy as np
    import oracle
    from oracle import train as T
    t64 = t16.astype(np.float64)
    if P > 1:
        x0, _ = _oracle_encode_par(levels, cap, coords, t64, None, F, P, want_out=True)
    else:
        x0 = oracle.Levels(levels, cap).forward(coords, t64)
    y, cache = T.mlp_forward(T.bf16_round(x0), layers)
    loss, dy = T.mse_loss(y, target.astype(np.float64), n_global)
    grads, dx0 = T.mlp_backward(dy, layers, cache)
    if P > 1:
        _, G = _oracle_encode_par(levels, cap, coords, t64, dx0, F, P)
    else:
        G = oracle.Levels(levels, cap).backward(coords, dx0, F)
    p, m, v = adam_state["table"]
    adam_state["table"] = T.adam_step(p, G, m, v, 1)
    for k, ((dW, db), (W_, b_)) in enumerate(zip(grads, layers)):
        T.adam_step(W_, dW, np.zeros_like(dW), np.zeros_like(dW), 1)
        T.adam_step(b_, db, np.zeros_like(db), np.zeros_like(db), 1)
    return loss


def cpu_oracle_baselines(W, max_procs=8):
    """SURVEY §8(d) "Oracle timing beside the GPU": the oracle, as it stands,
    on 2^18-point subsets of the HBM-regime encoder (cfg4 = cfg5's encoder:
    L=16, F=4, 160 M parameters) -- encode fwd+bwd, and the whole Oracle-T
    train step with dense Adam over every parameter -- plus Oracle-T on
    cfg3's full 2^18 batch; each on 1 core (BLAS limited to one thread) and
    on up to max_procs cores (encode split over forked processes, private
    gradient tables summed in process order; each table is 1.3 GB at cfg4)."""
    import numpy as np
    from threadpoolctl import threadpool_limits
    import oracle
    out = {"cpu_model": cpu_model(), "host_cores": len(os.sched_getaffinity(0))}
    P = max(1, min(len(os.sched_getaffinity(0)), max_procs))
    n = 1 << 18
    g = W.rng(123)
    for name, cfg, mlp in (("cfg4_cfg5", W.CFG4, W.MLP4), ("cfg3", W.CFG3, W.MLP3)):
        total = int(sum(W.table_sizes(cfg.levels, cfg.cap)))
        t16 = W.draw_table(g, total, cfg.F, "f16")
        coords = W.draw_coords(g, n)
        dout = g.standard_normal((n, cfg.L * cfg.F), dtype=np.float32)
        target = g.random(n, dtype=np.float32)
        layers = W.draw_mlp(g, mlp)
        res = {}
        if name == "cfg4_cfg5":
            t64 = t16.astype(np.float64)
            with threadpool_limits(1):
                t0 = time.perf_counter()
                lv = oracle.Levels(cfg.levels, cfg.cap)
                lv.forward(coords, t64)
                lv.backward(coords, dout, cfg.F)
                d1 = time.perf_counter() - t0
            t0 = time.perf_counter()
            _oracle_encode_par(cfg.levels, cfg.cap, coords, t64, dout, cfg.F, P)
            dP = time.perf_counter() - t0
            res["encode_fwd_bwd"] = {"unit": UNIT, "sample": f"{n} of cfg4's 2^22 points, fwd+bwd over the full "
                                                            f"40 M-entry F=4 table, fp64 C oracle",
                                     "one_core": {"value": n / d1, "cores": 1, "seconds": d1},
                                     "all_cores": {"value": n / dP, "cores": P, "seconds": dP}}
            del t64
        for label, procs in (("one_core", 1), ("all_cores", P)):
            state = {"table": (t16.astype(np.float64).reshape(-1, cfg.F), np.zeros((total, cfg.F)),
                               np.zeros((total, cfg.F)))}
            with threadpool_limits(1 if procs == 1 else None):
                t0 = time.perf_counter()
                _oracle_train_step(cfg.levels, cfg.cap, cfg.F, coords, target, t16, layers, state, n, procs)
                dt = time.perf_counter() - t0
            res.setdefault("train_step", {"unit": UNIT, "sample": f"{n} samples of the {name} train step "
                                          f"(Oracle-T: encode fwd, bf16 rounding, MLP {mlp.widths}, MSE, bwd, "
                                          f"encode bwd, dense Adam over {total * cfg.F + sum(W_.size + b_.size for W_, b_ in layers)} "
                                          f"parameters), fp64"})[label] = {"value": n / dt, "cores": procs,
                                                                           "seconds": dt}
            del state
        out[name] = res
    return out


# ------------------------------------------------------------------ ours
def cpu_baseline(cfg, case_coords, case_table, case_dout):
    import numpy as np
    import oracle
    n = len(case_coords)      # the full 2^20-point batch (~8 s of one core)
    lv = oracle.Levels(cfg.levels, cfg.cap)
    t64 = case_table.astype(np.float64)
    t0 = time.perf_counter()
    lv.forward(case_coords[:n], t64)
    lv.backward(case_coords[:n], case_dout[:n], cfg.F)
    dt = time.perf_counter() - t0
    return {"value": n / dt, "unit": UNIT, "cores": 1, "kind": "oracle", "cpu_model": cpu_model(),
            "sample": f"all {n} cfg2 points, fwd+bwd over the full tables, fp64 C, 1 thread, "
                      f"{dt:.1f} s"}


def microbench_roofline(fh, torch, enc, cfg, N, stream, hbm_peak):
    """§8(d): microbenchmarks of the encode's access shape (context: the
    kernel is not bounded by them).  Per level
    l, random x-pair gathers / vector reds over a T_l-entry buffer (same
    entry width, 8 pairs per thread) give a corner rate; streaming bytes go
    at the measured copy bandwidth.  t_roof = N * sum_l 16/rate_l + stream/BW."""
    F = cfg.F
    eb = F * 4
    n_thr = 1 << 20
    sink = torch.empty(n_thr, device="cuda")
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def timeit(fn, reps=3):
        best = 1e9
        for _ in range(reps):
            ev0.record(stream)
            fn()
            ev1.record(stream)
            ev1.synchronize()
            best = min(best, ev0.elapsed_time(ev1) / 1e3)
        return best

    # HBM copy ceiling with our own kernel (1 GiB -> 1 GiB)
    nb = 1 << 30
    a = torch.empty(nb, dtype=torch.uint8, device="cuda")
    b = torch.empty(nb, dtype=torch.uint8, device="cuda")
    t_copy = timeit(lambda: fh.bench_copy(b, a, nb, stream))
    bw_copy = 2 * nb / t_copy
    del a, b
    g_rate, r_rate, g_split, r_split = [], [], [], []
    for l in range(cfg.L):
        T = enc.level_info(l)["table_size"]
        buf = torch.zeros((T, F), device="cuda")
        fh.bench_gather(buf, T, eb, n_thr, sink, mode=1, seed=l, stream=stream)
        # mode 1: one aligned access per x-pair = the minimum-sector shape
        tg = timeit(lambda: fh.bench_gather(buf, T, eb, n_thr, sink, mode=1, seed=l, stream=stream))
        tr = timeit(lambda: fh.bench_red(buf, T, eb, n_thr, mode=1, seed=l, stream=stream))
        g_rate.append(16 * n_thr / tg)   # corners (2 per pair access) per second
        r_rate.append(16 * n_thr / tr)
        # mode 0 (two entry-wide accesses per pair), reported for context
        g_split.append(16 * n_thr / timeit(lambda: fh.bench_gather(buf, T, eb, n_thr, sink, mode=0, seed=l,
                                                                   stream=stream)))
        r_split.append(16 * n_thr / timeit(lambda: fh.bench_red(buf, T, eb, n_thr, mode=0, seed=l, stream=stream)))
        del buf
    # the L2's random-reduction op rate: one 16-byte red.v4 per x-pair at
    # uniform positions in an L2-resident 48 MiB buffer (8-byte entries,
    # mode 1) -- the unit the encode backward is bound by
    # (67 M reductions per launch, best of 5: a launch as long as the
    # backward pass itself, so ramp-up and tail do not understate the rate)
    n_red = 1 << 23
    rb = torch.zeros((48 << 20) // 4, device="cuda")
    fh.bench_red(rb, (48 << 20) // 8, 8, n_red, mode=1, seed=99, stream=stream)
    t_red = timeit(lambda: fh.bench_red(rb, (48 << 20) // 8, 8, n_red, mode=1, seed=99, stream=stream), reps=5)
    red_ops_per_s = 8 * n_red / t_red
    del rb
    stream_fwd = N * (16 + cfg.L * F * 4)
    stream_bwd = N * (16 + cfg.L * F * 4)
    t_fwd_lv = sum(N * 16 / g for g in g_rate) + stream_fwd / bw_copy
    t_bwd_lv = sum(N * 16 / r for r in r_rate) + stream_bwd / bw_copy
    # the encode's own shape: all levels in one launch, (sample, level)
    # threads level-fastest, 8 ideal x-pairs per thread inside each level's
    # range of the packed table (fh_bench_*_levels) -- the per-level runs
    # above overstate the coarse levels' contention, which the kernel's
    # level mix dilutes
    full = torch.zeros((enc.entries, F), device="cuda")
    msink = torch.empty(N * cfg.L, device="cuda")
    fh.bench_gather_levels(full, enc, eb, N, msink, stream=stream)
    tg_mix = timeit(lambda: fh.bench_gather_levels(full, enc, eb, N, msink, stream=stream))
    fh.bench_red_levels(full, enc, eb, N, stream=stream)
    tr_mix = timeit(lambda: fh.bench_red_levels(full, enc, eb, N, stream=stream))
    del full, msink
    t_fwd = tg_mix + stream_fwd / bw_copy
    t_bwd = tr_mix + stream_bwd / bw_copy
    return {
        "t_roof_fwd_ms": t_fwd * 1e3, "t_roof_bwd_ms": t_bwd * 1e3,
        "model": "level-mix microbenchmark (fh_bench_gather_levels / fh_bench_red_levels) + streamed bytes at the "
                 "measured copy bandwidth",
        "t_per_level_sum_fwd_ms": t_fwd_lv * 1e3, "t_per_level_sum_bwd_ms": t_bwd_lv * 1e3,
        # SURVEY §8(d) "expected counts": each x-pair as two entry-wide accesses (the
        # naive shape, per-level rates) -- the pair layout of DESIGN.md §8.1 beats it
        "t_split_pairs_fwd_ms": (sum(N * 16 / g for g in g_split) + stream_fwd / bw_copy) * 1e3,
        "t_split_pairs_bwd_ms": (sum(N * 16 / r for r in r_split) + stream_bwd / bw_copy) * 1e3,
        "mix_gather_corner_rate_G_per_s": round(N * cfg.L * 16 / tg_mix / 1e9, 2),
        "mix_red_corner_rate_G_per_s": round(N * cfg.L * 16 / tr_mix / 1e9, 2),
        "copy_gbs": bw_copy / 1e9, "hbm_peak_gbs": hbm_peak,
        "l2_red_op_ceiling_G_per_s": red_ops_per_s / 1e9,
        "gather_corner_rate_G_per_s": [round(g / 1e9, 2) for g in g_rate],
        "red_corner_rate_G_per_s": [round(r / 1e9, 2) for r in r_rate],
        "split_gather_corner_rate_G_per_s": [round(g / 1e9, 2) for g in g_split],
        "split_red_corner_rate_G_per_s": [round(r / 1e9, 2) for r in r_split],
    }


def hbm_regime_bench(fh, torch, W, steps, hbm_peak):
    """The metric's HBM regime: BASELINE.json configs[3] encoder (L=16, F=4
    fp16 tables capped at 2^22: 305 MiB of tables, 609 MiB of fp32 grads),
    2^22 uniform points, encode fwd (bf16 out, as in the train step) + bwd,
    L2 flushed.  Roofline: the kernels run L2-sized level-group passes, so per
    level the measured random-gather / red rate at that level's table size
    and entry width (8 B fp16x4 rows; 16 B fp32x4 grads, no pair merge) bounds
    the corner traffic, and the compulsory HBM bytes -- tables read once,
    grads read + written once, coordinates, encodings and upstream grads
    streamed -- go at the measured copy bandwidth."""
    cfg, N = W.CFG4, W.N_CFG4
    enc = fh.Encoder(cfg.levels, cfg.F, cfg.table_dtype, cfg.cap)
    g = torch.Generator("cuda").manual_seed(4)
    coords = torch.rand((N, 4), device="cuda", generator=g)
    table = ((torch.rand((enc.entries, cfg.F), device="cuda", generator=g) - 0.5) * 2e-4).half()
    out = torch.empty((N, cfg.L * cfg.F), device="cuda", dtype=torch.bfloat16)
    dout = torch.randn((N, cfg.L * cfg.F), device="cuda", generator=g)
    dt = torch.zeros((enc.entries, cfg.F), device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    tf = tb = 0.0
    for it in range(steps + 2):
        flush.fill_(it & 255)
        e[0].record()
        enc.fwd(coords, table, out, out_dtype="bf16")
        e[1].record()
        enc.bwd(coords, dout, dt, overwrite=True)
        e[2].record()
        torch.cuda.synchronize()
        if it >= 2:
            tf += e[0].elapsed_time(e[1])
            tb += e[1].elapsed_time(e[2])
    fwd_ms, bwd_ms = tf / steps, tb / steps
    # the same backward from a level-major dout ([L][N][F], FH_BWD_DOUT_LEVEL_MAJOR:
    # the train step's dL/d(enc) layout for F >= 4)
    dout_lm = dout.view(N, cfg.L, cfg.F).permute(1, 0, 2).contiguous()
    del dout
    tl = 0.0
    for it in range(steps + 2):
        flush.fill_(it & 255)
        e[1].record()
        enc.bwd(coords, dout_lm, dt, overwrite=True, level_major=True)
        e[2].record()
        torch.cuda.synchronize()
        if it >= 2:
            tl += e[1].elapsed_time(e[2])
    bwd_lm_ms = tl / steps
    del out, dout_lm, flush
    LF = cfg.L * cfg.F
    # compulsory HBM bytes of one pass: the table (fwd) or the fp32 grads
    # (bwd: read + written) once, plus the streamed coordinates and encodings /
    # upstream grads -- a lower bound on the DRAM traffic, so frac <= 1
    hbm_fwd = enc.entries * cfg.F * 2 + N * (16 + LF * 2)           # fp16 tables + coords + bf16 out
    hbm_bwd = enc.entries * cfg.F * 4 * 2 + N * (16 + LF * 4)       # grads RMW + coords + fp32 dout
    bw = hbm_peak * 1e9
    ncu = load_ncu_summary().get("cfg4", {})
    out = {"workload": "cfg4 encoder (BASELINE.json configs[3]): 2^22 points, L=16, F=4 fp16 tables cap 2^22 "
                       "(305 MiB) + fp32 grads (609 MiB); fwd (bf16 out) + bwd, L2 flushed",
           "fwd_ms": fwd_ms, "bwd_ms": bwd_ms, "samples_per_s": N / ((fwd_ms + bwd_ms) / 1e3),
           "bwd_ms_level_major_dout": bwd_lm_ms,
           "compulsory_hbm_bytes": {"fwd": hbm_fwd, "bwd": hbm_bwd},
           "hbm_frac_fwd": hbm_fwd / bw / (fwd_ms / 1e3), "hbm_frac_bwd": hbm_bwd / bw / (bwd_ms / 1e3),
           "note": "compulsory bytes / time / measured HBM peak: the lower bound of the DRAM traffic, so <= 1; the "
                   "passes are bound by L2 request / atomic throughput (see ncu)"}
    if ncu:
        out["ncu"] = ncu
    ncu_lm = load_ncu_summary().get("cfg4_lm", {})
    if ncu_lm:
        out["ncu_level_major_dout"] = ncu_lm
    return out


def train_step_bench(fh, torch, W, which, rank, world, dist, steps, warmup, dp_mode="nccl"):
    """All §8(a) rows in one step: Philox voxel sampling from the synthetic
    field, encode fwd (fp16 table -> bf16), tcgen05 MLP fwd + MSE + bwd,
    encode bwd, [NCCL all-reduce of the flat fp32 grads over NVLink when
    world > 1], fused Adam.
      cfg3: BASELINE.json configs[2], 256^3 x 32 Gaussian blobs, batch 2^18 (N=1)
      cfg5: BASELINE.json configs[4], configs[3] field + encoder, global
            batch 2^24 split over the ranks (strong scaling)."""
    from paper_2507_03836_b200 import dp
    if which == "cfg3":
        blobs = W.gaussian_blob_params(W.rng(0))
        field = fh.field_gaussian_blobs(256, 32, blobs)
        cfg, mlp, n_global = W.CFG3, W.MLP3, W.N_CFG3 * world
    else:
        field = fh.field_value_noise(640, 256, 256, 100, seed=0, band=0.02)
        cfg, mlp, n_global = W.CFG4, W.MLP4, 1 << 24
    n_local = n_global // world
    enc = fh.Encoder(cfg.levels, cfg.F, cfg.table_dtype, cfg.cap)
    gen = torch.Generator("cuda").manual_seed(0)           # identical init on every rank
    table0 = (torch.rand((enc.entries, cfg.F), device="cuda", generator=gen) * 2 - 1) * 1e-4
    peer = world > 1 and dp_mode in ("peer", "multicast")
    fused = world > 1 and dp_mode == "fused"
    tr = fh.Trainer(enc, table0, W.draw_mlp(W.rng(0), mlp), n_local, world=world,
                    alloc=dp.symm_alloc if peer else None)
    del table0
    coords = torch.empty((n_local, 4), device="cuda")
    target = torch.empty((n_local,), device="cuda")
    stream = torch.cuda.current_stream()
    # world > 1: per-backward-launch reduce-scatter of the table grads on a
    # communication stream, overlapped with the rest of the backward
    # (dp.OverlappedShardedDP; NCCL over NVLink/NVSwitch), all-reduce of the
    # tails + MLP grads, Adam on this rank's chunks, all-gather of the fp16
    # table shadow.  Falls back to dp.ShardedDP (no overlap) if the plan
    # needs more than 63 Adam ranges.
    sdp = None
    comm = None
    if fused:   # the library's own NCCL exchange (fh_trainer_set_comm), communicator from torch's libnccl
        uid = [fh.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        comm = fh.NcclComm(uid[0], world, rank)
        tr.set_comm(comm)
    elif peer and dp_mode == "multicast":
        # --dp multicast: the same through an NVLS multicast object (multimem.ld_reduce / multimem.st);
        # falls back to the peer-pointer form when the system gives torch no multicast object
        try:
            sdp = dp.MulticastShardedDP(tr)
        except ValueError:
            sdp = dp.PeerShardedDP(tr)
    elif peer:
        sdp = dp.PeerShardedDP(tr)     # --dp peer: fused reduce + Adam + all-gather over NVLink peer memory
    elif world > 1:
        try:
            sdp = dp.OverlappedShardedDP(tr)
        except ValueError:
            sdp = dp.ShardedDP(tr)

    def one(k, ev=None):
        if ev: ev[0].record(stream)
        fh.sample_voxels(field, n_local, seed=1234, subsequence=rank, offset=k, coords=coords, target=target)
        if ev: ev[1].record(stream)
        if comm is not None:   # fused: fwd_bwd + exchange + Adam + all-gather in one library call
            loss = tr.step(coords, target, n_global)
            if ev:
                for i in (2, 3, 4): ev[i].record(stream)
            return loss
        loss = tr.fwd_bwd(coords, target, n_global)
        if ev: ev[2].record(stream)
        if isinstance(sdp, (dp.OverlappedShardedDP, dp.PeerShardedDP)):
            if ev: ev[3].record(stream)   # the reduction already overlaps the backward
            sdp.reduce_and_apply()
        elif sdp:
            sdp.reduce()
            if ev: ev[3].record(stream)
            sdp.apply()
            sdp.gather()
        else:
            if ev: ev[3].record(stream)
            tr.apply()
        if ev: ev[4].record(stream)
        return loss

    losses = []
    for k in range(max(warmup, 3)):
        losses.append(one(k).item())
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(5)] for _ in range(steps)]
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    l0 = fh.kernel_launches()
    for k in range(steps):
        one(1000 + k, ev[k])
    torch.cuda.synchronize()
    launches = (fh.kernel_launches() - l0) / steps
    total = sum(e[0].elapsed_time(e[4]) for e in ev) / 1e3
    phase = [sum(e[i].elapsed_time(e[i + 1]) for e in ev) / steps for i in range(4)]
    if dist:
        t = torch.tensor([total], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total = float(t.item())
    # NEXT-1: the renderer's model evaluation V = model(S) (fh_infer) on the
    # same batch shape, after training
    yb = torch.empty((n_local,), device="cuda")
    for _ in range(3):
        tr.infer(coords, yb)
    ie0, ie1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ie0.record(stream)
    for _ in range(steps):
        tr.infer(coords, yb)
    ie1.record(stream)
    torch.cuda.synchronize()
    infer_ms = ie0.elapsed_time(ie1) / steps
    # renderer-sized batches (Alg. 1 marches <= 64 samples per ray): latency of
    # one fh_infer call, eager vs replayed from a CUDA graph
    small = {}
    for nb in (1 << 10, 1 << 12, 1 << 16):
        cs, ys = coords[:nb], yb[:nb]
        reps = 100
        ie0.record(stream)
        for _ in range(reps):
            tr.infer(cs, ys)
        ie1.record(stream)
        torch.cuda.synchronize()
        eager_us = ie0.elapsed_time(ie1) / reps * 1e3
        gs = torch.cuda.Stream()
        gs.wait_stream(stream)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.stream(gs):
            tr.infer(cs, ys, stream=gs)
            with torch.cuda.graph(graph, stream=gs):
                tr.infer(cs, ys, stream=gs)
        torch.cuda.synchronize()
        ie0.record(stream)
        for _ in range(reps):
            graph.replay()
        ie1.record(stream)
        torch.cuda.synchronize()
        small[str(nb)] = {"eager_us": eager_us, "graph_us": ie0.elapsed_time(ie1) / reps * 1e3}
        del graph
    # DP correctness: after the timed steps the replicas must be bit-identical
    same = dp.replicas_identical(tr.shadow_flat) and dp.replicas_identical(tr.mlp_master)
    if comm is not None:
        torch.cuda.synchronize()
        tr.set_comm(None)
        comm.destroy()
    last = tr.loss.clone()
    if dist:
        dist.all_reduce(last)
    st = tr.status()
    return {
        "workload": f"{which}: " + ("BASELINE.json configs[2] train_step (256^3x32 Gaussian blobs, L=16 F=2 fp16, "
                                    "MLP 32-64-64-1 bf16, batch 2^18)" if which == "cfg3" else
                                    "BASELINE.json configs[4] DP train_step (configs[3] field 640x256x256x100, "
                                    "L=16 F=4 fp16 cap 2^22, MLP 64-64-64-1, global batch 2^24)"),
        "value": n_global * steps / total, "unit": "samples/s", "ms_per_step": total * 1e3 / steps,
        "global_batch": n_global, "per_gpu_batch": n_local, "n_gpus": world,
        "scaling": "strong" if which == "cfg5" else "weak",
        "phase_ms": {"sample": phase[0], "fwd_bwd": phase[1], "grad_reduce": phase[2],
                     "adam_and_gather": phase[3]},
        "dp": ("fused in the library (fh_trainer_set_comm): per-level-group ncclReduceScatter overlapped with the "
               "backward + sharded Adam + in-place fp16 ncclAllGather" if comm is not None else
               "per-level-group NVLS multimem.ld_reduce + Adam + multimem.st of the fp16 shadow "
               "(fh_train_apply_multicast)" if isinstance(sdp, dp.MulticastShardedDP) else
               "per-level-group fused reduce + Adam + shadow broadcast over NVLink peer memory (fh_train_apply_peers)"
               if isinstance(sdp, dp.PeerShardedDP) else
               "per-backward-launch reduce-scatter overlapped with the backward + sharded Adam + all-gather (NCCL)"
               if isinstance(sdp, dp.OverlappedShardedDP) else
               "reduce-scatter + sharded Adam + all-gather (NCCL)" if world > 1 else "single GPU"),
        "infer": {"what": "fh_infer: encode fwd + tcgen05 MLP forward (Alg. 1 V = model(S))",
                  "ms": infer_ms, "samples_per_s": n_local / (infer_ms / 1e3),
                  "small_batch_latency": small},
        "loss_first_warmup": losses[0], "loss_last": float(last.item()), "status": int(st),
        "params": enc.param_count + tr.n_mlp, "gpu_launches_per_step": launches, "replicas_identical": bool(same),
    }


def paper_encoder_compare(fh, torch, W, steps):
    """NEXT-3: F-Hash vs the MHE baseline on a paper-shaped workload
    (Combustion-Seg FBB 200x110x54, 10 key frames, fold 2, F = 2; MHE with
    T = 2^20, 6 levels, one encoder per key frame -- PAPER.md Table 3 column
    P:619), batch 2^21 of voxel-aligned samples on key frames.
    Encode fwd + bwd, fp32 tables, L2 flushed before each step."""
    S, n, B = (200, 110, 54), 10, 1 << 21
    gen = torch.Generator("cuda").manual_seed(7)
    vox = [torch.randint(0, s, (B,), device="cuda", generator=gen) for s in S]
    k = torch.randint(0, n, (B,), device="cuda", generator=gen)
    coords = torch.stack([vox[0] / (S[0] - 1), vox[1] / (S[1] - 1), vox[2] / (S[2] - 1), k / (n - 1)],
                         1).float().contiguous()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    res = {}
    encs = {
        "fhash": fh.Encoder(fh.fold_schedule(S, n, 2), 2),
        # NEXT-2: the same encoder with the brick (tiled Z-order) linearization, P:174 / R21
        "fhash_brick": fh.Encoder(fh.fold_schedule(S, n, 2), 2, lin=fh.FH_LIN_BRICK),
        "mhe": fh.MHEEncoder(W.geometric(16, 200, 6), 2, 1 << 20, n),
    }
    for name, enc in encs.items():
        table = (torch.rand((enc.entries, 2), device="cuda", generator=gen) - 0.5) * 2e-4
        out = torch.empty((B, enc.L * 2), device="cuda")
        g = torch.randn((B, enc.L * 2), device="cuda", generator=gen)
        dt = torch.zeros_like(table)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        tot = 0.0
        for it in range(steps + 3):
            flush.fill_(it & 255)
            e0.record()
            enc.fwd(coords, table, out)
            enc.bwd(coords, g, dt, overwrite=True)
            e1.record()
            torch.cuda.synchronize()
            if it >= 3:
                tot += e0.elapsed_time(e1)
        ms = tot / steps
        # encoding_stats (fh_level_stats, S:330-338 / Fig. 4): collisions and bucket utilisation
        st = [enc.level_stats(l) for l in range(enc.L)]
        res[name] = {"levels": enc.L, "params": enc.param_count, "params_Mi": round(enc.param_count / 2 ** 20, 2),
                     "fwd_bwd_ms": ms, "samples_per_s": B / (ms / 1e3),
                     "collisions": sum(c for _, c, _ in st),
                     "utilisation_per_level": [round(u, 4) for _, _, u in st]}
        del table, out, g, dt
    res["workload"] = ("Combustion-Seg shape: FBB 200x110x54, 10 key frames, batch 2^21 voxel samples; "
                       "F-Hash fold 2 (Eqs. 4-8; Eq. 9 and brick linearization) vs MHE T=2^20 x 6 levels "
                       "x 10 frames; F=2 fp32")
    return res


def coreset_bench(fh, torch, W, steps, hbm_peak, with_cpu):
    """NEXT-4: GPU coreset selection (fh_coreset_build + fh_coreset_emit,
    PAPER §3.1, Eqs. 1-3) on 8 key frames of the cfg3 field (256^3 moving
    Gaussian blobs), segmentation feature at 0.5.  HBM-streaming: algorithmic
    bytes = 4 B/vertex volume read + 20 B/sample written + the occupancy bits."""
    import numpy as np
    blobs = W.gaussian_blob_params(W.rng(0))
    field = fh.field_gaussian_blobs(256, 32, blobs)
    keys = field[::4].contiguous()
    del field
    n = keys.shape[0]
    V = keys[0].numel()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    cs = fh.Coreset(keys, fh.FH_FEAT_SEGMENTATION, 0.5)
    M = cs.count
    coords = torch.empty((M, 4), device="cuda")
    vals = torch.empty((M,), device="cuda")
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    tot = 0.0
    launches = 0
    for it in range(steps + 2):
        flush.fill_(it & 255)
        l0 = fh.kernel_launches()
        e0.record()
        c2 = fh.Coreset(keys, fh.FH_FEAT_SEGMENTATION, 0.5)
        c2.emit(coords, vals)
        e1.record()
        torch.cuda.synchronize()
        launches = fh.kernel_launches() - l0
        if it >= 2:
            tot += e0.elapsed_time(e1)
    ms = tot / steps
    alg = n * V * 4 + M * 20 + n * cs.words * 4
    out = {"workload": "8 key frames of the cfg3 field (256^3 Gaussian blobs), segmentation >= 0.5; "
                       "build (feature, dilation, occupancy, FBB, counts) + emit (Eqs. 1-3 samples)",
           "vertices": n * V, "coreset_samples": M, "coreset_fraction": M / (n * V),
           "fbb": cs.fbb, "ms": ms, "vertices_per_s": n * V / (ms / 1e3),
           "roofline": {"bound": "hbm", "achieved_gbs": alg / (ms / 1e3) / 1e9, "peak_gbs": hbm_peak,
                        "frac": alg / (ms / 1e3) / 1e9 / hbm_peak, "algorithmic_bytes": alg},
           "gpu_launches": launches}
    if with_cpu:
        from oracle import coreset as C
        small = keys[:2, 96:128, 96:128, 96:128].cpu().numpy()
        t0 = time.perf_counter()
        C.build_coreset(small, C.SEGMENTATION, 0.5)
        dt = time.perf_counter() - t0
        out["cpu_baseline"] = {"value": small.size / dt, "unit": "vertices/s", "cores": 1, "kind": "oracle",
                               "sample": f"2 frames x 32^3 crop of the same volume, {dt:.1f} s"}
    del keys, cs, coords, vals, flush
    return out


def run_ours(args, rank, local_rank, world):
    import numpy as np
    import torch
    import workloads as W
    from paper_2507_03836_b200 import fhash as fh

    torch.cuda.set_device(local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    cfg = W.CFG2
    N = W.N_CFG2
    enc = fh.Encoder(cfg.levels, cfg.F, cfg.table_dtype, cfg.cap)
    case = W.encode_case(cfg, N, seed=rank)
    coords = torch.from_numpy(case.coords).cuda()
    table = torch.from_numpy(case.table).cuda()
    dout = torch.from_numpy(case.dout).cuda()
    out = torch.empty((N, cfg.L * cfg.F), device="cuda")
    dtable = torch.empty((enc.entries, cfg.F), device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    stream = torch.cuda.current_stream()

    def step():
        # dtable = the gradient: fh_encode_bwd_ex(FH_BWD_OVERWRITE) zeroes each
        # level group right before its reductions (include/fhash.h)
        enc.fwd(coords, table, out, stream=stream)
        enc.bwd(coords, dout, dtable, stream=stream, overwrite=True)

    for _ in range(max(args.warmup, 3)):
        flush.fill_(1)
        step()
    if enc.status_sync(stream) != fh.FH_OK:
        raise RuntimeError("domain flag set on synthetic inputs")

    K = args.steps
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(K)]
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    l0 = fh.kernel_launches()
    with ClockSampler(local_rank) as clk:
        for k in range(K):
            flush.fill_(k & 0xFF)
            e = ev[k]
            e[0].record(stream)
            e[1].record(stream)
            enc.fwd(coords, table, out, stream=stream)
            e[2].record(stream)
            enc.bwd(coords, dout, dtable, stream=stream, overwrite=True)
            e[3].record(stream)
        torch.cuda.synchronize()
    launches = fh.kernel_launches() - l0
    if dist:
        dist.barrier()
    fwd_ms = sum(e[1].elapsed_time(e[2]) for e in ev) / K
    bwd_ms = sum(e[2].elapsed_time(e[3]) for e in ev) / K
    step_ms = sum(e[0].elapsed_time(e[3]) for e in ev) / K
    total_s = step_ms * K / 1e3
    if dist:
        t = torch.tensor([total_s], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_s = float(t.item())
    status = enc.status_sync(stream)
    if status != fh.FH_OK:
        raise RuntimeError("domain flag set during timed region")
    value = N * world * K / total_s
    props = torch.cuda.get_device_properties(local_rank)
    me = {"rank": rank, "local_rank": local_rank, "device": props.name,
          "pci_bus_id": getattr(props, "pci_bus_id", None), "uuid": str(getattr(props, "uuid", "")),
          "device_ms_per_step": step_ms}
    ranks = [me]
    comm = {"backend": None, "world_size": 1}
    if dist:
        ranks = [None] * world
        dist.all_gather_object(ranks, me)
        comm = {"backend": dist.get_backend(), "world_size": dist.get_world_size(),
                "nccl_version": ".".join(str(v) for v in torch.cuda.nccl.version())}

    # e2e: the same step through the C ABI from pinned HOST buffers, copies
    # inside the timed region (fh_encode_step_host: H2D of the step's coords and
    # dout, fwd, bwd (dtable overwritten), D2H of out and dtable).  Steps
    # rotate over three streams with three device / host-output buffer sets,
    # so step k+1's H2D overlaps step k's kernels and step k-1's D2H (PCIe is
    # full duplex; with two sets the next H2D on a stream waits for that
    # stream's D2H); every step's copies stay inside the timed region.
    coords_h = torch.from_numpy(case.coords).pin_memory()
    dout_h = torch.from_numpy(case.dout).pin_memory()
    NS = int(os.environ.get("FH_E2E_STREAMS", "3"))   # streams / buffer sets the e2e steps rotate over
    streams = [torch.cuda.Stream() for _ in range(NS)]
    sets = [dict(c=coords, g=dout, o=out, dt=dtable)]
    for _ in range(NS - 1):
        sets.append(dict(c=torch.empty_like(coords), g=torch.empty_like(dout), o=torch.empty_like(out),
                         dt=torch.empty_like(dtable)))
    for b in sets:
        b["oh"] = torch.empty((N, cfg.L * cfg.F)).pin_memory()
        b["dth"] = torch.empty((enc.entries, cfg.F)).pin_memory()

    def e2e_step(k):
        b, st = sets[k % NS], streams[k % NS]
        enc.step_host(coords_h, dout_h, table, b["c"], b["g"], b["o"], b["dt"], b["oh"], b["dth"], st)

    ke = max(4, min(K, 10))
    for k in range(4):
        e2e_step(k)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for st in streams:
        st.wait_event(e0)
    for k in range(ke):
        e2e_step(k)
    for st in streams:
        j = torch.cuda.Event()
        j.record(st)
        stream.wait_event(j)
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_s = e0.elapsed_time(e1) / 1e3
    if dist:
        t = torch.tensor([e2e_s], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    if not torch.equal(sets[0]["oh"], sets[1]["oh"]):   # same inputs -> identical forward output
        raise RuntimeError("e2e: the two pipelined buffer sets disagree")
    e2e = {"value": N * world * ke / e2e_s, "unit": UNIT, "h2d_bytes_per_step": N * 16 + N * cfg.L * cfg.F * 4,
           "d2h_bytes_per_step": N * cfg.L * cfg.F * 4 + enc.entries * cfg.F * 4, "steps": ke,
           "api": "fh_encode_step_host (pinned host in/out), steps rotating over three streams / buffer sets"}

    # Train step (all §8(a) rows): free the encode buffers first.
    train = {}
    if not args.no_train:
        del coords_h, dout_h, sets, out, dout, dtable, flush
        torch.cuda.empty_cache()
        kt = max(3, min(K, 10))

        def leg(which):
            # The headline above is already measured: a failing train leg is
            # reported in its own key (traceback on stderr) instead of losing
            # the line.  Every rank runs the same code, so a failure here is
            # normally raised on all ranks alike.
            try:
                return train_step_bench(fh, torch, W, which, rank, world, dist, kt, args.warmup, args.dp)
            except Exception as ex:  # noqa: BLE001
                import traceback
                traceback.print_exc(file=sys.stderr)
                return {"error": f"{type(ex).__name__}: {ex}"[:400]}
            finally:
                torch.cuda.empty_cache()

        if world == 1:
            train["cfg3"] = leg("cfg3")
        train["cfg5"] = leg("cfg5")
    encoders = paper_encoder_compare(fh, torch, W, max(3, min(K, 10))) if not args.no_train else None
    torch.cuda.empty_cache()
    hbm_peak, peak_src = load_peaks()
    coreset = coreset_bench(fh, torch, W, max(3, min(K, 10)), hbm_peak,
                            with_cpu=(rank == 0 and not args.no_cpu_baseline)) if not args.no_train else None
    torch.cuda.empty_cache()

    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return

    mb = microbench_roofline(fh, torch, enc, cfg, N, stream, hbm_peak)
    hbm_regime = hbm_regime_bench(fh, torch, W, max(3, min(K, 10)), hbm_peak) if not args.no_train else None
    # Contract roofline of the dominant kernel: algorithmic bytes / launch time.
    LF4 = cfg.L * cfg.F * 4
    alg = {"fwd": N * (16 * cfg.L * cfg.F * 4 + 16 + LF4), "bwd": N * (16 * cfg.L * cfg.F * 4 + 16 + LF4)}
    dom = "bwd" if bwd_ms >= fwd_ms else "fwd"
    dom_ms = bwd_ms if dom == "bwd" else fwd_ms
    achieved = alg[dom] / (dom_ms / 1e3) / 1e9
    ncu = load_ncu_summary().get("cfg2", {})
    traffic = ncu.get("dram_bytes_per_pass", {}).get(dom)
    roofline = {"bound": "hbm", "kernel": f"encode {dom} pass (fh::{dom}_kernel<2> level groups"
                + (" + merge_shift_kernel)" if dom == "bwd" else ")"), "achieved": achieved, "peak": hbm_peak,
                "unit": "GB/s", "frac": achieved / hbm_peak, "traffic": traffic,
                "peak_source": peak_src,
                "algorithmic_bytes_per_launch": alg[dom], "launch_unit": "one encode pass (all its launches)",
                "note": "useful gather (or red) payload 16*L*F*4 B + coords 16 B + out/dout L*F*4 B per sample over the "
                        "measured HBM copy peak; the cfg2 tables are L2-resident, so the binding unit is the L2 "
                        "(l2_frac: ncu lts__throughput of the same launches, profiles/)"}
    # the backward issues one 16-byte reduction per x-pair of every (sample,
    # level) (F = 2 with the shifted pairs): 8 per cell
    red_ops = N * cfg.L * 8
    roofline["l2_red"] = {"what": "encode bwd: L2 reduction ops issued per second vs the measured random red.v4 op "
                                  "rate of an L2-resident buffer (the unit the backward is bound by)",
                          "ops_per_pass": red_ops, "achieved_G_per_s": red_ops / (bwd_ms / 1e3) / 1e9,
                          "ceiling_G_per_s": mb["l2_red_op_ceiling_G_per_s"],
                          "frac": red_ops / (bwd_ms / 1e3) / 1e9 / mb["l2_red_op_ceiling_G_per_s"]}
    if ncu:
        roofline["l2_frac"] = ncu.get("lts_throughput_frac", {}).get(dom)
        roofline["l2_evidence"] = {k: ncu[k] for k in ("source", "lts_throughput_frac", "l1tex2xbar_req_frac",
                                                        "l2_red_sectors_per_pass", "l2_hit_frac") if k in ncu}
    t_micro = mb["t_roof_fwd_ms"] + mb["t_roof_bwd_ms"]
    gather_microbench = {
        "what": "the encode's access shape without its index math (fh_bench_gather_levels / fh_bench_red_levels: "
                "one aligned x-pair access per corner pair, same level mix) + streamed bytes at the copy bandwidth; "
                "context, NOT a ceiling (the kernel may beat it)",
        "t_ms": t_micro, "t_measured_ms": fwd_ms + bwd_ms, "measured_over_microbench": (fwd_ms + bwd_ms) / t_micro,
        **{k: v for k, v in mb.items() if k not in ("t_roof_fwd_ms", "t_roof_bwd_ms")},
        "t_fwd_ms": mb["t_roof_fwd_ms"], "t_bwd_ms": mb["t_roof_bwd_ms"],
    }
    cpu = None
    cpu_all = None
    cpu_more = None
    if world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(cfg, case.coords, case.table, case.dout)
        try:
            cpu_all = cpu_baseline_all_cores(cfg, case.coords, case.table, case.dout)
        except Exception as ex:   # the all-cores run is context; never fail the bench on it
            cpu_all = {"unavailable": f"{type(ex).__name__}: {ex}"}
        if not args.no_train:
            try:
                cpu_more = cpu_oracle_baselines(W)
            except Exception as ex:   # context; never fail the bench on it
                cpu_more = {"unavailable": f"{type(ex).__name__}: {ex}"}
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K, "warmup": max(args.warmup, 3),
        "ms_per_step": total_s * 1e3 / K, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f32", "data": "synthetic", "config": config_block(cfg, N, world),
        "kernels_ms": {"zero_grad": "inside encode_bwd (FH_BWD_OVERWRITE)", "encode_fwd": fwd_ms, "encode_bwd": bwd_ms, "step": step_ms},
        "roofline": roofline, "gather_microbench": gather_microbench, "cpu_baseline": cpu, "cpu_baseline_all_cores": cpu_all,
        "cpu_oracle_baselines": cpu_more, "e2e": e2e,
        "gpu_launches": launches, "clocks": clk.summary(), "ranks": ranks, "comm": comm, "train_step": train,
        "paper_encoders": encoders, "coreset": coreset, "hbm_regime": hbm_regime,
    }
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


def free_port() -> int:
    import socket
    with socket.socket(socket.AF_INET, socket.SOCK_STREAM) as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def spawn_ranks(n: int, argv) -> int:
    """Re-launch this script with n ranks under torch.distributed.run (one
    process per GPU, rendezvous on 127.0.0.1).  NCCL's INIT lines (which
    report nranks and the rank -> device mapping) go to stderr."""
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()), os.path.abspath(__file__), *argv]
    return subprocess.call(cmd, env=env)


def launch_check(args, rank, world):
    """The N > 1 plumbing without GPU work: gloo rendezvous, a barrier, the
    max-over-ranks reduction of a per-rank time, and the per-rank record."""
    import socket
    import torch
    import torch.distributed as dist
    if world > 1:
        dist.init_process_group("gloo")
    t = 0.001 * (rank + 1)   # a rank-dependent "device time": the max must be the last rank's
    info = {"rank": rank, "local_rank": env_int("LOCAL_RANK", 0), "host": socket.gethostname(), "pid": os.getpid(),
            "device_ms": t * 1e3}
    ranks = [info]
    if world > 1:
        dist.barrier()
        tt = torch.tensor([t], dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t = float(tt.item())
        ranks = [None] * world
        dist.all_gather_object(ranks, info)
    if rank == 0:
        print(json.dumps({"launch_check": True, "metric": METRIC, "unit": UNIT, "n_gpus": world,
                          "max_rank_ms": t * 1e3, "ranks": ranks,
                          "comm": {"backend": "gloo" if world > 1 else None, "world_size": world}}), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=None, help="ranks (GPUs); default WORLD_SIZE or 1")
    ap.add_argument("--launch-check", action="store_true", help="launcher / rendezvous / reduction only (CPU, gloo)")
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-train", action="store_true", help="skip the train_step (cfg3 / cfg5) sub-benchmarks")
    ap.add_argument("--dp", default="nccl", choices=["nccl", "fused", "peer", "multicast"],
                    help="N>1 gradient path: NCCL reduce-scatter overlapped with the backward from Python (default), "
                         "the same exchange driven inside the library (fused, fh_trainer_set_comm), or the fused "
                         "peer-memory reduce + Adam + all-gather kernel (torch symmetric memory), or that step through "
                         "an NVLS multicast object (multimem.ld_reduce / multimem.st; falls back to peer without one)")
    args = ap.parse_args()
    if "WORLD_SIZE" not in os.environ and (args.gpus or 1) > 1:
        sys.exit(spawn_ranks(args.gpus, sys.argv[1:]))
    rank = env_int("RANK", 0)
    local_rank = env_int("LOCAL_RANK", 0)
    world = env_int("WORLD_SIZE", 1)
    if args.gpus is not None and args.gpus != world:
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if args.launch_check:
        launch_check(args, rank, world)
    elif args.impl == "reference":
        run_reference(args, rank, world)
    else:
        run_ours(args, rank, local_rank, world)


if __name__ == "__main__":
    main()
