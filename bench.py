"""Benchmark of the ILU / stri / spmv hot path on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl mine|reference]

One step = one pass of the hot path over the config's matrix, inputs
resident in HBM: refresh the factor values from the assembled matrix,
numeric factorization (sync-free kernel), forward + backward triangular
solve, spmv.  `value` is the factorization throughput in factor nonzeros
per second (BASELINE.json metric "ILU factor nnz/s, stri and spmv GB/s");
stri and spmv GB/s are reported under "paths".  Every matrix is larger
than the 126 MB L2, so no flush is needed between steps.

For N > 1 (torchrun, one process per GPU) every rank runs its own replica
of the single-matrix workload (factorization and stri of one matrix run on
one GPU: replicas only), `value` aggregates all ranks over the max-over-ranks
time.  --impl reference times the reference's CPU algorithm (the pinned C
oracle, threaded point-to-point version) on the host cores.
"""

from __future__ import annotations

import argparse
import ctypes
import hashlib
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

HBM_FALLBACK = 6650.0   # GB/s, B200_PROFILING.md fallback if MEASURED_PEAKS.json is absent


def peaks():
    p = os.path.join(REPO, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured"
    return HBM_FALLBACK, "fallback"


def alg_bytes(n, nnz_a, nnz_f):
    """SURVEY.md §8d algorithmic bytes (int32 indices, fp64 values)."""
    return dict(
        spmv=12 * nnz_a + 20 * n + 4,
        factor=20 * nnz_f + 8 * n + 4,
        stri=12 * nnz_f + 48 * n + 8,
    )


def build_config(cfg, rank=0, world=1, rmat_count=64, first=0):
    """Matrix + device plan of the config.  c5 (a batch of independent R-MAT
    systems) is sharded (dist.BatchShard): this rank builds the
    block-diagonal matrix of its contiguous block of seeds; `blocks` is the
    shard."""
    import paper_1812_06160_b200 as jv
    from paper_1812_06160_b200 import workloads as W
    from paper_1812_06160_b200.dist import BatchShard
    from paper_1812_06160_b200.plan import build_plan

    blocks = None
    if cfg == "c5":
        s = W.CONFIGS[cfg]
        blocks = BatchShard(rmat_count, rank, world, first)
        a, base = blocks.assemble(lambda sd: W.rmat(18, sd)), None
    else:
        a, base, s = W.config_matrix(cfg)
    t0 = time.perf_counter()
    if base == "rcm":
        base_perm = jv.rcm_order(a.pattern).perm
    elif base is None:
        base_perm = None
    else:
        base_perm = base.perm
    import torch
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    plan = build_plan(a, base_perm=base_perm, k=s["k"], tau=s["tau"],
                      min_level_rows=s["min_level_rows"])
    torch.cuda.synchronize()
    # setup, reported apart from the steps as the reference does
    # (pipeline.py:231-237): base order, then levels / partition / permutation /
    # symbolic pattern / assembly on the device
    build_config.setup = {"order_s": t1 - t0, "plan_s": time.perf_counter() - t1}
    return a, plan, s, blocks


def rhs(n, blocks):
    """b drawn in the original order (uniform[-1,1], seed 0 per system, as
    the reference's krylov.py:199 / SURVEY.md §8d), one draw per block."""
    if blocks is None:
        return np.random.default_rng(0).uniform(-1.0, 1.0, n)
    return np.concatenate([np.random.default_rng(0).uniform(-1.0, 1.0, m) for m in blocks.sizes])


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled while the GPU is busy."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        self.proc.wait(timeout=5)
        self.t.join(timeout=2)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def _median_runs(fn, budget_s, max_runs=5, prep=None):
    """Median wall time of fn() over up to max_runs runs within budget_s
    (at least one); prep() runs untimed before each."""
    ts = []
    deadline = time.perf_counter() + budget_s
    while len(ts) < max_runs and (not ts or time.perf_counter() < deadline):
        if prep is not None:
            prep()
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return statistics.median(ts), len(ts)


def cpu_baseline(cfg, plan, seconds=12.0, blocks=None):
    """The reference's algorithms on the host (the pinned C oracle) on the
    same matrix: factor (serial 1 core; point-to-point threads on all
    cores), stri pair (serial sweeps; p2p threaded sweeps), spmv (1 core,
    the reference's is single-threaded).  Each path: median of up to 5 runs
    within its share of `seconds`; value copies made outside the timing.
    For the c5 batch the sample is ONE system of the batch (the throughput
    units are per nonzero / per byte, so they carry over)."""
    import oracle
    from paper_1812_06160_b200 import device as dv

    ilu = plan.ilu
    n = ilu.n
    rs = dv.host_i64(ilu.row_start, n + 1)
    col = dv.host_i64(ilu.col, ilu.nnz)
    diag = dv.host_i64(ilu.diag_pos, n)
    val = dv.host_f64(plan.assembled, ilu.nnz)
    prs, pcol = plan.permuted.host_pattern()
    pval = dv.host_f64(plan.permuted.val, plan.permuted.nnz)
    sample = f"full {cfg} matrix"
    if blocks is not None:
        from paper_1812_06160_b200 import workloads as W
        sd = blocks.seeds[0]
        m = W.rmat(18, sd)
        fe = oracle.front_end(m.n, m.row_start, m.col, m.val)
        rs, col, diag, val = fe["row_start"], fe["col"], fe["diag"], fe["val"]
        prs, pcol, pval = fe["permuted"]
        n = m.n
        sample = f"one system of the c5 batch (R-MAT seed {sd})"
    tau = ilu.tau
    cores = os.cpu_count() or 1
    nnz_f, nnz_a = int(col.size), int(pcol.size)
    ab = alg_bytes(n, nnz_a, nnz_f)
    share = seconds / 5.0
    v = np.empty_like(val)
    refresh = lambda: np.copyto(v, val)
    fs, k1 = _median_runs(lambda: oracle.p2p(0, 1, rs, col, v, diag, tau, inplace=True), share,
                          prep=refresh)
    ft, k2 = _median_runs(lambda: oracle.p2p(0, cores, rs, col, v, diag, tau, inplace=True), share,
                          prep=refresh)
    fval, _ = oracle.factor_serial(rs, col, val, diag, tau)
    b = np.random.default_rng(0).uniform(-1.0, 1.0, n)
    ss, k3 = _median_runs(lambda: oracle.solve_backward(
        rs, col, fval, diag, oracle.solve_forward(rs, col, fval, b)), share)
    x = np.empty(n)

    def thr():
        np.copyto(x, b)
        oracle.p2p(1, cores, rs, col, fval, diag, vec=x, inplace=True)
        oracle.p2p(2, cores, rs, col, fval, diag, vec=x, inplace=True)
    st, k4 = _median_runs(thr, share)
    sp, k5 = _median_runs(lambda: oracle.spmv(prs, pcol, pval, b), share)
    GB = lambda nb, t: nb / t / 1e9
    return {
        "value": nnz_f / ft, "unit": "factor nnz/s", "cores": cores, "kind": "port",
        "sample": f"{sample}; pinned C restatement of the reference kernels; medians of "
                  f"{min(k1, k2, k3, k4, k5)}-5 runs",
        "serial_value": nnz_f / fs, "serial_cores": 1, "cpu_model": cpu_model(),
        "paths": {
            "factor": {"serial_ms": fs * 1e3, "threaded_ms": ft * 1e3, "threads": cores,
                       "serial_nnz_per_s": nnz_f / fs, "threaded_nnz_per_s": nnz_f / ft},
            "stri": {"serial_ms": ss * 1e3, "threaded_ms": st * 1e3, "threads": cores,
                     "serial_GBps": GB(ab["stri"], ss), "threaded_GBps": GB(ab["stri"], st),
                     "sweeps": "forward+backward (serial = solve_serial; threaded = solve_ls p2p)"},
            "spmv": {"serial_ms": sp * 1e3, "GBps": GB(ab["spmv"], sp), "threads": 1},
        },
    }


def digest(a, kind):
    a = np.ascontiguousarray(a, dtype=np.int64 if kind == "i" else np.float64)
    return hashlib.sha256(a.tobytes()).hexdigest()


def parity_check(cfg, ilu, plan, x, sy, blocks, n):
    """Bitwise digests of the timed arrays against the reference's full-size
    digests (tests/golden/full_digests.json); None when none apply."""
    from paper_1812_06160_b200 import device as dv
    dpath = os.path.join(REPO, "tests", "golden", "full_digests.json")
    if not os.path.exists(dpath):
        return None
    allg = json.load(open(dpath))
    if blocks is None:
        d = allg.get(cfg)
        if not d:
            return None
        return (digest(ilu.host_val(), "f") == d["digests"]["fval"]
                and digest(dv.host_f64(x, n), "f") == d["digests"]["x"]
                and digest(dv.host_f64(sy, n), "f") == d["digests"]["spmv_perm"])
    have = [sd for sd in blocks.seeds if f"c5_seed{sd}" in allg]
    parity_check.detail = {"systems_checked": len(have), "systems": len(blocks.seeds)}
    if not have:
        return None
    perm = dv.host_i64(plan.perm, n)
    rows = blocks.system_rows(perm)
    rs = dv.host_i64(ilu.row_start, n + 1)
    val = ilu.host_val()
    xh = dv.host_f64(x, n)
    syh = dv.host_f64(sy, n) if sy is not None else None   # None: no product in this step
    ok = True
    for sd in have:
        d = allg[f"c5_seed{sd}"]["digests"]
        r = rows[sd]
        ok &= digest(blocks.take_rows(rs, val, r), "f") == d["fval"]
        ok &= digest(xh[r], "f") == d["x"]
        if syh is not None:
            ok &= digest(syh[r], "f") == d["spmv_perm"]
    return bool(ok)


def measure_batch(world, rank, per_gpu, steps):
    """Batch sharding (SURVEY §8e, config 5's systems): every rank factors
    and solves its own `per_gpu` R-MAT systems (seeds rank*per_gpu + i) as
    one block-diagonal matrix, no collective on the hot path; per-GPU work
    fixed (weak scaling; at 8 GPUs x 8 systems this is the full c5 batch).
    Device time per step is the max over ranks; every system is checked
    bitwise against the reference's digests (all 64 seeds are pinned)."""
    import torch
    import torch.distributed as dist
    from paper_1812_06160_b200 import device as dv

    a, plan, s, shard = build_config("c5", rank, world, per_gpu * world)
    ilu = plan.ilu
    n = ilu.n
    perm = dv.host_i64(plan.perm, n)
    b = dv.f64(rhs(n, shard)[perm])
    y, x = dv.empty_f64(n), dv.empty_f64(n)

    def step():
        plan.reset_values()
        ilu.factor_async()
        ilu.solve_async(0, b, y)
        ilu.solve_async(1, y, x)
    step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(steps):
        step()
    e1.record()
    torch.cuda.synchronize()
    ms = torch.tensor([e0.elapsed_time(e1) / steps, float(ilu.nnz)], dtype=torch.float64,
                      device="cuda")
    if world > 1:
        dist.all_reduce(ms[:1], op=dist.ReduceOp.MAX)
        dist.all_reduce(ms[1:], op=dist.ReduceOp.SUM)
    step_ms, nnz_all = float(ms[0]), float(ms[1])
    ok = parity_check("c5", ilu, plan, x, None, shard, n)   # (this step has no spmv)
    det = dict(getattr(parity_check, "detail", {}))
    if world > 1:
        parts = [None] * world
        dist.all_gather_object(parts, (ok, det))
        ok = all(p[0] in (None, True) for p in parts) and any(p[0] is not None for p in parts)
        det = {"systems_checked": sum(p[1].get("systems_checked", 0) for p in parts),
               "systems": sum(p[1].get("systems", 0) for p in parts)}
    dv.check_hang()
    del plan, ilu
    return {"systems_per_gpu": per_gpu, "systems_total": per_gpu * world, "scaling": "weak",
            "step": "refresh + factor + forward + backward stri",
            "step_ms_max_over_ranks": step_ms, "factor_nnz_total": nnz_all,
            "nnz_per_s_aggregate": nnz_all / (step_ms / 1e3),
            "bitwise_vs_reference": ok, **det}


def measure_spmv_dist(plan, steps, world, rank):
    """Row-partitioned spmv of the config's (permuted) matrix over all ranks
    with one NCCL halo exchange per product (dist.DistSpmv): back-to-back
    (Krylov-like) and single-shot device time, max over ranks."""
    import torch
    import torch.distributed as dist
    from paper_1812_06160_b200 import device as dv
    from paper_1812_06160_b200 import dist as jd

    A = plan.permuted
    n = A.n
    rs, col = A.host_pattern()
    val = dv.host_f64(A.val, A.nnz)
    bounds = jd.row_partition(rs, world)
    hp = jd.plan_halo(rs, col, val, bounds, rank, world)
    sp = jd.DistSpmv(hp)
    x = np.random.default_rng(0).uniform(-1.0, 1.0, n)
    sp.x_local.copy_(dv.f64(x[hp.lo:hp.hi]))
    y = dv.empty_f64(max(hp.n_local, 1))
    for _ in range(5):
        sp(sp.x_local, y)
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(steps):
        sp(sp.x_local, y)
    e1.record()
    torch.cuda.synchronize()
    b2b = e0.elapsed_time(e1) / steps
    single = []
    for _ in range(min(steps, 20)):
        dist.barrier()
        torch.cuda.synchronize()
        e0.record()
        sp(sp.x_local, y)
        e1.record()
        torch.cuda.synchronize()
        single.append(e0.elapsed_time(e1))
    t = torch.tensor([b2b, statistics.median(single)], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    b2b, one = [float(v) for v in t.tolist()]
    # bitwise check of the distributed product against the whole-matrix one
    parts = [None] * world
    dist.all_gather_object(parts, (hp.lo, dv.host_f64(y, hp.n_local)))
    ok = None
    if rank == 0:
        import oracle
        full = np.zeros(n)
        for lo, part in parts:
            full[lo:lo + part.size] = part
        ok = bool(np.array_equal(full, oracle.spmv(rs, col, val, x)))
    nbytes = alg_bytes(n, A.nnz, 0)["spmv"]
    peak, _ = peaks()
    return {"ranks": world, "partition": "contiguous rows, nnz-balanced",
            "back_to_back_us": b2b * 1e3, "single_shot_us": one * 1e3,
            "GBps_aggregate": nbytes / (b2b * 1e-3) / 1e9,
            "frac_of_world_peak": nbytes / (b2b * 1e-3) / 1e9 / (peak * world),
            "single_shot_GBps": nbytes / (one * 1e-3) / 1e9,
            "halo_bytes_rank0": hp.halo_bytes, "peers_rank0": hp.stats["peers"],
            "boundary_rows_rank0": hp.stats["boundary_rows"], "bitwise_vs_oracle": ok}


def run_mine(args):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    from paper_1812_06160_b200 import device as dv

    a, plan, s, blocks = build_config(args.config, rank, world, args.rmat_count)
    setup = dict(build_config.setup)
    t_sched = time.perf_counter()
    batched = blocks is not None
    ilu = plan.ilu
    n, nnz_f, nnz_a = ilu.n, ilu.nnz, plan.permuted.nnz
    ab = alg_bytes(n, nnz_a, nnz_f)
    perm = dv.host_i64(plan.perm, n)
    b = dv.f64(rhs(n, blocks)[perm])
    y = dv.empty_f64(n)
    x = dv.empty_f64(n)
    sy = dv.empty_f64(n)
    ilu.factor_schedule()
    ilu.elim_lists()
    ilu.fwd_schedule()
    ilu.bwd_schedule()
    plan.permuted.tile_rows()

    def step(ev=None):
        plan.reset_values()
        if ev is not None:
            ev[0].record()
        ilu.factor_async()
        if ev is not None:
            ev[1].record()
        ilu.solve_async(0, b, y)
        if ev is not None:
            ev[2].record()
        ilu.solve_async(1, y, x)
        if ev is not None:
            ev[3].record()
        dv.spmv_dev(plan.permuted, b, sy)
        if ev is not None:
            ev[4].record()

    torch.cuda.synchronize()
    setup["schedules_s"] = time.perf_counter() - t_sched   # sweep schedules, elimination lists, spmv plan
    t_first = time.perf_counter()
    step()
    torch.cuda.synchronize()
    # first step: region / tail / single-CTA plans and the one-time path timing
    setup["first_step_s"] = time.perf_counter() - t_first
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    bad = dv.read_row_slot(ilu.err)
    dv.check_hang()

    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.3)
    for _ in range(max(args.warmup, 3)):   # keep the GPU busy while the sampler starts
        step()
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(5)] for _ in range(args.steps)]
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    from paper_1812_06160_b200 import _lib as _L
    _L.launch_counts.clear()
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_push("timed")   # ncu --nvtx --nvtx-include "timed/"
    t0.record()
    for k in range(args.steps):
        step(evs[k])
    t1.record()
    torch.cuda.nvtx.range_pop()
    launches = sum(_L.launch_counts.values())
    launch_detail = dict(_L.launch_counts)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = sampler.stop()
    total_ms = t0.elapsed_time(t1)
    f_ms = [e[0].elapsed_time(e[1]) for e in evs]
    fw_ms = [e[1].elapsed_time(e[2]) for e in evs]
    bw_ms = [e[2].elapsed_time(e[3]) for e in evs]
    sp_ms = [e[3].elapsed_time(e[4]) for e in evs]
    mine = torch.tensor([float(nnz_f), float(nnz_a), float(n)], dtype=torch.float64, device="cuda")
    times = torch.tensor([total_ms, sum(f_ms), sum(fw_ms) + sum(bw_ms), sum(sp_ms)],
                         dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(times, op=dist.ReduceOp.MAX)
        dist.all_reduce(mine, op=dist.ReduceOp.SUM)
    total_ms, f_sum, st_sum, sp_sum = [float(v) for v in times.tolist()]
    tot_nnz_f, tot_nnz_a, tot_n = [int(v) for v in mine.tolist()]
    K = args.steps
    f_avg, st_avg, sp_avg = f_sum / K / 1e3, st_sum / K / 1e3, sp_sum / K / 1e3   # seconds

    parity = parity_check(args.config, ilu, plan, x, sy, blocks, n)

    # the paper's CSR-LS baseline on this GPU (one launch per level, CUDA
    # graph), for comparison with the sync-free / region sweeps; same bits
    csrls = None
    if not batched:
        cy, cx = dv.empty_f64(n), dv.empty_f64(n)
        ilu.solve_csrls_async(0, b, cy)
        ilu.solve_csrls_async(1, cy, cx)
        ce = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        cf, cb = [], []
        for _ in range(5):
            ce[0].record()
            ilu.solve_csrls_async(0, b, cy)
            ce[1].record()
            ilu.solve_csrls_async(1, cy, cx)
            ce[2].record()
            torch.cuda.synchronize()
            cf.append(ce[0].elapsed_time(ce[1]) * 1e3)
            cb.append(ce[1].elapsed_time(ce[2]) * 1e3)
        csrls = {"fwd_us": statistics.median(cf), "bwd_us": statistics.median(cb),
                 "launches_per_sweep": ilu._csrls[0][3],
                 "bitwise_equal_to_step": bool(torch.equal(cx, x))}
    if world > 1:
        pl = [None] * world
        dist.all_gather_object(pl, parity)
        parity = None if all(p is None for p in pl) else all(p in (None, True) for p in pl)

    # end to end through the public API (host numpy buffers in, out)
    e2e = measure_e2e(a, plan, args)
    if world > 1:
        et = torch.tensor([e2e["ms"]], dtype=torch.float64, device="cuda")
        dist.all_reduce(et, op=dist.ReduceOp.MAX)
        e2e["ms"] = float(et.item())
        e2e["value"] = (tot_nnz_f if batched else world * nnz_f) / (e2e["ms"] / 1e3)

    multi = None
    if not batched and args.batch_per_gpu > 0:
        multi = {}
        if world > 1:
            try:
                multi["spmv_dist"] = measure_spmv_dist(plan, max(K, 20), world, rank)
            except Exception as e:   # never lose the main line to the extra measurement
                multi["spmv_dist"] = {"error": repr(e)[:200]}
        try:
            multi["batch"] = measure_batch(world, rank, args.batch_per_gpu, 3)
        except Exception as e:
            multi["batch"] = {"error": repr(e)[:200]}

    peak, peak_kind = peaks()
    # per-GPU algorithmic bytes (every rank factors its own matrix / shard)
    ach = ab["factor"] / f_avg / 1e9
    prof = load_profile(args.config) or {}

    def impl_of(sw):
        rp = ilu._region_for(sw)
        if rp is None:
            return "tickets"
        if rp is dv.SMALL:
            return "small"
        return "two_stage" if rp is dv.TWO_STAGE else ("cta" if rp is dv.CTA else "region")
    impl = {sw: impl_of(sw) for sw in ("factor", "fwd", "bwd")}

    # DAG depths and the measured cross-SM hop: depth x t_hop is the floor of
    # a sweep whose consecutive levels sit on different SMs
    hop_ns = ctypes.c_double(0.0)
    _L.call("jv_hop_latency", 20000, ctypes.byref(hop_ns))
    t_hop_us = hop_ns.value / 1e3
    fdepth = dv.levels_dev(ilu.pattern, False)[1]
    bdepth = dv.levels_dev(ilu.pattern, True)[1]
    tail = measure_tail(ilu, plan, K) if plan.n_upper < n else None

    def roof(nbytes, secs, depth, kernel, traffic_key):
        a = nbytes / secs / 1e9
        return {"bound": "hbm", "achieved": a, "peak": peak, "unit": "GB/s", "frac": a / peak,
                "frac_of_8TBs_nominal": a / 8000.0,
                "peak_kind": peak_kind, "alg_bytes": nbytes, "us": secs * 1e6,
                "traffic": prof.get(traffic_key), "kernel": kernel, "dag_depth": depth,
                "t_hop_us": t_hop_us, "depth_x_thop_us": depth * t_hop_us}
    # tau > 0: strict-lower positions left exactly 0 by the timed factorization
    # (dropped multipliers, fill included; full_digests.json stats.zero_l)
    zero_l = None
    if s["tau"] > 0 and not batched:
        rows = torch.repeat_interleave(torch.arange(n, device="cuda"),
                                       (ilu.row_start[1:n + 1] - ilu.row_start[:n]).long())
        low = torch.arange(nnz_f, device="cuda") < ilu.diag_pos[:n].long()[rows]
        zero_l = int(((ilu.val[:nnz_f] == 0.0) & low).sum().item())
    rooflines = {
        "factor": roof(ab["factor"], f_avg, fdepth,
                       {"tickets": "factor_kernel", "region": "region_kernel<0>",
                        "two_stage": "factor_kernel + tail_upper_kernel + corner",
                        "cta": "factor_cta_kernel"}[impl["factor"]],
                       "factor_dram_bytes"),
        "stri": roof(ab["stri"], st_avg, fdepth + bdepth,
                     f"fwd {impl['fwd']} + bwd {impl['bwd']}", "stri_dram_bytes"),
        "spmv": roof(ab["spmv"], sp_avg, 0,
                     "spmv_bulk_kernel" if _L.load().jv_spmv_impl_for(
                         plan.permuted.nnz, dv.ptr(plan.permuted.tile_rows())) else "spmv_stream_kernel",
                     "spmv_dram_bytes"),
    }
    if tail is not None:
        tail_nnz = int(dv.host_i64(ilu.row_start[plan.n_upper:], 1)[0])
        tb = 20 * (nnz_f - tail_nnz) + 8 * (n - plan.n_upper) + 4
        tail["stage1_roofline"] = roof(tb, tail["stage1_us"] / 1e6, 0, "tail_upper_kernel",
                                       "tail_dram_bytes")
        tail["stage1_roofline"]["note"] = ("alg bytes = the tail rows' share of the factor "
                                           "formula (20 nnz_tail + 8 n_tail + 4)")
    paths = {
        "impl": impl, "autotune_ms": {k: list(v) for k, v in ilu.autotune_ms.items()},
        "factor": {"us": f_avg * 1e6, "nnz_per_s": nnz_f / f_avg, "alg_bytes": ab["factor"],
                   "GBps": ab["factor"] / f_avg / 1e9, "frac": ab["factor"] / f_avg / 1e9 / peak},
        "stri": {"us": st_avg * 1e6, "alg_bytes": ab["stri"], "GBps": ab["stri"] / st_avg / 1e9,
                 "frac": ab["stri"] / st_avg / 1e9 / peak,
                 "fwd_us": sum(fw_ms) / K * 1e3, "bwd_us": sum(bw_ms) / K * 1e3},
        "stri_csrls_baseline": csrls,
        "tail": tail,
        "spmv": {"us": sp_avg * 1e6, "alg_bytes": ab["spmv"], "GBps": ab["spmv"] / sp_avg / 1e9,
                 "frac": ab["spmv"] / sp_avg / 1e9 / peak},
    }
    if batched:
        workload = f"c5:rmat18_x{args.rmat_count} (block-diagonal shard per rank)"
        value = tot_nnz_f / f_avg
        scaling = "strong"
        par = f"batch-sharded dp{world} ({len(blocks.seeds)} systems on rank {rank})"
    else:
        workload = f"{args.config}:{s['name']}"
        value = world * nnz_f / f_avg
        scaling = "weak"
        par = f"replicas{world}" + (" + row-partitioned spmv" if world > 1 else "")
    line = {
        "metric": "ILU factor nnz/s, stri and spmv GB/s (fp64) vs HBM roofline; 1/2/4/8 GPU",
        "value": value,
        "unit": "factor nnz/s",
        "n_gpus": world,
        "steps": K,
        "warmup": args.warmup,
        "ms_per_step": total_ms / K,
        "higher_is_better": True,
        "scaling": scaling,
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (seeded generator, SURVEY.md §8d recipe)",
        "config": {"workload": workload, "n": n, "nnz_a": nnz_a, "nnz_f": nnz_f,
                   "total_nnz_f": tot_nnz_f, "k": s["k"], "tau": s["tau"], "levels": plan.nlev,
                   "n_upper": plan.n_upper, "parallelism": par,
                   "l2": ("inputs > 126 MB L2, no flush needed"
                          if 8 * nnz_f + 12 * nnz_a > 126e6 else
                          "working set below the 126 MB L2: steps run L2-warm, no flush "
                          "(a parity-size config, not the bench line)")},
        "roofline": dict(rooflines["factor"]),
        "rooflines": rooflines,
        "paths": paths,
        "e2e": e2e,
        "setup": setup,
        "tau_zero_l": zero_l,
        "gpu_launches": launches,
        "gpu_launch_detail": launch_detail,
        "clocks": clocks,
        "parity_vs_reference": parity,
        "parity_detail": getattr(parity_check, "detail", None) if batched else None,
        "zero_pivot_row": bad,
    }
    if multi:
        line["multi_gpu"] = multi
    if world == 1 and rank == 0 and not args.no_cpu:
        cb = cpu_baseline(args.config, plan, seconds=args.cpu_seconds, blocks=blocks)
        cp = cb["paths"]
        cp["factor"]["gpu_speedup_vs_threaded"] = (nnz_f / f_avg) / cb["value"]
        cp["stri"]["gpu_speedup_vs_threaded"] = cp["stri"]["threaded_ms"] / 1e3 / st_avg
        cp["spmv"]["gpu_speedup_vs_serial"] = cp["spmv"]["serial_ms"] / 1e3 / sp_avg
        line["cpu_baseline"] = cb
    if rank == 0:
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


def measure_tail(ilu, plan, K):
    """The two-stage path timed on its own, whatever the
    autotune picked for the step: upper rows, then the segmented tail
    stage 1 and the corner, CUDA events on the stream; bitwise check
    against the step's factor values."""
    import torch
    from paper_1812_06160_b200 import device as dv

    want = ilu.val.clone()
    n_upper = plan.n_upper
    tp = ilu.tail_plan(n_upper)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    up, s1, cr = [], [], []
    for k in range(K + 2):
        plan.reset_values()
        ev[0].record()
        ilu.factor_two_stage_async(n_upper, ev=ev[1:])
        torch.cuda.synchronize()
        if k >= 2:
            up.append(ev[0].elapsed_time(ev[1]) * 1e3)
            s1.append(ev[1].elapsed_time(ev[2]) * 1e3)
            cr.append(ev[2].elapsed_time(ev[3]) * 1e3)
    same = bool(torch.equal(ilu.val, want))
    dv.check_hang()
    return {"n_upper": n_upper, "tail_rows": tp.nt, "corner_entries": tp.nc,
            "stage1_updates": tp.nops, "stage1_groups": tp.ngroups, "stage1_segments": tp.nsegs,
            "upper_us": statistics.median(up), "stage1_us": statistics.median(s1),
            "corner_us": statistics.median(cr),
            "two_stage_us": statistics.median(up) + statistics.median(s1) + statistics.median(cr),
            "bitwise_equal_to_step": same}


def measure_e2e(a, plan, args):
    """factor_serial through the drop-in API: host values uploaded, factored,
    downloaded every call (structure and schedules cached on the object)."""
    import paper_1812_06160_b200 as jv
    from paper_1812_06160_b200 import device as dv
    from paper_1812_06160_b200.csr import SparsityPattern
    from paper_1812_06160_b200.symbolic import IluFactors

    ilu = plan.ilu
    n = ilu.n
    pat = SparsityPattern(n, dv.host_i64(ilu.row_start, n + 1), dv.host_i64(ilu.col, ilu.nnz))
    assembled = dv.host_f64(plan.assembled, ilu.nnz)
    f = IluFactors(n, pat, assembled.copy(), dv.host_i64(ilu.diag_pos, n),
                   jv.Permutation(dv.host_i64(plan.perm, n)), ilu.tau, ilu.milu)
    for _ in range(4):   # factor_serial times whole vs streamed transfers on its first four calls
        f.val[:] = assembled
        jv.factor_serial(f)
    ts = []
    for _ in range(max(3, min(args.steps, 10))):
        f.val[:] = assembled
        t0 = time.perf_counter()
        jv.factor_serial(f)
        ts.append(time.perf_counter() - t0)
    t = statistics.median(ts)
    # the reference's Krylov pattern (pipeline.py:300, krylov.py:200):
    # precond = lambda r: apply_preconditioner(factors, r), host vectors in
    # and out; the factors stay resident between calls (symbolic.py)
    precond = lambda r: jv.apply_preconditioner(f, r)  # noqa: E731
    r = np.random.default_rng(1).uniform(-1.0, 1.0, n)
    uploads = []
    real_upload = dv.upload_f64
    dv.upload_f64 = lambda dst, src: (uploads.append(src.size), real_upload(dst, src))[1]
    try:
        precond(r)
        uploads.clear()
        tp = []
        for _ in range(max(3, min(args.steps, 10))):
            t0 = time.perf_counter()
            precond(r)
            tp.append(time.perf_counter() - t0)
    finally:
        dv.upload_f64 = real_upload
    return {"value": ilu.nnz / t, "unit": "factor nnz/s",
            "h2d_bytes_per_step": 8 * ilu.nnz, "d2h_bytes_per_step": 8 * ilu.nnz,
            "api": "paper_1812_06160_b200.factor_serial(IluFactors with host numpy values)",
            "ms": t * 1e3,
            "precond_lambda": {"api": "lambda r: apply_preconditioner(factors, r), host r and z",
                               "ms_per_call": statistics.median(tp) * 1e3,
                               "h2d_bytes_per_call": 8 * n, "d2h_bytes_per_call": 8 * n,
                               "factor_value_uploads_in_timed_calls": len(uploads)}}


def load_profile(cfg):
    p = os.path.join(REPO, "profiles", "ncu_summary.json")
    if not os.path.exists(p):
        return None
    return json.load(open(p)).get(cfg)


def run_reference(args):
    """The reference's CPU algorithm (pinned C oracle, threaded p2p factor,
    all host threads) on the same config; rank 0 only."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle
    from paper_1812_06160_b200 import workloads as W
    from oracle import front_end

    if args.config == "c5":
        # one system of the batch per step (nnz/s is per nonzero, the
        # systems are independent): the bounded sample of the workload
        a, base, s = W.rmat(18, 0), None, W.CONFIGS["c5"]
    else:
        a, base, s = W.config_matrix(args.config)
    if base == "rcm":
        sym_rs, sym_col = oracle.symmetrize(a.n, a.row_start, a.col)
        base_perm = oracle.rcm(sym_rs, sym_col)
    elif base is None:
        base_perm = None
    else:
        base_perm = base.perm
    fe = front_end(a.n, a.row_start, a.col, a.val, base_perm=base_perm, k=s["k"], tau=s["tau"],
                   min_level_rows=s["min_level_rows"])
    rs, col, diag, val = fe["row_start"], fe["col"], fe["diag"], fe["val"]
    nnz_f = col.size
    cores = os.cpu_count() or 1
    v = np.empty_like(val)
    for _ in range(args.warmup):
        np.copyto(v, val)
        oracle.p2p(0, cores, rs, col, v, diag, s["tau"], inplace=True)
    ts = []
    for _ in range(args.steps):
        np.copyto(v, val)      # the refresh is not part of the factorization
        t0 = time.perf_counter()
        oracle.p2p(0, cores, rs, col, v, diag, s["tau"], inplace=True)
        ts.append(time.perf_counter() - t0)
    t = sum(ts) / len(ts)
    rate = nnz_f / t
    print(json.dumps({
        "impl": "reference",
        "metric": "ILU factor nnz/s, stri and spmv GB/s (fp64) vs HBM roofline; 1/2/4/8 GPU",
        "value": rate, "unit": "factor nnz/s", "n_gpus": int(os.environ.get("WORLD_SIZE", "1")),
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded generator, SURVEY.md §8d recipe)",
        "config": {"workload": f"{args.config}:{s['name']}", "n": a.n, "nnz_f": nnz_f},
        "cpu_baseline": {"value": rate, "unit": "factor nnz/s", "cores": cores, "kind": "port",
                         "cpu_model": cpu_model(),
                         "sample": (f"one R-MAT system of the c5 batch per step" if args.config == "c5"
                                    else f"full {args.config} factorization per step") +
                                   ", threaded p2p restatement of factor_p2p_kernel"},
        "e2e": {"value": rate, "unit": "factor nnz/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c2")
    ap.add_argument("--impl", default="mine", choices=["mine", "reference"])
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--rmat-count", type=int, default=64, help="c5 batch size")
    ap.add_argument("--batch-per-gpu", type=int, default=4,
                    help="R-MAT systems per GPU of the multi_gpu.batch measurement (0: off)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_mine(args)


if __name__ == "__main__":
    main()
