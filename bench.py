#!/usr/bin/env python3
"""Benchmark of the filter hot path (BASELINE.json metric) -> ONE JSON line on rank 0.

A step = one pass of the whole hot path over the workload:
  tf_build_filter (the library's path choice: lattice-ordered centroids such as config 5 take
  the lattice build -- detect, verify, per-type tables, count, scan, fill with Hs; anything
  else the cell list -- bbox, keys, radix sort, cell start, count, scan, fill with Hs)
  + APPLIES x (tf_sensitivity_filter + tf_density_filter)
`build_cell_list` times the cell-list path on the same input after the timed region
(--build-path selects the path used inside the step).
on config 5 by default (12M Kuhn-tet centroids, rmin 1.5, 20 applies; BASELINE.json
configs[4] -- the configuration the north-star targets are quoted on), inputs resident in
HBM. value = algorithmic bytes of the step / step time (GB/s; bytes model SURVEY.md 8(d)).

Multi-GPU (`torchrun --nproc-per-node N bench.py --gpus N`): ONE problem (the same config)
sharded over the N ranks (NEXT-4, paper_2012_08208_b200/sharded.py): device slab plan, local build,
and every apply with an NCCL point-to-point halo exchange overlapped with the interior rows
(strong scaling); time = max over ranks; value = the whole problem's algorithmic bytes / that time.
`--dry-run --gpus N` runs the same sharded step with N shards as threads on one GPU (a loopback
transport instead of NCCL): a functional check of the multi-GPU path, not a measurement.

`--impl reference` times the CPU oracle (test infrastructure, oracle/) on a bounded
sample of the same workload instead (the reference arm of this tier).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

HBM_NOMINAL_GBS = 8000.0
METRIC = "filter build nnz/s and apply GB/s (fraction of 8 TB/s HBM) at 1 B200"


# ------------------------------------------------------------------ bytes model

def sens_bytes(n, nnz):
    return 12 * nnz + 8 * (n + 1) + 32 * n


def dens_bytes(n, nnz):
    return 12 * nnz + 8 * (n + 1) + 24 * n


def build_bytes(n, nnz, dim):
    return 8 * dim * n + 12 * nnz + 8 * (n + 1) + 8 * n


def step_bytes(n, nnz, dim, applies):
    return build_bytes(n, nnz, dim) + applies * (sens_bytes(n, nnz) + dens_bytes(n, nnz))


# ------------------------------------------------------------------ distributed plumbing

def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def init_dist(backend):
    """Process group for N > 1 (None at N = 1). NCCL: the rank's GPU (LOCAL_RANK) is made current
    and bound to the group first, so every collective (barriers included) runs on it."""
    import torch.distributed as dist
    ws, rank, local = dist_env()
    if ws > 1 and not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        kw = {}
        if backend == "nccl":
            import torch
            torch.cuda.set_device(local)
            kw["device_id"] = torch.device("cuda", local)
        dist.init_process_group(backend=backend, rank=rank, world_size=ws, **kw)
    return dist if ws > 1 else None


def reduce_max(value: float, dist=None, device=None) -> float:
    """Max over ranks (timing rule: the job is as slow as its slowest rank)."""
    if dist is None:
        return value
    import torch
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def aggregate(per_rank_units: float, world: int, max_seconds: float) -> float:
    """Whole-job throughput: units processed by all ranks / slowest rank's time."""
    return per_rank_units * world / max_seconds


# ------------------------------------------------------------------ clocks (NVML, sampled during timing)

class ClockSampler:
    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
        0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
        0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
    }

    def __init__(self, index=0, period=0.1):
        self.samples, self.reasons = [], 0
        self.period = period
        self._stop = threading.Event()
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # pragma: no cover - no NVML
            self.err = str(e)

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                self.reasons |= self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.ok:
            self.t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"]}
        names = [v for k, v in self.REASONS.items() if self.reasons & k and k != 0x1]
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz, "reasons": names,
                "samples": len(self.samples)}


def measured_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs: torch copy, read+write bytes)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md: 6.65 TB/s)"


def ncu_traffic():
    """Per-launch DRAM bytes of the dominant kernel from the committed ncu --set full summary."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        d = json.load(open(p))
        return d.get("k_spmv_sens_bytes_per_launch"), d.get("source")
    except Exception:
        return None, None


# ------------------------------------------------------------------ workload

def load_workload(cfg):
    c, x, dc, rmin = synth.workload(cfg)
    return c, x, dc, rmin, synth.CONFIGS[cfg]


# ------------------------------------------------------------------ CPU oracle baseline

def host_cpu():
    try:
        model = next(l.split(":", 1)[1].strip() for l in open("/proc/cpuinfo") if l.startswith("model name"))
    except Exception:
        model = "unknown CPU"
    return f"{model} ({os.cpu_count()} logical cores on the host)"


def oracle_sample(c, x, dc, rmin, applies, rows_per_step, steps, seed_cfg, threads=1):
    """Time the oracle (as it stands) on a bounded sample of the workload: the cell list over
    all N points (setup, charged pro rata), then for `rows_per_step` seeded rows: the row build
    (count + fill) and `applies` sensitivity + density applies. threads > 1 runs the same
    oracle calls on contiguous row chunks in host threads (ctypes releases the GIL; the oracle's
    row functions only read the cell list): SURVEY 8(d)'s multicore CPU baseline, no oracle
    change. Returns (GB/s of the sample's algorithmic bytes, per-step seconds list, description)."""
    import oracle
    from concurrent.futures import ThreadPoolExecutor
    n, dim = c.shape
    t0 = time.perf_counter()
    cl = oracle.CellList(c, rmin)
    t_setup = time.perf_counter() - t0
    all_rows = synth.sample_rows(seed_cfg, n, rows_per_step * steps)

    def work(rows):
        H = cl.rows(rows)
        for _ in range(applies):
            oracle.apply_sensitivity(H, x, dc)
            oracle.apply_density(H, x)
        return H.nnz

    vals, times = [], []
    with ThreadPoolExecutor(threads) as ex:
        # one untimed pass first (first-touch page faults of a fresh cell list / buffers)
        warm = np.sort(all_rows[:max(1, min(len(all_rows), rows_per_step // 4))])
        list(ex.map(work, [ch for ch in np.array_split(warm, threads) if ch.size]))
        for s in range(steps):
            rows = np.sort(all_rows[s * rows_per_step:(s + 1) * rows_per_step])
            chunks = [ch for ch in np.array_split(rows, threads) if ch.size]
            t0 = time.perf_counter()
            nnz = sum(ex.map(work, chunks))
            dt = time.perf_counter() - t0 + t_setup * len(rows) / n
            m = len(rows)
            b = (8 * dim * m + 12 * nnz + 8 * m + 8 * m) + applies * (
                (12 * nnz + 8 * m + 32 * m) + (12 * nnz + 8 * m + 24 * m))
            vals.append(b / dt / 1e9)
            times.append(dt)
    cl.close()
    how = "single-threaded" if threads == 1 else f"{threads} host threads over row chunks"
    desc = (f"{rows_per_step} seeded rows per step (stream S(c,5,0)) of the same workload: row build "
            f"+ {applies}x(sensitivity+density) on those rows; cell-list setup over all {n} points "
            f"({t_setup:.2f} s, single thread) charged pro rata; one untimed warm-up pass; C oracle "
            f"(-O2 -ffp-contract=off), {how}, "
            f"on {host_cpu()}")
    return statistics.median(vals), times, desc


# ------------------------------------------------------------------ GPU arm

def run_ours(args):
    import torch
    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    dist = init_dist("nccl")
    device = torch.device("cuda", local)
    import paper_2012_08208_b200 as tf

    c, x, dc, rmin, meta = load_workload(args.config)
    n, dim = c.shape
    applies = args.applies if args.applies is not None else meta["applies"]
    cd = torch.from_numpy(c).to(device)
    xd = torch.from_numpy(x).to(device)
    dcd = torch.from_numpy(dc).to(device)
    out_s = torch.empty_like(xd)
    out_d = torch.empty_like(xd)
    stream = torch.cuda.current_stream()

    ev = lambda: torch.cuda.Event(enable_timing=True)
    rec = {"build": [], "sens": [], "dens": []}

    def step(record):
        e0, e1 = ev(), ev()
        e0.record(stream)
        f = tf.tf_build_filter(cd, rmin, path=args.build_path)
        e1.record(stream)
        pairs = []
        for _ in range(applies):
            a, b, d = ev(), ev(), ev()
            a.record(stream)
            f.sensitivity(xd, dcd, out=out_s)
            b.record(stream)
            f.density(xd, out=out_d)
            d.record(stream)
            pairs.append((a, b, d))
        if record:
            rec["_pending"] = (e0, e1, pairs)
        return f

    # warm-up (untimed)
    nnz = None
    for _ in range(args.warmup):
        f = step(False)
        nnz = f.nnz
        f.close()
    torch.cuda.synchronize()

    # timed: K steps bracketed by barrier + synchronize; events on the launching stream
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    k0 = tf.kernel_launches()
    filters_launches = 0
    with ClockSampler(local) as clk:
        t_start, t_end = ev(), ev()
        t_start.record(stream)
        for _ in range(args.steps):
            f = step(True)
            nnz = f.nnz
            f.close()  # frees on the device (stream-ordered pool), inside the step
            e0, e1, pairs = rec.pop("_pending")
            rec.setdefault("_all", []).append((e0, e1, pairs))
        t_end.record(stream)
        torch.cuda.synchronize()
    launches = tf.kernel_launches() - k0
    if dist:
        dist.barrier()
    # the general (cell-list) build on the same input, outside the timed region
    fb = tf.tf_build_filter(cd, rmin)
    build_path = fb.stats()["path"]
    fb.close()
    t_cl = []
    for it in range(0 if args.no_build_cell_list else 4):
        e0, e1 = ev(), ev()
        e0.record(stream)
        fb = tf.tf_build_filter(cd, rmin, path="cell_list")
        e1.record(stream)
        torch.cuda.synchronize()
        fb.close()
        if it:
            t_cl.append(e0.elapsed_time(e1) / 1e3)
    elapsed = t_start.elapsed_time(t_end) / 1e3
    for e0, e1, pairs in rec["_all"]:
        rec["build"].append(e0.elapsed_time(e1) / 1e3)
        for a, b, d in pairs:
            rec["sens"].append(a.elapsed_time(b) / 1e3)
            rec["dens"].append(b.elapsed_time(d) / 1e3)
    t_max = reduce_max(elapsed, dist, device)

    sb = step_bytes(n, nnz, dim, applies)
    value = aggregate(sb * args.steps, ws, t_max) / 1e9
    t_sens = statistics.mean(rec["sens"])
    t_dens = statistics.mean(rec["dens"])
    t_build = statistics.mean(rec["build"])
    peak, peak_src = measured_peak()
    sens_gbs = sens_bytes(n, nnz) / t_sens / 1e9
    traffic, traffic_src = ncu_traffic()

    # self-check of what was timed (after the timed region): 1,000 seeded rows of a handle built
    # through the timed path and of the general cell-list handle, CSR bitwise and both filters
    # within 1e-10 of the oracle's row functions; a mismatch fails the run
    check = verify_rows(tf, c, x, dc, rmin, cd, xd, dcd, args, device) if (rank == 0 and not args.no_check) else None
    res = {}
    if not args.no_e2e:  # every rank (its own GPU and host buffers); max time over ranks
        res["e2e"] = run_e2e(tf, c, x, dc, rmin, applies, n, nnz, dim, args, dist, ws, device)
    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        v, times, desc = oracle_sample(c, x, dc, rmin, applies, args.cpu_rows, 1, args.config)
        cpu = {"value": v, "unit": "GB/s", "cores": 1, "kind": "oracle", "sample": desc,
               "seconds": times}
        th = max(1, min(os.cpu_count() or 1, 64))
        if th > 1:  # the same oracle loops over row chunks on all host cores
            vp, tp, dp = oracle_sample(c, x, dc, rmin, applies, args.cpu_rows, 1, args.config, th)
            cpu["parallel"] = {"value": vp, "unit": "GB/s", "cores": th, "kind": "oracle, row chunks in host threads",
                               "sample": dp, "seconds": tp}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_max / args.steps * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": meta["name"], "config_index": args.config, "n": n, "dim": dim,
                       "rmin": rmin, "nnz": nnz, "applies_per_step": applies,
                       "step": "build + applies x (sensitivity + density)",
                       "l2": "inputs larger than L2 (CSR %.1f GB >> 126 MB L2); no flush" % (12 * nnz / 1e9),
                       "parallelism": f"replicas{ws}"},
            "build": {"ms": t_build * 1e3, "nnz_per_s": nnz / t_build,
                      "gbs": build_bytes(n, nnz, dim) / t_build / 1e9,
                      "frac_of_8tbs": build_bytes(n, nnz, dim) / t_build / 1e9 / HBM_NOMINAL_GBS,
                      "path": build_path if args.build_path == "auto" else args.build_path},
            "build_cell_list": None if not t_cl else {
                "ms": statistics.mean(t_cl) * 1e3, "nnz_per_s": nnz / statistics.mean(t_cl),
                "gbs": build_bytes(n, nnz, dim) / statistics.mean(t_cl) / 1e9,
                "frac_of_8tbs": build_bytes(n, nnz, dim) / statistics.mean(t_cl) / 1e9 / HBM_NOMINAL_GBS,
                "note": "the general path (any centroids), same input, timed after the step loop"},
            "apply": {"sensitivity_us": t_sens * 1e6, "sensitivity_gbs": sens_gbs,
                      "sensitivity_frac_of_8tbs": sens_gbs / HBM_NOMINAL_GBS,
                      "density_us": t_dens * 1e6, "density_gbs": dens_bytes(n, nnz) / t_dens / 1e9,
                      "density_frac_of_8tbs": dens_bytes(n, nnz) / t_dens / 1e9 / HBM_NOMINAL_GBS,
                      "iters_per_s": 1.0 / (t_sens + t_dens)},
            "roofline": {"kernel": "k_spmv<sensitivity>", "bound": "hbm", "achieved": sens_gbs, "peak": peak,
                         "unit": "GB/s", "frac": sens_gbs / peak, "traffic": traffic,
                         "algorithmic_bytes_per_launch": sens_bytes(n, nnz), "peak_source": peak_src,
                         "traffic_source": traffic_src},
            "cpu_baseline": cpu,
            "gpu_launches": launches,
            "clocks": clk.summary(),
            "check": check,
        }
        line.update(res)
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


def verify_rows(tf, c, x, dc, rmin, cd, xd, dcd, args, device, count=1000):
    """Compare `count` seeded rows (stream S(cfg,5,0), synth.sample_rows) of the timed path's CSR
    and both filters -- and of the cell-list path's CSR -- with the oracle's cell-list row functions
    (test infrastructure, run here outside every timed region). Raises on any mismatch."""
    import torch

    import oracle
    n = c.shape[0]
    rows = np.sort(synth.sample_rows(args.config, n, count))
    ref = oracle.CellList(c, rmin).rows(rows)
    want_s = oracle.apply_sensitivity(ref, x, dc)
    want_d = oracle.apply_density(ref, x)
    rt = torch.from_numpy(rows).to(device)
    out = {"rows": int(rows.size), "stream": "synth.sample_rows(config, n, 1000)", "csr": "bitwise"}
    for label, path in (("timed", args.build_path), ("cell_list", "cell_list")):
        f = tf.tf_build_filter(cd, rmin, path=path)
        rowptr, cols, vals, hs = f.csr()
        starts = rowptr[rt]
        lens = rowptr[rt + 1] - starts
        total = int(lens.sum())
        seg0 = torch.repeat_interleave(torch.cumsum(lens, 0) - lens, lens)
        idx = torch.repeat_interleave(starts, lens) + (torch.arange(total, device=device) - seg0)
        rp = np.zeros(rows.size + 1, np.int64)
        rp[1:] = np.cumsum(lens.cpu().numpy())
        ok = (np.array_equal(rp, ref.rowptr) and np.array_equal(cols[idx].cpu().numpy(), ref.cols)
              and np.array_equal(vals[idx].cpu().numpy(), ref.vals))
        hs_rel = float(np.max(np.abs(hs[rt].cpu().numpy() - ref.hs) / np.abs(ref.hs)))
        s = f.sensitivity(xd, dcd)[rt].cpu().numpy()
        d = f.density(xd)[rt].cpu().numpy()
        rel = max(float(np.max(np.abs(s - want_s) / np.abs(want_s))), float(np.max(np.abs(d - want_d) / np.abs(want_d))))
        path_name = f.stats()["path"]
        f.close()
        if not ok or hs_rel > 1e-12 or rel > 1e-10:
            raise SystemExit(f"bench self-check FAILED ({label} path {path_name}): csr_equal={ok} "
                             f"hs_rel={hs_rel:.3e} out_rel={rel:.3e}")
        out[label] = {"path": path_name, "hs_max_rel": hs_rel, "outputs_max_rel": rel}
    return out


def run_sharded(args):
    """One problem over N shards (NEXT-4). A step = the device slab plan + local centroid gather +
    local build + APPLIES x (sensitivity + density), each apply with its halo exchange. Real run:
    one process per GPU under torchrun, NCCL transport. Dry run: N threads on one GPU, loopback."""
    import threading

    import torch
    import paper_2012_08208_b200 as tf
    from paper_2012_08208_b200 import sharded

    c, x, dc, rmin, meta = load_workload(args.config)
    n, dim = c.shape
    applies = args.applies if args.applies is not None else meta["applies"]
    if args.dry_run:
        world, dist = args.gpus, None
        hub = sharded.LoopbackTransport(world)
        ranks = list(range(world))
        device = torch.device("cuda", 0)
        torch.cuda.set_device(device)
    else:
        world, rank, local = dist_env()
        torch.cuda.set_device(local)
        dist = init_dist("nccl")
        ranks = [rank]
        device = torch.device("cuda", local)
    cd = torch.from_numpy(c).to(device)
    xg, dcg = torch.from_numpy(x).to(device), torch.from_numpy(dc).to(device)
    res = {}

    def body(k):
        stream = torch.cuda.Stream(device) if args.dry_run else torch.cuda.current_stream(device)
        transport = hub.endpoint(k) if args.dry_run else sharded.DistTransport()
        ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
        with torch.cuda.stream(stream):
            def step(record):
                e0, e1, e2 = ev(), ev(), ev()
                e0.record(stream)
                sf = sharded.ShardedFilter(cd, rmin, k, world, transport)
                e1.record(stream)
                ids = sf.plan.owned_ids.long()
                xo, dco = xg[ids], dcg[ids]
                for _ in range(applies):
                    sf.sensitivity(xo, dco)
                    sf.density(xo)
                e2.record(stream)
                info = (sf.plan.n_owned, sf.plan.n_interior, sf.plan.n_halo,
                        int(sf.filter.csr()[0][sf.plan.n_owned].item()) if sf.filter else 0)
                sf.close()
                return (e0, e1, e2), info
            for _ in range(args.warmup):
                step(False)
            torch.cuda.synchronize(device)
            if dist:
                dist.barrier()
            torch.cuda.synchronize(device)
            t0, t1 = ev(), ev()
            l0 = tf.kernel_launches()
            with ClockSampler(device.index if device.index is not None else 0) as clk:
                t0.record(stream)
                evs = []
                for _ in range(args.steps):
                    e, info = step(True)
                    evs.append(e)
                t1.record(stream)
                torch.cuda.synchronize(device)
            launches = tf.kernel_launches() - l0
        res[k] = dict(launches=launches, clocks=clk.summary(), elapsed=t0.elapsed_time(t1) / 1e3, build=[a.elapsed_time(b) / 1e3 for a, b, _ in evs],
                      apply=[b.elapsed_time(c_) / 1e3 / applies for _, b, c_ in evs], info=info)

    if args.dry_run:
        th = [threading.Thread(target=body, args=(k,)) for k in ranks]
        for t in th:
            t.start()
        for t in th:
            t.join()
    else:
        body(ranks[0])
    mine = [res[k] for k in ranks]
    t_max = max(r["elapsed"] for r in mine)
    t_max = reduce_max(t_max, dist, device)
    owned_nnz = sum(r["info"][3] for r in mine)
    halo = [r["info"][2] for r in mine]
    if dist:
        t = torch.tensor([float(owned_nnz)], dtype=torch.float64, device=device)
        dist.all_reduce(t)
        owned_nnz = int(t.item())
    nnz = owned_nnz  # the owned rows of all shards are the global rows
    b_build = max(statistics.mean(r["build"]) for r in mine)
    b_apply = max(statistics.mean(r["apply"]) for r in mine)
    value = step_bytes(n, nnz, dim, applies) * args.steps / t_max / 1e9
    rank0 = (args.dry_run or dist_env()[1] == 0)
    if rank0:
        line = {
            "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": 1 if args.dry_run else world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_max / args.steps * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": meta["name"], "config_index": args.config, "n": n, "dim": dim, "rmin": rmin,
                       "nnz": nnz, "applies_per_step": applies, "shards": world,
                       "step": "shard plan + local build + applies x (sensitivity + density), halo exchange per apply",
                       "l2": "inputs larger than L2 (CSR %.1f GB over all shards); no flush" % (12 * nnz / 1e9),
                       "parallelism": f"slabs{world}" + (" (dry run: threads on one GPU, loopback transport)"
                                                         if args.dry_run else " (NCCL point-to-point halo)")},
            "shard": {"plan_build_ms_max": b_build * 1e3, "iteration_ms_max": b_apply * 1e3,
                      "halo_points": halo if args.dry_run else None},
            "dry_run": bool(args.dry_run),
            "gpu_launches": mine[0]["launches"],
            "clocks": mine[0]["clocks"],
            "e2e": None,
            "e2e_note": "the host-buffer path (tf_build_filter_host / tf_filter_iteration_host) is single-GPU; "
                        "the sharded run keeps its inputs resident on every rank",
        }
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


def run_e2e(tf, c, x, dc, rmin, applies, n, nnz, dim, args, dist=None, ws=1, device=None):
    """Same step through the C ABI's host-buffer variants: H2D of centroids / x / dc from
    pinned memory and D2H of every filtered field inside the timed region. Under torchrun every
    rank runs it on its own GPU; each step is bracketed by a barrier and timed as the max over
    ranks, and the value is the whole-job aggregate (like `value`)."""
    import torch
    cp = torch.from_numpy(c).pin_memory().numpy()
    xp = torch.from_numpy(x).pin_memory().numpy()
    dcp = torch.from_numpy(dc).pin_memory().numpy()
    os_ = torch.empty(n, dtype=torch.float64).pin_memory().numpy()
    od = torch.empty(n, dtype=torch.float64).pin_memory().numpy()

    def step():
        f = tf.tf_build_filter_host(cp, rmin)
        for _ in range(applies):
            tf.tf_filter_iteration_host(f, xp, dcp, os_, od)  # x, dc up once; both results down
        f.close()

    step()  # warm-up
    torch.cuda.synchronize()
    ts = []
    for _ in range(args.e2e_steps):
        if dist is not None:
            dist.barrier()
        t0 = time.perf_counter()
        step()
        torch.cuda.synchronize()
        ts.append(reduce_max(time.perf_counter() - t0, dist, device))
    t = statistics.median(ts)
    h2d = 8 * dim * n + applies * (16 * n)
    d2h = applies * (8 * n + 8 * n)
    return {"value": aggregate(step_bytes(n, nnz, dim, applies), ws, t) / 1e9, "unit": "GB/s",
            "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "steps": args.e2e_steps, "seconds_per_step": t,
            "timer": "host wall clock around the blocking C-ABI *_host calls, max over ranks"}


# ------------------------------------------------------------------ reference arm (the oracle)

def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    c, x, dc, rmin, meta = load_workload(args.config)
    n, dim = c.shape
    applies = args.applies if args.applies is not None else meta["applies"]
    v, times, desc = oracle_sample(c, x, dc, rmin, applies, args.cpu_rows, args.warmup + args.steps, args.config)
    timed = times[args.warmup:]
    vals = v
    line = {
        "impl": "reference", "metric": METRIC, "value": vals, "unit": "GB/s", "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": statistics.mean(timed) * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": meta["name"], "config_index": args.config, "n": n, "dim": dim, "rmin": rmin,
                   "applies_per_step": applies, "step": "bounded sample, see cpu_baseline.sample",
                   "parallelism": "cpu single thread"},
        "cpu_baseline": {"value": vals, "unit": "GB/s", "cores": 1, "kind": "oracle", "sample": desc},
        "e2e": {"value": vals, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--applies", type=int, default=None)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-rows", type=int, default=200000)
    ap.add_argument("--build-path", choices=["auto", "cell_list", "lattice"], default="auto")
    ap.add_argument("--no-build-cell-list", action="store_true", help="skip the build_cell_list leg")
    ap.add_argument("--no-check", action="store_true", help="skip the post-run oracle row check (launch lists)")
    ap.add_argument("--dry-run", action="store_true",
                    help="with --gpus N > 1: the sharded path with N shards as threads on one GPU")
    args = ap.parse_args(argv)
    if args.warmup < 3 and args.impl == "ours":
        print("warning: timing rules need --warmup >= 3", file=sys.stderr)
    if args.impl == "reference":
        run_reference(args)
    elif args.gpus > 1 and (args.dry_run or dist_env()[0] > 1):
        run_sharded(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
