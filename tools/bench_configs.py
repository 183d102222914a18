#!/usr/bin/env python3
"""Per-config measurements (BASELINE.json: "report ... on the seeded synthetic centroid
sets"): build nnz/s and GB/s, sensitivity / density apply GB/s and iterations/s, each as a
fraction of the 8 TB/s HBM roofline, for configs 1-5 on one B200.

Timing: CUDA events on the launching stream, warm-up first, median of the repetitions.
"hot" = back-to-back repetitions (small configs stay L2-resident); "cold" = a 512 MB buffer
is written between repetitions to flush the 126 MB L2. Writes JSON to stdout.
"""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import synth  # noqa: E402
import paper_2012_08208_b200 as tf  # noqa: E402

HBM = 8000.0


def timed(fn, reps, flush=None, stream=None):
    s = stream or torch.cuda.current_stream()
    out = []
    for _ in range(reps):
        if flush is not None:
            flush.add_(1.0)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        fn()
        b.record(s)
        torch.cuda.synchronize()
        out.append(a.elapsed_time(b) / 1e3)
    return statistics.median(out)


def main():
    dev = torch.device("cuda:0")
    flush = torch.zeros(64 * 1024 * 1024, dtype=torch.float64, device=dev)  # 512 MB
    res = []
    for cfg in (1, 2, 3, 4, 5):
        c, x, dc, rmin, meta = bench.load_workload(cfg)
        n, dim = c.shape
        cd, xd, dcd = (torch.from_numpy(a).to(dev) for a in (c, x, dc))
        out = torch.empty_like(xd)
        f = tf.tf_build_filter(cd, rmin)
        nnz = f.nnz
        f.close()
        reps_b = 5 if cfg < 5 else 3

        def build():
            g = tf.tf_build_filter(cd, rmin)
            g.close()

        t_build = timed(build, reps_b)

        def build_cl():
            g = tf.tf_build_filter(cd, rmin, path="cell_list")
            g.close()

        t_build_cl = timed(build_cl, reps_b)
        f = tf.tf_build_filter(cd, rmin)
        for _ in range(3):
            f.sensitivity(xd, dcd, out=out)
            f.density(xd, out=out)
        torch.cuda.synchronize()
        reps = 50 if cfg < 5 else 20
        row = {"config": cfg, "workload": meta["name"], "n": n, "nnz": nnz, "rmin": rmin,
               "build_ms": t_build * 1e3, "build_nnz_per_s": nnz / t_build,
               "build_gbs": bench.build_bytes(n, nnz, dim) / t_build / 1e9,
               "build_cell_list_ms": t_build_cl * 1e3,
               "build_cell_list_frac_8tbs": bench.build_bytes(n, nnz, dim) / t_build_cl / 1e9 / HBM}
        row["build_frac_8tbs"] = row["build_gbs"] / HBM
        for mode, fl in (("hot", None), ("cold", flush)):
            ts = timed(lambda: f.sensitivity(xd, dcd, out=out), reps, fl)
            td = timed(lambda: f.density(xd, out=out), reps, fl)
            row[f"sens_us_{mode}"] = ts * 1e6
            row[f"sens_gbs_{mode}"] = bench.sens_bytes(n, nnz) / ts / 1e9
            row[f"dens_us_{mode}"] = td * 1e6
            row[f"dens_gbs_{mode}"] = bench.dens_bytes(n, nnz) / td / 1e9
            row[f"sens_frac_8tbs_{mode}"] = row[f"sens_gbs_{mode}"] / HBM
            row[f"dens_frac_8tbs_{mode}"] = row[f"dens_gbs_{mode}"] / HBM
            row[f"iters_per_s_{mode}"] = 1.0 / (ts + td)
        row["stats"] = f.stats()
        f.close()
        res.append(row)
        print(json.dumps(row), flush=True)
        del cd, xd, dcd, out
        torch.cuda.empty_cache()


def stencil_rows():
    """Matrix-free stencil (row a10) on configs 1 and 3: own bytes (x, dc read, out written)
    and CSR-equivalent GB/s, labelled."""
    dev = torch.device("cuda:0")
    flush = torch.zeros(64 * 1024 * 1024, dtype=torch.float64, device=dev)
    for cfg, dims in ((1, (2, 60, 20, 1)), (3, (3, 160, 80, 80))):
        c, x, dc, rmin, meta = bench.load_workload(cfg)
        n = c.shape[0]
        xd, dcd = torch.from_numpy(x).to(dev), torch.from_numpy(dc).to(dev)
        out = torch.empty_like(xd)
        f = tf.tf_build_stencil(*dims, 1.0, rmin)
        for _ in range(3):
            f.sensitivity(xd, dcd, out=out)
        row = {"stencil_config": cfg, "n": n, "nnz_equiv": f.nnz}
        for mode, fl in (("hot", None), ("cold", flush)):
            ts = timed(lambda: f.sensitivity(xd, dcd, out=out), 50, fl)
            td = timed(lambda: f.density(xd, out=out), 50, fl)
            row[f"sens_us_{mode}"] = ts * 1e6
            row[f"sens_own_gbs_{mode}"] = 24 * n / ts / 1e9
            row[f"sens_csr_equiv_gbs_{mode}"] = bench.sens_bytes(n, f.nnz) / ts / 1e9
            row[f"dens_us_{mode}"] = td * 1e6
            row[f"dens_own_gbs_{mode}"] = 16 * n / td / 1e9
            row[f"dens_csr_equiv_gbs_{mode}"] = bench.dens_bytes(n, f.nnz) / td / 1e9
        print(json.dumps(row), flush=True)
        f.close()


def graph_rows():
    """Configs 1-3 with the applies captured in a CUDA graph (20 iterations of sensitivity +
    density per graph): removes the per-call host overhead that dominates the small configs."""
    dev = torch.device("cuda:0")
    for cfg in (1, 2, 3):
        c, x, dc, rmin, meta = bench.load_workload(cfg)
        n = c.shape[0]
        xd, dcd = torch.from_numpy(x).to(dev), torch.from_numpy(dc).to(dev)
        os_, od = torch.empty_like(xd), torch.empty_like(xd)
        f = tf.tf_build_filter(torch.from_numpy(c).to(dev), rmin)
        st = torch.cuda.Stream()
        st.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(st):
            f.sensitivity(xd, dcd, out=os_)
            f.density(xd, out=od)
        torch.cuda.current_stream().wait_stream(st)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        iters = 20
        with torch.cuda.graph(g):
            for _ in range(iters):
                f.sensitivity(xd, dcd, out=os_)
                f.density(xd, out=od)
        g.replay()
        torch.cuda.synchronize()
        t = timed(g.replay, 10) / iters
        print(json.dumps({"graph_config": cfg, "n": n, "nnz": f.nnz, "iteration_us": t * 1e6,
                          "iters_per_s": 1.0 / t,
                          "gbs": (bench.sens_bytes(n, f.nnz) + bench.dens_bytes(n, f.nnz)) / t / 1e9}), flush=True)
        f.close()


def oc_rows():
    """NEXT-1 OC update (30 bisection passes + final write) on configs 3 and 5."""
    dev = torch.device("cuda:0")
    for cfg in (3, 5):
        n = synth.centroids(cfg).shape[0] if cfg != 5 else 12_000_000
        x = synth.density(cfg, n)
        dcf = synth.sensitivity(cfg, x)
        xd, dd = torch.from_numpy(x).to(dev), torch.from_numpy(dcf).to(dev)
        xn = torch.empty_like(xd)
        for _ in range(2):
            tf.tf_oc_update(xd, dd, 0.5, x_new=xn)
        t = timed(lambda: tf.tf_oc_update(xd, dd, 0.5, x_new=xn), 10)
        it = 30
        bytes_ = it * 16 * n + 24 * n
        print(json.dumps({"oc_config": cfg, "n": n, "us": t * 1e6, "iterations": it,
                          "bytes_model": "30 x 16N (x, dc per pass) + 24N (final pass)",
                          "gbs": bytes_ / t / 1e9, "frac_8tbs": bytes_ / t / 1e9 / HBM}), flush=True)


def helmholtz_rows():
    """NEXT-3 Helmholtz filter (sensitivity use, rtol 1e-12) on the config-2 and config-5 meshes:
    build ms, solve us, CG iterations, and bytes per CG iteration (CSR 12 B/nnz + 8 B/row,
    vectors 104 B/node: z and p_old gathered once per node, p and q written; u, r, q, p, dinv
    read and u, r, z written in the update) against the 8 TB/s roofline."""
    dev = torch.device("cuda:0")
    flush = torch.zeros(64 * 1024 * 1024, dtype=torch.float64, device=dev)
    for cfg, (nodes, cells), rmin in ((2, synth.tri_mesh(300, 100, "right"), 2.5),
                                      (5, synth.kuhn_mesh(200, 100, 100), 1.5)):
        n = cells.shape[0]
        R = tf.helmholtz_radius(rmin)
        nd, cd = torch.from_numpy(nodes).to(dev), torch.from_numpy(cells).to(dev)
        x = torch.from_numpy(synth.density(cfg, n)).to(dev)
        dc = torch.from_numpy(synth.sensitivity(cfg, synth.density(cfg, n))).to(dev)
        tf.tf_helmholtz_build(nd, cd, R).close()
        holder = {}

        def build():
            holder["h"] = tf.tf_helmholtz_build(nd, cd, R)
        tb = timed(build, 3)
        h = holder["h"]
        out = torch.empty_like(x)
        info = h._info(dev)
        h.sensitivity(x, dc, out=out, info=info)
        t = timed(lambda: h.sensitivity(x, dc, out=out, info=info), 10, flush=flush)
        inf = h.decode_info(info)
        it = inf["iterations"]
        per_it = 12 * h.nnz + 8 * h.n_nodes + 104 * h.n_nodes
        print(json.dumps({"helmholtz_config": cfg, "cells": n, "nodes": h.n_nodes, "nnz": h.nnz, "R": R,
                          "build_ms": tb * 1e3, "solve_us_cold": t * 1e6, "iterations": it,
                          "rel_residual": inf["rel_residual"], "us_per_iteration": t * 1e6 / max(1, it),
                          "bytes_per_iteration": per_it,
                          "iteration_gbs": per_it * it / t / 1e9 if it else None,
                          "iteration_frac_8tbs": per_it * it / t / 1e9 / HBM if it else None}), flush=True)
        h.close()


def lattice_rows():
    """Matrix-free periodic lattice (tf_build_lattice) vs the stored CSR on configs 2 and 5
    (cold L2): the same filters without streaming H (x, dc, out only: 24 B/cell sensitivity)."""
    dev = torch.device("cuda:0")
    flush = torch.zeros(64 * 1024 * 1024, dtype=torch.float64, device=dev)
    for cfg, (nx, ny, nz, offs, dim) in ((2, (300, 100, 1, synth.tri_lattice_offsets("right"), 2)),
                                         (5, (200, 100, 100, synth.kuhn_lattice_offsets(), 3))):
        c, x, dc, rmin = synth.workload(cfg)
        xd, dd = torch.from_numpy(x).to(dev), torch.from_numpy(dc).to(dev)
        out = torch.empty_like(xd)
        f = tf.tf_build_lattice(dim, nx, ny, nz, 1.0, offs, rmin)
        f.sensitivity(xd, dd, out=out)
        ls = timed(lambda: f.sensitivity(xd, dd, out=out), 10, flush=flush)
        ld = timed(lambda: f.density(xd, out=out), 10, flush=flush)
        g = tf.tf_build_filter(torch.from_numpy(c).to(dev), rmin)
        g.sensitivity(xd, dd, out=out)
        cs = timed(lambda: g.sensitivity(xd, dd, out=out), 10, flush=flush)
        cd = timed(lambda: g.density(xd, out=out), 10, flush=flush)
        n = x.shape[0]
        print(json.dumps({"lattice_config": cfg, "n": n, "nnz_equiv": f.nnz, "types": int(offs.shape[0]),
                          "sens_us_cold": ls * 1e6, "dens_us_cold": ld * 1e6, "csr_sens_us_cold": cs * 1e6,
                          "csr_dens_us_cold": cd * 1e6, "sens_speedup": cs / ls, "dens_speedup": cd / ld,
                          "sens_own_gbs": 24 * n / ls / 1e9, "dens_own_gbs": 16 * n / ld / 1e9}), flush=True)
        f.close()
        g.close()


def both_rows():
    """tf_filter_both: both filters in one pass over H, against the two separate calls (cold L2).
    Algorithmic bytes: 12 nnz + 8(N+1) + 40N (CSR once; x, dc, Hs read; two outputs written)."""
    dev = torch.device("cuda:0")
    flush = torch.zeros(64 * 1024 * 1024, dtype=torch.float64, device=dev)
    for cfg in (3, 4, 5):
        c, x, dc, rmin = bench.load_workload(cfg)[:4]
        n = c.shape[0]
        f = tf.tf_build_filter(torch.from_numpy(c).to(dev), rmin)
        xd, dd = torch.from_numpy(x).to(dev), torch.from_numpy(dc).to(dev)
        so, do = torch.empty_like(xd), torch.empty_like(xd)
        f.both(xd, dd, so, do)
        tb = timed(lambda: f.both(xd, dd, so, do), 10, flush=flush)

        def sep():
            f.sensitivity(xd, dd, out=so)
            f.density(xd, out=do)
        ts = timed(sep, 10, flush=flush)
        byt = 12 * f.nnz + 8 * (n + 1) + 40 * n
        print(json.dumps({"both_config": cfg, "n": n, "nnz": f.nnz, "both_us_cold": tb * 1e6,
                          "separate_us_cold": ts * 1e6, "speedup": ts / tb, "both_gbs": byt / tb / 1e9,
                          "both_frac_8tbs": byt / tb / 1e9 / HBM, "iters_per_s": 1.0 / tb}), flush=True)
        f.close()


if __name__ == "__main__":
    if os.environ.get("LATTICE_ONLY"):
        lattice_rows()
        sys.exit(0)
    if os.environ.get("BOTH_ONLY"):
        both_rows()
        sys.exit(0)
    if os.environ.get("HELM_ONLY"):
        helmholtz_rows()
        sys.exit(0)
    if os.environ.get("OC_ONLY"):
        oc_rows()
        sys.exit(0)
    if os.environ.get("GRAPH_ONLY"):
        graph_rows()
        sys.exit(0)
    if not os.environ.get("STENCIL_ONLY"):
        main()
    stencil_rows()
    graph_rows()
    oc_rows()
    helmholtz_rows()
    both_rows()
    lattice_rows()
