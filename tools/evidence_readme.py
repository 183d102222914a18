"""Turn one `tools/evidence.sh` run (gpurun_out/ev_*) into profiles/<round>/: copy the raw files,
summarise the ncu captures, refresh profiles/ncu_traffic.json and write README.md.
Usage: python tools/evidence_readme.py r01   (after bringing gpurun_out/ back from the box)."""
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EV = os.path.join(ROOT, "gpurun_out")
HBM = 8000.0


def last_json(path):
    return json.loads(open(path).read().strip().splitlines()[-1])


def ncu(args, out):
    with open(out, "w") as f:
        subprocess.run(["ncu", *args], stdout=f, stderr=subprocess.DEVNULL, check=True)


def summary_blocks(path):
    blocks, cur = [], None
    for line in open(path):
        if line.strip().startswith("Kernel Name"):
            cur = {"name": line.split(None, 2)[2].strip()}
            blocks.append(cur)
        elif cur is not None and line.strip() and not line.startswith("----"):
            parts = line.split()
            if len(parts) >= 2:
                try:
                    cur[parts[0]] = float(parts[1])
                    cur[parts[0] + "_unit"] = parts[2] if len(parts) > 2 else ""
                except ValueError:
                    pass
    return blocks


SURVEY_KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
               "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
               "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
               "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
               "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
               "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active"]


def write_survey_metrics(raw, out):
    """SURVEY 8(d)'s ncu metric list (DRAM bytes and throughput, L2 hit rate, fp64 pipe) per kernel."""
    import csv
    rows = list(csv.reader(open(raw)))
    h, units = rows[0], rows[1]
    keys = [k for k in SURVEY_KEYS if k in h]
    with open(out, "w") as f:
        f.write("# SURVEY 8(d) ncu metrics per kernel (ncu --set full --clock-control none; config 5 bench step: "
                "lattice build + 2 applies, then the cell-list build leg); source: tools/evidence.sh capture\n")
        f.write("kernel | " + " | ".join(f"{k} [{units[h.index(k)]}]" for k in keys) + "\n")
        for r in rows[2:]:
            f.write(r[h.index("Kernel Name")][:40] + " | " + " | ".join(r[h.index(k)] for k in keys) + "\n")


def main(rnd):
    dst = os.path.join(ROOT, "profiles", rnd)
    os.makedirs(dst, exist_ok=True)
    for a, b in [("ev_bench.json", "bench.json"), ("ev_bench_ref.json", "bench_reference.json"),
                 ("ev_build_inst_groups.csv", "build_inst_groups.csv"), ("ev_build_inst_bins.csv", "build_inst_bins.csv"),
                 ("ev_build_paths.jsonl", "build_paths.jsonl"), ("ev_build_trace.log", "build_trace.log"),
                 ("ev_cl_check.jsonl", "cl_check.jsonl"), ("ev_apply_mid.jsonl", "apply_mid.jsonl"),
                 ("ev_bench_dry2.json", "bench_dry_run_2shards.json"),
                 ("ev_bench_dry4_c3.json", "bench_dry_run_4shards_c3.json"),
                 ("ev_configs.jsonl", "configs.jsonl"), ("ev_clocks.csv", "clocks_during_bench.csv"),
                 ("ev_launches.csv", "launches.csv"), ("ev_pytest_gpu.log", "pytest_gpu.log"),
                 ("ev_smoke.log", "smoke.log")]:
        if os.path.exists(os.path.join(EV, a)):
            shutil.copy(os.path.join(EV, a), os.path.join(dst, b))
    rep = os.path.join(EV, "ev_prof.ncu-rep")
    raw = os.path.join(EV, "ev_prof_raw.csv")  # exported on the GPU box (the report itself is too large to bring back)
    if not os.path.exists(raw):
        raw = "/tmp/ev_raw.csv"
        ncu(["-i", rep, "--page", "raw", "--csv"], raw)
    with open(os.path.join(dst, "ncu_full_summary.txt"), "w") as f:
        subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_summary.py"), raw], stdout=f, check=True)
    write_survey_metrics(raw, os.path.join(dst, "survey_metrics.txt"))
    for k in ("k_spmv", "k_cl_fill", "k_cl_count", "k_lat_fill_exact"):
        src = os.path.join(EV, f"ev_src_{k}.csv")
        if not os.path.exists(src):
            src = f"/tmp/src_{k}.csv"
            ncu(["-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k", f"regex:{k}", "-c", "1"], src)
        with open(os.path.join(dst, f"{k}_source_hot.txt"), "w") as f:
            r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_source_hot.py"), src], stdout=f)
        if r.returncode != 0:
            os.remove(os.path.join(dst, f"{k}_source_hot.txt"))  # kernel not in this capture
    with open(os.path.join(dst, "sass_evidence.txt"), "w") as f:
        subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sass_evidence.py")], stdout=f, check=True)
    with open(os.path.join(dst, "launches_summary.txt"), "w") as f:
        subprocess.run([sys.executable, os.path.join(ROOT, "tools", "launch_summary.py"),
                        os.path.join(dst, "launches.csv")], stdout=f, check=True)

    blocks = summary_blocks(os.path.join(dst, "ncu_full_summary.txt"))
    empty = {"name": "(not captured)", "gpu__time_duration.sum": float("nan"), "dram__bytes_read.sum": float("nan"),
             "dram__bytes_write.sum": float("nan")}
    pick = lambda pat: next((b for b in blocks if pat in b["name"]), empty)  # noqa: E731
    sens, dens, fill, count = pick("k_spmv<1"), pick("k_spmv<0"), pick("k_cl_fill"), pick("k_cl_count")
    latfill = pick("k_lat_fill_exact")
    gb = 1e9
    traffic = {
        "source": f"ncu --set full --clock-control none, config 5 (profiles/{rnd}/ncu_full_summary.txt)",
        "k_spmv_sens_bytes_per_launch": (sens["dram__bytes_read.sum"] + sens["dram__bytes_write.sum"]) * gb,
    }
    for key, b in (("k_cl_count", count), ("k_cl_fill", fill), ("k_lat_fill_exact", latfill), ("k_spmv_sens", sens),
                   ("k_spmv_dens", dens)):
        traffic[key] = {"dram_read_bytes": b["dram__bytes_read.sum"] * gb,
                        "dram_write_bytes": b["dram__bytes_write.sum"] * gb,
                        "duration_ms_cold_serialised": b["gpu__time_duration.sum"]}
    json.dump(traffic, open(os.path.join(ROOT, "profiles", "ncu_traffic.json"), "w"), indent=1)

    d = last_json(os.path.join(dst, "bench.json"))
    ref = last_json(os.path.join(dst, "bench_reference.json"))
    rows = [json.loads(l) for l in open(os.path.join(dst, "configs.jsonl")) if l.strip()]
    ap, bd, cl, e2e = d["apply"], d["build"], d["clocks"], d["e2e"]
    peak = d["roofline"]["peak"]
    L = []
    w = L.append
    w(f"# Round {rnd[1:].lstrip('0')} evidence (B200, sm_100a)\n")
    w("All numbers from one `gpurun` call (`tools/evidence.sh`, summarised by `tools/evidence_readme.py`) "
      "on a fresh B200 with the committed code.\n")
    w(f"## bench.py ({d['config']['workload']}: nnz {d['config'].get('nnz', 0):,}; step = build + "
      f"{d['config'].get('applies_per_step', 20)} × (sensitivity + density))\n")
    w(f"* value **{d['value']:.0f} GB/s** (algorithmic bytes of the step / step time), {d['ms_per_step']:.1f} ms per step, "
      f"{d['gpu_launches']} libtopofilt launches in the timed region")
    w(f"* build ({bd.get('path', 'cell_list')} path) {bd['ms']:.2f} ms = {bd['nnz_per_s']:.3e} nnz/s = "
      f"**{100 * bd['frac_of_8tbs']:.1f}% of 8 TB/s**")
    if "build_cell_list" in d:
        bc = d["build_cell_list"]
        w(f"* the general cell-list build on the same input (`build_cell_list`, timed after the step loop): "
          f"{bc['ms']:.2f} ms = {bc['nnz_per_s']:.3e} nnz/s = {100 * bc['frac_of_8tbs']:.1f}% of 8 TB/s")
    w(f"* sensitivity apply {ap['sensitivity_us']:.0f} µs = {ap['sensitivity_gbs']:.0f} GB/s = "
      f"**{100 * ap['sensitivity_frac_of_8tbs']:.1f}% of 8 TB/s** ({100 * ap['sensitivity_gbs'] / peak:.1f}% of the measured "
      f"{peak:.0f} GB/s copy peak)")
    w(f"* density apply {ap['density_us']:.0f} µs = {ap['density_gbs']:.0f} GB/s = **{100 * ap['density_frac_of_8tbs']:.1f}% "
      f"of 8 TB/s**; {ap['iters_per_s']:.0f} iterations/s (both filters)")
    w(f"* clocks during the timed region: median {cl['sm_mhz']} MHz of {cl['sm_max_mhz']}, reasons {cl['reasons']} "
      "(nvidia-smi trace: `clocks_during_bench.csv`)")
    w(f"* e2e through the C-ABI host-buffer calls (pinned memory, PCIe copies in the timed region): "
      f"{e2e['value']:.0f} GB/s ({1e3 * e2e['seconds_per_step']:.0f} ms per step)")
    w(f"* cpu_baseline (oracle, {d['cpu_baseline']['cores']} core, sampled rows): {d['cpu_baseline']['value']:.2f} GB/s; "
      f"reference arm (`--impl reference`, same oracle): {ref['value']:.2f} GB/s")
    w(f"* roofline object: {json.dumps({k: d['roofline'][k] for k in ('kernel', 'bound', 'achieved', 'peak', 'frac', 'traffic')})}\n")
    w("## Launch list (`launches.csv`, ncu gpu__time_duration, cold/serialised; one step = build + 2 applies)\n")
    w("```")
    w(open(os.path.join(dst, "launches_summary.txt")).read().rstrip())
    w("```\n")
    w("## ncu --set full (`ncu_full_summary.txt`, `*_source_hot.txt`)\n")
    w("| kernel | duration (ncu) | DRAM read | DRAM write | issue active | DRAM % of peak |")
    w("|---|---|---|---|---|---|")
    for nm, b in (("k_spmv sensitivity", sens), ("k_spmv density", dens), ("k_lat_fill_exact (lattice build)", latfill),
                  ("k_cl_fill (cell-list build)", fill), ("k_cl_count (cell-list build)", count)):
        w(f"| {nm} | {b['gpu__time_duration.sum']:.3f} ms | {b['dram__bytes_read.sum']:.2f} GB | "
          f"{b['dram__bytes_write.sum']:.3f} GB | {b.get('smsp__issue_active.avg.pct_of_peak_sustained_active', 0):.0f}% | "
          f"{b.get('gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed', 0):.0f}% |")
    w("\nAlgorithmic bytes per apply launch: sensitivity 12.843 GB, density 12.747 GB (DESIGN.md §4.5). "
      "SASS evidence (`sass_evidence.txt`): `UBLKCP.S.G` (TMA bulk copies global->shared) + `SYNCS.*` (mbarriers) "
      "in the apply; `UBLKCP.G.S` (TMA bulk store shared->global of the weights) + `LDS.128`/`STG.E.128` in the "
      "lattice fill; `FADD2/FMUL2/FFMA2` (packed fp32x2) in the cell-list count/fill.\n")
    w("## All configs (`configs.jsonl`, `tools/bench_configs.py`)\n")
    w("| cfg | N | nnz | build path | build ms | build nnz/s | cell-list build ms | sens cold µs (% of 8 TB/s) | "
      "dens cold µs (% of 8 TB/s) |")
    w("|---|---|---|---|---|---|---|---|---|")
    for r in rows:
        if "config" in r:
            w(f"| {r['config']} | {r['n']:,} | {r['nnz']:,} | {r['stats'].get('path', '')} | {r['build_ms']:.3f} | "
              f"{r['build_nnz_per_s']:.2e} | {r.get('build_cell_list_ms', float('nan')):.3f} | "
              f"{r['sens_us_cold']:.1f} ({100 * r['sens_frac_8tbs_cold']:.1f}%) | "
              f"{r['dens_us_cold']:.1f} ({100 * r['dens_frac_8tbs_cold']:.1f}%) |")
    w("\nConfigs 1–2 are launch-bound (µs-scale applies).\n")
    st = [r for r in rows if "stencil_config" in r]
    if st:
        w("Matrix-free stencil (row a10), cold: " + "; ".join(
            f"config {r['stencil_config']}: sensitivity {r['sens_us_cold']:.1f} µs, density {r['dens_us_cold']:.1f} µs "
            f"(CSR-equivalent {r['sens_csr_equiv_gbs_cold']:.0f} GB/s)" for r in st) + ".\n")
    gr = [r for r in rows if "graph_config" in r]
    if gr:
        w("CUDA-graph replay of one iteration (sensitivity + density): " + "; ".join(
            f"config {r['graph_config']}: {r['iteration_us']:.1f} µs" for r in gr) + ".\n")
    oc = [r for r in rows if "oc_config" in r]
    if oc:
        w("OC update with bisection (NEXT-1): " + "; ".join(
            f"config {r['oc_config']} (N={r['n']:,}): {r['us']:.0f} µs for {r['iterations']} passes" for r in oc) + ".\n")
    hz = [r for r in rows if "helmholtz_config" in r]
    if hz:
        w("Helmholtz PDE filter (NEXT-3, sensitivity use, rtol 1e-12): " + "; ".join(
            f"config-{r['helmholtz_config']} mesh ({r['cells']:,} cells, {r['nodes']:,} nodes): build {r['build_ms']:.1f} ms, "
            f"solve {r['solve_us_cold']:.0f} µs cold, {r['iterations']} CG iterations "
            f"({100 * r['iteration_frac_8tbs']:.0f}% of 8 TB/s on 12 B/nnz + 112 B/node per iteration)" for r in hz) + ".\n")
    bo = [r for r in rows if "both_config" in r]
    if bo:
        w("Both filters in one pass over H (`tf_filter_both`, bitwise the separate calls), cold: " + "; ".join(
            f"config {r['both_config']}: {r['both_us_cold']:.0f} µs vs {r['separate_us_cold']:.0f} µs separate "
            f"({r['speedup']:.2f}×, {100 * r['both_frac_8tbs']:.0f}% of 8 TB/s on its own bytes)" for r in bo) + ".\n")
    la = [r for r in rows if "lattice_config" in r]
    if la:
        w("Matrix-free periodic lattice (`tf_build_lattice`), cold: " + "; ".join(
            f"config {r['lattice_config']} ({r['types']} cells per cube): sensitivity {r['sens_us_cold']:.0f} µs, "
            f"density {r['dens_us_cold']:.0f} µs vs stored CSR {r['csr_sens_us_cold']:.0f} / {r['csr_dens_us_cold']:.0f} µs "
            f"({r['sens_speedup']:.1f}× / {r['dens_speedup']:.1f}×)" for r in la) + ".\n")
    hrep = os.path.join(EV, "ev_hz.ncu-rep")
    if os.path.exists(hrep):
        ncu(["-i", hrep, "--page", "raw", "--csv"], "/tmp/ev_hz_raw.csv")
        with open(os.path.join(dst, "k_hz_apply_ncu_summary.txt"), "w") as f:
            subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_summary.py"), "/tmp/ev_hz_raw.csv"],
                           stdout=f, check=True)
        ncu(["-i", hrep, "--page", "source", "--csv", "--print-source", "cuda,sass"], "/tmp/ev_hz_src.csv")
        with open(os.path.join(dst, "k_hz_apply_source_hot.txt"), "w") as f:
            subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_source_hot.py"), "/tmp/ev_hz_src.csv"],
                           stdout=f, check=True)
        hb = summary_blocks(os.path.join(dst, "k_hz_apply_ncu_summary.txt"))[0]
        w(f"Helmholtz apply kernel under ncu (`k_hz_apply_ncu_summary.txt`): {hb['gpu__time_duration.sum']:.3f} ms, "
          f"DRAM {hb['dram__bytes_read.sum']:.2f} GB read + {hb['dram__bytes_write.sum']:.2f} GB written, "
          f"{hb.get('gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed', 0):.0f}% of DRAM peak.\n")
    mrep = os.path.join(EV, "ev_mf.ncu-rep")
    if os.path.exists(mrep):
        ncu(["-i", mrep, "--page", "raw", "--csv"], "/tmp/ev_mf_raw.csv")
        with open(os.path.join(dst, "matrix_free_ncu_summary.txt"), "w") as f:
            subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_summary.py"), "/tmp/ev_mf_raw.csv"],
                           stdout=f, check=True)
        mb = summary_blocks(os.path.join(dst, "matrix_free_ncu_summary.txt"))
        w("Matrix-free kernels under ncu (`matrix_free_ncu_summary.txt`, one sensitivity apply each): " + "; ".join(
            f"{b['name'].split('(')[0].split('::')[-1]}: {b['gpu__time_duration.sum']:.1f} "
            f"{b['gpu__time_duration.sum_unit']}, DRAM {b['dram__bytes_read.sum']:.1f} "
            f"{b['dram__bytes_read.sum_unit']} read" for b in mb) + " (vs the stored-CSR k_spmv sensitivity above).\n")
    sp = os.path.join(EV, "ev_shard_probe.jsonl")
    if os.path.exists(sp):
        shutil.copy(sp, os.path.join(dst, "shard_probe.jsonl"))
        rows = [json.loads(l) for l in open(sp) if l.strip()]
        one = next(r for r in rows if r["world"] == 1)
        w("NEXT-4 slab sharding, projected (`shard_probe.jsonl`, `tools/shard_probe.py`; config 5, the middle "
          "rank's owned-row applies measured on one B200, the halo exchange projected at 770 GB/s, not "
          f"overlapped): 1 GPU {one['sens_us'] + one['dens_us']:.0f} µs per iteration; " + "; ".join(
              f"{r['world']} ranks: {r['iteration_us_projected']:.0f} µs ({r['speedup_projected_vs_1gpu']:.2f}×; "
              f"halo {100 * r['halo_frac']:.0f}% of owned, {r['halo_mb_per_sens_apply']:.1f} MB per apply; "
              f"all local rows {r['sens_us_all_local_rows'] + r['dens_us_all_local_rows']:.0f} vs owned rows "
              f"{r['sens_us'] + r['dens_us']:.0f} µs)" for r in rows if r["world"] > 1) + ".\n")
    dp = os.path.join(EV, "ev_dense_probe.jsonl")
    if os.path.exists(dp):
        shutil.copy(dp, os.path.join(dst, "dense_probe.jsonl"))
    dp = os.path.join(dst, "dense_probe.jsonl")
    if os.path.exists(dp):
        drows = [json.loads(l) for l in open(dp) if l.strip().startswith("{")]
        w("Ablation, the paper's all-pairs build on the same GPU (`dense_probe.jsonl`, `tools/dense_probe.py`; "
          "`TF_BUILD_DENSE`: every pair visited as the paper's distance matrix does, exact fp64 pair tests, "
          "no N x N storage) against the cell list: " + "; ".join(
              f"{r['input']} (n = {r['n']:,}): {r['dense_ms']:.2f} ms vs {r['cell_list_ms']:.2f} ms "
              f"({r['speedup_cell_list']:.0f}x; the fp64 distance matrix would take {r['edm_bytes_fp64'] / 1e9:.1f} GB)"
              for r in drows) + ".\n")
    probe = os.path.join(EV, "ev_helm_probe.log")
    if os.path.exists(probe):
        shutil.copy(probe, os.path.join(dst, "helm_probe.log"))
    open(os.path.join(dst, "README.md"), "w").write("\n".join(L) + "\n")
    print(f"wrote profiles/{rnd}/README.md")


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "r01")
