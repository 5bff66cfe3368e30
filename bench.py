#!/usr/bin/env python
"""FS-FEM hot-path benchmark (BASELINE.json metric) on B200.

One step = the whole hot path on one synthetic cantilever:
    fsfem_build_faces -> fsfem_assemble_csr (symbolic + numeric) -> fsfem_apply_bc
    -> fsfem_pcg_solve (Jacobi-PCG to ||r||/||f|| <= 1e-10)
with inputs resident in HBM.  `value` = faces pushed through the whole path per second
(N_f * steps / device time, max over ranks); the JSON line also carries the two throughputs
the metric names (numeric-assembly faces/s and PCG iterations/s), the SpMV roofline,
the end-to-end number through the C ABI with pinned host buffers, and the CPU oracle baseline.

Usage: python bench.py [--gpus N] [--steps K] [--warmup W] [--config 4] [--impl fsfem|reference]
Multi-GPU: python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from fsfem_inputs import CONFIGS, config_mesh  # noqa: E402

E_MOD, NU = 1.0e6, 0.3
METRIC = "FS-FEM faces assembled/s + PCG iterations/s at ~2M tets; % of HBM roofline"
SAMPLE_X_CELLS = 25  # CPU-oracle sample: the first 25 of cfg4's 200 x-cells (same spacing)


def workload_name(cfg: int) -> str:
    nx, ny, nz = CONFIGS[cfg]["grid"]
    extra = []
    if CONFIGS[cfg].get("jitter"):
        extra.append(f"jitter {CONFIGS[cfg]['jitter']}h")
    if CONFIGS[cfg].get("node_perm_seed") is not None:
        extra.append("random node/tet order")
    return (f"cfg{cfg}: cantilever 10x1x1, {nx}x{ny}x{nz} hexes x 6 Kuhn T4, E=1e6 nu=0.3, clamped x=0, "
            f"tip load P=-1" + (", " + ", ".join(extra) if extra else ""))


# ------------------------------------------------------------------ clocks during the timed region
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except (OSError, FileNotFoundError):
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
            self.t.join(timeout=2)

    def summary(self) -> dict:
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.lines:
            p = [x.strip() for x in line.split(",")]
            if len(p) < 9:
                continue
            try:
                sm.append(float(p[1]))
                mx = float(p[2])
            except ValueError:
                continue
            for n, v in zip(names, p[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ------------------------------------------------------------------ CPU oracle baseline
def oracle_sample(cfg: int, sample_iters: int = 20) -> dict:
    """Time the oracle (as it stands) on a slab of the workload and scale to the full config.

    Sample: cfg's first SAMPLE_X_CELLS x-cells at the same spacing.  Scaled per stage by
    N_t (faces), N_f (assembly), nnz (BCs, PCG per iteration); the PCG iteration count of the
    full problem is the oracle's own, recorded by scripts/oracle_full_solve.py."""
    from oracle import Oracle
    full = config_mesh(cfg)
    m = config_mesh(cfg, x_cells=SAMPLE_X_CELLS if cfg >= 3 else None)
    o = Oracle(m.xyz, m.tets)
    t0 = time.perf_counter()
    o.build_faces()
    t_faces = time.perf_counter() - t0
    t0 = time.perf_counter()
    _, rp, _, _ = o.assemble_fs(E_MOD, NU)
    t_asm = time.perf_counter() - t0
    nnz_s = int(rp[-1])
    t0 = time.perf_counter()
    o.apply_bc(m.dirichlet, m.loads, 0)
    t_bc = time.perf_counter() - t0
    t0 = time.perf_counter()
    _, rep = o.pcg(1e-30, sample_iters, allow_not_converged=True)
    t_pcg = time.perf_counter() - t0
    it_s = max(1, rep["iterations"])
    from fsfem_inputs import kuhn_counts
    c = kuhn_counts(*full.grid)
    cs = kuhn_counts(*m.grid)
    gold = os.path.join(ROOT, "tests", "golden", f"oracle_cfg{cfg}.json")
    iters_full = json.load(open(gold))["pcg"]["iterations"] if os.path.exists(gold) else None
    t_full = (t_faces * c["n_tets"] / cs["n_tets"] + t_asm * c["n_faces"] / cs["n_faces"]
              + t_bc * c["nnz_fs"] / nnz_s)
    t_iter_full = t_pcg / it_s * c["nnz_fs"] / nnz_s
    if iters_full is not None:
        t_full += iters_full * t_iter_full
    return dict(t_step_s=t_full, faces_per_s=c["n_faces"] / t_full if iters_full else None,
                assembly_faces_per_s=cs["n_faces"] / t_asm, pcg_it_per_s=1.0 / t_iter_full,
                iters_full=iters_full, wall_s=t_faces + t_asm + t_bc + t_pcg,
                sample=(f"oracle on a slab of cfg{cfg} ({m.grid[0]}x{m.grid[1]}x{m.grid[2]} hexes, {m.n_tets} tets, "
                        f"same spacing): faces + full assembly + BCs + {it_s} PCG iterations, scaled by N_t, N_f, "
                        f"nnz and the oracle's own full-size iteration count ({iters_full})"))


def cpu_cores() -> int:
    n = os.environ.get("OMP_NUM_THREADS")
    return int(n) if n else (os.cpu_count() or 1)


def cpu_info() -> dict:
    """CPU model, sockets, physical cores and logical CPUs of this host, read at run time."""
    model, phys, cores = None, set(), set()
    try:
        cur = {}
        for line in open("/proc/cpuinfo"):
            if ":" not in line:
                if cur:
                    phys.add(cur.get("physical id", "0"))
                    cores.add((cur.get("physical id", "0"), cur.get("core id", cur.get("processor"))))
                cur = {}
                continue
            k, v = [t.strip() for t in line.split(":", 1)]
            cur[k] = v
            if k == "model name" and model is None:
                model = v
        if cur:
            phys.add(cur.get("physical id", "0"))
            cores.add((cur.get("physical id", "0"), cur.get("core id", cur.get("processor"))))
    except OSError:
        pass
    return {"model": model, "sockets": len(phys) or None, "physical_cores": len(cores) or None,
            "logical_cpus": os.cpu_count()}


def oracle_sample_threads(cfg: int, threads: int) -> dict:
    """oracle_sample in a fresh process with OMP_NUM_THREADS=threads (the oracle's OpenMP loops
    read it at load time; results are identical for any thread count)."""
    env = dict(os.environ, OMP_NUM_THREADS=str(threads), OMP_PROC_BIND="close", OMP_PLACES="cores")
    code = (f"import json, sys; sys.path.insert(0, {ROOT!r}); import bench; "
            f"print(json.dumps(bench.oracle_sample({cfg})))")
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, check=True).stdout
    d = json.loads(out.strip().splitlines()[-1])
    d["threads"] = threads
    return d


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    for _ in range(args.warmup):
        oracle_sample(args.config, sample_iters=5)
    vals = []
    samples = []
    for _ in range(args.steps):
        s = oracle_sample(args.config)
        vals.append(s["t_step_s"])
        samples.append(s)
    t = float(np.mean(vals))
    wall = float(np.mean([x["wall_s"] for x in samples]))
    nf = config_faces(args.config)
    v = nf / t
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "faces/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": wall * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(args),
            "components": {"assembly_faces_per_s": samples[-1]["assembly_faces_per_s"],
                           "pcg_it_per_s": samples[-1]["pcg_it_per_s"], "pcg_iterations": samples[-1]["iters_full"]},
            "extrapolated": True,
            "extrapolated_ms_per_full_step": t * 1e3,
            "note": ("each step runs the oracle on a bounded slab of the workload; ms_per_step is that measured "
                     "wall time, value is the workload's faces divided by the full-step time extrapolated from "
                     "the slab phase by phase (extrapolated_ms_per_full_step; a full cfg4 oracle step takes minutes)"),
            "cpu": cpu_info(),
            "cpu_baseline": {"value": v, "unit": "faces/s", "cores": cpu_cores(), "kind": "oracle",
                             "sample": samples[-1]["sample"]},
            "e2e": {"value": v, "unit": "faces/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def workload_config(args) -> dict:
    """The workload description both arms print (the driver compares the two config objects):
    only what the arguments and the mesh's closed-form counts fix."""
    from fsfem_inputs import kuhn_counts
    c = kuhn_counts(*CONFIGS[args.config]["grid"])
    world = int(os.environ.get("WORLD_SIZE", "1"))
    nnz = c["nnz_fs"] if args.method == "fs" else c["nnz_fem"]
    return {"workload": workload_name(args.config), "n_nodes": c["n_nodes"], "n_tets": c["n_tets"],
            "n_faces": c["n_faces"], "nnz": nnz,
            "parallelism": f"row-block x{world} ({args.exchange})" if world > 1 else "single GPU",
            "l2": ("inputs larger than L2 (CSR values alone 8*nnz bytes > 126 MB)" if 8 * nnz > 126e6 else
                   "inputs smaller than L2: the operator stays L2-resident between iterations"),
            "bc": args.bc, "tol": args.tol, "deterministic_dots": bool(args.deterministic),
            "method": "FS-FEM" if args.method == "fs" else "FEM-T4 (comparison)"}


def config_faces(cfg: int) -> int:
    from fsfem_inputs import kuhn_counts
    return kuhn_counts(*CONFIGS[cfg]["grid"])["n_faces"]


def load_peaks() -> tuple[float, str]:
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        return float(json.load(open(p))["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


SPMV_KERNELS = {0: "k_spmv_small<true> (warp per node, PCG SpMV + p.q)",
                1: "k_spmv<true> (gather, PCG SpMV + p.q)",
                2: "k_spmv_df<true> (dataflow push, PCG SpMV + p.q)"}


def traffic_from_profile(cfg: int, kernel: int):
    """DRAM bytes per launch (dram__bytes_read.sum + dram__bytes_write.sum) of the kernel from
    the committed ncu capture (profiles/spmv_dram_traffic.json), or None."""
    p = os.path.join(ROOT, "profiles", "spmv_dram_traffic.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d.get(f"cfg{cfg}_kernel{kernel}")
    return None


def asm_traffic_from_profile(cfg: int, what: str = ""):
    """DRAM bytes of one numeric assembly (ncu dram__bytes_read.sum + dram__bytes_write.sum), or with
    what="fp64_pipe_pct" its FP64 pipe utilisation, from the committed capture
    (profiles/asm_dram_traffic.json), or None."""
    p = os.path.join(ROOT, "profiles", "asm_dram_traffic.json")
    if os.path.exists(p):
        return json.load(open(p)).get(f"cfg{cfg}" + (f"_{what}" if what else ""))
    return None


def run_gpu(args):
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        dist.init_process_group("nccl")
    torch.cuda.set_device(local)
    from paper_2001_08849_b200 import (FsFem, fsfem_apply_bc, fsfem_assemble_csr, fsfem_build_faces,
                                       fsfem_nccl_get_unique_id, fsfem_pcg_solve, load_library)
    load_library()
    m = config_mesh(args.config)
    stream = torch.cuda.current_stream()
    g = FsFem(device=local, stream=stream.cuda_stream)
    if world > 1:
        uid = [fsfem_nccl_get_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        g.comm_init(uid[0], rank, world)
        g.set_exchange(1 if args.exchange == "halo" else 0)
    if args.deterministic:
        g.set_deterministic(True)
    if args.method == "fem":
        g.set_method(1)  # FSFEM_METHOD_FEM_T4, for comparison runs only
    bc_mode = 1 if args.bc == "penalty" else 0
    dev = torch.device("cuda", local)
    xyz_d = torch.from_numpy(m.xyz).to(dev)
    tets_d = torch.from_numpy(m.tets).to(dev)
    dir_d = torch.from_numpy(m.dirichlet).to(dev)
    loads_d = torch.from_numpy(m.loads.reshape(-1).copy()).to(dev)
    u_d = torch.zeros(3 * m.n_nodes, dtype=torch.float64, device=dev)

    def step(xyz, tets, dirichlet, loads, u):
        nf, ni = fsfem_build_faces(g.ctx, xyz, tets)
        rb, nr, nnz = fsfem_assemble_csr(g.ctx, E_MOD, NU)
        fsfem_apply_bc(g.ctx, dirichlet, loads, bc_mode)
        rep = fsfem_pcg_solve(g.ctx, u, True, args.tol, 0)
        return nf, nnz, rep

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def timed(k, inputs):
        reps = []
        barrier()
        l0 = g.report()["kernel_launches"]
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        for _ in range(k):
            reps.append(step(*inputs))
        ev1.record(stream)
        barrier()
        ms = ev0.elapsed_time(ev1)
        launches = g.report()["kernel_launches"] - l0
        if world > 1:
            t = torch.tensor([ms], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms, reps, launches

    dev_inputs = (xyz_d, tets_d, dir_d, loads_d, u_d)
    for _ in range(args.warmup):
        step(*dev_inputs)
    with ClockSampler(local) as clk:
        ms, reps, launches = timed(args.steps, dev_inputs)
    nf, nnz, _ = reps[-1]
    value = nf * args.steps / (ms / 1e3)

    def agg(key):
        return float(np.mean([r[2][key] for r in reps]))

    t_num, t_pcg = agg("t_numeric_ms"), agg("t_pcg_ms")
    iters = agg("iterations")
    spmv_ms = sum(r[2]["t_spmv_ms"] for r in reps)
    spmv_n = sum(r[2]["spmv_launches"] for r in reps)
    spmv_dev_ms = sum(r[2]["t_spmv_dev_ms"] for r in reps)
    spmv_dev_n = sum(r[2]["spmv_dev_launches"] for r in reps)
    vals_local = torch.tensor([t_num, t_pcg, spmv_ms / max(spmv_n, 1), spmv_dev_ms / max(spmv_dev_n, 1)],
                              dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(vals_local, op=dist.ReduceOp.MAX)
    t_num, t_pcg, spmv_avg_ms, spmv_dev_avg_ms = [float(x) for x in vals_local.tolist()]

    # end to end through the C ABI with pinned host buffers (H2D of inputs, D2H of u per step)
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()  # noqa: E731
    host_inputs = (pin(m.xyz), pin(m.tets), pin(m.dirichlet), pin(m.loads.reshape(-1)),
                   torch.zeros(3 * m.n_nodes, dtype=torch.float64).pin_memory())
    e2e = None
    if not args.no_e2e:
        step(*host_inputs)
        ms_e2e, _, _ = timed(args.steps, host_inputs)
        e2e = {"value": nf * args.steps / (ms_e2e / 1e3), "unit": "faces/s",
               "h2d_bytes_per_step": int(m.xyz.nbytes + m.tets.nbytes + m.dirichlet.nbytes + m.loads.nbytes),
               "d2h_bytes_per_step": int(8 * 3 * m.n_nodes)}

    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return 0

    peak, peak_kind = load_peaks()
    last = reps[-1][2]
    # algorithmic bytes as the library counts them for its symmetric block storage
    spmv_bytes = int(last["spmv_bytes"])
    cluster_loop = int(last["pcg_loop"]) == 2
    kind = int(last["spmv_kernel"])
    if cluster_loop:
        # the whole recurrence is one launch of the cluster kernel: its bytes per iteration are the
        # SpMV's plus the vector traffic of S9 (88 B per dof beyond the SpMV's x read / y write)
        it_bytes = spmv_bytes + 88 * 3 * m.n_nodes
        achieved = it_bytes * iters / (t_pcg / 1e3) / 1e9
        roof = {"kernel": "k_pcg_cluster (whole PCG loop in one thread-block-cluster launch)", "bound": "hbm",
                "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak, "traffic": None,
                "algorithmic_bytes_per_iteration": it_bytes, "iterations_per_launch": iters,
                "avg_launch_ms": t_pcg, "peak_kind": peak_kind, "launches_per_step": 1,
                "share_of_step": t_pcg / (ms / args.steps),
                "timing": "CUDA events around the PCG loop of every timed step (fsfem_report.t_pcg_ms)",
                "note": "operator and vectors are L2-resident at this size; the HBM peak is an upper bound only"}
    achieved = spmv_bytes / (max(spmv_avg_ms, 1e-12) / 1e3) / 1e9
    roof_spmv = {"kernel": SPMV_KERNELS.get(kind, str(kind)), "bound": "hbm", "achieved": achieved, "peak": peak,
            "unit": "GB/s", "frac": achieved / peak, "traffic": traffic_from_profile(args.config, kind),
            "algorithmic_bytes_per_launch": spmv_bytes, "avg_launch_ms": spmv_avg_ms, "launches_timed": spmv_n,
            "peak_kind": peak_kind, "launches_per_step": iters + 1,
            "share_of_step": spmv_dev_ms / max(spmv_dev_n, 1) * (iters + 1) / (ms / args.steps),
            "timing": "CUDA events around the second SpMV of every 32-iteration CUDA-graph batch (after an update kernel, like every SpMV but the batch's first), live in the timed steps",
            "device_timer": {"avg_launch_ms": spmv_dev_avg_ms, "launches": spmv_dev_n,
                             "achieved": spmv_bytes / (max(spmv_dev_avg_ms, 1e-12) / 1e3) / 1e9,
                             "frac": spmv_bytes / (max(spmv_dev_avg_ms, 1e-12) / 1e3) / 1e9 / peak,
                             "how": "%globaltimer from CTA 0's start to the last CTA's end of EVERY PCG SpMV (fire-and-forget reductions)"},
            "full_csr_equivalent_bytes": 12 * nnz + 32 * 3 * m.n_nodes}
    if not cluster_loop:
        roof = roof_spmv
    asm_bytes = int(last["assembly_bytes"])
    asm_aux = int(last["assembly_aux_bytes"])
    survey_bytes = 24 * m.n_nodes + 16 * m.n_tets + 8 * nnz  # mesh + full CSR values
    roof_asm = {"kernel": "k_asm_tile<0> (numeric assembly S2-S4 + S6, tiles)", "bound": "hbm",
                "achieved": asm_bytes / (t_num / 1e3) / 1e9, "peak": peak, "unit": "GB/s",
                "frac": asm_bytes / (t_num / 1e3) / 1e9 / peak, "algorithmic_bytes_per_launch": asm_bytes,
                "aux_bytes_per_launch": asm_aux, "avg_launch_ms": t_num,
                "frac_survey_full_csr_bytes": survey_bytes / (t_num / 1e3) / 1e9 / peak,
                "traffic": asm_traffic_from_profile(args.config),
                "fp64_pipe_pct_ncu": asm_traffic_from_profile(args.config, "fp64_pipe_pct"),
                "timing": "CUDA events around the numeric assembly of every timed step (fsfem_report.t_numeric_ms)"}
    cfgd = workload_config(args)
    if world == 1 and (cfgd["n_faces"] != nf or cfgd["nnz"] != nnz):
        raise RuntimeError(f"mesh sizes differ from the closed form: faces {nf} vs {cfgd['n_faces']}, "
                           f"nnz {nnz} vs {cfgd['nnz']}")
    line = {"metric": METRIC, "value": value, "unit": "faces/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": cfgd,
            "pcg": ("Jacobi-PCG (standard recurrence, whole loop in one thread-block-cluster kernel)"
                    if cluster_loop else
                    "Jacobi-PCG (standard recurrence, host-polled CUDA-graph batches of 32 iterations)"),
            "components": {"assembly_faces_per_s": nf / (t_num / 1e3), "assembly_ms": t_num,
                           "assembly_hbm_frac": asm_bytes / (t_num / 1e3) / 1e9 / peak,
                           "pcg_it_per_s": iters / (t_pcg / 1e3), "pcg_iterations": iters, "pcg_ms": t_pcg,
                           "faces_ms": agg("t_faces_ms"), "symbolic_ms": agg("t_symbolic_ms"), "bc_ms": agg("t_bc_ms"),
                           "cold_faces_per_s": nf / ((agg("t_faces_ms") + agg("t_symbolic_ms") + t_num) / 1e3),
                           "true_rel_residual": reps[-1][2]["true_rel_residual"]},
            "roofline": roof, "roofline_assembly": roof_asm, "e2e": e2e, "gpu_launches": int(launches),
            "clocks": clk.summary()}
    if world == 1 and not args.no_cpu_baseline:
        allc = cpu_cores()
        s_all = oracle_sample_threads(args.config, allc)
        s_one = oracle_sample_threads(args.config, 1)
        line["cpu_baseline"] = {"value": s_all["faces_per_s"], "unit": "faces/s", "cores": allc, "kind": "oracle",
                                "sample": s_all["sample"] + " (extrapolated from the slab; the oracle's faces, "
                                "assembly and BCs are single-threaded, its SpMV/PCG loops use all threads)",
                                "assembly_faces_per_s": s_all["assembly_faces_per_s"],
                                "pcg_it_per_s": s_all["pcg_it_per_s"], "wall_s": s_all["wall_s"],
                                "one_thread": {"value": s_one["faces_per_s"], "pcg_it_per_s": s_one["pcg_it_per_s"],
                                               "assembly_faces_per_s": s_one["assembly_faces_per_s"],
                                               "wall_s": s_one["wall_s"]},
                                "cpu": cpu_info()}
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=4, choices=[1, 2, 3, 4, 5])
    ap.add_argument("--impl", default="fsfem", choices=["fsfem", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--exchange", default="allgather", choices=["allgather", "halo"],
                    help="multi-GPU exchange of the search direction (fsfem_set_exchange)")
    ap.add_argument("--bc", default="modify", choices=["modify", "penalty"],
                    help="Dirichlet treatment (fsfem_apply_bc mode; PAPER.md:243-245)")
    ap.add_argument("--tol", type=float, default=1e-10, help="PCG relative residual (north star: 1e-10)")
    ap.add_argument("--deterministic", action="store_true",
                    help="GPU-count-invariant dots (fsfem_set_deterministic)")
    ap.add_argument("--method", default="fs", choices=["fs", "fem"],
                    help="fs = FS-FEM (the product); fem = the FEM-T4 companion (comparison only)")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_gpu(args)


if __name__ == "__main__":
    sys.exit(main())
