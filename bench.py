"""Benchmark of the B200 implicit MPM Newton step (BASELINE.json metric:
implicit Newton steps/s and Jacobian nnz assembled/s).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl product|reference] [--config cfg4|cfg1]

A bench step is one implicit load step (MpmSim::step, mpm_solver.hpp:402-407:
binning + Newton-Krylov solve to tol 1e-10 + G2P) of the cfg 4 3D strip
footing (128x128x64 cells, 8,388,608 particles, fp64), the load ramped over 20
increments. value = Newton iterations / s (each iteration = Jacobian assembly
+ linear solve + line-search residual, mpm_solver.hpp:297-348) summed over all
ranks' slabs; with N ranks each owns one 8.39M-particle slab (weak scaling).
Inputs are resident in HBM for `value`; `e2e` goes through the C ABI with
host buffers (particle upload + step + particle download per step).
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)
PEAKS = os.path.join(REPO, "MEASURED_PEAKS.json")
REF_TOOL = os.path.join(REPO, "oracle", "_ref", "impm_ref")
METRIC = "implicit Newton steps/s"
UNIT = "Newton iterations/s (8.39M-particle 3D slabs)"
SLAB_PARTICLES = 8_388_608


def peaks():
    try:
        with open(PEAKS) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# --------------------------------------------------------------- clocks ---
class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region: one
    `nvidia-smi --query-gpu=... -lms 200` process started before and stopped
    after (the profiling recipe's clocks line), so sampling costs one NVML
    query per 200 ms instead of a process start per sample."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device=0):
        self.device = device
        self.rows = []
        self._p = None
        self._t = None

    def _read(self):
        try:
            for line in self._p.stdout:
                line = line.strip()
                if line:
                    self.rows.append([c.strip() for c in line.split(",")])
        except Exception:
            pass

    def __enter__(self):
        try:
            self._p = subprocess.Popen(["nvidia-smi", "-i", str(self.device), "--query-gpu=" + self.Q,
                                        "--format=csv,noheader,nounits", "-lms", "200"],
                                       stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
        except Exception:
            self._p = None
        return self

    def __exit__(self, *a):
        if self._p is not None:
            self._p.terminate()  # our own child process
            try:
                self._p.wait(timeout=5)
            except Exception:
                self._p.kill()
            if self._t is not None:
                self._t.join(timeout=5)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 5 + i and r[5 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


# ---------------------------------------------------------- CPU baseline ---
def sample_spec(path, cells=(12, 12, 6), steps=20):
    """cfg 4 scaled down for the CPU reference: same physical domain (64 x 64
    x 32 m), same material and loads, coarser grid (h = 64/12 m)."""
    h = 64.0 / cells[0]
    with open(path, "w") as f:
        f.write(f"""dim = 3
cells = {cells[0]},{cells[1]},{cells[2]}
h = {h}
ppc = 2
material = neo_hookean
E = 10e6
nu = 0.3
rho = 2000
bc = column
t_hat = 100e3
strip_fraction = 0.125
strip_axes = 1
steps = {steps}
tol = 1e-10
""")
    return int(np.prod(cells)) * 8


def run_reference_sample(budget_s, replicas=1):
    """Times the reference's own MpmSim::step (oracle/_ref, built from
    /root/reference/proj/src) on the scaled cfg 4 sample; `replicas`
    concurrent single-threaded processes. Returns (value in UNIT, info)."""
    if not os.path.exists(REF_TOOL):
        return None, {"error": "oracle/_ref/impm_ref not built"}
    with tempfile.TemporaryDirectory() as tmp:
        spec = os.path.join(tmp, "sample.spec")
        P = sample_spec(spec)
        procs = [subprocess.Popen([REF_TOOL, "bench", spec, str(budget_s)], stdout=subprocess.PIPE,
                                  stderr=subprocess.PIPE, text=True) for _ in range(replicas)]
        outs = [p.communicate(timeout=budget_s * 20 + 600) for p in procs]
    rates, infos = [], []
    for out, err in outs:
        line = [l for l in out.splitlines() if l.startswith("{")]
        if not line:
            return None, {"error": err.strip()[-300:]}
        info = json.loads(line[-1])
        infos.append(info)
        rates.append(info["newton_per_s"])
    # per-slab-equivalent: iterations/s x (sample particles / slab particles)
    value = sum(rates) * P / SLAB_PARTICLES
    nnz_rate = sum(i["nnz_per_s"] for i in infos)
    return value, {"particles": P, "newton_iterations": sum(i["newton_iterations"] for i in infos),
                   "step_seconds": max(i["step_seconds"] for i in infos), "replicas": replicas,
                   "nnz_per_s": nnz_rate, "newton_per_s_sample": sum(rates)}


# ------------------------------------------------------------- product ----
def make_sim(prob, device, profile, comm=None):
    """Single GPU: MpmSim on the whole problem. N > 1: this rank's SlabSim of
    the cfg 5 problem (axis-0 slab decomposition over NCCL)."""
    import paper_2507_09435_b200 as impm

    opts = prob.options
    opts.profile = profile
    if comm is None:
        sim = impm.MpmSim(prob.grid, prob.particles, prob.material, opts, device=device)
        sim.fixed[:] = prob.fixed
    else:
        from paper_2507_09435_b200.distributed import SlabSim

        sim = SlabSim(prob.grid, comm, prob.meta["cuts"], prob.particles, prob.meta["ids"], prob.material, opts,
                      device=device)
        sim.set_fixed_global(prob.fixed)
    sim.gravity = prob.gravity
    return sim


def ncu_traffic(name):
    """DRAM bytes (dram__bytes_read.sum + dram__bytes_write.sum) per launch of
    a kernel class from the committed ncu capture of the CURRENT kernels
    (profiles/r02/traffic.json, written by scripts/ncu_traffic.py), or None."""
    path = os.path.join(REPO, "profiles", "r02", "traffic.json")
    try:
        with open(path) as f:
            t = json.load(f)[name]
        return {"traffic_bytes": t["traffic_bytes"], "source": t.get("source", path)}
    except (OSError, KeyError, ValueError, TypeError):
        return None


def spmv_bytes(info, D):
    """algorithmic bytes of one compacted box-BSR SpMV launch: the stored
    (structurally nonzero) block values + their slot ids, per-row act_list and
    block count, x gathered once per active node, y written once."""
    rows = info["rows"]
    stored_values = info["row_values"]  # all rows, fp64
    return stored_values * 8 + stored_values // (D * D) + rows * (4 + 4 + D * 8 + D * 8 + D)


def fp64_peak():
    """DFMA peak (TFLOP/s): profiles/r02/fp64_peak.json (scripts/fp64_peak.cu
    on this pool's B200), else the nominal 37 TFLOP/s (148 SMs x 64 DFMA/clk x
    1.965 GHz x 2)."""
    path = os.path.join(REPO, "profiles", "r02", "fp64_peak.json")
    try:
        with open(path) as f:
            return float(json.load(f)["dfma_tflops"]), "measured (profiles/r02/fp64_peak.json)"
    except (OSError, KeyError, ValueError):
        return 37.2, "nominal"


def kernel_table(kt, rec, info, D, P, n_nodes, peak, symmetric_nh=True):
    """One row per kernel class of the profiled load step: CUDA-event time,
    launches, SURVEY.md 8(d) algorithmic bytes per launch, achieved GB/s and
    fraction of the measured HBM peak. K6 (tangent + assembly) counts as one
    launch per Jacobian: 184 B/particle of state reads + 8 B per
    reference-pattern nnz written (8(d) K6, ~1.31 kB/particle in 3D)."""
    total = sum(v[0] for k, v in kt.items() if k not in ("vcycle_level0", "vcycle_level1", "vcycle_coarse",
                                                          "galerkin", "mg_power", "mg_coarsest"))
    its = max(rec.iterations, 1)
    ref_nnz = rec.nnz_assembled / its  # per Jacobian
    n_jac = kt["assemble"][1]
    rows = []

    def row(name, kernel, ms, n, byt, model, key, flops=None):
        per = ms / n if n else None
        ach = byt / (per / 1e3) / 1e9 if (byt and per) else None
        tr = ncu_traffic(key) if key else None
        r = {"class": name, "kernel": kernel, "ms_total": ms, "launches": n, "ms_per_launch": per,
             "bytes_per_launch": byt, "bytes_model": model, "achieved_gbs": ach,
             "frac": ach / peak if ach else None, "share": ms / total if total else None, "traffic_key": key,
             "ncu_dram_bytes_per_launch": tr["traffic_bytes"] if tr else None}
        if flops and per:
            fpk, src = fp64_peak()
            r["fp64"] = {"flops_per_launch": flops, "achieved_tflops": flops / (per / 1e3) / 1e12,
                         "peak_tflops": fpk, "frac": flops / (per / 1e3) / 1e12 / fpk, "peak_source": src}
        rows.append(r)

    jm = kt["tangent"][0] + kt["assemble"][0]
    row("jacobian", ("K6 Jacobian: k_tangent_nh3q (factored closed-form tangent) + k_assemble_nh3f (bin per CTA, "
                     "block pair per thread, colour-batched BSR upper blocks) + k_zero_rows + k_mirror_lower + "
                     "k_diag_inverse") if symmetric_nh else
        ("K6 Jacobian: k_tangent (dual-number dP/dG) + k_assemble_bins_staged (colour-batched BSR, full blocks: "
         "nonsymmetric J) + k_diag_inverse"),
        jm, n_jac, (184 * P + 8 * ref_nnz) if n_jac else None,
        "SURVEY 8(d) K6: 184 B/particle state + 8 B x reference-pattern nnz",
        "jacobian" if symmetric_nh else None)  # ncu traffic of the neo-Hookean Jacobian only
    row("spmv", "k_spmv<double> (compacted box-BSR y = J x, outer Krylov)", kt["spmv"][0], kt["spmv"][1],
        spmv_bytes(info, D), "stored block values x 8 + slot ids + 33 B/row", "cg")
    nres = kt["residual_particles"][1]
    row("residual", "K5 residual: k_residual_bins_staged (+ per-particle pass)", kt["residual_particles"][0] +
        kt["residual_nodes"][0], nres, (184 * P + 16 * D * n_nodes) if nres else None,
        "SURVEY 8(d) K5: 184 B/particle + 16 F B/node", None)
    row("commit", "K9 G2P k_commit", kt["commit"][0], kt["commit"][1], 384 * P if kt["commit"][1] else None,
        "SURVEY 8(d) K9: 184 + 200 B/particle", "commit")
    # fine level of the V-cycle: two fp16 row-scaled sweeps (residual, Jacobi)
    # per V-cycle + zero-start smoothing, restriction, prolongation; the
    # profiler opens two level-0 scopes per V-cycle
    sv, rows_ = info["row_values"], info["rows"]
    vl0 = kt.get("vcycle_level0", (0.0, 0))
    row("vcycle_level0", "MG fine level: k_spmv<__half> residual + Jacobi sweeps, k_jacobi0, k_restrict, "
        "k_prolong_add", vl0[0], vl0[1], (2 * sv + sv // (D * D) + 250 * rows_) if vl0[1] else None,
        "per scope (half a V-cycle): fp16 values 2 B x stored + slot ids + ~250 B/row of vectors and Dinv",
        "vcycle_level0")
    row("vcycle", "MG V-cycle, all levels (fp16/fp32 level sweeps, restriction, prolongation, coarsest solve)",
        kt["vcycle"][0], kt["vcycle"][1], None, "-", None)
    row("mg_setup", "MG setup (Galerkin PtAP, power estimate)", kt["mg_setup"][0], kt["mg_setup"][1], None, "-",
        "gap")
    row("krylov_vector", "Krylov BLAS-1 (dots, axpys)", kt["krylov_vector"][0], kt["krylov_vector"][1], None,
        "-", None)
    return rows


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="product", choices=["product", "reference"])
    ap.add_argument("--config", default="cfg4", choices=["cfg4", "cfg1"])
    ap.add_argument("--material", default="neo_hookean",
                    choices=["neo_hookean", "cam_clay", "drucker_prager", "hencky_j2", "hencky"],
                    help="cfg4/cfg5 material: neo-Hookean (pinned substitute, default) or an unpinned extension")
    ap.add_argument("--e2e-steps", type=int, default=None, help="timed end-to-end load steps (default: --steps)")
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    if args.e2e_steps is None:
        args.e2e_steps = args.steps

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        if rank != 0:
            return
        nproc = os.cpu_count() or 1
        budget = max(10.0, 5.0 * (args.steps + args.warmup))
        value, info = run_reference_sample(budget, replicas=nproc)
        if value is None:
            print(json.dumps({"impl": "reference", "unavailable": info.get("error", "reference build missing")}))
            return
        sample = (f"cfg4 scaled to 12x12x6 cells ({info['particles']} particles), {info['replicas']} concurrent "
                  f"single-thread replicas of the reference MpmSim::step, {budget:.0f}s each; rate scaled by "
                  f"particle ratio to one 8.39M-particle slab (extrapolated; LU cost is superlinear, so this "
                  f"flatters the CPU)")
        out = {"metric": METRIC, "value": value, "unit": UNIT, "impl": "reference", "n_gpus": args.gpus,
               "steps": args.steps, "warmup": args.warmup, "ms_per_step": None, "higher_is_better": True,
               "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
               "config": {"workload": "cfg4 3D strip footing (neo-Hookean substitute for MCC)", "sample": sample},
               "cpu_baseline": {"value": value, "unit": UNIT, "cores": nproc, "kind": "reference", "sample": sample},
               "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
               "nnz_per_s": info["nnz_per_s"] * info["particles"] / SLAB_PARTICLES}
        print(json.dumps(out))
        return

    import torch

    dist = None
    if world > 1:
        import torch.distributed as dist

        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    device = local if world > 1 else 0
    torch.cuda.set_device(device)

    from paper_2507_09435_b200 import _abi, workloads

    # Load schedule: the reference ramps the load as k / steps and never
    # re-solves a load it has reached (scenarios.cpp:130-131). The bench runs
    # warmup + steps device load steps, one profiled step and (on a fresh sim)
    # warmup + e2e_steps end-to-end steps, so the ramp has at least that many
    # increments and every step advances the load.
    n_total = max(20, args.warmup + max(args.steps + 1, args.e2e_steps))

    comm = None
    if world > 1:
        # cfg 5: one cfg 4 slab per GPU, stacked along axis 0, one NCCL
        # communicator of the library (halos + dot partials on the sim stream)
        from paper_2507_09435_b200.distributed import Communicator

        def bcast(payload):
            box = [payload]
            dist.broadcast_object_list(box, src=0)
            return box[0]

        comm = Communicator.nccl(rank, world, device, broadcast=bcast)
        if args.config != "cfg4":
            raise SystemExit("multi-GPU runs use the cfg 5 slab workload (--config cfg4)")
        prob = workloads.footing3d_slab(world, rank, material=args.material, steps=n_total)
    elif args.config == "cfg4":
        prob = workloads.footing3d(material=args.material, steps=n_total)
    else:
        prob = workloads.column2d_nh(steps=n_total)
    D = prob.grid.dim
    sim = make_sim(prob, device, profile=False, comm=comm)
    stream = torch.cuda.current_stream(device)
    sim.set_stream(stream.cuda_stream)
    assert prob.load_steps == n_total

    def scale(k):
        if k > n_total:
            raise RuntimeError(f"load step {k} beyond the {n_total}-increment ramp")
        return k / n_total

    # warm-up load steps
    k = 0
    for _ in range(args.warmup):
        k += 1
        sim.step(scale(k))
    sim.kernel_times(reset=True)
    L = _abi.lib()
    launches0 = L.impm_launch_count()
    if dist:
        dist.barrier()
    torch.cuda.synchronize(device)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    recs = []
    with ClockSampler(device) as clocks:
        ev0.record(stream)
        for _ in range(args.steps):
            k += 1
            recs.append(sim.step(scale(k)))
        ev1.record(stream)
        torch.cuda.synchronize(device)
    if dist:
        dist.barrier()
    ms = ev0.elapsed_time(ev1)
    launches = L.impm_launch_count() - launches0
    # one more load step with per-kernel CUDA events (not in the timed region:
    # the events would perturb the headline number)
    opts = prob.options
    opts.profile = True
    sim.set_options(opts)
    sim.kernel_times(reset=True)
    k += 1
    prof_rec = sim.step(scale(k))
    torch.cuda.synchronize(device)
    kt = sim.kernel_times()
    info = sim.matrix_info()
    opts.profile = False
    sim.set_options(opts)
    its = sum(r.iterations for r in recs)
    kry = sum(r.krylov_iterations for r in recs)
    nnz = sum(r.nnz_assembled for r in recs)
    t = torch.tensor([ms], dtype=torch.float64, device=f"cuda:{device}")
    tot_its = torch.tensor([float(its)], dtype=torch.float64, device=f"cuda:{device}")
    if dist:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.all_reduce(tot_its, op=dist.ReduceOp.SUM)
    ms_max = float(t.item())
    value = float(tot_its.item()) / (ms_max / 1e3)

    # per-kernel table and the roofline of the dominant kernel, from the live
    # CUDA events of the profiled load step (events on the sim stream)
    peak, peak_kind = peaks()
    P = int(prob.particles.shape[0])
    table = kernel_table(kt, prof_rec, info, D, P, int(prob.grid.node_count()), peak,
                         symmetric_nh=prob.material.kind == "neo_hookean")
    dom = max((r for r in table if r["bytes_per_launch"]), key=lambda r: r["ms_total"])
    tr = ncu_traffic(dom["traffic_key"])
    asm_ms, _ = kt["assemble"]
    tan_ms, _ = kt["tangent"]
    nnz_rate = prof_rec.nnz_assembled / ((asm_ms + tan_ms) / 1e3) if asm_ms + tan_ms > 0 else None

    # end-to-end through the C ABI with host buffers
    e2e = None
    if args.e2e_steps > 0:
        # migration can grow a slab's particle count: headroom in the buffers
        rows = prob.particles.shape[0] if comm is None else int(prob.particles.shape[0] * 1.1) + 1024
        bufs = [torch.empty((rows, prob.particles.shape[1]), dtype=torch.float64, pin_memory=True).numpy()
                for _ in range(2)]
        bufs[0][: prob.particles.shape[0]] = prob.particles
        sim2 = make_sim(prob, device, profile=False, comm=comm)
        sim2.set_stream(stream.cuda_stream)
        e_its = 0
        st_ = {"i": 0, "n": prob.particles.shape[0], "ids": prob.meta.get("ids") if comm is not None else None,
               "h2d": 0, "d2h": 0}

        def upload():  # H2D of this step's inputs (pinned host AoS)
            h = bufs[st_["i"]][: st_["n"]]
            st_["h2d"] = h.nbytes
            if comm is None:
                sim2.set_particles(h)
            else:
                sim2.set_particles(h, st_["ids"])

        def download():  # D2H of the step's result (particle state) into the other buffer
            o = bufs[1 - st_["i"]]
            n = sim2.n_particles if comm is not None else st_["n"]
            if comm is None:
                sim2._h.call("impm_sim_get_particles", _abi.ptr(o), n, o.strides[0])
            else:
                ids_out = np.empty(n, dtype=np.int64)
                sim2._h.call("impm_sim_get_particles_ids", _abi.ptr(o), _abi.ptr(ids_out), n, o.strides[0])
                st_["ids"] = ids_out
            st_["d2h"] = n * o.strides[0]
            st_["n"] = n
            st_["i"] = 1 - st_["i"]

        # successive load steps with the particle state living in host memory
        # between steps (upload the last downloaded state, step the next
        # increment, download), after the same warm-up as the device leg: the
        # timed increments are the same ones
        ke = 0
        for _ in range(args.warmup):
            ke += 1
            upload()
            sim2.step(scale(ke))
            download()
        torch.cuda.synchronize(device)
        phase = {"upload": 0.0, "step": 0.0, "download": 0.0}
        t0 = time.perf_counter()
        for j in range(args.e2e_steps):
            ke += 1
            ta = time.perf_counter()
            upload()
            tb = time.perf_counter()
            e_its += sim2.step(scale(ke)).iterations
            tc = time.perf_counter()
            download()
            td = time.perf_counter()
            phase["upload"] += tb - ta
            phase["step"] += tc - tb
            phase["download"] += td - tc
        torch.cuda.synchronize(device)
        el = time.perf_counter() - t0
        e_t = torch.tensor([el], dtype=torch.float64, device=f"cuda:{device}")
        e_i = torch.tensor([float(e_its)], dtype=torch.float64, device=f"cuda:{device}")
        if dist:
            dist.all_reduce(e_t, op=dist.ReduceOp.MAX)
            dist.all_reduce(e_i, op=dist.ReduceOp.SUM)
        e2e = {"value": float(e_i.item()) / float(e_t.item()), "unit": UNIT,
               "h2d_bytes_per_step": int(st_["h2d"]), "d2h_bytes_per_step": int(st_["d2h"]),
               "newton_iterations": int(e_its), "seconds": float(e_t.item()),
               "phase_seconds": {k_: round(v_, 4) for k_, v_ in phase.items()},
               "note": "particle state round-trips through pinned host memory every load step"}
        del sim2

    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return

    cpu = None
    if not args.no_cpu and world == 1:
        v, cinfo = run_reference_sample(args.cpu_budget, replicas=1)
        if v is not None:
            cpu = {"value": v, "unit": UNIT, "cores": 1, "kind": "reference",
                   "sample": (f"reference MpmSim::step (oracle/_ref, built from /root/reference/proj/src, banded-LU "
                              f"substitute for Eigen SparseLU) on cfg4 scaled to 12x12x6 cells "
                              f"({cinfo['particles']} particles), {cinfo['newton_iterations']} Newton iterations in "
                              f"{cinfo['step_seconds']:.1f}s, 1 thread; scaled by particle ratio to one slab"),
                   "nnz_per_s_sample": cinfo["nnz_per_s"]}
        else:
            cpu = {"value": None, "unit": UNIT, "cores": 1, "kind": "reference", "sample": cinfo.get("error")}

    state_gb = prob.particles.nbytes / 1e9
    bsr_gb = info["rows"] * info["row_stride"] * 8 / 1e9 if "row_stride" in info else info["row_values"] * 8 / 1e9
    l2_note = (f"inputs larger than L2 (particle state {state_gb:.1f} GB, BSR {bsr_gb:.1f} GB per slab)"
               if state_gb + bsr_gb > 0.126 else
               f"inputs fit in L2 (particle state {1e3 * state_gb:.0f} MB, BSR {1e3 * bsr_gb:.0f} MB): "
               "a latency-bound configuration, reported as measured")
    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": prob.name, "note": prob.note, "particles_per_gpu": int(prob.particles.shape[0]),
                   "grid_nodes": int(prob.grid.node_count()), "active_rows": info["rows"],
                   "stored_blocks_per_row": info["row_values"] / max(info["rows"], 1) / D ** 2,
                   "free_dofs": int(sim.n_dofs()), "load_increments": n_total,
                   "parallelism": "1 slab per GPU" if world == 1 else
                   (f"{world} axis-0 slabs of one (128*{world})x128x64-cell problem (cfg 5): NCCL 2-plane halos, "
                    f"summed dot partials, rank-local MG (block Jacobi across slabs), particle migration"),
                   "l2": l2_note},
        "newton_iterations": its, "krylov_iterations": kry,
        "nnz_per_s": nnz_rate, "nnz_assembled": nnz,
        "roofline": {"bound": "hbm", "kernel": dom["kernel"], "achieved": dom["achieved_gbs"], "peak": peak,
                     "unit": "GB/s", "frac": dom["frac"], "traffic": tr["traffic_bytes"] if tr else None,
                     "traffic_source": (tr or {}).get("source"),
                     "bytes_per_launch": dom["bytes_per_launch"], "bytes_model": dom["bytes_model"],
                     "avg_launch_ms": dom["ms_per_launch"], "launches": dom["launches"],
                     "share_of_step": dom["share"], "peak_source": peak_kind,
                     "fp64": dom.get("fp64")},
        "kernels": table,
        "profiled_step": {"newton_iterations": prof_rec.iterations, "krylov_iterations": prof_rec.krylov_iterations,
                          "seconds": prof_rec.seconds},
        "kernel_ms": {k_: v_[0] for k_, v_ in kt.items()},
        "kernel_launches_by_class": {k_: v_[1] for k_, v_ in kt.items()},
        "gpu_launches": int(launches),
        "e2e": e2e,
        "cpu_baseline": cpu,
        "clocks": clocks.summary(),
    }
    print(json.dumps(out))
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
