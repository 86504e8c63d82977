"""Benchmark of the per-Newton linear-solve hot path on B200 (driver contract).

Workload (BASELINE.json config 5): stiff FEM box make_box_tets(68,68,68),
985,527 DOF, E = 1e8, x = 0 face pinned, first-Newton stable Neo-Hookean
matrix; right-hand side b = M dt^2 g (the first Newton step from rest). One *step* is
one Newton linear solve through the C-ABI with the triplet stream resident in
HBM: filter_pinned -> assembly (sort + reduce) -> MAS build (block_edges +
hierarchy + restriction + batched inversion) -> PCG to rel_tol 1e-4
(restart 250). Multi-GPU: one independent scene per rank (the cfg5 batch,
weak scaling), no data-path collective; NCCL only gathers per-scene stats and
the max-over-ranks timing.

  value        PCG iterations / s over the PCG loops (metric's first half)
  ms_per_step  one full Newton solve (assembly + MAS build + PCG)
  e2e          the same metric through the host-pointer C-ABI calls, per whole
               Newton solve (adipc_gpu_assemble_filtered / build_preconditioner / adipc_gpu_pcg with
               pinned host buffers; H2D of the stream and b, D2H of x inside)
  roofline     dominant PCG kernel, algorithmic bytes / CUDA-event time
  cpu_baseline the reference's own hot-path code compiled in place into
               oracle/_ref (kind "reference"; Eigen replaced by the subset in
               oracle/eigen_shim), else the oracle restatement (kind "port"),
               on all host cores

`--impl reference` times that CPU implementation alone, same metric/config:
`value` = its PCG-loop rate on a bounded sample of iterations; `e2e` = the
same unit as the GPU arm's e2e, PCG iterations per second of one whole Newton
linear solve (assembly + MAS build + PCG to rel_tol, ~340 iterations, timed
once; `--no-full-solve` skips it).
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

MEASURED = os.path.join(ROOT, "MEASURED_PEAKS.json")
REL_TOL, RESTART, MAX_ITERS, CAPACITY, MAX_LEVELS = 1e-4, 250, 100000, 16, 4
METRIC = "PCG iterations/sec + ms per Newton solve; HBM GB/s vs roofline; speedup vs host CPU"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-full-solve", action="store_true", help="reference arm: skip the whole-solve e2e timing")
    ap.add_argument("--config", default="cfg5_stiff_box")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cache", action="store_true", help="rebuild the MAS hierarchy every step")
    ap.add_argument("--no-solve-order", action="store_true",
                    help="run the MAS/PCG in the reference slot numbering (A/B of the solve-order renumbering)")
    ap.add_argument("--cpu-iters", type=int, default=10, help="PCG iterations per CPU sample step")
    ap.add_argument("--no-producer", action="store_true", help="skip the device element-Hessian producer timing")
    ap.add_argument("--no-hybrid", action="store_true",
                    help="skip the cfg4_hybrid_1m Newton-solve line (the north star's ~1M-DOF hybrid scene)")
    ap.add_argument("--no-geom", action="store_true",
                    help="skip the geometric hybrid Newton iteration (real contact: broad phase + producers on the device)")
    ap.add_argument("--selftest", action="store_true",
                    help="launcher / rendezvous / stats-gather self-test without GPU work (CPU tests, gloo)")
    return ap.parse_args()


def peaks():
    try:
        with open(MEASURED) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def gather_scene_stats(stats, world, dist):
    """Batch of independent scenes, one per rank (replicas):
    the only collective is an all-gather of each scene's stats; the job time
    is the max over ranks, the work (PCG iterations) the sum over ranks."""
    if dist is not None and world > 1:
        gathered = [None] * world
        dist.all_gather_object(gathered, stats)
    else:
        gathered = [stats]
    agg = {"max_total_ms": max(g["total_ms"] for g in gathered),
           "max_pcg_ms": max(g["pcg_ms"] for g in gathered),
           "iters": sum(g["iters"] for g in gathered),
           "converged": all(g.get("conv", True) for g in gathered)}
    return gathered, agg


def ncu_traffic():
    """DRAM bytes per launch by kernel class from the committed ncu capture."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            return json.load(f)["bytes_per_launch"]
    except Exception:
        return {}


# ----------------------------------------------------------------- clocks ---
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.samples = []
        self.sampler = None
        self._stop = threading.Event()
        self._t = None

    def _nvml(self):
        """NVML handle (nvidia-ml-py) for 20 ms sampling, or None: nvidia-smi
        then (one process per sample, ~0.3 s each)."""
        try:
            import pynvml as N
            N.nvmlInit()
            return N, N.nvmlDeviceGetHandleByIndex(self.index)
        except Exception:
            return None

    def _run(self):
        nv = self._nvml()
        self.sampler = "nvml" if nv else "nvidia-smi"
        bits = (0x8, 0x40, 0x20, 0x4)  # hw_slowdown, hw_thermal, sw_thermal, sw_power_cap (NVML event reasons)
        while not self._stop.is_set():
            try:
                if nv:
                    N, h = nv
                    get = getattr(N, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                        N.nvmlDeviceGetCurrentClocksThrottleReasons
                    r = get(h)
                    self.samples.append([str(N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM)),
                                         str(N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM))] +
                                        ["Active" if r & b else "Not Active" for b in bits])
                else:
                    out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                    f = [x.strip() for x in out.stdout.strip().split(",")]
                    if len(f) >= 6:
                        self.samples.append(f)
            except Exception:
                pass
            self._stop.wait(0.02 if nv else 0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=6)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if "Active" in s[2 + i]
                          and "Not" not in s[2 + i]})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples), "sampler": self.sampler}


# ------------------------------------------------------------- byte model ---
def byte_model(n, U, levels):
    """Algorithmic (compulsory) bytes per PCG iteration by kernel class
    (DESIGN.md 'byte model'): fp64 values, u32/i32 indices,
    explicit inverses as stored (symmetric-packed, (3f)(3f+1)/2 doubles)."""
    inv, nodes, parts = [], [], []
    for L in levels:
        fill = np.bincount(L["part_of"], minlength=L["n_parts"]).astype(np.int64)
        d = 3 * fill  # symmetric-packed inverses: d(d+1)/2 doubles, padded to even
        inv.append(int(np.sum(((d * (d + 1) // 2 + 1) // 2) * 2) * 8))
        nodes.append(int(L["n_nodes"]))
        parts.append(int(L["n_parts"]))
    nl = len(levels)
    nxt = lambda l: nodes[l + 1] if l + 1 < nl else 0  # noqa: E731
    vec = 24 * n
    spmv = 80 * U + vec + vec                      # A (72 B + 2 x u32 per block), p read, Ap written
    # update pass (solve order: unit-stride): x r/w, p, r r/w, Ap, r_1 write,
    # level-1 children lists + offsets, subdomain bounds
    update = 4 * n + 6 * vec + 24 * nxt(0) + 4 * (n + nxt(0) + parts[0])
    # preconditioner, every level in one launch: level 0 (D0^-1, r read, z write,
    # subdomain bounds) + each coarse level (D_l^-1, member list, r_l read, y_l
    # write, RED targets of the update pass)
    precond = inv[0] + 4 * n + 2 * vec + sum(
        inv[l] + 4 * nodes[l] + 48 * nodes[l] + 24 * nxt(l) + 4 * (nodes[l] + nxt(l) + parts[l])
        for l in range(1, nl))
    # z read, p r/w, Ap cleared, agg map + y_l gather per coarse level
    final = 4 * vec + sum(4 * n + 24 * nodes[l] for l in range(1, nl))
    return {"spmv": spmv, "update": update, "precond": precond, "final": final,
            "total": spmv + update + precond + final, "inv_bytes": inv}


# --------------------------------------------------------------- scenes ---
def make_problem(config, seed):
    """The rank's scene. cfg5: the batch of SURVEY.md §8d — rank r solves the
    scene of seed 5 + r (seed 5 unjittered, the others with a +-1e-3 h vertex
    jitter); other configs are the same scene on every rank."""
    import scenegen as scenes

    if config == "cfg5_stiff_box":
        return scenes.cfg5_batch_scene(seed)
    return scenes.CONFIGS[config]()


WORKLOADS = {
    "cfg5_stiff_box": "cfg5: stiff FEM box 68^3 cells, 985,527 DOF, E=1e8, PCG-only Newton solve, MAS cemas16 "
                      "(4 levels), rel_tol 1e-4, restart 250; batch of scenes seeds 5.. (one per GPU)",
}


def workload_config(args, sc, world):
    """The `config` object, identical in both arms (same keys, same values)."""
    return {"workload": WORKLOADS.get(args.config, args.config), "config": args.config,
            "n_block_rows": int(sc.n_blocks), "triplets": int(len(sc.keys)),
            "contact_node_blocks": int(len(sc.node_keys)),
            "l2": "inputs larger than L2 (A 203 MB + symmetric-packed MAS inverses 214 MB per scene, 126 MB L2)",
            "parallelism": f"{world} independent scenes (replicas of the single-GPU solve)",
            "seeds": list(range(5, 5 + world))}


def cpu_reference(sc, rank_seed, cpu_iters, steps, warmup, sample_note=True, full_solve=False):
    """The reference's CPU implementation of the path, all host threads:
    oracle/_ref (its own headers compiled in place, kind "reference") when
    present, else the oracle restatement (kind "port"). One-time assembly +
    MAS build, then timed steps of `cpu_iters` PCG iterations each (the
    bounded sample). full_solve: also one whole PCG solve to the bench's
    tolerance, so a whole Newton linear solve (assembly + MAS build + PCG —
    the unit of the GPU arm's e2e) is timed end to end."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle_py as O

    kind = "reference" if O.reference_available() else "port"
    with O.use_backend("reference" if kind == "reference" else "restated"):
        cores = O.lib().oracle_max_threads()
        par = O.ExecPolicy(deterministic=False, threads=cores)
        # filter_pinned is private to IncrementalPotential in the reference
        # (not exported by oracle/_ref): the restated filter runs untimed
        fk, fv = O.filter_pinned(sc.keys, sc.vals, sc.pinned)
        t0 = time.perf_counter()
        sk, sv = O.sort_stream(fk, fv, par)
        rows, cols, blocks = O.fast_hash_reduction(sk, sv, sc.n_blocks, par)
        t_asm = time.perf_counter() - t0
        # the level-0 partition by the reference's own partition_block_graph
        # (partition.hpp:88-159, in oracle/_ref) — untimed, once per scene
        part_of, n_parts = O.partition_block_graph(sc.n_blocks, sc.rest_edges, CAPACITY)
        t0 = time.perf_counter()
        A = O.Matrix(sc.n_blocks, rows, cols, blocks)
        H = O.Hierarchy(part_of, n_parts, CAPACITY, O.block_edges(rows, cols), MAX_LEVELS)
        M = O.MasPreconditioner(A, H)
        t_build = time.perf_counter() - t0
        import scenegen as S

        b = S.gravity_rhs(sc)
        times = []
        for s in range(warmup + steps):
            t0 = time.perf_counter()
            _, r = O.pcg_solve(A, b, M, 1e-30, RESTART, cpu_iters, par)
            dt = time.perf_counter() - t0
            if s >= warmup:
                times.append(dt)
        # the same loop sample on ONE host thread
        t0 = time.perf_counter()
        O.pcg_solve(A, b, M, 1e-30, RESTART, cpu_iters, O.ExecPolicy(deterministic=False, threads=1))
        it_s_1t = cpu_iters / (time.perf_counter() - t0)
        full = None
        if full_solve:
            t0 = time.perf_counter()
            _, rf = O.pcg_solve(A, b, M, REL_TOL, RESTART, MAX_ITERS, par)
            t_pcg = time.perf_counter() - t0
            full = {"iters": int(rf["iters"]), "pcg_s": t_pcg, "converged": bool(rf["converged"]),
                    "newton_solve_s": t_asm + t_build + t_pcg}
    it_s = cpu_iters / float(np.mean(times))
    what = ("oracle/_ref: the reference's own sparse/precond/solver headers compiled -O2 -fopenmp against "
            "oracle/eigen_shim" if kind == "reference" else "oracle restatement (oracle/oracle.hpp)")
    return {"value": it_s, "unit": "PCG iterations/s", "cores": cores, "kind": kind,
            "sample": f"{what}; {steps} steps x {cpu_iters} PCG iterations (MAS-preconditioned, cfg5 matrix) after "
                      f"a one-time assembly ({t_asm:.2f} s) and MAS build ({t_build:.2f} s); the reference's "
                      f"serial stages (radix sort, O scan, restriction, LLT, hierarchy, PCG vector ops) stay serial",
            "assembly_s": t_asm, "mas_build_s": t_build, "full_solve": full, "value_1_thread": it_s_1t}


# ------------------------------------------------------------ hybrid scene ---
HYBRID = "cfg4_hybrid_1m"


def hybrid_cpu(sc, cpu_iters, full_solve):
    """The reference's CPU path on the hybrid scene: two_level_abd_reduce of
    the contact node stream appended to the DOF stream
    (incremental_potential.hpp:322-394), filter_pinned, sort + reduce, the
    hierarchy + MAS build, then PCG (a bounded sample of `cpu_iters`
    iterations; full_solve: also the whole solve to rel_tol)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle_py as O
    import scenegen as S

    kind = "reference" if O.reference_available() else "port"
    with O.use_backend("reference" if kind == "reference" else "restated"):
        cores = O.lib().oracle_max_threads()
        par = O.ExecPolicy(deterministic=False, threads=cores)
        t0 = time.perf_counter()
        tk, tv = O.two_level_abd_reduce(sc.node_keys, sc.node_vals, sc.n_fem, sc.n_bodies, sc.abd_body, sc.jac36, par)
        t_two = time.perf_counter() - t0
        keys = np.concatenate([sc.keys, tk])
        vals = np.concatenate([sc.vals, tv])
        del tk, tv
        fk, fv = O.filter_pinned(keys, vals, sc.pinned)  # restated (private in the reference): untimed
        del keys, vals
        t0 = time.perf_counter()
        sk, sv = O.sort_stream(fk, fv, par)
        rows, cols, blocks = O.fast_hash_reduction(sk, sv, sc.n_blocks, par)
        t_asm = time.perf_counter() - t0 + t_two
        del sk, sv, fk, fv
        part_of, n_parts = O.partition_block_graph(sc.n_blocks, sc.rest_edges, CAPACITY)
        t0 = time.perf_counter()
        A = O.Matrix(sc.n_blocks, rows, cols, blocks)
        H = O.Hierarchy(part_of, n_parts, CAPACITY, O.block_edges(rows, cols), MAX_LEVELS)
        M = O.MasPreconditioner(A, H)
        t_build = time.perf_counter() - t0
        b = O.srbk_spmv(sc.n_blocks, rows, cols, blocks, S.ballistic_direction(sc), O.ExecPolicy(deterministic=True))
        t0 = time.perf_counter()
        _, r = O.pcg_solve(A, b, M, 1e-30, RESTART, cpu_iters, par)
        it_s = cpu_iters / (time.perf_counter() - t0)
        full = None
        if full_solve:
            t0 = time.perf_counter()
            _, rf = O.pcg_solve(A, b, M, REL_TOL, RESTART, MAX_ITERS, par)
            t_pcg = time.perf_counter() - t0
            full = {"iters": int(rf["iters"]), "pcg_s": t_pcg, "converged": bool(rf["converged"]),
                    "newton_solve_s": t_asm + t_build + t_pcg}
    return {"value": it_s, "unit": "PCG iterations/s", "cores": cores, "kind": kind,
            "sample": f"{'oracle/_ref (the reference headers)' if kind == 'reference' else 'oracle restatement'}; "
                      f"two-level reduction + sort/reduce ({t_asm:.2f} s), MAS build ({t_build:.2f} s), "
                      f"{cpu_iters} PCG iterations" + (", then the whole PCG solve" if full else ""),
            "assembly_s": t_asm, "two_level_s": t_two, "mas_build_s": t_build, "full_solve": full}


def hybrid_gpu(args, local_rank, with_cpu):
    """cfg4_hybrid_1m on this GPU: a step = one Newton linear solve of the
    hybrid scene through the C ABI with the DOF stream and the contact node
    stream resident in HBM: two_level_abd_reduce + append + filter + sort +
    reduce (adipc_gpu_assemble_contact_device), a COLD MAS build (no hierarchy
    reuse: contacts change the pattern every Newton iteration, and the
    reference rebuilds the hierarchy every iteration, newton.hpp:243-255),
    PCG to rel_tol on b = A x*, x* the free-fall step."""
    import torch

    from paper_2411_06224_b200 import _lib
    from paper_2411_06224_b200 import api as P
    from paper_2411_06224_b200.context import Context
    import scenegen as S

    dev = torch.device("cuda", local_rank)
    sc = make_problem(HYBRID, 4)
    stream = torch.cuda.Stream(dev)
    ctx = Context(local_rank, stream=stream)
    ctx.set_option(_lib.OPT_PROFILE, 0)
    ctx.set_option(_lib.OPT_CACHE_HIERARCHY, 0)
    l0 = P.partition_block_graph(sc.n_blocks, sc.rest_edges, CAPACITY)
    ctx.set_level0_partition(l0.part_of, l0.n_parts, CAPACITY, MAX_LEVELS)
    with torch.cuda.stream(stream):
        d = {k: torch.from_numpy(v).to(dev) for k, v in dict(
            keys=sc.keys.view(np.int64), vals=sc.vals, nk=sc.node_keys.view(np.int64), nv=sc.node_vals,
            body=sc.abd_body, jac=sc.jac36, pin=sc.pinned).items()}
    stream.synchronize()

    def assemble():
        return ctx.assemble_contact(d["keys"], d["vals"], d["nk"], d["nv"], sc.n_fem, sc.n_bodies, d["body"],
                                    d["jac"], sc.n_blocks, d["pin"])

    U, n_tiles = assemble()
    n, _ = ctx.matrix_info()
    xs = torch.from_numpy(S.ballistic_direction(sc)).to(dev)
    d_b = torch.empty_like(xs)
    d_x = torch.empty_like(xs)
    with torch.cuda.stream(stream):
        ctx.spmv(xs, d_b)
    stream.synchronize()

    def step():
        assemble()
        ctx.build_preconditioner(_lib.PRECOND_MAS)
        _, res = ctx.pcg(d_b, REL_TOL, RESTART, MAX_ITERS, x=d_x)
        return res, ctx.timings()

    for _ in range(args.warmup):
        step()
    levels = ctx.precond_levels()
    bm = byte_model(n, U, levels)
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    recs = []
    ev0.record(stream)
    for _ in range(args.steps):
        recs.append(step())
    ev1.record(stream)
    torch.cuda.synchronize()
    total_ms = ev0.elapsed_time(ev1)
    iters = sum(r.iters for r, _ in recs)
    t = {k: sum(tt[k] for _, tt in recs) / args.steps for k in recs[0][1]}
    err = float(torch.linalg.norm(d_x - xs) / torch.linalg.norm(xs))
    pcg_iter_s = t["pcg_ms"] / 1e3 / max(iters / args.steps, 1)
    # e2e: the same solve through the host-pointer C ABI (pinned buffers):
    # both streams cross PCIe every Newton iteration, x comes back
    import ctypes as C

    L = _lib.gpu()
    h = {k: v.cpu().pin_memory() for k, v in d.items()}
    h_b, h_x = d_b.cpu().pin_memory(), torch.empty(3 * n, dtype=torch.float64).pin_memory()
    Uo, nto, it, rr, cv = C.c_int64(), C.c_int64(), C.c_int(), C.c_double(), C.c_int()

    def e2e_step():
        ctx._check(L.adipc_gpu_assemble_contact(
            ctx.h, h["keys"].data_ptr(), h["vals"].data_ptr(), len(sc.keys), h["nk"].data_ptr(), h["nv"].data_ptr(),
            len(sc.node_keys), sc.n_fem, sc.n_bodies, len(sc.abd_body), h["body"].data_ptr(), h["jac"].data_ptr(),
            sc.n_blocks, h["pin"].data_ptr(), C.byref(Uo), C.byref(nto)))
        ctx._check(L.adipc_gpu_build_preconditioner(ctx.h, _lib.PRECOND_MAS))
        ctx._check(L.adipc_gpu_pcg(ctx.h, h_b.data_ptr(), REL_TOL, RESTART, MAX_ITERS, h_x.data_ptr(), C.byref(it),
                                   C.byref(rr), C.byref(cv)))
        return it.value

    e2e_step()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e_iters = sum(e2e_step() for _ in range(args.steps))
    e2e_ms = (time.perf_counter() - t0) * 1000.0 / args.steps
    h2d = sum(v.numel() * v.element_size() for v in h.values()) + h_b.numel() * 8
    out = {"config": HYBRID,
           "workload": "hybrid affine-deformable coupling at ~1M DOF: 8 FEM blocks 34^3 cells (E=1e8) + 40 ABD gears "
                       "(kappa 1e8), 105K contact stencils -> two_level_abd_reduce; cold MAS build every Newton "
                       "iteration; b = A x*, x* the free-fall step",
           "n_block_rows": int(sc.n_blocks), "dof": 3 * int(sc.n_blocks), "triplets": int(len(sc.keys)),
           "contact_node_blocks": int(len(sc.node_keys)), "contact_tiles": int(n_tiles), "U": int(U),
           "levels": [(int(L_["n_nodes"]), int(L_["n_parts"])) for L_ in levels],
           "ms_per_newton_solve": total_ms / args.steps,
           "assembly_ms": t["assemble_ms"], "mas_build_cold_ms": t["build_ms"],
           "mas_build_cold_host_ms": t["build_host_ms"], "pcg_ms": t["pcg_ms"],
           "pcg_iters_per_solve": iters / args.steps, "pcg_iters_per_s": iters / (t["pcg_ms"] * args.steps / 1e3),
           "converged": all(r.converged for r, _ in recs), "x_err_vs_xstar": err,
           "roofline_pcg_iteration": {"bound": "hbm", "bytes_per_iter": bm["total"],
                                      "achieved": bm["total"] / pcg_iter_s / 1e9, "peak": peaks()[0], "unit": "GB/s",
                                      "frac": bm["total"] / pcg_iter_s / 1e9 / peaks()[0],
                                      "iter_us": pcg_iter_s * 1e6},
           "e2e": {"ms_per_newton_solve": e2e_ms, "pcg_iters_per_solve": e_iters / args.steps,
                   "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(3 * n * 8),
                   "path": "adipc_gpu_assemble_contact + adipc_gpu_build_preconditioner + adipc_gpu_pcg "
                           "(host pointers, pinned)"}}
    ctx.close()
    if with_cpu:
        cb = hybrid_cpu(sc, args.cpu_iters, full_solve=False)
        # per Newton solve on the CPU: its own assembly + MAS build + the GPU's
        # iteration count at the sampled CPU iteration rate
        cpu_solve_s = cb["assembly_s"] + cb["mas_build_s"] + out["pcg_iters_per_solve"] / cb["value"]
        out["cpu_baseline"] = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample", "assembly_s",
                                                  "two_level_s", "mas_build_s")}
        out["cpu_baseline"]["ms_per_newton_solve_est"] = cpu_solve_s * 1e3
        out["speedup_newton_solve_vs_cpu"] = cpu_solve_s * 1e3 / out["ms_per_newton_solve"]
        out["speedup_e2e_newton_solve_vs_cpu"] = cpu_solve_s * 1e3 / e2e_ms
    return out


# ------------------------------------------------- geometric hybrid scene ---
GEOM = "geom_hybrid_1m"
GEOM_WORKLOAD = ("geometric hybrid at ~1M DOF: 2x2x2 FEM blocks 34^3 cells (E=1e8, 343,000 vertices, 1.89M tets) + "
                 "5x5 affine bodies (kappa 1e8) resting on them, every interface dhat/2 = 0.5 mm apart; one Newton "
                 "iteration from host state: contact-node positions, broad phase, contact + element + body "
                 "producers, gradient lift, two-level reduction + sort + reduce, cold MAS build, PCG on -grad")


def geom_cpu(full_solve=True):
    """The reference's CPU path for one Newton iteration of the geometric
    hybrid scene (IncrementalPotential::assemble composed from oracle/_ref's
    compiled reference pieces — element stencils, broad phase, contact
    stencils, two-level reduction, sort, reduction — then the hierarchy + MAS
    build and the whole PCG solve), all host threads."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle_py as O
    from scenegen.geom import GeomHybrid

    g = GeomHybrid()
    kind = "reference" if O.reference_available() else "port"
    with O.use_backend("reference" if kind == "reference" else "restated"):
        cores = O.lib().oracle_max_threads()
        par = O.ExecPolicy(deterministic=False, threads=cores)
        t0 = time.perf_counter()
        _, grad, rows, cols, blocks, cnt = O.ip_assemble(g, g.state(), par)
        t_asm = time.perf_counter() - t0
        part_of, n_parts = O.partition_block_graph(g.n_blocks, g.rest_edges, CAPACITY)
        t0 = time.perf_counter()
        A = O.Matrix(g.n_blocks, rows, cols, blocks)
        H = O.Hierarchy(part_of, n_parts, CAPACITY, O.block_edges(rows, cols), MAX_LEVELS)
        M = O.MasPreconditioner(A, H)
        t_build = time.perf_counter() - t0
        out = {"config": GEOM, "kind": kind, "cores": cores, "assembly_s": t_asm, "mas_build_s": t_build,
               "U": int(len(rows)), **{k: int(v) for k, v in cnt.items()}}
        if full_solve:
            t0 = time.perf_counter()
            _, r = O.pcg_solve(A, -grad, M, REL_TOL, RESTART, MAX_ITERS, par)
            out.update(pcg_s=time.perf_counter() - t0, iters=int(r["iters"]), converged=bool(r["converged"]))
            out["newton_iteration_s"] = t_asm + t_build + out["pcg_s"]
    out["sample"] = ("one Newton iteration: " + ("oracle/_ref (the reference's compiled code)" if kind == "reference"
                     else "oracle restatement") + "; assembly = element + body stencils with PSD projection, "
                     "broad phase, contact stencils, two-level reduction, sort, reduction")
    return out


def geom_gpu(args, local_rank):
    """geom_hybrid_1m on this GPU through the device IncrementalPotential
    (potential.py over the C ABI): a step = one Newton iteration's linear
    solve from the HOST state — H2D of [x; q], assemble (positions, broad
    phase, contact / element / body producers, lift, two-level + sort +
    reduce), a cold MAS build, PCG on -grad, D2H of the direction."""
    import torch

    from paper_2411_06224_b200 import _lib
    from paper_2411_06224_b200 import api as P
    from paper_2411_06224_b200.context import Context
    from paper_2411_06224_b200.potential import IncrementalPotential
    from scenegen.geom import GeomHybrid

    g = GeomHybrid()
    dev = torch.device("cuda", local_rank)
    stream = torch.cuda.Stream(dev)
    ctx = Context(local_rank, stream=stream)
    ctx.set_option(_lib.OPT_PROFILE, 0)
    ctx.set_option(_lib.OPT_CACHE_HIERARCHY, 0)
    l0 = P.partition_block_graph(g.n_blocks, g.rest_edges, CAPACITY)
    ctx.set_level0_partition(l0.part_of, l0.n_parts, CAPACITY, MAX_LEVELS)
    with torch.cuda.stream(stream):
        t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
        mesh = {"mass": t(g.mass), "tets": t(g.tets), "rest_inv9": t(g.rest_inv9), "rest_volume": t(g.rest_volume),
                "tet_begin": g.tet_begin, "mu": [g.mu], "lam": [g.lam],
                "bodies": {"reduced_mass": t(g.reduced_mass.transpose(0, 2, 1)), "kappa": t(g.kappa_abd),
                           "volume": t(g.body_volume)}}
        ip = IncrementalPotential(ctx, mesh, {"verts": t(g.surf_verts), "edges": t(g.edges), "tris": t(g.tris)},
                                  {"n_fem": g.n_fem, "abd_body": t(g.abd_body), "jac36": t(g.jac36)}, g.dt,
                                  pinned=t(g.pinned))
        ip.set_targets(t(g.x_tilde.reshape(-1)), t(g.q_tilde))
        ip.set_contact(g.dhat, g.kappa)
        d_state = torch.empty(3 * g.n_blocks, dtype=torch.float64, device=dev)
        d_dir, d_rhs, d_res = (torch.empty_like(d_state) for _ in range(3))
    stream.synchronize()
    h_state = torch.from_numpy(g.state()).pin_memory()
    h_dir = torch.empty(3 * g.n_blocks, dtype=torch.float64).pin_memory()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]

    def newton():
        with torch.cuda.stream(stream):
            ev[0].record(stream)
            d_state.copy_(h_state, non_blocking=True)
            _, grad = ip.assemble(d_state)
            ev[1].record(stream)
            ctx.build_preconditioner(_lib.PRECOND_MAS)
            ev[2].record(stream)
            torch.neg(grad, out=d_rhs)
            _, res = ctx.pcg(d_rhs, REL_TOL, RESTART, MAX_ITERS, x=d_dir)
            ev[3].record(stream)
            h_dir.copy_(d_dir, non_blocking=True)
            ev[4].record(stream)
        stream.synchronize()
        return res, [ev[i].elapsed_time(ev[i + 1]) for i in range(4)]

    for _ in range(args.warmup):
        newton()
    ip.profile = True  # one profiled iteration: the assemble phases
    newton()
    asm_phases = dict(ip.last["phase_ms"])
    ip.profile = False
    launches0 = Context.kernel_launches()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    recs = [newton() for _ in range(args.steps)]
    wall_ms = (time.perf_counter() - t0) * 1000.0 / args.steps
    launches = (Context.kernel_launches() - launches0) / args.steps
    ph = np.mean([r[1] for r in recs], axis=0)
    with torch.cuda.stream(stream):  # size-independent check: ||A d + grad|| / ||grad||
        ctx.spmv(d_dir, d_res)
        rel = float(torch.linalg.norm(d_res - d_rhs) / torch.linalg.norm(d_rhs))
    n, U = ctx.matrix_info()
    levels = ctx.precond_levels()
    out = {"config": GEOM, "workload": GEOM_WORKLOAD, "dof": 3 * int(g.n_blocks), "tets": int(len(g.tets)),
           "bodies": int(g.n_bodies), "surface": {"verts": int(len(g.surf_verts)), "edges": int(len(g.edges)),
                                                   "tris": int(len(g.tris))},
           "U": int(U), "candidates_pt": ip.last["n_pt"], "candidates_ee": ip.last["n_ee"],
           "contact_node_blocks": ip.last["node_blocks"], "contact_tiles": ip.last["contact_tiles"],
           "levels": [(int(L_["n_nodes"]), int(L_["n_parts"])) for L_ in levels],
           "ms_per_newton_iteration": wall_ms, "assemble_ms": float(ph[0]), "assemble_phases_ms": asm_phases,
           "mas_build_cold_ms": float(ph[1]),
           "pcg_ms": float(ph[2]), "d2h_ms": float(ph[3]),
           "pcg_iters": float(np.mean([r[0].iters for r in recs])),
           "converged": all(r[0].converged for r in recs), "true_rel_residual": rel,
           "gpu_launches_per_iteration": launches,
           "h2d_bytes_per_step": 3 * 8 * int(g.n_blocks), "d2h_bytes_per_step": 3 * 8 * int(g.n_blocks),
           "timing": "wall clock per step around H2D .. D2H with a stream sync (host-pointer e2e); phases by "
                     "CUDA events on the context stream"}
    ctx.close()
    return out


# -------------------------------------------------------------- main arm ---
def run_ours(args, rank, world, local_rank, dist):
    import torch

    from paper_2411_06224_b200 import _lib
    from paper_2411_06224_b200 import api as P
    from paper_2411_06224_b200.context import Context

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    sc = make_problem(args.config, 5 + rank)
    stream = torch.cuda.Stream(dev)
    ctx = Context(local_rank, stream=stream)
    ctx.set_option(_lib.OPT_PROFILE, 0)  # timed steps: graph-replayed iterations, no profiling events
    ctx.set_option(_lib.OPT_SOLVE_ORDER, 0 if args.no_solve_order else 1)
    l0 = P.partition_block_graph(sc.n_blocks, sc.rest_edges, CAPACITY)
    ctx.set_level0_partition(l0.part_of, l0.n_parts, CAPACITY, MAX_LEVELS)

    with torch.cuda.stream(stream):
        d_keys = torch.from_numpy(sc.keys.view(np.int64)).to(dev)
        d_vals = torch.from_numpy(sc.vals).to(dev)
        d_pin = torch.from_numpy(sc.pinned).to(dev)
    stream.synchronize()
    # filter_pinned + sort + reduce on the device-resident raw stream
    # (incremental_potential.hpp:255-257)
    ctx.assemble_filtered(d_keys, d_vals, sc.n_blocks, d_pin)
    n, U = ctx.matrix_info()
    # the first Newton step from rest: b = M dt^2 g, pinned slots zero
    import scenegen as S

    d_b = torch.from_numpy(S.gravity_rhs(sc)).to(dev)
    d_x = torch.empty(3 * n, dtype=torch.float64, device=dev)
    d_res = torch.empty(3 * n, dtype=torch.float64, device=dev)
    stream.synchronize()

    def step():
        ctx.assemble_filtered(d_keys, d_vals, sc.n_blocks, d_pin)
        ctx.build_preconditioner(_lib.PRECOND_MAS)
        _, res = ctx.pcg(d_b, REL_TOL, RESTART, MAX_ITERS, x=d_x)
        t = ctx.timings()
        prof = ctx.pcg_profile()
        return res, t, prof

    # first two warm-up steps: cold MAS builds (hierarchy from the pattern) —
    # the first one also pays the process's one-time allocations and module
    # loads, the second is a new-pattern rebuild in a running solver; later
    # steps reuse the hierarchy while the pattern hash is unchanged (it is a
    # pure function of the pattern), as a Newton loop without contact changes
    cold = first = None
    for i in range(args.warmup):
        _, t, _ = step()
        if i == 0:
            first = cold = t
        if i == 1:
            cold = t
        if i == 0 and not args.no_cache:
            ctx.set_option(_lib.OPT_CACHE_HIERARCHY, 1)
    levels = ctx.precond_levels()
    bm = byte_model(n, U, levels)

    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = Context.kernel_launches()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    recs = []
    with ClockSampler(local_rank) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            recs.append(step())
        ev1.record(stream)
        torch.cuda.synchronize()
    if dist:
        dist.barrier()
    launches = Context.kernel_launches() - launches0
    total_ms = ev0.elapsed_time(ev1)
    iters = sum(r.iters for r, _, _ in recs)
    pcg_ms = sum(t["pcg_ms"] for _, t, _ in recs)
    asm_ms = sum(t["assemble_ms"] for _, t, _ in recs)
    build_ms = sum(t["build_ms"] for _, t, _ in recs)
    build_host_ms = sum(t["build_host_ms"] for _, t, _ in recs)
    # kernel-class breakdown for the roofline: one more solve, same inputs, with
    # CUDA events bracketing every kernel class (direct launches, not graphs)
    ctx.set_option(_lib.OPT_PROFILE, 1)
    _, _, prof = step()
    ctx.set_option(_lib.OPT_PROFILE, 0)
    res_last = recs[-1][0]
    # size-independent check at full size: true residual of the returned x
    with torch.cuda.stream(stream):
        ctx.spmv(d_x, d_res)
    stream.synchronize()
    xerr = float(torch.linalg.norm(d_b - d_res) / torch.linalg.norm(d_b))
    # the step after the solve (newton.hpp:257-290, step.cu) on this direction:
    # step_inf_norm + apply_direction through the C ABI (host-visible latency)
    d_state = torch.zeros_like(d_x)
    stream.synchronize()
    t_ps = time.perf_counter()
    for _ in range(10):
        ctx.step_inf_norm(d_x, n, 0)
        ctx.apply_direction(d_state, d_x, 1.0, d_res)
    post_solve_us = (time.perf_counter() - t_ps) / 10 * 1e6

    stats = dict(total_ms=total_ms, pcg_ms=pcg_ms, iters=iters, asm_ms=asm_ms, build_ms=build_ms,
                 launches=launches, conv=bool(res_last.converged), rel=float(res_last.rel_residual), xerr=xerr)
    gathered, agg = gather_scene_stats(stats, world, dist)
    max_total, max_pcg, all_iters = agg["max_total_ms"], agg["max_pcg_ms"], agg["iters"]

    out = None
    if rank == 0:
        hbm, peak_src = peaks()
        kernels = {}
        for key, bkey in (("spmv", "spmv"), ("update", "update"), ("precond", "precond"), ("final", "final")):
            ms = prof[key + "_ms"]
            it = max(prof["iters"], 1)
            avg_s = ms / it / 1000.0
            kernels[key] = {"bytes_per_launch": bm[bkey], "avg_ms": ms / it,
                            "achieved_gbs": bm[bkey] / avg_s / 1e9 if avg_s > 0 else None}
        dom = max(kernels, key=lambda k: kernels[k]["avg_ms"])
        dk = kernels[dom]
        # per-iteration time inside the timed region (CUDA graphs, kernels chained
        # by programmatic dependent launch), per scene; and the per-class event
        # sum of the profiled solve (direct launches, no overlap) for reference
        iter_s = (max_pcg / 1000.0) / max(all_iters / world, 1)
        iter_s_classes = (prof["spmv_ms"] + prof["update_ms"] + prof["precond_ms"] + prof["final_ms"]) / max(prof["iters"], 1) / 1e3
        out = {
            "metric": METRIC,
            "value": all_iters / (max_pcg / 1000.0),
            "unit": "PCG iterations/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": max_total / args.steps,
            "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": "f64",
            "data": "synthetic (reference generators: make_box_tets + stable Neo-Hookean first-Newton matrix; "
                    "b = M dt^2 g, the first Newton step from rest)",
            "config": workload_config(args, sc, world),
            "ms_per_newton_solve": (sum(g["build_ms"] + g["pcg_ms"] for g in gathered[:1]) / args.steps),
            "assembly_ms": asm_ms / args.steps,
            "mas_build_ms": build_ms / args.steps,
            "mas_build_host_ms": build_host_ms / args.steps,
            "mas_build_cold_ms": cold["build_ms"] if cold else None,
            "mas_build_cold_host_ms": cold["build_host_ms"] if cold else None,
            "mas_build_first_ms": first["build_ms"] if first else None,
            "hierarchy_cache": not args.no_cache,
            "post_solve_us": post_solve_us,
            "pcg_ms": pcg_ms / args.steps,
            "pcg_iters_per_solve": iters / args.steps,
            "converged": all(g["conv"] for g in gathered),
            "rel_residual": res_last.rel_residual,
            "true_rel_residual_b_minus_Ax": xerr,
            "per_rank": gathered,
            "gpu_launches": launches,
            "kernels": kernels,
            "kernels_note": "per-class CUDA-event times from one extra profiled solve on the same stream and inputs "
                            "right after the timed steps (profiling events force direct launches instead of the "
                            "timed region's CUDA graphs)",
            "roofline": {"bound": "hbm", "kernel": dom, "achieved": dk["achieved_gbs"], "peak": hbm,
                         "peak_source": peak_src, "unit": "GB/s",
                         "frac": (dk["achieved_gbs"] / hbm) if dk["achieved_gbs"] else None,
                         "algorithmic_bytes_per_launch": dk["bytes_per_launch"],
                         "traffic": ncu_traffic().get(dom), "traffic_source": "profiles/ncu_traffic.json"},
            "roofline_pcg_iteration": {"bound": "hbm", "bytes_per_iter": bm["total"],
                                       "achieved": bm["total"] / iter_s / 1e9, "peak": hbm, "unit": "GB/s",
                                       "frac": bm["total"] / iter_s / 1e9 / hbm, "iter_us": iter_s * 1e6,
                                       "iter_us_class_sum": iter_s_classes * 1e6},
            # context for the fractions above: the read bandwidth ONE kernel of
            # this size reaches on this B200 with a cold, CLEAN L2 and no
            # compute (tools/stream_read_bench.cu, r02: 50 MB 3.7 TB/s, 200 MB
            # 6.0; the r01 figures 3.2 / 4.65 had the flush's dirty lines
            # written back inside the timed kernel)
            "roofline_practical": {"unit": "GB/s", "single_kernel_read_200MB": 6030.0,
                                   "dominant_kernel_frac": kernels[dom]["achieved_gbs"] / 6030.0,
                                   "source": "tools/stream_read_bench.cu"},
            "clocks": clk.summary(),
        }
    def gathered(obj):
        if dist:
            g = [None] * world
            dist.all_gather_object(g, obj)
            return g
        return [obj]

    pr = None
    if not args.no_producer and args.config == "cfg5_stiff_box" and len(sc.tets):
        pr = producer_gpu(args, ctx, sc, d_b, stream, dev)
        if rank == 0:
            out["producer"] = pr
    # e2e through the host-pointer C-ABI (pinned host buffers)
    if not args.no_e2e:
        e2e = run_e2e(args, ctx, sc, d_b, stream, dev)
        g = gathered(e2e)
        gp = gathered(pr) if pr is not None else None
        if rank == 0:
            tot = max(x["ms"] for x in g)
            stream_e2e = {"value": sum(x["iters"] for x in g) / (tot / 1000.0), "unit": "PCG iterations/s",
                          "h2d_bytes_per_step": g[0]["h2d"], "d2h_bytes_per_step": g[0]["d2h"],
                          "ms_per_step": tot / args.steps,
                          "path": "adipc_gpu_assemble_filtered + adipc_gpu_build_preconditioner "
                                  "+ adipc_gpu_pcg (host pointers, pinned): the host-produced 1.54 GB triplet "
                                  "stream crosses PCIe every Newton iteration"}
            if gp is not None:
                # a Newton iteration's inputs are the positions: the element
                # Hessians are produced on the device (§8f #1), so only x goes in
                # and the direction comes out — strictly more of the reference's
                # work than its own timed window (which excludes element evaluation)
                ptot = max(x["newton_solve_from_host_positions_ms"] for x in gp) * args.steps
                out["e2e"] = {"value": sum(x["pcg_iters_per_solve"] * args.steps for x in gp) / (ptot / 1000.0),
                              "unit": "PCG iterations/s", "h2d_bytes_per_step": gp[0]["h2d_bytes_per_step"],
                              "d2h_bytes_per_step": gp[0]["d2h_bytes_per_step"], "ms_per_step": ptot / args.steps,
                              "path": gp[0]["path"] + " (element Hessians produced on the device from the positions)"}
                out["e2e_host_stream"] = stream_e2e
            else:
                out["e2e"] = stream_e2e
    ctx.close()
    return out, sc


def producer_gpu(args, ctx, sc, d_b, stream, dev):
    """§8f #1 on the benchmarked scene: the device element-Hessian producer
    (inertia + stable Neo-Hookean stencils + PSD projection, emission in the
    reference's order, energy.cu) replaces the host triplet stream. Times the
    producer alone, the whole assemble() (produce + filter + sort + reduce),
    and a whole Newton linear solve from HOST positions (H2D of x, assemble,
    MAS build, PCG, D2H of the direction): the PCIe traffic per Newton
    iteration drops from the 1.54 GB stream to two position vectors."""
    import torch

    from paper_2411_06224_b200 import _lib
    import scenegen as S

    inv9, vol = S.tet_rest_data(sc.verts, sc.tets)
    n, nt = len(sc.mass), len(sc.tets)
    with torch.cuda.stream(stream):
        mesh = {"mass": torch.from_numpy(sc.mass).to(dev), "tets": torch.from_numpy(sc.tets).to(dev),
                "rest_inv9": torch.from_numpy(inv9).to(dev), "rest_volume": torch.from_numpy(vol).to(dev),
                "tet_begin": [0, nt], "mu": [sc.mu], "lam": [sc.lam]}
        d_pin = torch.from_numpy(sc.pinned).to(dev)
        d_xt = torch.from_numpy(S.inertial_target(sc)).to(dev)
        d_x = torch.from_numpy(np.ascontiguousarray(sc.verts.reshape(-1))).to(dev)
        keys = torch.empty(n + 10 * nt, dtype=torch.int64, device=dev)
        vals = torch.empty((n + 10 * nt, 9), dtype=torch.float64, device=dev)
        grad = torch.empty(3 * n, dtype=torch.float64, device=dev)
        d_dir = torch.empty(3 * n, dtype=torch.float64, device=dev)
        d_rhs = torch.empty(3 * n, dtype=torch.float64, device=dev)
    stream.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def timed(fn, reps):
        fn()
        torch.cuda.synchronize()
        ev0.record(stream)
        for _ in range(reps):
            fn()
        ev1.record(stream)
        torch.cuda.synchronize()
        return ev0.elapsed_time(ev1) / reps

    emit_ms = timed(lambda: ctx.fem_emit(mesh, d_x, d_xt, 1e-4, keys, vals, grad, pinned=d_pin), args.steps)
    # a later Newton iteration: a deformed mesh (vertices moved by up to 1 % of
    # a cell) makes nearly every stencil indefinite -> the projection pass runs
    h_cell = float(np.abs(sc.verts[1] - sc.verts[0]).max())
    d_xdef = d_x + torch.from_numpy(np.random.default_rng(1).uniform(-0.01 * h_cell, 0.01 * h_cell,
                                                                    3 * n)).to(dev)
    emit_def_ms = timed(lambda: ctx.fem_emit(mesh, d_xdef, d_xt, 1e-4, keys, vals, grad, pinned=d_pin), args.steps)
    asm_ms = timed(lambda: ctx.fem_assemble(mesh, d_x, d_xt, 1e-4, grad, pinned=d_pin), args.steps)
    # whole Newton linear solve from host positions: x in, direction out
    h_x = torch.from_numpy(np.ascontiguousarray(sc.verts.reshape(-1))).pin_memory()
    h_dir = torch.empty(3 * n, dtype=torch.float64).pin_memory()

    def newton():
        with torch.cuda.stream(stream):
            d_x.copy_(h_x, non_blocking=True)
            ctx.fem_assemble(mesh, d_x, d_xt, 1e-4, grad, pinned=d_pin)
            ctx.build_preconditioner(_lib.PRECOND_MAS)
            torch.neg(grad, out=d_rhs)
            _, res = ctx.pcg(d_rhs, REL_TOL, RESTART, MAX_ITERS, x=d_dir)
            h_dir.copy_(d_dir, non_blocking=True)
        stream.synchronize()
        return res.iters

    newton()
    t0 = time.perf_counter()
    iters = sum(newton() for _ in range(args.steps))
    newton_ms = (time.perf_counter() - t0) * 1000.0 / args.steps
    return {"what": "device element-Hessian producer (SURVEY 8f #1): inertia + 1,886,592 stable Neo-Hookean stencils "
                    "with PSD projection, stream in the reference's emission order",
            "tets": nt, "stream_entries": n + 10 * nt, "fem_emit_ms": emit_ms, "fem_assemble_ms": asm_ms,
            "fem_emit_deformed_ms": emit_def_ms,
            "stream_bytes_written": 80 * (n + 10 * nt),
            "emit_write_gbs": 80 * (n + 10 * nt) / (emit_ms / 1e3) / 1e9,
            "newton_solve_from_host_positions_ms": newton_ms, "pcg_iters_per_solve": iters / args.steps,
            "e2e_pcg_iters_per_s": iters / (newton_ms * args.steps / 1e3),
            "h2d_bytes_per_step": 3 * n * 8, "d2h_bytes_per_step": 3 * n * 8,
            "path": "H2D x + adipc_gpu_fem_assemble_device + adipc_gpu_build_preconditioner + adipc_gpu_pcg_device "
                    "+ D2H direction"}


def run_e2e(args, ctx, sc, d_b, stream, dev):
    import torch

    from paper_2411_06224_b200 import _lib

    L = _lib.gpu()
    import ctypes as C

    T = len(sc.keys)
    h_keys = torch.from_numpy(sc.keys.view(np.int64)).pin_memory()
    h_vals = torch.from_numpy(sc.vals).pin_memory()
    h_pin = torch.from_numpy(sc.pinned).pin_memory()
    h_b = d_b.cpu().pin_memory()
    h_x = torch.empty_like(h_b).pin_memory()
    U = C.c_int64()
    it, rr, cv = C.c_int(), C.c_double(), C.c_int()

    def step():
        # filter_pinned + sort + reduce from the host stream (one H2D of it)
        ctx._check(L.adipc_gpu_assemble_filtered(ctx.h, h_keys.data_ptr(), h_vals.data_ptr(), T, sc.n_blocks,
                                                 h_pin.data_ptr(), 1, C.byref(U)))
        ctx._check(L.adipc_gpu_build_preconditioner(ctx.h, _lib.PRECOND_MAS))
        ctx._check(L.adipc_gpu_pcg(ctx.h, h_b.data_ptr(), REL_TOL, RESTART, MAX_ITERS, h_x.data_ptr(), C.byref(it),
                                   C.byref(rr), C.byref(cv)))
        return it.value

    for _ in range(max(1, args.warmup // 2)):
        step()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    iters = 0
    for _ in range(args.steps):
        iters += step()
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t0) * 1000.0
    n3 = 3 * sc.n_blocks
    h2d = T * 80 + sc.n_blocks + n3 * 8  # raw stream (keys + values) + pins + b
    d2h = n3 * 8                          # x
    return {"ms": ms, "iters": iters, "h2d": int(h2d), "d2h": int(d2h)}


def spawn_ranks(n):
    """`bench.py --gpus N` without an external launcher: start N ranks of this
    script (RANK / LOCAL_RANK / WORLD_SIZE / MASTER_* set, rendezvous on
    127.0.0.1), forward their output, and return the worst exit code."""
    import socket

    so = socket.socket()
    so.bind(("127.0.0.1", 0))
    port = so.getsockname()[1]
    so.close()
    procs = []
    for r in range(n):
        env = dict(os.environ, RANK=str(r), LOCAL_RANK=str(r), WORLD_SIZE=str(n), LOCAL_WORLD_SIZE=str(n),
                   MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        procs.append(subprocess.Popen([sys.executable, os.path.abspath(__file__), *sys.argv[1:]], env=env))
    rc = 0
    for p in procs:
        rc = max(rc, p.wait())
    return rc


def selftest(args, rank, world, dist):
    """Launcher / rendezvous / max-over-ranks self-test (no GPU work): every
    rank reports synthetic timings for its seed; rank 0 prints the gathered
    aggregate. Used by the CPU tests at world size 2 over gloo."""
    stats = dict(total_ms=10.0 + rank, pcg_ms=5.0 + rank, iters=100 + rank, conv=True, seed=5 + rank)
    gathered, agg = gather_scene_stats(stats, world, dist)
    if rank == 0:
        print(json.dumps({"selftest": True, "n_gpus": world, "seeds": [g["seed"] for g in gathered], **agg}),
              flush=True)


def main():
    args = parse()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(spawn_ranks(args.gpus))
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if args.selftest:
        import torch.distributed as tdist

        if world > 1:
            tdist.init_process_group("gloo")
        selftest(args, rank, world, tdist if world > 1 else None)
        if world > 1:
            tdist.barrier()
            tdist.destroy_process_group()
        return
    if args.impl == "reference":
        if rank != 0:
            return
        # the reference arm loads only oracle/ libraries: the reference's own
        # hot-path code (oracle/_ref) and the scene generators built under
        # oracle/build — nothing from the product package
        import scenegen as scenes

        scenes.use_library("oracle")
        sc = make_problem(args.config, 5)
        cb = cpu_reference(sc, 5, args.cpu_iters, args.steps, args.warmup, full_solve=not args.no_full_solve)
        full = cb["full_solve"]
        # e2e in the GPU arm's unit: PCG iterations per second of whole Newton
        # linear solves (assembly + MAS build + PCG); `value` stays the PCG-loop rate
        e2e_value = full["iters"] / full["newton_solve_s"] if full else cb["value"]
        line = {"metric": METRIC, "value": cb["value"], "unit": "PCG iterations/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 * args.cpu_iters / cb["value"],
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic (same generator and seed as the GPU arm)",
                "config": workload_config(args, sc, world),
                "impl": "reference",
                "cpu_baseline": {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample", "value_1_thread")},
                "assembly_s": cb["assembly_s"], "mas_build_s": cb["mas_build_s"], "full_solve": full,
                "ms_per_newton_solve": 1000.0 * (cb["mas_build_s"] + full["pcg_s"]) if full else None,
                "e2e": {"value": e2e_value, "unit": "PCG iterations/s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0,
                        "scope": "one whole Newton linear solve (assembly + MAS build + PCG to rel_tol), timed"
                                 if full else "PCG-loop sample only"}}
        if not args.no_hybrid and args.config == "cfg5_stiff_box":
            hy = hybrid_cpu(make_problem(HYBRID, 4), args.cpu_iters, full_solve=not args.no_full_solve)
            hf = hy["full_solve"]
            line["hybrid"] = {"config": HYBRID, "pcg_iters_per_s": hy["value"],
                              "cpu_baseline": {k: hy[k] for k in ("value", "unit", "cores", "kind", "sample")},
                              "assembly_s": hy["assembly_s"], "two_level_s": hy["two_level_s"],
                              "mas_build_s": hy["mas_build_s"], "full_solve": hf,
                              "ms_per_newton_solve": 1000.0 * hf["newton_solve_s"] if hf else None}
        if not args.no_geom and args.config == "cfg5_stiff_box":
            line["geom"] = geom_cpu(full_solve=not args.no_full_solve)
        print(json.dumps(line), flush=True)
        return
    dist = None
    if world > 1:
        import torch
        import torch.distributed as tdist

        torch.cuda.set_device(local_rank)
        tdist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        dist = tdist
    out, sc = run_ours(args, rank, world, local_rank, dist)
    if not args.no_hybrid and args.config == "cfg5_stiff_box":
        hy = hybrid_gpu(args, local_rank, with_cpu=(rank == 0 and world == 1 and not args.no_cpu_baseline))
        if rank == 0:
            out["hybrid"] = hy
    if not args.no_geom and args.config == "cfg5_stiff_box":
        ge = geom_gpu(args, local_rank)
        if rank == 0:
            out["geom"] = ge
    if rank == 0:
        if world == 1 and not args.no_cpu_baseline:
            cb = cpu_reference(sc, 5, args.cpu_iters, 2, 1)
            out["cpu_baseline"] = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample", "value_1_thread")}
            out["cpu_baseline"]["assembly_s"] = cb["assembly_s"]
            out["cpu_baseline"]["mas_build_s"] = cb["mas_build_s"]
            out["speedup_pcg_iters_per_s_vs_cpu"] = out["value"] / cb["value"]
        print(json.dumps(out), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
