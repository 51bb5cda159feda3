"""bench.py -- SGBEM V-matrix assembly throughput (entries/s, FP64) on B200.

Workload (BASELINE.json configs[3], "C4"): closed ellipse (semi-axes 2, 1;
16 control points, cubic), p = 3, 32768 uniform elements -> N = 32768,
n_q = 65536, dense A = 8.6 GB.  One STEP = one full assembly of A on the
device: pair-moment table (cold), circulant log-part tables, fused K1 grid +
banded contraction (IK1), fused log part (IK2), symmetrise/scale epilogue.
Inputs are the O(N) precompute of ``build_discretization`` (host, timed
separately as ``precompute_s``); the output (8.6 GB) exceeds L2 (126 MB) and
is rewritten every step, so no L2 flush is needed.

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]

N > 1: one rank per GPU (``--gpus N`` re-runs itself under torchrun when no
launcher set WORLD_SIZE).  The upper-triangle tile pairs are split into equal
contiguous ranges dealt cyclically over ranks and chunks; each rank assembles
its ranges with no communication, and a packed all-gather of the upper tiles
per chunk (half the bytes of full rows) overlaps the next chunk's compute; the
received tiles are unpacked and mirrored on a side stream (total work fixed ->
"strong").  The line adds ``distributed_ms`` (assembly / gathered / total /
epilogue, max over ranks, received bytes per rank).  ``--impl reference`` times the CPU oracle port of the
reference algorithm (oracle/wq_oracle.py, row-block restatement) on a
bounded row sample of the same workload (rank 0 only).
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
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

METRIC = "SGBEM V-matrix assembly entries/s (FP64)"
UNIT = "entries/s"
FP64_DATASHEET_TFLOPS = 37.2  # 148 SM x 64 DFMA/clk x 2 x 1.965 GHz
SURVEY_W_C4 = 9.62e11         # algorithmic flop-eq of the C4 assembly


def workload(n_el: int, p: int = 3, geometry: str = "ellipse"):
    import paper_1703_10016_b200 as W
    if geometry == "ellipse":
        th = 2 * np.pi * np.arange(16) / 16
        cp = np.column_stack([2 * np.cos(th), np.sin(th)])
        bp = np.linspace(0, 1, 17)
    else:
        th = 2 * np.pi * np.arange(32) / 32
        r = 1 + 0.3 * np.cos(5 * th)
        cp = np.column_stack([r * np.cos(th), r * np.sin(th)])
        bp = np.linspace(0, 1, 33)
    curve = W.load_curve({"degree": 3, "closed": True, "breakpoints": bp.tolist(),
                          "control_points": cp.tolist()})
    space = W.make_cyclic_basis(p, np.linspace(0, 1, n_el + 1))
    return curve, space


def _label(args) -> str:
    """Workload name of a closed-curve run (C4 at the defaults)."""
    c4 = args.geometry == "ellipse" and args.p == 3 and args.n_el == 32768
    c2 = args.geometry == "ellipse" and args.p == 3 and args.n_el == 1024
    c3 = args.geometry == "star" and args.n_el == 4096
    tag = "C4: " if c4 else "C2: " if c2 else f"C3 (p={args.p}): " if c3 else ""
    geo = ("closed ellipse 2x1 (16 ctrl pts, cubic)" if args.geometry == "ellipse"
           else "closed star r = 1 + 0.3 cos 5t (32 ctrl pts, cubic)")
    return f"{tag}{geo}, p={args.p}, {args.n_el} uniform elements"


def workload_c5(n_el: int = 16384, p: int = 4, seed: int = 0, zone: float = 0.2,
                ratio: float = 0.9, growth_elems: int = 60):
    """BASELINE.json configs[4] ("C5"): open slit [-1, 1] x {0}, degree p,
    n_el elements graded geometrically (ratio per element) toward both ends
    over the outer `zone` fraction, growth from the end element capped at the
    interior width after `growth_elems` elements (the literal 0.9^3277
    underflows); every interior knot doubled with probability
    0.25 from np.random.default_rng(seed).random(n_el - 1) (4030 doubles ->
    N = 20418 at the defaults)."""
    import paper_1703_10016_b200 as W
    ng = int(round(zone * n_el))
    w = np.ones(n_el)
    fac = ratio ** np.maximum(0, growth_elems - np.arange(ng))
    w[:ng] = fac
    w[n_el - ng:] = fac[::-1]
    bp = np.concatenate([[0.0], np.cumsum(w)])
    bp = -1.0 + 2.0 * bp / bp[-1]
    mult = np.where(np.random.default_rng(seed).random(n_el - 1) < 0.25, 2, 1)
    curve = W.load_curve({"degree": 1, "knots": [-1, -1, 1, 1], "control_points": [[-1, 0], [1, 0]]})
    return curve, W.make_open_basis(p, bp, mult)


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
            self.thread.join(timeout=2)

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def fp64_peak_tflops(torch, _lib):
    """Measured DFMA throughput (burst) of this GPU: the roofline denominator."""
    blocks = 148 * 16
    out = torch.empty(blocks, dtype=torch.float64, device="cuda")
    iters = 20000
    _lib.call("wq_fp64_peak", iters, blocks, _lib.ptr(out), _lib.stream_handle())
    torch.cuda.synchronize()
    best = 0.0
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        _lib.call("wq_fp64_peak", iters, blocks, _lib.ptr(out), _lib.stream_handle())
        e1.record()
        torch.cuda.synchronize()
        best = max(best, blocks * 256 * iters * 64 * 2 / (e0.elapsed_time(e1) * 1e-3) / 1e12)
    return best


def kernel_flops(disc):
    """Algorithmic flop-eq per launch of the two dominant kernels (DESIGN.md
    'roofline'): DFMA = 2, DADD/DMUL = 1, ln = 44 (libdevice fast path,
    SURVEY F9)."""
    N, nq = disc.space.dim, disc.nodes.n
    wg = disc.rules.WG
    c_k1 = 4 + 1 + 44 + 1                     # dist^2, x 1/p^2, ln, x 1/2
    nb = -(-N // 64)
    sym = (nb + 1) / (2.0 * nb)                # ik1_sym computes the upper-triangle tiles only
    ik1 = (c_k1 * nq * nq + 2 * wg * (nq * N + N * N)) * sym
    from paper_1703_10016_b200 import assembly as AS
    lp = AS._log_part(disc)
    if lp.path == "circulant":
        K = lp.U.shape[1] * (lp.da + 1)            # (p+1)(P+1) = 64 at p = 3
        ws = lp.s_w.shape[1]
        ik2 = 2 * (K + ws) * N * N + 2 * ws * N * N   # Phi (Theta H^-1 + F S), then S^T Phi
    else:
        ik2 = None
    return {"ik1": ik1, "ik2": ik2}


def x2_executed_flops(disc):
    """FP64 tensor flops the x2 kernel (x2ws_kernel; x2v4_kernel issues the same) executes
    per launch: per tile pair 2 orientations x 8 (phi NSTEPS x NKB + band 8 x KS/4) DMMA
    m8n8k4 of 512 flops (wq_fast.cu X2Cfg)."""
    p = disc.space.degree
    NA = p + 13
    NAPAD = -(-NA // 4) * 4
    WSPAD = -(-(2 * p + 1) // 4) * 4
    nsteps = ((p + 1) * NAPAD + WSPAD) // 4
    nkb = (64 + 2 * p + 14) // 8
    ks4 = -(-(8 + 2 * p) // 4)
    nb = -(-disc.space.dim // 64)
    pairs = nb * (nb + 1) // 2
    return float(pairs * 8 * 2 * (nsteps * nkb + 8 * ks4) * 512)


def committed_traffic(dom):
    """dram read+write bytes per launch of the dominant kernel from the
    committed ncu --set full capture (profiles/r*_traffic.json), or None."""
    import glob
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_traffic.json")))
    if not files:
        return None
    try:
        data = json.load(open(files[-1]))
        key = {"ik1": "ik1_sym_kernel", "ik2": "x2ws_kernel"}[dom]
        return data[key]["total"]
    except (OSError, ValueError, KeyError):
        return None


REF_DIR = os.path.join(ROOT, "baseline", "_ref")


def reference_ladder(sizes, with_ebe=True, ebe_max=1024):
    """The UNMODIFIED reference (``wqbem`` installed into baseline/_ref) through
    its own public API on this host's cores: build_discretization
    (rule_seconds, assembly.py:147-172), assemble_weighted_matrix cold (first
    call, pair-table lru_cache empty) and warm, with the reference's own
    seconds (assembly.py:248-259), and the element-by-element
    assemble_baseline_matrix(ng=12) with its own timer (assembly.py:418-538),
    on the ellipse p = 3 ladder (N = 1024 is config 2) and config 1; plus a
    power-law fit of the weighted path's seconds to config 4 (N = 32768),
    labelled as an extrapolation (the reference cannot run it)."""
    if not os.path.isdir(os.path.join(REF_DIR, "wqbem")):
        return {"unavailable": "baseline/_ref not installed (pip install --target baseline/_ref)"}
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    import wqbem
    from wqbem import assembly as RA
    from wqbem.geometry import load_curve
    from wqbem.splines import make_cyclic_basis, make_open_basis
    th = 2 * np.pi * np.arange(16) / 16
    ell = load_curve({"degree": 3, "closed": True, "breakpoints": np.linspace(0, 1, 17).tolist(),
                      "control_points": np.column_stack([2 * np.cos(th), np.sin(th)]).tolist()})
    slit = load_curve({"degree": 1, "knots": [-1, -1, 1, 1], "control_points": [[-1, 0], [1, 0]]})
    cases = [("C1 slit p=2", slit, make_open_basis(2, np.linspace(-1, 1, 65)))]
    cases += [(f"ellipse p=3 N={n}" + (" (C2)" if n == 1024 else ""), ell,
               make_cyclic_basis(3, np.linspace(0, 1, n + 1))) for n in sizes]
    rows = []
    for name, curve, space in cases:
        N = space.dim
        t0 = time.perf_counter()
        disc = RA.build_discretization(curve, space, 1)
        build_s = time.perf_counter() - t0
        from wqbem import quadrature as RQ
        for fn in (getattr(RQ, "_unit_pair_stack", None),):
            if fn is not None and hasattr(fn, "cache_clear"):
                fn.cache_clear()
        _, _, cold = RA.assemble_weighted_matrix(disc)
        _, _, warm = RA.assemble_weighted_matrix(disc)
        rec = {"case": name, "N": N, "build_s": build_s, "rule_seconds": disc.rule_seconds,
               "weighted_cold_s": cold, "weighted_warm_s": warm,
               "weighted_entries_per_s": N * N / warm}
        if with_ebe and N <= ebe_max:
            _, _, ebe = RA.assemble_baseline_matrix(curve, space, ng=12)
            rec.update(ebe_s=ebe, ebe_entries_per_s=N * N / ebe)
        rows.append(rec)
        del disc
    lad = [r for r in rows if r["case"].startswith("ellipse")]
    fit = None
    lad = lad[-2:]    # the two largest sizes: closest to the asymptotic law (N^2.5-3)
    if len(lad) >= 2:
        x = np.log([r["N"] for r in lad])
        y = np.log([r["weighted_warm_s"] for r in lad])
        k, c = np.polyfit(x, y, 1)
        t4 = float(np.exp(c + k * np.log(32768)))
        fit = {"law": f"seconds ~ N^{k:.2f} (fit over N = {[r['N'] for r in lad]})",
               "c4_seconds_extrapolated": t4, "c4_entries_per_s_extrapolated": 32768 ** 2 / t4,
               "label": "EXTRAPOLATION: the reference cannot run C4 (550 GB pair tensor, SURVEY F6)"}
        e = [r for r in rows if r["case"].startswith("ellipse") and "ebe_s" in r][-2:]
        if len(e) >= 2:
            k2, c2 = np.polyfit(np.log([r["N"] for r in e]), np.log([r["ebe_s"] for r in e]), 1)
            t5 = float(np.exp(c2 + k2 * np.log(32768)))
            fit.update(ebe_law=f"seconds ~ N^{k2:.2f}", ebe_c4_seconds_extrapolated=t5,
                       ebe_c4_entries_per_s_extrapolated=32768 ** 2 / t5)
    return {"package": f"wqbem {wqbem.__version__} (unmodified, baseline/_ref)",
            "cores": os.cpu_count(),
            "blas_threads": os.environ.get("OPENBLAS_NUM_THREADS", "unset (all cores)"),
            "cases": rows, "c4_fit": fit}


def run_reference(args):
    """CPU oracle port (reference algorithm, row-block restatement) on a
    bounded row sample of the same workload; rank 0 only.  The line also
    carries the unmodified reference timed on the ladder it can run
    (``reference_ladder``)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import wq_oracle as O
    curve, space = workload(args.n_el, args.p, args.geometry)
    oc = O.Curve(curve.basis, curve.control_points)
    ob = O.Basis(space.degree, space.knots, space.closed)
    t0 = time.perf_counter()
    cr = O.CirculantRows(oc, ob)
    setup = time.perf_counter() - t0
    N = space.dim
    R = args.ref_rows
    rng = np.random.default_rng(0)
    for _ in range(args.warmup):
        cr.m_rows(rng.integers(0, N, 1))
    times = []
    for k in range(args.steps):
        rows = rng.integers(0, N, R)
        t0 = time.perf_counter()
        cr.a_rows(rows)
        times.append(time.perf_counter() - t0)
    t = float(np.mean(times))
    value = R * N / t
    cores = os.cpu_count()
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (deterministic analytic geometry, BASELINE.json configs[3])",
        "config": {"workload": f"C4 ellipse p={args.p} N={N}", "N": N,
                   "sample_rows_per_step": R},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": f"{R} random rows of A per step (row-block restatement of "
                                   f"assemble_weighted_matrix + scale_and_symmetrize), setup "
                                   f"{setup:.1f}s untimed (rules + lru-cached pair table, as "
                                   f"the reference's warm path)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    if args.ref_ladder:
        t0 = time.perf_counter()
        line["reference_ladder"] = reference_ladder([int(x) for x in args.ref_ladder.split(",")])
        line["reference_ladder"]["wall_s"] = time.perf_counter() - t0
    print(json.dumps(line), flush=True)


def launcher_check(world: int) -> int:
    """``--launcher-check``: the rank plumbing alone (CPU, gloo): every rank
    joins the group, the world size matches --gpus, rank 0 prints one line."""
    import torch
    import torch.distributed as dist
    dist.init_process_group("gloo")
    assert dist.get_world_size() == world
    t = torch.tensor([dist.get_rank() + 1.0])
    dist.all_reduce(t)
    if dist.get_rank() == 0:
        print(json.dumps({"launcher": "ok", "world": world, "rank_sum": float(t.item())}), flush=True)
    dist.destroy_process_group()
    return 0


def spawn_ranks(n: int) -> int:
    """``--gpus N`` without a launcher: re-run this command under torchrun
    with one rank per GPU (rendezvous on 127.0.0.1) and return its status."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.abspath(__file__)] + sys.argv[1:]
    rc = subprocess.call(cmd)
    if rc:
        raise SystemExit(rc)
    return rc


def main():
    ap = argparse.ArgumentParser(description=__doc__.split("\n")[0])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--n-el", type=int, default=32768)
    ap.add_argument("--p", type=int, default=3)
    ap.add_argument("--geometry", default="ellipse", choices=["ellipse", "star"])
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--chunks", type=int, default=4,
                    help="N > 1: pair-range chunks per rank (all-gather pipelining depth)")
    ap.add_argument("--ref-rows", type=int, default=8)
    ap.add_argument("--ref-ladder", default="256,512,1024",
                    help="--impl reference: N of the unmodified-reference ladder ('' = skip)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--launcher-check", action="store_true",
                    help="only check the one-rank-per-GPU launch (CPU, gloo)")
    ap.add_argument("--graph", default="auto", choices=["auto", "on", "off"],
                    help="replay the 1-GPU assembly as a CUDA graph (auto: N <= 8192)")
    ap.add_argument("--workload", default="c4", choices=["c4", "c5"],
                    help="c4: the headline (BASELINE metric config); c5: graded open slit with "
                         "double knots (configs[4]), 1 GPU, no reference arm (the reference raises)")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_c5(args) if args.workload == "c5" else run_reference(args)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn_ranks(args.gpus)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}: launch one rank per GPU")
    if args.launcher_check:
        return launcher_check(world)
    if args.workload == "c5":
        return run_c5(args)

    import torch
    import torch.distributed as dist
    import paper_1703_10016_b200 as W
    from paper_1703_10016_b200 import _lib, assembly as AS, distributed as D

    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        assert dist.get_world_size() == args.gpus, "one NCCL rank per GPU"

    curve, space = workload(args.n_el, args.p, args.geometry)
    t0 = time.perf_counter()
    disc = W.build_discretization(curve, space, 1)
    AS._log_part(disc)
    precompute_s = time.perf_counter() - t0
    N = space.dim

    alpha = -1.0 / (4.0 * np.pi)
    launches = {"n": 0}
    chunks = args.chunks
    X = torch.empty((N, N), dtype=torch.float64, device="cuda")
    pg = None
    if world == 1:
        per_step = 9   # pair table, 5 circulant-table kernels, zext, ik1_sym, x2_pairs
    else:
        # equal tile-pair ranges dealt cyclically; chunk c's packed upper-triangle
        # all-gather overlaps chunk c+1's compute, unpacks on a side stream
        pg = D.packed_gather(N, world, chunks)
        mine = sum(1 for c in range(chunks) if pg.block(c, rank)[1] > pg.block(c, rank)[0])
        unp = sum(1 for c in range(chunks) for r in range(world)
                  if r != rank and pg.block(c, r)[1] > pg.block(c, r)[0])
        per_step = 7 + 3 * mine + unp   # tables, (ik1_pairs, x2_pairs_range, pack) per own block, unpacks

    graph = None
    if world == 1 and (args.graph == "on" or (args.graph == "auto" and N <= 8192)):
        # launch/host-bound sizes: the whole assembly replays as one CUDA graph
        try:
            graph = AS.AssemblyGraph(disc, X)
        except Exception as exc:   # capture unsupported: eager launches
            print(f"bench: CUDA graph capture failed ({exc}); eager launches", file=sys.stderr)
            graph = None

    def step(marks=None):
        if graph is not None:
            graph.replay()
        elif world == 1:
            AS._assemble_into(disc, X)
        else:
            D.assemble_distributed_pipelined(disc, X, chunks=chunks, zext=AS._zext_table(disc),
                                             marks=marks)
        launches["n"] += per_step

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    AS._check_flag(AS._smooth(disc))
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches["n"] = 0
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        time.sleep(0.3)  # let nvidia-smi start sampling before the timed region
        e0.record()
        for _ in range(args.steps):
            step()
        e1.record()
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = e0.elapsed_time(e1) / args.steps
    ms = max_over_ranks(torch, dist, world, ms)
    gpu_launches = launches["n"]
    value = N * N / (ms * 1e-3)

    dist_split = None
    if world > 1:
        dist_split = distributed_split(torch, dist, disc, X, chunks, pg, step)
    # ---- per-kernel split + roofline of the dominant kernel (1 GPU layout) ----
    peak = fp64_peak_tflops(torch, _lib)
    split = kernel_split(torch, _lib, AS, disc, X, alpha)
    names = ["tables", "ik1_sym", "x2_pairs"]
    fl = kernel_flops(disc)
    dom = "ik1" if split[1] >= split[2] else "ik2"
    dom_ms = split[1] if dom == "ik1" else split[2]
    achieved = fl[dom] / (dom_ms * 1e-3) / 1e12
    executed = x2_executed_flops(disc) if dom == "ik2" else None
    roofline = {"bound": "fp64", "kernel": {"ik1": "ik1_sym_kernel", "ik2": "x2ws_kernel"}[dom],
                "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
                "executed_flop_per_launch": executed,
                "executed_frac": (executed / (dom_ms * 1e-3) / 1e12 / peak) if executed else None,
                "executed_note": "DMMA flops the kernel issues (skew and band padding included), "
                                 "executed / time / peak ~ the DMMA pipe's active fraction",
                "peak_source": "measured DFMA probe (wq_fp64_peak, burst); MEASURED_PEAKS.json has "
                               "no FP64 entry", "peak_datasheet": FP64_DATASHEET_TFLOPS,
                "traffic": committed_traffic(dom), "traffic_unit": "bytes per launch (ncu, profiles/)"}
    # fixed W for C4, x (N+1)/(2N) when the symmetry of A is exploited
    survey_frac = SURVEY_W_C4 * (N + 1) / (2.0 * N) / (ms * 1e-3) / (peak * 1e12 * world) \
        if (args.n_el == 32768 and args.p == 3) else None

    # ---- end to end through the public API with host buffers ----
    e2e = None
    if args.e2e_steps > 0:
        e2e = end_to_end(torch, dist, W, AS, D, disc, X, args, world, rank, chunks)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(args, N)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (deterministic analytic geometry, BASELINE.json configs[3])",
            "config": {"workload": _label(args), "N": N, "nq": disc.nodes.n,
                       "cuda_graph": graph is not None,
                       "parallelism": (f"{world} NCCL ranks: equal upper-triangle tile-pair ranges "
                                       f"x {chunks} chunks, packed upper-tile all-gather per chunk "
                                       "overlapped with compute, unpack + mirror on a side stream")
                       if world > 1 else "single GPU",
                       "l2": (f"{N * N * 8 / 1e9:.2g} GB output > 126 MB L2, rewritten every step "
                              "(no flush needed)") if N * N * 8 > 126e6 else
                             (f"{N * N * 8 / 1e6:.3g} MB output fits L2 (launch-bound size; "
                              "not an L2-flushed timing)")},
            "clocks": clk.summary(),
            "gpu_launches": gpu_launches,
            "split_ms": dict(zip(names, [float(x) for x in split])),
            "distributed_ms": dist_split,
            "roofline": roofline,
            "fp64_roofline_fraction_survey_W": survey_frac,
            "fp64_roofline_fraction_survey_W_note": (
                "SURVEY 8(d) fixed W (prices every ln at 44 flop-eq, libdevice's count) / step "
                "time / peak; the kernels execute 8 FP64 operations per ln, so this figure can "
                "exceed 1 -- kept for continuity with the survey's target only; "
                "roofline.frac and roofline.executed_frac are the measured ones"),
            "precompute_s": precompute_s,
            "e2e": e2e,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def max_over_ranks(torch, dist, world, v):
    if world == 1:
        return float(v)
    t = torch.tensor([float(v)], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def distributed_split(torch, dist, disc, X, chunks, pg, step, reps=3):
    """SURVEY 8(d)(i)-(ii) at N > 1, max over ranks: assembly_ms (start until
    this rank's last pair range is computed and packed), gathered_ms (until the
    last chunk's all-gather has landed), total_ms (until every received block is
    unpacked and mirrored); epilogue_ms = total - gathered.  Received NVLink
    bytes per rank from the packed layout."""
    world = dist.get_world_size()
    acc = np.zeros(3)
    for _ in range(reps):
        ev = {}

        def marks(name):
            e = torch.cuda.Event(enable_timing=True)
            e.record()          # current stream: main for "computed", the unpack stream inside
            ev[name] = e

        dist.barrier()
        torch.cuda.synchronize()
        start = torch.cuda.Event(enable_timing=True)
        start.record()
        step(marks)
        torch.cuda.synchronize()
        acc += [start.elapsed_time(ev["computed"]), start.elapsed_time(ev["gathered"]),
                start.elapsed_time(ev["done"])]
    acc /= reps
    out = [max_over_ranks(torch, dist, world, v) for v in acc]
    return {"assembly_ms": out[0], "gathered_ms": out[1], "total_ms": out[2],
            "epilogue_ms": out[2] - out[1], "recv_bytes_per_rank": pg.recv_bytes(),
            "full_rows_bytes_per_rank": (world - 1) * disc.space.dim ** 2 * 8 // world,
            "chunks": chunks}


def kernel_split(torch, _lib, AS, disc, X, alpha, reps=3):
    """Per-kernel times of the single-GPU launch layout (tables, ik1_sym,
    x2_pairs), CUDA events on the launching stream."""
    N = disc.space.dim
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
    split = np.zeros(3)
    sm = AS._smooth(disc)
    lp, dd = AS._logpart_dev(disc)
    orig_call = _lib.call
    table_ms = []

    def table_call(name, *a):
        # per-launch events: host-side Python between the table kernels stays out of the split
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0.record()
        r = orig_call(name, *a)
        t1.record()
        table_ms.append((t0, t1))
        return r

    for _ in range(reps):
        _lib.call = table_call
        try:
            zext = AS._zext_table(disc)
        finally:
            _lib.call = orig_call
        ev[0].record()
        ev[1].record()
        _lib.call("wq_ik1_sym", AS.ctypes_ref(sm["struct"]), _lib.ptr(X), N, sm["span64"],
                  _lib.ptr(sm["flag"]), _lib.stream_handle())
        ev[2].record()
        # the production log-part kernel (assembly._assemble_v2)
        _lib.call("wq_x2_pairs", N, disc.space.degree, lp.da + 1, lp.nApad, lp.s_w.shape[1],
                  lp.uext.shape[1], lp.zstride, _lib.ptr(dd["uext"]), _lib.ptr(zext),
                  _lib.ptr(dd["s_w"]), alpha, 2.0, _lib.ptr(X), N, _lib.stream_handle())
        ev[3].record()
        torch.cuda.synchronize()
        split += [sum(a.elapsed_time(b) for a, b in table_ms)] + [ev[k].elapsed_time(ev[k + 1])
                                                                 for k in (1, 2)]
        table_ms.clear()
    return split / reps


def end_to_end(torch, dist, W, AS, D, disc, X, args, world, rank, chunks):
    """The same metric through the public API with host buffers: every step
    copies the O(N) inputs host -> device from pinned memory, assembles, and
    reads the result back.  1 GPU: ``assemble_matrix_to_host`` streams finished
    row blocks to a pinned host array while the next assemble (8.6 GB D2H at
    PCIe speed).  N GPUs: the distributed assembly, then each rank reads its
    1/N share of the rows back over its own PCIe link (the union is A on the
    host side); wall time max over ranks."""
    N = disc.space.dim
    sm = AS._smooth(disc)
    lp, dd = AS._logpart_dev(disc)
    inputs = [v for v in list(sm.values()) + list(dd.values())
              if isinstance(v, torch.Tensor) and v.is_cuda and v.numel() > 1]
    pinned = [t.cpu().pin_memory() for t in inputs]
    h2d = sum(t.numel() * t.element_size() for t in pinned)
    if world == 1:
        host = AS.pinned_host_matrix(N)   # pages on the GPU's NUMA node

        def run():
            W.assemble_matrix_to_host(disc, out=host, work=X)
        d2h = N * N * 8
    else:
        r0, r1 = N * rank // world, N * (rank + 1) // world
        host = AS.pinned_host_matrix(r1 - r0, N)

        def run():
            D.assemble_distributed_pipelined(disc, X, chunks=chunks)
            host.copy_(X[r0:r1], non_blocking=True)
        d2h = N * N * 8                   # summed over ranks (each reads its share)
    run()                                 # untimed warm-up of the host path
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.e2e_steps):
        for src, dst in zip(pinned, inputs):
            dst.copy_(src, non_blocking=True)
        run()
        torch.cuda.synchronize()
    t = (time.perf_counter() - t0) / args.e2e_steps
    if world > 1:
        import torch as _t
        tt = _t.tensor([t], dtype=_t.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t = float(tt.item())
    out = {"value": N * N / t, "unit": UNIT, "h2d_bytes_per_step": int(h2d * world),
           "d2h_bytes_per_step": int(d2h), "ms_per_step": t * 1e3,
           "path": "assemble_matrix_to_host (streamed row blocks)" if world == 1 else
                   "assemble_distributed_pipelined + per-rank D2H of a 1/N row share"}
    if world == 1:
        out["cold_call"] = cold_call(torch, W, AS, args, host, X)
    return out


def cold_call(torch, W, AS, args, host, X):
    """One complete drop-in call from the curve and space objects, nothing
    cached: build_discretization (O(N) host precompute), the log-part host
    ingredients, the uploads, the device assembly with the pair table cold, and
    the streamed D2H of A -- what a user's first assemble call costs."""
    curve, space = workload(args.n_el, args.p, args.geometry)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    disc = W.build_discretization(curve, space, 1)
    t1 = time.perf_counter()
    AS._log_part(disc)
    t2 = time.perf_counter()
    W.assemble_matrix_to_host(disc, out=host, work=X)
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    N = space.dim
    return {"value": N * N / (t3 - t0), "unit": UNIT, "ms": (t3 - t0) * 1e3,
            "build_discretization_ms": (t1 - t0) * 1e3, "log_part_host_ms": (t2 - t1) * 1e3,
            "upload_assemble_d2h_ms": (t3 - t2) * 1e3}


SURVEY_W_C5 = 5.46e11         # algorithmic flop-eq of the C5 assembly


def run_c5(args):
    """Config 5: the general (graded-mesh) device path, one step = one full
    assembly of A (lattice Theta / D from the unit gap table, graded outer
    elements by per-pair blocks, banded fit solves, IK1, symmetrise).  N > 1:
    cyclic row blocks of the general path (replicated D / F) with the chunked
    in-place NCCL all-gather.  The reference cannot run it
    (quadrature.py:489-491)."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        if rank == 0:
            print(json.dumps({"impl": "reference", "unavailable": "the reference raises "
                              "ConstructionError on graded meshes (quadrature.py:489-491)"}))
        return
    import torch
    import torch.distributed as dist
    import paper_1703_10016_b200 as W
    from paper_1703_10016_b200 import _lib, assembly as AS, distributed as D
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    curve, space = workload_c5()
    t0 = time.perf_counter()
    disc = W.build_discretization(curve, space, 1)
    AS._log_part(disc)
    precompute_s = time.perf_counter() - t0
    N = space.dim
    chunks = 4
    if world == 1:
        X = torch.empty((N, N), dtype=torch.float64, device="cuda")

        def step():
            AS._assemble_into(disc, X)
    else:
        sub, n_pad = D.cyclic_blocks(N, world, chunks)
        Xpad = torch.empty((n_pad, N), dtype=torch.float64, device="cuda")

        def step():
            D.assemble_distributed_pipelined(disc, Xpad, chunks=chunks)
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    AS._check_flag(AS._smooth(disc))
    # launches per step and per-entry-point split (host-synchronous, attribution only)
    orig = _lib.call
    split, count = {}, {"n": 0}

    def timed(name, *a):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        r = orig(name, *a)
        e1.record()
        torch.cuda.synchronize()
        split[name] = split.get(name, 0.0) + e0.elapsed_time(e1)
        count["n"] += 1
        return r

    _lib.call = timed
    step()
    _lib.call = orig
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        time.sleep(0.3)
        e0.record()
        for _ in range(args.steps):
            step()
        e1.record()
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = e0.elapsed_time(e1) / args.steps
    t_dev = torch.tensor([ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t_dev, op=dist.ReduceOp.MAX)
    ms = float(t_dev.item())
    peak = fp64_peak_tflops(torch, _lib)
    # SURVEY 8(d)'s W counts the K1 grid (c_pair nq^2 + the IK1 contraction, c_pair = 67 open);
    # on this unit-speed straight slit K1 vanishes identically and is not evaluated, so that
    # work is taken out of W rather than credited
    W = SURVEY_W_C5
    k1_skipped = AS._K1_SHORTCUT and AS._k1_vanishes(disc)
    if k1_skipped:
        nq, wbar = disc.nodes.n, 2 * space.degree + 1
        W -= 67.0 * nq * nq + 2.0 * wbar * (nq * N + N * N)
    e2e = None
    if world == 1 and args.e2e_steps > 0:
        # public API with host buffers: H2D of the O(N) inputs from pinned memory, assembly,
        # D2H of the 3.3 GB matrix into a pinned host array
        sm = AS._smooth(disc)
        lp, dd = AS._logpart_dev(disc)
        inputs = [v for v in list(sm.values()) + list(dd.values())
                  if isinstance(v, torch.Tensor) and v.is_cuda and v.numel() > 1]
        pinned = [t.cpu().pin_memory() for t in inputs]
        host = AS.pinned_host_matrix(N)
        W_ = __import__("paper_1703_10016_b200")
        W_.assemble_matrix_to_host(disc, out=host, work=X)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            for src, dst in zip(pinned, inputs):
                dst.copy_(src, non_blocking=True)
            W_.assemble_matrix_to_host(disc, out=host, work=X)
            torch.cuda.synchronize()
        t_e2e = (time.perf_counter() - t0) / args.e2e_steps
        e2e = {"value": N * N / t_e2e, "unit": UNIT,
               "h2d_bytes_per_step": int(sum(t.numel() * t.element_size() for t in pinned)),
               "d2h_bytes_per_step": int(N * N * 8), "ms_per_step": t_e2e * 1e3,
               "path": "assemble_matrix_to_host (assemble, then one D2H copy)"}
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline_c5(args)
    if rank == 0:
        line = {
            "metric": METRIC, "value": N * N / (ms * 1e-3), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (analytic slit, seeded knot multiplicities, BASELINE.json configs[4])",
            "config": {"workload": "C5: open slit [-1,1]x{0}, p=4, 16384 elements graded 0.9 "
                                   "toward both ends (growth capped at the interior width after "
                                   "60 elements), interior knots doubled w.p. 0.25 "
                                   "(default_rng(0))", "N": N, "nq": disc.nodes.n,
                       "parallelism": (f"general-path cyclic row blocks x{world}, {chunks} chunks, "
                                       "replicated D/F, in-place NCCL all-gather") if world > 1
                       else "single GPU",
                       "l2": "3.3 GB output > 126 MB L2, rewritten every step"},
            "clocks": clk.summary(),
            "gpu_launches": count["n"] * args.steps,
            "split_ms": {k: round(v, 3) for k, v in sorted(split.items(), key=lambda t: -t[1])},
            "roofline": {"bound": "fp64",
                         "kernel": "whole step (SURVEY 8(d) W for C5"
                                   + (", less the K1 grid, identically zero here)" if k1_skipped else ")"),
                         "achieved": W / (ms * 1e-3) / 1e12 / world, "peak": peak,
                         "unit": "TFLOP/s per GPU", "W_flop": W,
                         "frac": W / (ms * 1e-3) / 1e12 / world / peak, "traffic": None},
            "precompute_s": precompute_s,
            "e2e": e2e,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def cpu_baseline_c5(args, rows: int = 2):
    """C5 on this host: the oracle's row restatement for graded open meshes
    (oracle.GeneralRows: pair moments by the reference recipe, FFT correlation
    on the width lattice, banded fit solves), timed on a bounded row sample;
    its O(N) setup (rules, gap table) reported separately."""
    try:
        from oracle import wq_oracle as O
    except ImportError:
        return None
    sp = O.config5_space()
    slit = O.Curve(O.open_basis(1, np.array([-1.0, 1.0])), [[-1, 0], [1, 0]])
    t0 = time.perf_counter()
    gr = O.GeneralRows(slit, sp)
    setup = time.perf_counter() - t0
    sample = np.random.default_rng(2).integers(0, sp.dim, rows)
    t0 = time.perf_counter()
    gr.a_rows(sample)
    t = time.perf_counter() - t0
    return {"value": rows * sp.dim / t, "unit": UNIT, "cores": os.cpu_count(), "kind": "port",
            "sample": f"{rows} rows of A ({rows * sp.dim} entries) via oracle.GeneralRows, {t:.1f}s "
                      f"(its per-call Theta / D matvecs over every element pair dominate); setup "
                      f"{setup:.1f}s untimed; the reference itself raises on graded meshes"}


def cpu_baseline(args, N):
    """Oracle port timed on this host on a bounded row sample (10-30 s)."""
    try:
        from oracle import wq_oracle as O
    except ImportError:
        return None
    curve, space = workload(args.n_el, args.p, args.geometry)
    cr = O.CirculantRows(O.Curve(curve.basis, curve.control_points),
                         O.Basis(space.degree, space.knots, space.closed))
    rows = np.random.default_rng(1).integers(0, N, args.ref_rows)
    cr.a_rows(rows[:1])
    t0 = time.perf_counter()
    cr.a_rows(rows)
    t = time.perf_counter() - t0
    return {"value": len(rows) * N / t, "unit": UNIT, "cores": os.cpu_count(), "kind": "port",
            "sample": f"{len(rows)} rows of A ({len(rows) * N} entries) via the oracle row-block "
                      f"restatement, {t:.1f}s; setup (rules, pair table) untimed"}


if __name__ == "__main__":
    main()
