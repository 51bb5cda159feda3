"""bench.py -- SGBEM V-matrix assembly entries/s (FP64) on B200 (v1)."""
import argparse, json, os, sys, time
import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def ellipse():
    import paper_1703_10016_b200 as W
    th = 2 * np.pi * np.arange(16) / 16
    return W.load_curve({"degree": 3, "closed": True, "breakpoints": np.linspace(0, 1, 17).tolist(),
                         "control_points": np.column_stack([2 * np.cos(th), np.sin(th)]).tolist()})


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--n", type=int, default=32768)
    ap.add_argument("--impl", default="b200")
    a = ap.parse_args()
    import torch
    import paper_1703_10016_b200 as W
    from paper_1703_10016_b200 import assembly as AS, _lib
    t0 = time.perf_counter()
    space = W.make_cyclic_basis(3, np.linspace(0, 1, a.n + 1))
    disc = W.build_discretization(ellipse(), space, 1)
    AS._log_part(disc)
    t_pre = time.perf_counter() - t0
    N = space.dim
    X = torch.empty((N, N), dtype=torch.float64, device="cuda")
    for _ in range(a.warmup):
        AS._assemble_into(disc, X)
    torch.cuda.synchronize()
    AS._check_flag(AS._smooth(disc))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.steps):
        AS._assemble_into(disc, X)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.steps
    # phase split
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    ph = np.zeros(3)
    for _ in range(3):
        ev[0].record(); AS._ik1_into(disc, X); ev[1].record()
        AS._ik2_x2_into(disc, X, accumulate=True); ev[2].record()
        _lib.call("wq_symmetrize", _lib.ptr(X), N, -1.0 / (4 * np.pi), _lib.stream_handle()); ev[3].record()
        torch.cuda.synchronize()
        ph += [ev[0].elapsed_time(ev[1]), ev[1].elapsed_time(ev[2]), ev[2].elapsed_time(ev[3])]
    ph /= 3
    # fp64 peak
    out = torch.empty(148 * 16, dtype=torch.float64, device="cuda")
    iters = 20000
    _lib.call("wq_fp64_peak", iters, 148 * 16, _lib.ptr(out), _lib.stream_handle())
    torch.cuda.synchronize()
    e0.record(); _lib.call("wq_fp64_peak", iters, 148 * 16, _lib.ptr(out), _lib.stream_handle()); e1.record()
    torch.cuda.synchronize()
    peak = 148 * 16 * 256 * iters * 64 * 2 / (e0.elapsed_time(e1) * 1e-3) / 1e12
    print(json.dumps({"metric": "entries/s", "value": N * N / (ms * 1e-3), "ms_per_step": ms, "N": N,
                      "phases_ms": {"ik1": ph[0], "ik2": ph[1], "sym": ph[2]}, "fp64_peak_tflops": peak,
                      "precompute_s": t_pre}))


if __name__ == "__main__":
    main()
