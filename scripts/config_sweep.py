"""Measure every BASELINE.json config on one B200: device time, density matrices/s, algorithmic
TF/s and fraction of the measured bf16 peak, and accuracy per precision mode.

Accuracy references (measurement only; the CPU oracle stays test infrastructure):
  * fp64 recursion: the same MLSP2 polynomial evaluated with torch float64 GEMMs on the GPU
    (X0 = (1 - mu0) I - (beta/beta0)(H - mu I); A += d X; X = a X^2 + b X + c I; D = A + X),
  * exact Fermi matrix V diag(f(lambda)) V^T from torch.linalg.eigh (float64), reported, not gated.
Every row carries the nvidia-smi clocks / throttle reasons sampled while it was timed, the
fraction of the measured bf16 peak (burst: each row times its kernels alone), and -- for the
single-matrix configs -- the paper's comparator on the same box: cuSOLVER diagonalisation
(torch.linalg.eigh -> cusolverDn{D,S}syevd) plus the D = V f(lambda) V^T assembly.
Writes one JSON document (stdout, or --out).

    python scripts/config_sweep.py [--out profiles/r2_configs.json] [--quick]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2605_08523_b200 import engine as E  # noqa: E402
from paper_2605_08523_b200.hamiltonians import tight_binding, batch_params  # noqa: E402
from bench import ClockSampler  # noqa: E402

DEV = torch.device("cuda", 0)


def peaks():
    try:
        with open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except Exception:
        return {"bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}


def recursion_f64(H: torch.Tensor, mu: float, kT: float, model: E.Mlsp2Model) -> torch.Tensor:
    n = H.shape[0]
    I = torch.eye(n, dtype=torch.float64, device=H.device)
    s = (1.0 / kT) / model.beta0
    X = (1.0 - model.mu0) * I - s * (H - mu * I)
    A = torch.zeros_like(X)
    for a, b, c, d in model.abcd:
        A = A + d * X
        X = a * (X @ X) + b * X + c * I
    return A + X


def fermi_exact(H: torch.Tensor, mu: float, kT: float) -> torch.Tensor:
    lam, V = torch.linalg.eigh(H)
    f = 1.0 / (1.0 + torch.exp(torch.clamp((lam - mu) / kT, -700, 700)))
    return (V * f) @ V.T


def errors(D: torch.Tensor, R: torch.Tensor) -> dict:
    d = D - R
    tr_r = torch.trace(R).item()
    return {"max_abs": d.abs().max().item(),
            "fro_rel": (torch.linalg.norm(d) / torch.linalg.norm(R)).item(),
            "trace_rel": abs(torch.trace(D).item() - tr_r) / abs(tr_r)}


def timed(H_dev, mu, kT, model, mode, reps):
    D = torch.empty_like(H_dev)
    E.compute_density_matrices_device(H_dev, mu, kT, model, mode, D_dev=D)
    torch.cuda.synchronize()
    ts = []
    with ClockSampler(0) as clk:
        clk.mark("start")
        t_end = time.perf_counter() + 0.3  # at least ~0.3 s under load so the clock sampler sees it
        while len(ts) < reps or time.perf_counter() < t_end:
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record()
            _, status, _ = E.compute_density_matrices_device(H_dev, mu, kT, model, mode, D_dev=D)
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b) / 1e3)
        clk.mark("end")
    st = status.cpu().numpy()
    assert (st == 0).all(), st
    return float(np.median(ts)), D, clk.summary()


def cusolver_time(H: torch.Tensor, mu: float, kT: float, dtype, reps: int = 3) -> float:
    """Paper's comparator: cusolverDn{D,S}syevd (torch.linalg.eigh) + D = V f V^T, median seconds."""
    Hd = H.to(dtype)
    fermi_exact(Hd, mu, kT)
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        fermi_exact(Hd, mu, kT)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) / 1e3)
    return float(np.median(ts))


def run_case(name, n, B, mode, model, pk, reps, ref_idx=(0,), exact=True, mu=None, kT=None, cusolver=False):
    if mu is None:
        mu, kT = np.zeros(B), np.full(B, 0.01)
    seeds = [1234] if B == 1 else [10000 + k for k in range(B)]
    H = np.stack([tight_binding(n, seed=s) for s in seeds])
    H_dev = torch.from_numpy(H).to(DEV)
    t, D, clocks = timed(H_dev, mu, kT, model, mode, reps)
    F = B * E.algorithmic_flops(n, model.layer_count, mode)
    out = {"config": name, "n": n, "batch": B, "mode": mode.name, "seconds": t,
           "matrices_per_s": B / t, "algorithmic_tflops": F / t / 1e12,
           "frac_of_burst_bf16": F / t / 1e12 / pk["bf16_tflops"],
           "frac_of_sustained_bf16": F / t / 1e12 / pk.get("bf16_tflops_sustained", pk["bf16_tflops"]),
           "fp32_equiv_gemm_tflops": B * model.layer_count * 2.0 * n ** 3 / t / 1e12, "clocks": clocks,
           "k2_kernel": E.k2_kernel_name(n, mode)}
    if cusolver:
        td = cusolver_time(H_dev[0], float(mu[0]), float(kT[0]), torch.float64)
        ts_ = cusolver_time(H_dev[0], float(mu[0]), float(kT[0]), torch.float32)
        out["cusolver"] = {"dsyevd_plus_D_s": td, "ssyevd_plus_D_s": ts_,
                           "speedup_vs_dsyevd": td / (t / B), "speedup_vs_ssyevd": ts_ / (t / B),
                           "note": "torch.linalg.eigh (cusolverDn{D,S}syevd) + V f(lambda) V^T on the same B200; "
                                   "the paper's comparator (PAPER.md:682-688: 16x / 9x vs D, 5x / 2x vs S on RTX 6000 Ada)"}
    errs, errs_exact = [], []
    for k in ref_idx:
        R = recursion_f64(H_dev[k], float(mu[k]), float(kT[k]), model)
        errs.append(errors(D[k], R))
        if exact:
            errs_exact.append(errors(D[k], fermi_exact(H_dev[k], float(mu[k]), float(kT[k]))))
        del R
    out["error_vs_fp64_recursion"] = {key: max(e[key] for e in errs) for key in errs[0]}
    if errs_exact:
        out["error_vs_exact_fermi"] = {key: max(e[key] for e in errs_exact) for key in errs_exact[0]}
    out["error_sample"] = list(ref_idx)
    del H_dev, D
    torch.cuda.empty_cache()
    print(json.dumps(out), file=sys.stderr, flush=True)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out")
    ap.add_argument("--quick", action="store_true", help="skip N=16384 and the 512-matrix batch")
    args = ap.parse_args()
    model = E.load_model("M1500")
    pk = peaks()
    F32E, BF16, FP16 = E.PrecisionMode.MIXED_EMULATED, E.PrecisionMode.BF16, E.PrecisionMode.FP16
    rows = []
    rows.append(run_case("configs[0] N=256 single", 256, 1, F32E, model, pk, 20))
    rows.append(run_case("configs[0] N=256 single", 256, 1, BF16, model, pk, 20))
    rows.append(run_case("configs[1] N=1024 single", 1024, 1, F32E, model, pk, 10, cusolver=True))
    rows.append(run_case("configs[1] N=1024 batch 16 (bench)", 1024, 16, F32E, model, pk, 10, ref_idx=(0, 7)))
    for n in (4096, 8192):
        for mode in (F32E, BF16, FP16):
            rows.append(run_case("configs[2] N=%d single" % n, n, 1, mode, model, pk, 3, cusolver=mode == F32E))
    # outside the north star's tensor-core modes: DOUBLE / SINGLE (library GEMM path)
    for mode in (E.PrecisionMode.DOUBLE, E.PrecisionMode.SINGLE):
        for n in (1024, 4096):
            rows.append(run_case("PrecisionMode %s N=%d single" % (mode.name, n), n, 1, mode, model, pk, 3))
    if not args.quick:
        mu, kT = batch_params(512)
        for mode in (F32E, BF16):
            rows.append(run_case("configs[3] 512 x N=512, mu/kT per matrix", 512, 512, mode, model, pk, 3,
                                 ref_idx=(0, 5, 11, 23, 100, 511), mu=mu, kT=kT))
        for mode in (F32E, BF16):
            rows.append(run_case("configs[4] N=16384 single (1 GPU)", 16384, 1, mode, model, pk, 1, exact=False))
    doc = {"gpu": torch.cuda.get_device_name(0), "peaks": pk, "model": "M1500 (beta0=1500, mu0=1/3, L=30)",
           "when": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime()), "rows": rows}
    txt = json.dumps(doc, indent=1)
    if args.out:
        with open(args.out, "w") as f:
            f.write(txt + "\n")
    print(txt)


if __name__ == "__main__":
    main()
