"""Development tool: time the GPU calibration step (mobi_joint_step, csrc/calib.cu) at a LLaMA3-8B q/o
shape, its fp64 GEMM against cuBLAS DGEMM (torch.matmul) on the same shape, and the reference's CPU
joint_forward + joint_backward (oracle/_ref) on a bounded sample.  Prints one JSON line."""
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))
from paper_2602_20191_b200 import joint_step  # noqa: E402
from test_oracle import joint_case  # noqa: E402


def flops(out, inn, T, h, E):
    fwd = E * 2 * T * out * inn + 2 * T * inn * h + 2 * T * h * (E - 1)
    bwd = E * 2 * out * inn * T + 2 * T * inn * h + 4 * T * h * (E - 1)
    return fwd + bwd


def gpu_time(c, sched, t, reps=5):
    d = {k: (torch.from_numpy(np.ascontiguousarray(v)).cuda() if k in ("w", "w1", "b1", "w2", "b2", "x", "y_fp") else v)
         for k, v in c.items()}
    joint_step(**d, sched=sched, t=t)
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        joint_step(**d, sched=sched, t=t)
        ts.append(time.perf_counter() - t0)
    return float(np.median(ts))


def main():
    out, inn, T, h, E = 4096, 4096, 512, 1024, 4
    sched = (8.0, 3.0, 100, 0, 1e-5)
    c = joint_case(out=out, inn=inn, T=T, h=h, gs=128, seed=1)
    tg = gpu_time(c, sched, 10)
    fl = flops(out, inn, T, h, E)
    # cuBLAS DGEMM on the dominant product shape (T x in) x (in x out)
    a = torch.randn(T, inn, dtype=torch.float64, device="cuda")
    b = torch.randn(inn, out, dtype=torch.float64, device="cuda")
    for _ in range(3):
        a @ b
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        a @ b
    e1.record()
    torch.cuda.synchronize()
    cublas_tf = 2 * T * inn * out * 10 / (e0.elapsed_time(e1) * 1e-3) / 1e12
    r = {"what": "calibration step (joint_forward + joint_backward), fp64", "shape": dict(out=out, inn=inn, T=T, h=h, E=E),
         "gpu_ms": tg * 1e3, "gflop": fl / 1e9, "gpu_tflops": fl / tg / 1e12, "cublas_dgemm_tflops": cublas_tf}
    # reference CPU on a bounded sample, and the GPU on the same sample
    from oracle import oracle as O
    so, si, sT, sh = 512, 512, 64, 128
    cs = joint_case(out=so, inn=si, T=sT, h=sh, gs=128, seed=1)
    ref = O.reference()
    t0 = time.perf_counter()
    ref.joint_step(**cs, sched=sched, t=10)
    tr = time.perf_counter() - t0
    r["sample"] = dict(out=so, inn=si, T=sT, h=sh, E=E, ref_cpu_ms=tr * 1e3, ref_cpu_threads=1,
                       gpu_ms=gpu_time(cs, sched, 10) * 1e3, gflop=flops(so, si, sT, sh, E) / 1e9)
    print(json.dumps(r))


if __name__ == "__main__":
    main()
