"""Development tool: run every production kernel variant once at small shapes, for
compute-sanitizer (racecheck / synccheck / memcheck) on the B200:

  compute-sanitizer --tool racecheck python tools/sanitize_paths.py

Covers the decode router (6- and 4-deep rings) + slice-plane GEMV (T=1, 16; 1, 2 and 8 row tiles per
CTA), the merged-code stream-K decode GEMV, the 1-CTA tcgen05 router with the cluster K-split and the
split-K GEMM (T=40), the CTA-pair router (N=128 and N=256) and the CTA-pair GEMM (T=300..1300), the
bulk-copy gather, the stable permutation, the device radix-select for delta and the GPU decompose.
Each forward is also compared with the CUDA-core reference GEMM (debug impl 1) on the same masks, so a
sanitizer-perturbed schedule that corrupts results fails loudly.
"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))
from gpu_helpers import make_layer, make_x  # noqa: E402
from paper_2602_20191_b200 import calibrate_threshold, permute_by_slice  # noqa: E402
from paper_2602_20191_b200.layer import decompose  # noqa: E402

GENERIC = [((4, 2, 2), 300), ((1, 1, 1, 1, 1, 1, 1, 1), 40)]  # per-slice CUDA-core path
CASES = [  # (out, in, h, T, what)
    (256, 512, 128, 1, "decode router + slice planes"),
    (256, 512, 128, 16, "slice planes, two 8-token groups"),
    (8192, 1024, 64, 8, "slice planes, 2 row tiles per CTA"),
    (4768, 512, 64, 1, "slice planes, 2 row tiles per CTA, last CTA half empty"),
    (20000, 128, 16, 2, "slice planes, 8 row tiles per CTA"),
    (1024, 14336, 3584, 1, "down-size decode router: 448 CTAs, 4-deep ring"),
    (1024, 14336, 3584, 4, "stream-K merged-code decode (planes' activations do not fit)"),
    (256, 1024, 256, 40, "1-CTA router cluster K-split + split-K GEMM"),
    (256, 512, 2048, 1024, "pair router N=128 + pair GEMM"),
    (256, 256, 4096, 1280, "pair router N=256 + pair GEMM"),
    (512, 384, 96, 700, "1-CTA router + pair GEMM, several units per pair"),
]


def main():
    only = sys.argv[1] if len(sys.argv) > 1 else None
    for out, inn, h, T, what in CASES:
        if only and only not in what:
            continue
        _, layer = make_layer(out, inn, gs=128, hidden=h, seed=out + T)
        xb, _ = make_x(T, inn, seed=T + 3)
        delta = calibrate_threshold(layer.score(xb), 1 / 6)
        y, m = layer.forward(xb, delta, return_masks=True)
        plan = layer.last_plan()
        layer.set_debug_impl(1)
        y_ref = layer.forward_masked(xb, m)
        layer.set_debug_impl(0)
        torch.cuda.synchronize()
        d = (y.float() - y_ref.float()).norm() / y_ref.float().norm()
        print(f"{what:52s} {out}x{inn} h={h} T={T}: plan {plan} rel vs simt {d:.2e}", flush=True)
        assert d < 1e-2, what
        layer.close()
    from paper_2602_20191_b200 import MobiLayer
    from oracle import oracle as O
    for sb, T in GENERIC:
        if only and only != "generic":
            continue
        L = O.synthetic_layer(192, 320, seed=4, group_size=64, slice_bits=sb)
        layer = MobiLayer.from_stack(L["codes"], L["slice_bits"], L["scale"], L["zero"], 64, L["w1"], L["b1"],
                                     L["w2"], L["b2"], device=0)
        xb, _ = make_x(T, 320, seed=T)
        delta = calibrate_threshold(layer.score(xb), 1 / 6)
        y, m = layer.forward(xb, delta, return_masks=True)
        layer.route(xb, delta)
        torch.cuda.synchronize()
        print(f"generic {sb} T={T}: plan {layer.last_plan()}", flush=True)
        layer.close()
    masks = torch.randint(0, 8, (333,), dtype=torch.uint8, device="cuda") * 2 + 1
    perm, inv, groups = permute_by_slice(masks)
    s = torch.randn(200000, device="cuda")
    calibrate_threshold(s, 1 / 6)
    w = torch.randn(64, 256, dtype=torch.float64, device="cuda") * 0.02
    decompose(w, 128, [2, 2, 2, 2], 4.0)
    torch.cuda.synchronize()
    print("sanitize paths ok")


if __name__ == "__main__":
    main()
