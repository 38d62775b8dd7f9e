"""Mint the golden fixtures in tests/golden/ from the REFERENCE ITSELF.

Run in the build container (needs /root/reference):  python tests/golden/make_golden.py

Everything numeric here is computed by oracle/_ref/libmobi_ref.so -- the
unmodified reference headers compiled where they lie -- and by the reference
CLI (oracle/_ref/mobi) for the toy checkpoint.  The committed fixtures then pin
the C restatement (oracle/mobi_oracle.c) and the GPU path on boxes where the
reference sources are absent.

Fixtures:
  toy_default_seed1.mobi   `mobi calibrate configs/toy_default.cfg --seed 1` (BASELINE config 1)
  toy_stream.npz           layer-by-layer hot path over calib batch 0 of that checkpoint at
                           target bits {2, 3, 4}: X_l, S_l, delta_l, G_l, masks, perm, Y_l
  qo_T4.npz                4096x4096 synthetic layer (SURVEY 8(d) recipe, seed 7), T=4 tokens:
                           S, delta(rho=1/6), G, Y, plus codes/scale/zero checksums
  small_cases.npz          reference unit-test-shaped cases (random_stack n=8 / n=6, all-on,
                           all-off, mixed gates; permute_by_slice {1,3,1,3})
"""
from __future__ import annotations

import hashlib
import shutil
import subprocess
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle import oracle as O  # noqa: E402
from paper_2602_20191_b200 import checkpoint as ckpt  # noqa: E402

GOLD = Path(__file__).resolve().parent
TOY_CFG = "/root/reference/proj/configs/toy_default.cfg"


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def silu(x):
    return x / (1.0 + np.exp(-x))


def toy(ref):
    O.build()
    run = Path("/tmp/mobi_golden_toy")
    shutil.rmtree(run, ignore_errors=True)
    subprocess.run([str(O.HERE / "_ref" / "mobi"), "calibrate", TOY_CFG, "--out", str(run), "--seed", "1"],
                   check=True, stdout=subprocess.DEVNULL)
    shutil.copy(run / "checkpoint.mobi", GOLD / "toy_default_seed1.mobi")
    ck = ckpt.load(GOLD / "toy_default_seed1.mobi")
    c = ck.config
    x0, _ = O.gen_calibset(1, c["seqlen"], c["model_dim"], c["outlier_frac"], c["outlier_scale"], c["seed"])
    out = {}
    for target in (2.0, 3.0, 4.0):
        h = x0[0]
        rho = ref.ratio_from_target_bits(target, c["slice_bits"])
        for li, L in enumerate(ck.layers):
            codes = ref.layer_stack(L.planes, L.cols, L.slice_bits)
            s = ref.score(h, L.w1, L.b1, L.w2, L.b2)
            delta = ref.calibrate_threshold(s, rho)
            g = ref.gate_hard(s, delta)
            y = ref.forward_elastic(h, codes, L.slice_bits, L.base_scale, L.base_zero, L.group_size, g)
            masks = O.masks_from_gates(g)
            _, perm, inv, groups = ref.permute_by_slice(h, masks)
            key = f"t{int(target)}_l{li}"
            out[key + "_x"] = h
            out[key + "_s"] = s
            out[key + "_delta"] = np.array(delta)
            out[key + "_g"] = g
            out[key + "_masks"] = masks
            out[key + "_perm"] = perm
            out[key + "_y"] = y
            out[key + "_avg_bits"] = np.array(ref.avg_bits(g, L.slice_bits))
            h = y if li + 1 == len(ck.layers) else silu(y)
    for li, L in enumerate(ck.layers):
        out[f"l{li}_codes"] = ref.layer_stack(L.planes, L.cols, L.slice_bits)
    np.savez_compressed(GOLD / "toy_stream.npz", **out)


def qo(ref):
    L = O.synthetic_layer(4096, 4096, seed=7, backend=ref)
    x, _ = O.gen_calibset(1, 4, 4096, 0.05, 8.0, 11)
    x = x[0]
    s = ref.score(x, L["w1"], L["b1"], L["w2"], L["b2"])
    delta = ref.calibrate_threshold(s, 1.0 / 6.0)
    g = ref.gate_hard(s, delta)
    y = ref.forward_elastic(x, L["codes"], L["slice_bits"], L["scale"], L["zero"], 128, g)
    np.savez_compressed(GOLD / "qo_T4.npz", x=x, s=s, delta=np.array(delta), g=g, y=y,
                        codes_sha=np.array(sha(L["codes"])), scale_sha=np.array(sha(L["scale"])),
                        zero_sha=np.array(sha(L["zero"])), w1_sha=np.array(sha(L["w1"])),
                        clamp_counts=L["clamp_counts"], scale_head=L["scale"][:64], zero_head=L["zero"][:64])


def small(ref):
    rng = O.Rng(8)
    out = {}
    for n, tag in ((8, "n8"), (6, "n6")):
        w = rng.normal(n * n).reshape(n, n)
        scale, zero = ref.params_from_clip(w, n, 2, 40.0)
        codes, _, _ = ref.decompose(w, n, scale, zero, [2, 2, 2, 2])
        x = rng.normal(5 * n).reshape(5, n)
        gm = np.zeros((5, 3))
        gm[0, 0] = gm[1, 0] = gm[1, 1] = gm[2, 2] = 1.0
        gm[3] = 1.0
        for name, g in (("on", np.ones((5, 3))), ("off", np.zeros((5, 3))), ("mixed", gm)):
            out[f"{tag}_{name}_y"] = ref.forward_elastic(x, codes, [2, 2, 2, 2], scale, zero, n, g)
            out[f"{tag}_{name}_g"] = g
        out[f"{tag}_w"], out[f"{tag}_x"], out[f"{tag}_codes"] = w, x, codes
        out[f"{tag}_scale"], out[f"{tag}_zero"] = scale, zero
    toks = np.arange(4, dtype=np.float64).reshape(4, 1)
    permuted, perm, inv, groups = ref.permute_by_slice(toks, np.array([1, 3, 1, 3], np.uint8))
    out["perm_1313"] = perm
    out["perm_1313_groups"] = np.array(groups)
    np.savez_compressed(GOLD / "small_cases.npz", **out)


if __name__ == "__main__":
    ref = O.reference()
    toy(ref)
    qo(ref)
    small(ref)
    print("golden fixtures written to", GOLD)
