"""Generate tests/golden/ fixtures by running the UNMODIFIED reference (oracle/_ref).

Run in the build container (where /root/reference exists):
    make -C oracle ref && python tools/make_golden.py

Inputs are regenerated from seeds with the reference's counter-based generator
(fill_random, tensor.cpp:65-96), so only seeds, shapes and expected outputs are stored.
Outputs: tests/golden/golden.npz (arrays) and tests/golden/golden.json (hashes, metadata).
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import RefLib  # noqa: E402

GOLD = os.path.join(ROOT, "tests", "golden")
INPUT_STREAM = 0x696E707574  # bench.cpp:76-77 "input"


def pm1(ref, shape, seed):
    """A +-1 matrix from the reference generator: sign(fill_random)."""
    return ref.sign(ref.fill_random(shape, seed))


def main():
    ref = RefLib()
    arrays, meta = {}, {"reference_isa": ref.isa, "cases": {}}

    # --- encoder KATs (test_binarize.cpp:62-103)
    arrays["kat_rows_ones"] = ref.pack(np.ones((1, 32), np.float32), "rows")
    arrays["kat_rows_minus"] = ref.pack(-np.ones((1, 32), np.float32), "rows")
    alt = np.where(np.arange(32) % 2 == 0, 1.0, -1.0).astype(np.float32)[None]
    arrays["kat_rows_alt"] = ref.pack(alt, "rows")
    col33 = np.ones((33, 1), np.float32)
    col33[32] = -1
    arrays["kat_cols_33"] = ref.pack(col33, "cols")

    # --- random encoder cases incl. adversarial floats
    enc = []
    for i, (r, c) in enumerate([(1, 1), (7, 70), (33, 31), (64, 300), (300, 27), (2, 9216)]):
        x = ref.fill_random((r, c), 1000 + i)
        x.flat[:: max(1, x.size // 7)] = 0.0  # zeros -> +1
        if x.size > 4:
            x.flat[1] = -0.0   # -0.0 -> +1 (v >= 0)
            x.flat[2] = np.nan  # NaN -> -1
            x.flat[3] = np.inf
            x.flat[4] = -np.inf
        if x.size > 6:
            x.flat[5] = np.float32(1e-45)   # denormal
            x.flat[6] = np.float32(-1e-45)
        arrays[f"enc{i}_x"] = x
        arrays[f"enc{i}_rows"] = ref.pack(x, "rows", apply_sign=True)
        arrays[f"enc{i}_cols"] = ref.pack(x, "cols", apply_sign=True)
        enc.append([r, c])
    meta["cases"]["encode"] = enc

    # --- xnor_gemm: the acceptance sweep's lengths (acceptance.cpp:61-79) + larger K
    gemm = []
    shapes = [(1, 1, 1), (3, 4, 31), (5, 7, 32), (16, 16, 33), (9, 13, 40), (2, 3, 64),
              (11, 5, 96), (16, 9, 100), (64, 1024, 576), (33, 65, 1000), (130, 70, 9216)]
    for i, (m, n, L) in enumerate(shapes):
        w = ref.pack(pm1(ref, (m, L), 2000 + i), "rows")
        x = ref.pack(pm1(ref, (L, n), 3000 + i), "cols")
        arrays[f"gemm{i}_w"], arrays[f"gemm{i}_x"] = w, x
        arrays[f"gemm{i}_out"] = ref.xnor_gemm(w, x, L)
        gemm.append([m, n, L])
    meta["cases"]["gemm"] = gemm

    # --- im2col KAT (test_lowering.cpp:55-66)
    x = np.arange(1, 10, dtype=np.float32).reshape(1, 1, 3, 3)
    arrays["kat_im2col"] = ref.im2col(x, 0, [2, 2, 1, 1, 0, 0, 1, 1])

    # --- binary conv layers (network.cpp:65-79), incl. cfg2 (64 -> 64, 32x32, batch 1)
    convs = []
    geoms = [((2, 3, 6, 6), [3, 3, 1, 1, 1, 1, 3, 5]),
             ((1, 1, 4, 4), [1, 1, 1, 1, 0, 0, 1, 1]),
             ((3, 5, 9, 7), [3, 2, 2, 1, 1, 0, 5, 7]),
             ((2, 4, 8, 8), [5, 5, 1, 1, 2, 2, 4, 3]),
             ((1, 64, 32, 32), [3, 3, 1, 1, 1, 1, 64, 64])]
    for i, (shape, g) in enumerate(geoms):
        xs, ws, bs = 4000 + i, 5000 + i, 6000 + i
        xx = ref.fill_random(shape, xs)
        K = g[0] * g[1] * g[6]
        pw = ref.pack(ref.fill_random((g[7], K), ws), "rows", apply_sign=True)
        b = ref.fill_random((g[7],), bs)
        y = ref.conv_forward_binary(xx, pw, b, g)
        key = f"conv{i}"
        if y.size <= 20000:
            arrays[f"{key}_out"] = y
        convs.append({"shape": list(shape), "geom": g, "seeds": [xs, ws, bs], "fnv1a": ref.fnv1a(y)})
    meta["cases"]["conv"] = convs

    # --- binary linear layers (network.cpp:121-126), incl. cfg1 (M = N = K = 1024)
    lins = []
    for i, (K, N, M) in enumerate([(8, 6, 4), (33, 6, 4), (100, 17, 29), (1024, 1024, 1024)]):
        xs, ws, bs = 7000 + i, 8000 + i, 9000 + i
        xx = ref.fill_random((K, N), xs)
        pw = ref.pack(ref.fill_random((M, K), ws), "rows", apply_sign=True)
        b = ref.fill_random((M,), bs)
        y = ref.linear_forward_packed(xx, pw, b)
        if y.size <= 20000:
            arrays[f"lin{i}_out"] = y
        lins.append({"K": K, "N": N, "M": M, "seeds": [xs, ws, bs], "fnv1a": ref.fnv1a(y)})
    meta["cases"]["linear"] = lins

    # --- networks: default VGG-small (cfg3 topology) and three spec files
    nets = []
    net = ref.net_default(1)
    for B in (1, 4):
        xin = ref.fill_random((B, 3, 32, 32), ref.mix64(1, INPUT_STREAM))
        lg = net.forward(xin)
        arrays[f"net_default_b{B}"] = lg
        nets.append({"name": "default", "seed": 1, "batch": B, "fnv1a": ref.fnv1a(lg)})
    for spec in ("tiny_spec", "pad_injected_spec", "strided_spec"):
        path = os.path.join(GOLD, f"{spec}.json")
        js = json.load(open(path))
        n = ref.net_file(path)
        xin = ref.fill_random(tuple(js["input_shape"]), ref.mix64(js["seed"], INPUT_STREAM))
        lg = n.forward(xin)
        arrays[f"net_{spec}"] = lg
        nets.append({"name": spec, "seed": js["seed"], "batch": js["input_shape"][0],
                     "fnv1a": ref.fnv1a(lg)})
    meta["cases"]["network"] = nets

    # --- RNG pins (tensor.cpp:65-77)
    meta["mix64"] = {f"{s},{c}": ref.mix64(s, c) for s, c in [(0, 0), (1, 0), (1, 1), (7, 123456789),
                                                              (2**63, 5)]}
    arrays["fill_random_s42"] = ref.fill_random((257,), 42)

    np.savez_compressed(os.path.join(GOLD, "golden.npz"), **arrays)
    with open(os.path.join(GOLD, "golden.json"), "w") as f:
        json.dump(meta, f, indent=1)
    sz = os.path.getsize(os.path.join(GOLD, "golden.npz"))
    print(f"wrote {len(arrays)} arrays ({sz/1024:.0f} KiB) and golden.json")


if __name__ == "__main__":
    main()
