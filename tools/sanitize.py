"""compute-sanitizer driver: one forward of the default network per engine setting and batch,
each checked against the oracle (run under `compute-sanitizer --tool memcheck|racecheck|synccheck`).

    python tools/sanitize.py [quick]   # quick: the default setting at batches 1 and 5 only
    python tools/sanitize.py tma       # the TMA-fed kernels: xnor4t CTA pairs, lin4 TMA-loaded images
"""
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_1911_04477_b200 as bnn  # noqa: E402
from oracle import Oracle  # noqa: E402

orc = Oracle()
lib = bnn.load()
SETTINGS = {"default": {}, "split16": {"split": 16, "lin4": 0}, "nosplit": {"split": 1, "lin4": 0},
            "nohalo": {"halo": 0}, "halostream": {"halo": 2}, "nolin4": {"lin4": 0},
            "swapall": {"swap": 2, "halo": 0}, "noswap": {"swap": 0, "halo": 0}, "nosmall": {"small": 0},
            "nopixpopc": {"pix": 0}, "pixf32": {"pix": 1}, "pixpacked": {"pix": 2}, "halo0": {"halo0": 1},
            "nopair": {"pair": 0, "halo": 0}, "pair224": {"pair": 3, "halo": 0}, "fp4all": {"fp4": 2}, "nofp4": {"fp4": 0}}
QUICK = len(sys.argv) > 1 and sys.argv[1] == "quick"
if QUICK:
    SETTINGS = {"default": {}}
bad = 0
if len(sys.argv) > 1 and sys.argv[1] == "tma":
    SETTINGS = {}
    lib.bnn_set_gemm_policy(3)  # xnor4t: CTA pairs when there are >= 2 row tiles
    for (m, n, L) in ((300, 481, 257), (129, 241, 2050), (1024, 600, 1030)):
        w = orc.pack(orc.fill_random((m, L), m), "rows", True)
        xx = orc.pack(orc.fill_random((L, n), n), "cols", True)
        got = bnn.xnor_gemm(bnn.PackedBitMatrix(m, L, "rows", w), bnn.PackedBitMatrix(L, n, "cols", xx), L)
        ok = np.array_equal(got, orc.xnor_gemm(w, xx, L)) and lib.bnn_last_gemm_kernel().decode() == "xnor4t_kernel"
        bad += not ok
        print("xnor4t", m, n, L, ok, flush=True)
    lib.bnn_set_gemm_policy(0)
    G = [{"kind": "affine_norm"}, {"kind": "htanh"}, {"kind": "sign"}]
    layers = [{"kind": "linear", "out_features": 992}] + G + [{"kind": "linear", "out_features": 544}] + G + \
             [{"kind": "linear", "out_features": 10}]
    for mode, b in ((2, 5), (1, 600)):  # forced TMA-loaded images / auto (e2m1 epilogue hand-off)
        lib.bnn_set_fused_lin4(mode)
        net = bnn.Network(layers, (2336, 1, 1), 41)
        net.set_engine("fused")
        x = orc.fill_random((b, 2336, 1, 1), 7)
        ok = np.array_equal(net.forward(x), orc.net(layers, (2336, 1, 1), 41).forward(x))
        bad += not ok
        print("lin4 tma", mode, b, ok, flush=True)
    lib.bnn_set_fused_lin4(1)
for name, st in SETTINGS.items():
    lib.bnn_set_fused_split(st.get("split", 0))
    lib.bnn_set_fused_halo(st.get("halo", 1))
    lib.bnn_set_fused_halo0(st.get("halo0", 0))
    lib.bnn_set_fused_lin4(st.get("lin4", 1))
    lib.bnn_set_fused_swap(st.get("swap", 1))
    lib.bnn_set_fused_small_logits(st.get("small", 1))
    lib.bnn_set_fused_pix_popc(st.get("pix", 3))
    lib.bnn_set_fused_fp4_pair(st.get("pair", 1))
    lib.bnn_set_fused_fp4(st.get("fp4", 1))
    for b in ((1, 5) if QUICK else (1, 5, 130)):
        net = bnn.Network(seed=1)
        x = orc.fill_random((b, 3, 32, 32), orc.mix64(1, 0x696E707574))
        ok = np.array_equal(net.forward(x), orc.net(seed=1).forward(x))
        bad += not ok
        print(name, b, ok, flush=True)
net = bnn.Network(seed=1)
net.set_engine("float")
x = orc.fill_random((2, 3, 32, 32), 3)
print("float", net.forward(x).shape)
sys.exit(1 if bad else 0)
