"""compute-sanitizer driver: one forward of the default network per engine setting and batch,
each checked against the oracle (run under `compute-sanitizer --tool memcheck|racecheck|synccheck`).

    python tools/sanitize.py [quick]   # quick: the default setting at batches 1 and 5 only
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
