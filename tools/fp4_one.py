import sys
import numpy as np
sys.path.insert(0, ".")
import paper_1911_04477_b200 as bnn  # noqa: E402
from oracle import Oracle  # noqa: E402
orc = Oracle(); lib = bnn.load()
lib.bnn_set_fused_fp4(int(sys.argv[1]) if len(sys.argv) > 1 else 1)
net = bnn.Network(seed=1)
x = orc.fill_random((1, 3, 32, 32), orc.mix64(1, 0x696E707574))
try:
    got = net.forward(x)
    want = orc.net(seed=1).forward(x)
    print("equal", np.array_equal(got, want), np.abs(got - want).max())
except Exception as e:
    print("ERR", e)
