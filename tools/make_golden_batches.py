"""Golden logits for the default network at the benchmarked batch sizes, from the UNMODIFIED
reference (oracle/_ref). Run in the build container (where /root/reference exists):

    make -C oracle ref && python tools/make_golden_batches.py

The reference's network_forward is per-image independent (network.cpp:71-78) and the bench
input is the counter-based fill_random stream (bench.cpp:68-78), so batch B's logits are the
first B columns of the largest batch's: one reference run over 65536 images gives every
batch's FNV-1a logits hash (bench.cpp:23-33). Writes tests/golden/default_net_batches.json
(hashes) and tests/golden/default_net_b256.npy (the full [10, 256] logits of the headline batch).
"""
from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import RefLib  # noqa: E402

GOLD = os.path.join(ROOT, "tests", "golden")
INPUT_STREAM = 0x696E707574
BATCHES = [1, 2, 3, 4, 64, 129, 256, 511, 512, 513, 1000, 1024, 2048, 4096, 8192, 16384, 65536]


def main():
    ref = RefLib()
    net = ref.net_default(1)
    big = max(BATCHES)
    x = ref.fill_random((big, 3, 32, 32), ref.mix64(1, INPUT_STREAM))
    t0 = time.time()
    chunk = 512  # bounded memory: the reference materialises every layer's float activations
    lg = np.concatenate([net.forward(x[i:i + chunk], batch_threads=os.cpu_count() or 1)
                         for i in range(0, big, chunk)], axis=1)
    dt = time.time() - t0
    hashes = {str(b): ref.fnv1a(np.ascontiguousarray(lg[:, :b])) for b in BATCHES}
    meta = {"network": "build_default_network(Binary, seed 1)", "input": "fill_random(B,3,32,32, mix64(1, 'input'))",
            "reference_isa": ref.isa, "fnv1a": hashes, "seconds": round(dt, 1)}
    with open(os.path.join(GOLD, "default_net_batches.json"), "w") as f:
        json.dump(meta, f, indent=1)
    np.save(os.path.join(GOLD, "default_net_b256.npy"), np.ascontiguousarray(lg[:, :256]))
    print(f"{big} images in {dt:.1f} s; wrote {len(hashes)} hashes")


if __name__ == "__main__":
    main()
