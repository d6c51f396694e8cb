"""Time the K3 GEMM kernels on device-resident packed operands (CUDA events).

    python tools/gemm_bench.py [--shapes M,N,K ...] [--iters 20]
Prints one JSON line per (shape, kernel) with ms per launch and T bops/s (2 per bit-MAC).
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1911_04477_b200 as bnn  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shapes", nargs="*", default=["1024,1024,1024", "4096,1024,9216", "4096,1024,4096",
                                                    "1000,1024,4096", "4096,4096,4096", "128,262144,1152",
                                                    "8192,8192,8192"])
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--kernels", default="popc,umma,tma")
    a = ap.parse_args()
    lib = bnn.load()
    s = torch.cuda.current_stream().cuda_stream
    for sh in a.shapes:
        M, N, L = (int(v) for v in sh.split(","))
        wpl = (L + 31) // 32
        w = torch.randint(-2**31, 2**31 - 1, (M, wpl), dtype=torch.int32, device="cuda")
        x = torch.randint(-2**31, 2**31 - 1, (N, wpl), dtype=torch.int32, device="cuda")
        if L % 32:
            mask = (1 << (L % 32)) - 1
            w[:, -1] &= mask
            x[:, -1] &= mask
        out = torch.empty((M, N), dtype=torch.int32, device="cuda")
        ref = None
        for k in a.kernels.split(","):
            lib.bnn_set_gemm_policy({"popc": 1, "umma": 2, "tma": 3}[k])
            run = lambda: bnn._lib.check(lib.bnn_xnor_gemm_s32(w.data_ptr(), wpl, x.data_ptr(), wpl, M, N, L,
                                                               out.data_ptr(), N, s))
            for _ in range(3):
                run()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(a.iters):
                run()
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / a.iters
            dev_ms = None
            try:  # device-only: the calls captured into one CUDA graph (host overhead excluded)
                st = torch.cuda.Stream()
                g = torch.cuda.CUDAGraph()
                with torch.cuda.stream(st):
                    run_s = lambda: bnn._lib.check(lib.bnn_xnor_gemm_s32(w.data_ptr(), wpl, x.data_ptr(), wpl, M, N, L,
                                                                         out.data_ptr(), N, st.cuda_stream))
                    run_s()
                    st.synchronize()
                    with torch.cuda.graph(g, stream=st):
                        for _ in range(5):
                            run_s()
                    g.replay()
                    st.synchronize()
                    e0.record(st)
                    g.replay()
                    e1.record(st)
                    st.synchronize()
                dev_ms = e0.elapsed_time(e1) / 5
            except Exception as e:  # noqa: BLE001
                dev_ms = f"not capturable: {e}"
            same = None
            if ref is None:
                ref = out.clone()
            else:
                same = bool(torch.equal(ref, out))
            print(json.dumps({"M": M, "N": N, "L": L, "kernel": lib.bnn_last_gemm_kernel().decode(),
                              "ms": round(ms, 4), "Tbops": round(2 * M * N * L / ms / 1e9, 1),
                              "device_ms": dev_ms if not isinstance(dev_ms, float) else round(dev_ms, 4),
                              "device_Tbops": round(2 * M * N * L / dev_ms / 1e9, 1) if isinstance(dev_ms, float) else None,
                              "matches_first": same}), flush=True)
    lib.bnn_set_gemm_policy(0)


if __name__ == "__main__":
    main()
