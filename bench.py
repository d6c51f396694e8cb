"""Benchmark driver: BNN VGG-small CIFAR-10 inference (binary conv/FC hot path) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--batch B] [--impl ours|reference]

Workload (BASELINE.json configs[2], the images/sec half of the headline metric): the
reference's default network (build_default_network, network.cpp:422-465: six binary 3x3 convs
128/128p/256/256p/512/512p + binary FC 1024/1024/10 with affine-htanh-sign between layers),
seed 1, synthetic 32x32x3 input from the reference generator (fill_random with the bench
input stream, bench.cpp:68-78), batch B per GPU (default 256). A step = one full
network_forward of one batch through the fused engine (one tcgen05 launch per weighted layer,
replayed as a CUDA graph). Multi-GPU (torchrun): each rank runs its contiguous batch shard
independently with replicated packed weights; the only collective is the final NCCL logits
gather.

Timing: W warm-up steps, then K steps bracketed by barrier + cuda.synchronize; each step is
timed with CUDA events on the launching stream, L2 is flushed before every step (a 256 MiB
write, outside the events); value = images of all ranks / the MAX over ranks of the summed
step times. A second, separately timed pass records per-layer CUDA events for the breakdown
and the dominant kernel's per-launch time (roofline). Parity: the logits of the last TIMED
step, assembled across ranks into the global [10, world*B] matrix, are hashed (FNV-1a,
bench.cpp:23-33) and compared with the unmodified reference's hash of the same batch
(tests/golden/default_net_batches.json) and, at the headline batch, with the reference run live.

--impl reference: the UNMODIFIED reference CPU implementation (oracle/_ref, compiled from
/root/reference/proj) on this host's cores, rank 0 only, the same batch per step.

--stub-oracle (tests only): the same N>1 driver path on CPU processes over gloo, with the
device forward replaced by the compiled reference / C oracle (tests/test_multigpu.py).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

INPUT_STREAM = 0x696E707574  # bench.cpp:76-77
IMG = 3 * 32 * 32
L2_FLUSH_BYTES = 256 << 20
METRIC = "BNN CIFAR-10 (VGG-small, binary conv/FC) inference images/sec"
WORKLOAD = "cfg3 BNN VGG-small CIFAR-10 forward (BASELINE.json configs[2]), all binary conv/FC layers"
GOLDEN = os.path.join(ROOT, "tests", "golden", "default_net_batches.json")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--batch", type=int, default=256, help="images per GPU per step")
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="target CPU time of the cpu_baseline sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-sweep", action="store_true")
    ap.add_argument("--sweep", default="1,64,1024,4096,16384,65536", help="per-GPU batch sweep (cfg5)")
    ap.add_argument("--no-configs", action="store_true", help="skip the per-config section (cfg1/2/4, K1/K2)")
    ap.add_argument("--stub-oracle", action="store_true", help=argparse.SUPPRESS)
    return ap.parse_args()


def dist_env():
    return int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")), int(os.environ.get("LOCAL_RANK", "0"))


def golden_hash(total: int):
    try:
        return json.load(open(GOLDEN))["fnv1a"].get(str(total))
    except (OSError, ValueError):
        return None


def cpu_info():
    """CPU model and the ISA flags that pick the reference's popcount path."""
    model, flags = None, set()
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name") and model is None:
                model = line.split(":", 1)[1].strip()
            elif line.startswith("flags") and not flags:
                flags = set(line.split(":", 1)[1].split())
    except OSError:
        pass
    keep = ["popcnt", "avx2", "fma", "avx512f", "avx512bw", "avx512vl", "avx512_vpopcntdq", "avx512_bitalg"]
    return {"model": model, "threads": os.cpu_count(), "isa_flags": [f for f in keep if f in flags]}


# ------------------------------------------------------------------------ clocks


class ClockSampler:
    """SM clock + throttle reasons sampled (NVML, every 5 ms) while the timed region runs."""

    def __init__(self, index: int):
        self.index, self.samples, self.reasons, self.stop_ev = index, [], set(), threading.Event()
        self.smax, self.err = None, None

    def start(self):
        try:
            import pynvml as nv

            nv.nvmlInit()
            self.nv = nv
            self.h = nv.nvmlDeviceGetHandleByIndex(self.index)
            self.smax = nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM)
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        except Exception as e:  # no NVML: record why
            self.err = f"nvml unavailable: {e}"

    def _run(self):
        nv = self.nv
        names = {nv.nvmlClocksEventReasonHwSlowdown: "hw_slowdown",
                 nv.nvmlClocksEventReasonHwThermalSlowdown: "hw_thermal_slowdown",
                 nv.nvmlClocksEventReasonSwThermalSlowdown: "sw_thermal_slowdown",
                 nv.nvmlClocksEventReasonSwPowerCap: "sw_power_cap",
                 nv.nvmlClocksEventReasonHwPowerBrakeSlowdown: "hw_power_brake"}
        while not self.stop_ev.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, n in names.items():
                    if r & bit:
                        self.reasons.add(n)
            except Exception:
                pass
            time.sleep(0.005)

    def stop(self):
        if self.err:
            return {"sm_mhz": None, "sm_max_mhz": None, "samples": 0, "reasons": [self.err]}
        self.stop_ev.set()
        self.t.join(timeout=2)
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None, "sm_max_mhz": self.smax,
                "samples": len(self.samples), "reasons": sorted(self.reasons), "source": "nvml, 5 ms"}


# ------------------------------------------------------------------ CPU baseline


def cpu_reference_rate(seconds: float, seed: int):
    """The UNMODIFIED reference network_forward(Binary) on this host's cores (batch-sharded over
    all host threads; the reference is re-entrant; threads = 1 GEMM setting)."""
    from oracle import RefLib

    ref = RefLib()
    net = ref.net_default(seed)
    cores = os.cpu_count() or 1
    x = ref.fill_random((cores, 3, 32, 32), ref.mix64(seed, INPUT_STREAM))
    t0 = time.perf_counter()
    net.forward(x, batch_threads=cores)
    rounds = max(1, int(seconds / max(time.perf_counter() - t0, 1e-3)))
    n = cores * rounds
    x = ref.fill_random((n, 3, 32, 32), ref.mix64(seed, INPUT_STREAM))
    t0 = time.perf_counter()
    net.forward(x, batch_threads=cores)
    dt = time.perf_counter() - t0
    return n / dt, cores, ref.isa, f"{n} images of the same network and input stream"


# ------------------------------------------------------------------ peaks


def measured_peaks():
    """Roofline denominators from the driver-written MEASURED_PEAKS.json: dense bf16 cuBLAS
    (burst) x4 for FP4 (kind::mxf4) and x2 for int8 (B200 dense FP4 : int8 : bf16 = 4 : 2 : 1),
    HBM copy bandwidth; the B200_PROFILING.md fallback when the file is absent."""
    try:
        pk = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        return {"bf16": pk["bf16_tflops"], "int8": 2 * pk["bf16_tflops"], "fp4": 4 * pk["bf16_tflops"],
                "hbm_gbs": pk["hbm_gbs"], "source": "MEASURED_PEAKS.json (bf16 burst x2 int8, x4 FP4; hbm_gbs)"}
    except (OSError, ValueError, KeyError):
        return {"bf16": 1590.0, "int8": 3180.0, "fp4": 6360.0, "hbm_gbs": 6650.0,
                "source": "fallback: B200_PROFILING.md 1.59 PFLOP/s bf16, 6.65 TB/s"}


def probe_peaks(lib, S):
    """In-run probes at this run's clocks: the tcgen05 dispatch rates the engine's kernels issue
    (kind::mxf4 and kind::i8, M=128 N=256), and cuBLASLt int8 (torch._int_mm 8192^3)."""
    import ctypes as C

    import torch

    from paper_1911_04477_b200 import _lib

    out = {}
    a, b = C.c_double(), C.c_double()
    for kind, name in ((1, "tcgen05_mxf4_tops"), (0, "tcgen05_i8_tops")):
        try:
            _lib.check(lib.bnn_probe_umma_peak(kind, 256, C.byref(a), C.byref(b), S))
            out[name] = a.value / 1e12
            out[name.replace("_tops", "_cycles_per_mma")] = b.value
        except Exception as e:
            out[name] = f"unavailable: {e}"
    try:
        n = 8192
        x = torch.randint(-64, 64, (n, n), dtype=torch.int8, device="cuda")
        y = torch.randint(-64, 64, (n, n), dtype=torch.int8, device="cuda")
        for _ in range(3):
            torch._int_mm(x, y)
        torch.cuda.synchronize()
        best = 1e9
        for _ in range(10):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            torch._int_mm(x, y)
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        out["cublaslt_int8_tops"] = 2 * n ** 3 / (best * 1e-3) / 1e12
        del x, y
    except Exception as e:
        out["cublaslt_int8_tops"] = f"unavailable: {e}"
    return out


# ------------------------------------------------------------ per-config section


FC_STACK = [{"kind": "linear", "out_features": 4096}, {"kind": "linear", "out_features": 4096},
            {"kind": "linear", "out_features": 1000}]  # BASELINE.json configs[3]


def _dev_time(fn, st, flush, iters):
    """Mean ms of fn() over iters runs on stream st, each timed with CUDA events and preceded by
    an L2 flush (a 256 MiB write outside the events)."""
    import torch

    with torch.cuda.stream(st):
        for _ in range(3):
            fn()
        st.synchronize()
        tot = 0.0
        for i in range(iters):
            flush.fill_(float(i))
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            fn()
            e1.record(st)
            st.synchronize()
            tot += e0.elapsed_time(e1)
    return tot / iters


def _graph_time(fn, st, flush, reps=20):
    """Device ms per call of fn() (a stream-ordered C-ABI call on st): `reps` calls captured into
    one CUDA graph and replayed between CUDA events, so host-side call overhead (ctypes, argument
    checks, launch) is not in the number; L2 is flushed before the replay (outside the events),
    the calls inside run back to back (operands L2-warm after the first). None if the call
    sequence cannot be captured."""
    import torch

    try:
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(st):
            fn()
            st.synchronize()
            with torch.cuda.graph(g, stream=st):
                for _ in range(reps):
                    fn()
            g.replay()
            st.synchronize()
            tot = 0.0
            for i in range(3):
                flush.fill_(float(i))
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(st)
                g.replay()
                e1.record(st)
                st.synchronize()
                tot += e0.elapsed_time(e1)
        return tot / 3 / reps
    except Exception:  # not capturable: report the host-visible timing only
        return None


def _max_over_ranks(v: float, world: int, dev) -> float:
    if world == 1:
        return v
    import torch
    import torch.distributed as dist

    t = torch.tensor([v], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def measure_configs(lib, dev, st, flush, seed, peaks, cpu, world, rank):
    """BASELINE.json's other named shapes on this GPU (device-resident inputs, L2 flushed before
    every timed call). At N > 1 the batch-like dimension is sharded across ranks with replicated
    weights (cfg1's N columns, cfg4's images; cfg2's single image runs as
    independent replicas), each rank times its share, and the job time is the max over ranks.
    At N = 1 also: the HBM-bound encoders' achieved bandwidth, the K3 pipe probes, the float
    control group, and the unmodified reference CPU path on the same shapes (cpu set)."""
    import ctypes as C

    import numpy as np
    import torch

    import paper_1911_04477_b200 as bnn
    from paper_1911_04477_b200 import _lib
    from paper_1911_04477_b200.shard import shard_range

    S = st.cuda_stream
    out = {}
    hbm = peaks["hbm_gbs"]
    int8_peak, fp4_peak = peaks["int8"], peaks["fp4"]

    def fill(shape, sd, offset=0):
        t = torch.empty(shape, dtype=torch.float32, device=dev)
        _lib.check(lib.bnn_fill_random_f32(sd, offset, t.numel(), t.data_ptr(), S))
        return t

    def packed_rows(M, K, sd):
        w = fill((M, K), sd)
        wpl = (K + 31) // 32
        pw = torch.empty((M, wpl), dtype=torch.int32, device=dev)
        _lib.check(lib.bnn_sign_pack_rows_f32(w.data_ptr(), M, K, pw.data_ptr(), wpl, S))
        return pw, wpl

    ref = None
    if cpu and world == 1:
        try:
            from oracle import RefLib

            ref = RefLib()
        except Exception as e:
            out["cpu_reference"] = f"unavailable: {e}"
    cores = os.cpu_count() or 1

    def cpu_ms(fn, reps=3):
        fn()
        t0 = time.perf_counter()
        for _ in range(reps):
            fn()
        return 1e3 * (time.perf_counter() - t0) / reps

    # cfg1: single binary linear layer, encode + xnor GEMM (+ bias), M = N = K = 1024; the N
    # (batch) columns are split across ranks
    M = N = K = 1024
    c0, nc = shard_range(N, world, rank)
    xfull = fill((K, N), bnn.mix64(seed, 11))
    x = xfull[:, c0:c0 + nc].contiguous()
    del xfull
    pw, wpl = packed_rows(M, K, bnn.mix64(seed, 12))
    bias = fill((M,), bnn.mix64(seed, 13))
    y = torch.empty((M, nc), dtype=torch.float32, device=dev)
    lines = torch.empty((nc, wpl), dtype=torch.int32, device=dev)
    acc = torch.empty((M, nc), dtype=torch.int32, device=dev)
    f_lin = lambda: _lib.check(lib.bnn_linear_forward_packed_f32(x.data_ptr(), K, nc, pw.data_ptr(), wpl, M,
                                                                 bias.data_ptr(), y.data_ptr(), S))
    f_enc = lambda: _lib.check(lib.bnn_sign_pack_cols_f32(x.data_ptr(), K, nc, lines.data_ptr(), wpl, S))
    f_gemm = lambda: _lib.check(lib.bnn_xnor_gemm_s32(pw.data_ptr(), wpl, lines.data_ptr(), wpl, M, nc, K,
                                                      acc.data_ptr(), nc, S))
    ms = _max_over_ranks(_dev_time(f_lin, st, flush, 20), world, dev)
    gemm_kernel = lib.bnn_last_gemm_kernel().decode()
    ms_enc = _max_over_ranks(_dev_time(f_enc, st, flush, 20), world, dev)
    ms_gemm = _max_over_ranks(_dev_time(f_gemm, st, flush, 20), world, dev)
    dev_lin, dev_enc, dev_gemm = (_graph_time(f, st, flush) for f in (f_lin, f_enc, f_gemm))
    bops = 2.0 * M * N * K
    c1 = {"shape": "linear_forward_packed x[1024,1024] f32, W 1024x1024 packed (BASELINE configs[0])",
          "sharding": f"{world} rank(s) x {nc} columns", "ms": ms, "binary_tops": bops / (ms * 1e-3) / 1e12,
          "gemm_kernel": gemm_kernel, "encode_ms": ms_enc, "xnor_gemm_ms": ms_gemm,
          "xnor_gemm_tops": bops / (ms_gemm * 1e-3) / 1e12,
          "xnor_gemm_frac_of_int8_peak": (bops / (ms_gemm * 1e-3) / 1e12) / int8_peak,
          "device_ms": {"linear_forward_packed": dev_lin, "encode": dev_enc, "xnor_gemm": dev_gemm,
                        "timer": "graph of 20 back-to-back C-ABI calls, per call (host call overhead excluded)"},
          "xnor_gemm_device_tops": bops / (dev_gemm * 1e-3) / 1e12 if dev_gemm else None}
    if ref is not None:
        xh = x.cpu().numpy()
        ph = pw.cpu().numpy().view(np.uint32)
        bh = bias.cpu().numpy()
        c1["cpu_reference_ms"] = cpu_ms(lambda: ref.linear_forward_packed(xh, ph, bh, threads=cores))
        c1["cpu_reference_threads"] = cores
        c1["parity_vs_reference"] = bool(np.array_equal(y.cpu().numpy(), ref.linear_forward_packed(xh, ph, bh)))
    out["cfg1_linear_1024"] = c1
    del x, y, lines, acc

    # cfg2: binary 3x3 conv 64 -> 64 on 32x32, batch 1 (encode + im2col + xnor GEMM + epilogue);
    # one image does not shard: at N > 1 every rank serves its own batch-1 request (replicas)
    g = _lib.ConvGeom(3, 3, 1, 1, 1, 1, 64, 64)
    xc = fill((1, 64, 32, 32), bnn.mix64(seed, 21))
    pwc, wplc = packed_rows(64, 576, bnn.mix64(seed, 22))
    bc = fill((64,), bnn.mix64(seed, 23))
    yc = torch.empty((1, 64, 32, 32), dtype=torch.float32, device=dev)
    f_conv = lambda: _lib.check(lib.bnn_conv_forward_binary_f32(xc.data_ptr(), 1, 64, 32, 32, pwc.data_ptr(), wplc,
                                                                bc.data_ptr(), C.byref(g), yc.data_ptr(), S))
    ms = _max_over_ranks(_dev_time(f_conv, st, flush, 30), world, dev)
    c2 = {"shape": "conv_forward_binary x[1,64,32,32], 3x3 pad 1, D=64 (BASELINE configs[1])", "ms": ms,
          "sharding": "replicas (one image per request)" if world > 1 else "single GPU",
          "requests_per_s": world / (ms * 1e-3),
          "binary_tops": world * 2.0 * 64 * 576 * 1024 / (ms * 1e-3) / 1e12,
          "gemm_kernel": lib.bnn_last_gemm_kernel().decode(), "note": "75.5 M bops per request: latency bound",
          "device_ms": _graph_time(f_conv, st, flush)}
    if ref is not None:
        xh, ph, bh = xc.cpu().numpy(), pwc.cpu().numpy().view(np.uint32), bc.cpu().numpy()
        geo = [3, 3, 1, 1, 1, 1, 64, 64]
        c2["cpu_reference_ms"] = cpu_ms(lambda: ref.conv_forward_binary(xh, ph, bh, geo, threads=cores), reps=10)
        c2["cpu_reference_threads"] = cores
        c2["parity_vs_reference"] = bool(np.array_equal(yc.cpu().numpy(), ref.conv_forward_binary(xh, ph, bh, geo)))
    out["cfg2_conv_64_32x32_b1"] = c2

    # cfg4: AlexNet-sized binary FC stack 9216 -> 4096 -> 4096 -> 1000, batch 1024 (images split
    # across ranks)
    Bf = 1024
    i0, nb = shard_range(Bf, world, rank)
    net = bnn.Network(FC_STACK, (9216, 1, 1), seed)
    xf = fill((nb, 9216, 1, 1), bnn.mix64(seed, INPUT_STREAM), i0 * 9216)
    yf = torch.empty((1000, nb), dtype=torch.float32, device=dev)
    ms = _max_over_ranks(_dev_time(lambda: net.forward_device(xf, yf, S), st, flush, 20), world, dev)
    fc_bops = 2.0 * Bf * (9216 * 4096 + 4096 * 4096 + 4096 * 1000)
    c4 = {"shape": "NetworkSpec [1024, 9216, 1, 1] -> linear 4096 -> 4096 -> 1000 (BASELINE configs[3])",
          "sharding": f"{world} rank(s) x {nb} images", "ms": ms, "images_per_s": Bf / (ms * 1e-3),
          "binary_tops": fc_bops / (ms * 1e-3) / 1e12, "frac_of_int8_peak": (fc_bops / (ms * 1e-3) / 1e12) / int8_peak,
          "frac_of_fp4_peak": (fc_bops / (ms * 1e-3) / 1e12) / fp4_peak,
          "engine": net.engine, "launches": net.last_launches(),
          "kernels": [net_kernel for net_kernel in (lib.bnn_net_layer_kernel(net.handle, i).decode() for i in range(3))]}
    if ref is not None:
        import tempfile

        spec = {"input_shape": [1, 9216, 1, 1], "seed": seed, "binarize_weights": False, "kernel": "binary",
                "layers": FC_STACK}
        with tempfile.NamedTemporaryFile("w", suffix=".json", delete=False) as fh:
            json.dump(spec, fh)
            path = fh.name
        try:
            rnet = ref.net_file(path)
            nb_cpu = 64  # bounded sample: the reference's linear layers cost the same per image
            xh = xf[:nb_cpu].cpu().numpy()
            t0 = time.perf_counter()
            want = rnet.forward(xh, threads=cores)
            dt = time.perf_counter() - t0
            c4["cpu_reference_images_per_s"] = nb_cpu / dt
            c4["cpu_reference_threads"] = cores
            c4["cpu_reference_sample"] = f"{nb_cpu} images"
            c4["parity_vs_reference"] = bool(np.array_equal(yf[:, :nb_cpu].cpu().numpy(), want))
        finally:
            os.unlink(path)
    out["cfg4_fc_stack_b1024"] = c4
    del xf, yf, net
    if world > 1:
        return out

    # The paper's comparison: the binary network vs the float control group
    # (ExecKernel::Float, CUDA-core FP32 without vendor libraries, csrc/control.cu) on this GPU
    Bc = 256
    netf = bnn.Network(seed=seed)
    netf.set_engine("float")
    xc2 = fill((Bc, 3, 32, 32), bnn.mix64(seed, INPUT_STREAM))
    yc2 = torch.empty((10, Bc), dtype=torch.float32, device=dev)
    ms_f = _dev_time(lambda: netf.forward_device(xc2, yc2, S), st, flush, 3)
    netb = bnn.Network(seed=seed)
    ms_b = _dev_time(lambda: netb.forward_device(xc2, yc2, S), st, flush, 20)
    out["control_group_vgg_b256"] = {
        "shape": "default network (cfg3) batch 256: binary fused engine vs float control group",
        "float_ms": ms_f, "float_images_per_s": Bc / (ms_f * 1e-3), "binary_ms": ms_b,
        "binary_images_per_s": Bc / (ms_b * 1e-3), "binary_over_float": ms_f / ms_b,
        "paper": "GTX 1080 Ti: binary 3.57 s vs control 11.23 s per 10k images (3.1x), PAPER.md:193-197"}
    del netf, netb, xc2, yc2

    # K1 encoder, HBM-bound: pack_cols(sign(X)) of a 1 GiB float matrix (> L2)
    Lk, Nk = 16384, 16384
    xe = torch.empty((Lk, Nk), dtype=torch.float32, device=dev)
    _lib.check(lib.bnn_fill_random_f32(bnn.mix64(seed, 31), 0, xe.numel(), xe.data_ptr(), S))
    wple = Lk // 32
    le = torch.empty((Nk, wple), dtype=torch.int32, device=dev)
    ms = _dev_time(lambda: _lib.check(lib.bnn_sign_pack_cols_f32(xe.data_ptr(), Lk, Nk, le.data_ptr(), wple, S)),
                   st, flush, 5)
    byt = Lk * Nk * 4 + Nk * wple * 4
    msr = _dev_time(lambda: _lib.check(lib.bnn_sign_pack_rows_f32(xe.data_ptr(), Lk, Nk, le.data_ptr(), wple, S)),
                    st, flush, 5)
    out["k1_sign_pack"] = {"shape": "float [16384, 16384] (1 GiB) -> packed", "bytes": byt,
                           "cols_ms": ms, "cols_gbs": byt / (ms * 1e-3) / 1e9, "cols_frac_hbm": byt / (ms * 1e-3) / 1e9 / hbm,
                           "rows_ms": msr, "rows_gbs": byt / (msr * 1e-3) / 1e9,
                           "rows_frac_hbm": byt / (msr * 1e-3) / 1e9 / hbm, "hbm_peak_gbs": hbm,
                           "peak_source": peaks["source"]}
    del xe, le

    # K2 binary im2col: x [256, 128, 32, 32] (128 MiB, > L2) -> packed K = 1152 lines
    g2 = _lib.ConvGeom(3, 3, 1, 1, 1, 1, 128, 128)
    xi = torch.empty((256, 128, 32, 32), dtype=torch.float32, device=dev)
    _lib.check(lib.bnn_fill_random_f32(bnn.mix64(seed, 41), 0, xi.numel(), xi.data_ptr(), S))
    li = torch.empty((256 * 1024, 36), dtype=torch.int32, device=dev)
    ms = _dev_time(lambda: _lib.check(lib.bnn_im2col_sign_pack_f32(xi.data_ptr(), 256, 128, 32, 32, C.byref(g2),
                                                                   li.data_ptr(), 36, S)), st, flush, 5)
    byt = xi.numel() * 4 + li.numel() * 4
    out["k2_im2col_sign_pack"] = {"shape": "x [256,128,32,32] f32 -> 262144 lines x 36 words", "bytes": byt, "ms": ms,
                                  "gbs": byt / (ms * 1e-3) / 1e9, "frac_hbm": byt / (ms * 1e-3) / 1e9 / hbm,
                                  "note": "algorithmic bytes = input once + packed output"}
    del xi, li

    # K3 pipe candidates (SURVEY §7 hard part 1): LOP3+POPC vs emulated b1 mma.sync vs tcgen05
    a, b = C.c_double(), C.c_double()
    _lib.check(lib.bnn_probe_popc_peak(C.byref(a), C.byref(b), S))
    popc = a.value / 1e12
    _lib.check(lib.bnn_probe_bmma_peak(C.byref(a), C.byref(b), S))
    bmma = a.value / 1e12
    out["k3_pipes_tbops"] = {"popc_lop3": popc, "b1_mma_sync_emulated": bmma,
                             "tcgen05_i8": peaks.get("probe", {}).get("tcgen05_i8_tops"),
                             "tcgen05_mxf4": peaks.get("probe", {}).get("tcgen05_mxf4_tops"),
                             "chosen": "tcgen05 kind::mxf4 (e2m1 operands, exact) for the packed-input convs "
                                       "(halo4 / swap4), the linear layers (lin4) and the standalone xnor_gemm "
                                       "above 2^26 bit-MACs (xnor4; xnor4t, TMA-fed, above 2^32); LOP3+POPC below it and for the pixel-input "
                                       "first conv and the logits",
                             "ncu_pipe_counters": "profiles/r02_k3_pipes_ncu.json"}

    # K3 on large GEMMs (the north star's ">= 50 % of the chosen pipe's peak for large GEMMs"):
    # standalone xnor_gemm (s32 output, the reference's IntMatrix) through the C ABI, AUTO policy
    # (the TMA-fed FP4 kernel, operands expanded once into HBM scratch inside the call)
    lg = {}
    for (Mg, Ng, Lg) in ((8192, 8192, 8192), (4096, 1024, 9216)):
        wplg = Lg // 32
        wg = torch.randint(-2**31, 2**31 - 1, (Mg, wplg), dtype=torch.int32, device=dev)
        xg = torch.randint(-2**31, 2**31 - 1, (Ng, wplg), dtype=torch.int32, device=dev)
        og = torch.empty((Mg, Ng), dtype=torch.int32, device=dev)
        fg = lambda: _lib.check(lib.bnn_xnor_gemm_s32(wg.data_ptr(), wplg, xg.data_ptr(), wplg, Mg, Ng, Lg,
                                                      og.data_ptr(), Ng, S))
        msg = _dev_time(fg, st, flush, 10)
        kern = lib.bnn_last_gemm_kernel().decode()
        tops = 2.0 * Mg * Ng * Lg / (msg * 1e-3) / 1e12
        e = {"ms": msg, "binary_tops": tops, "frac_of_fp4_peak": tops / fp4_peak, "kernel": kern}
        got = og.clone()
        _lib.check(lib.bnn_set_gemm_policy(1))  # the integer-pipe kernel on the same operands
        fg()
        _lib.check(lib.bnn_set_gemm_policy(0))
        st.synchronize()
        e["equal_to_popc_kernel"] = bool(torch.equal(got, og))
        if ref is not None:  # a 256 x 256 corner against the unmodified reference
            wh = wg[:256].cpu().numpy().view(np.uint32)
            xh = xg[:256].cpu().numpy().view(np.uint32)
            e["corner_parity_vs_reference"] = bool(np.array_equal(got[:256, :256].cpu().numpy(),
                                                                  ref.xnor_gemm(wh, xh, Lg, threads=cores)))
        lg[f"{Mg}x{Ng}x{Lg}"] = e
        del wg, xg, og, got
    out["k3_large_gemm"] = lg
    return out


# ---------------------------------------------------------------------- engines
# The headline loop is written once over an engine: the device (the product path) or, for the
# CPU tests of the N > 1 driver logic, a stub whose forward is the reference on the host.


class DeviceEngine:
    def __init__(self, args, world, rank, local):
        import torch

        import paper_1911_04477_b200 as bnn
        from paper_1911_04477_b200 import _lib

        self.torch, self.bnn, self._lib = torch, bnn, _lib
        torch.cuda.set_device(local)
        self.dev = torch.device("cuda", local)
        self.lib = bnn.load()
        self.st = torch.cuda.Stream(device=self.dev)
        self.S = self.st.cuda_stream
        self.net = bnn.Network(seed=args.seed)
        self.flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device=self.dev)

    def make_input(self, seed, offset, n):
        x = self.torch.empty((n, 3, 32, 32), dtype=self.torch.float32, device=self.dev)
        self._lib.check(self.lib.bnn_fill_random_f32(self.bnn.mix64(seed, INPUT_STREAM), offset, n * IMG,
                                                     x.data_ptr(), self.S))
        return x

    def logits_buffer(self, shape):
        return self.torch.empty(shape, dtype=self.torch.float32, device=self.dev)

    def forward(self, x, out):
        self.net.forward_device(x, out, self.S)

    def stream_ctx(self):
        return self.torch.cuda.stream(self.st)

    def synchronize(self):
        self.torch.cuda.synchronize()

    def before_step(self, i):
        self.flush.fill_(float(i))  # > L2 (126 MB): every step starts cold

    def timer(self):
        torch = self.torch
        st = self.st

        class T:
            def __init__(self):
                self.a, self.b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

            def start(self):
                self.a.record(st)

            def stop(self):
                self.b.record(st)

            def ms(self):
                return self.a.elapsed_time(self.b)

        return T()

    def hash(self, host_logits):
        return self.bnn.fnv1a_hash(host_logits)


class StubEngine:
    """CPU stand-in for tests: the same driver logic, the reference (or the C oracle) as the
    forward, perf_counter timing, gloo collectives."""

    def __init__(self, args, world, rank, local):
        import torch

        self.torch = torch
        self.dev = torch.device("cpu")
        try:
            from oracle import RefLib

            self.ref = RefLib()
            self.netf = self.ref.net_default(args.seed)
        except Exception:
            from oracle import Oracle

            self.ref = Oracle()
            self.netf = self.ref.net(seed=args.seed)

    def make_input(self, seed, offset, n):
        import numpy as np

        from oracle import Oracle

        orc = Oracle()
        x = np.empty((n, 3, 32, 32), np.float32)
        orc.lib.orc_fill_random(x.size, orc.mix64(seed, INPUT_STREAM), offset, x.ctypes.data)
        return x

    def logits_buffer(self, shape):
        return self.torch.empty(shape, dtype=self.torch.float32)

    def forward(self, x, out):
        out.copy_(self.torch.from_numpy(self.netf.forward(x)))

    def stream_ctx(self):
        import contextlib

        return contextlib.nullcontext()

    def synchronize(self):
        pass

    def before_step(self, i):
        pass

    def timer(self):
        class T:
            def start(self):
                self.t0 = time.perf_counter()

            def stop(self):
                self.t1 = time.perf_counter()

            def ms(self):
                return 1e3 * (self.t1 - self.t0)

        return T()

    def hash(self, host_logits):
        from oracle import Oracle

        import numpy as np

        a = np.ascontiguousarray(host_logits, np.float32)
        return int(Oracle().lib.orc_fnv1a(a.ctypes.data, a.size))


def headline(eng, args, world, rank):
    """W warm-up steps, K timed steps (per-step timers, max over ranks of the sum), then the
    parity of the LAST TIMED step's output: the per-rank logits gathered by the step's own
    collective are assembled into the global [F, world*B] matrix and hashed."""
    import torch
    import torch.distributed as dist

    from paper_1911_04477_b200.shard import assemble_gathered, input_offset, shard_range

    B = args.batch
    assert shard_range(B * world, world, rank)[1] == B
    x = eng.make_input(args.seed, input_offset(B * world, world, rank), B)
    logits = eng.logits_buffer((10, B))
    gathered = eng.logits_buffer((world, 10, B)) if world > 1 else None

    def step():
        eng.forward(x, logits)
        if world > 1:  # the only collective: the final logits gather
            if gathered.is_cuda:
                dist.all_gather_into_tensor(gathered, logits)
            else:  # gloo (the CPU test of this driver)
                dist.all_gather(list(gathered.unbind(0)), logits)

    clocks = None
    with eng.stream_ctx():
        for _ in range(max(args.warmup, 3)):
            step()
        eng.synchronize()
        timers = [eng.timer() for _ in range(args.steps)]
        if isinstance(eng, DeviceEngine):
            clocks = ClockSampler(torch.cuda.current_device())
            clocks.start()
        if world > 1:
            dist.barrier()
        eng.synchronize()
        for i in range(args.steps):
            eng.before_step(i)
            timers[i].start()
            step()
            timers[i].stop()
        eng.synchronize()
        if world > 1:
            dist.barrier()
    clk = clocks.stop() if clocks else None
    total_ms = _max_over_ranks(sum(t.ms() for t in timers), world, eng.dev)
    # parity of the timed output (rank 0): global [F, world*B] in the reference's layout
    full = assemble_gathered(gathered) if world > 1 else logits
    parity = None
    if rank == 0:
        lg = full.cpu().numpy()
        want = golden_hash(world * B)
        got = eng.hash(lg)
        parity = {"timed_output": f"logits of the last timed step, [10, {world * B}] assembled over {world} rank(s)",
                  "fnv1a": f"0x{got:016x}",
                  "reference_fnv1a": None if want is None else f"0x{want:016x}",
                  "match": None if want is None else bool(got == want)}
    return total_ms, clk, parity, logits, x


def live_reference_check(lg, B, seed, n=256):
    """The first min(B, n) columns of the timed logits against the compiled reference run now."""
    import numpy as np

    from oracle import RefLib

    ref = RefLib()
    k = min(B, n)
    x = ref.fill_random((k, 3, 32, 32), ref.mix64(seed, INPUT_STREAM))
    want = ref.net_default(seed).forward(x, batch_threads=os.cpu_count() or 1)
    return bool(np.array_equal(np.ascontiguousarray(lg[:, :k]), want)), k


# ---------------------------------------------------------------------- ours


def run_ours(args):
    import ctypes as C

    import torch
    import torch.distributed as dist

    world, rank, local = dist_env()
    if args.stub_oracle:
        if world > 1:
            dist.init_process_group("gloo")
        eng = StubEngine(args, world, rank, local)
        total_ms, _, parity, _, _ = headline(eng, args, world, rank)
        if rank == 0:
            ok = bool(parity and parity["match"])
            print(json.dumps({"metric": METRIC, "value": world * args.batch * args.steps / (total_ms * 1e-3),
                              "unit": "images/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
                              "ms_per_step": total_ms / args.steps, "higher_is_better": True, "scaling": "weak",
                              "vs_baseline": None, "data": "synthetic", "impl": "stub-oracle (CPU test of the driver)",
                              "config": {"workload": WORKLOAD, "batch_per_gpu": args.batch,
                                         "global_batch": args.batch * world},
                              "parity": parity, "parity_vs_oracle": ok}), flush=True)
        if world > 1:
            dist.destroy_process_group()
        return

    import numpy as np

    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    eng = DeviceEngine(args, world, rank, local)
    lib, net, st, S, dev, flush = eng.lib, eng.net, eng.st, eng.S, eng.dev, eng.flush
    from paper_1911_04477_b200 import _lib

    B = args.batch
    engine = net.engine
    n_layers = len(net.layers)
    total_ms, clk, parity, logits, x = headline(eng, args, world, rank)
    launches_per_step = net.last_launches()
    images = world * B * args.steps
    value = images / (total_ms * 1e-3)
    ms_per_step = total_ms / args.steps
    if rank == 0 and B <= 4096:
        try:  # the headline batch's timed logits against the reference run live on this host
            ok, k = live_reference_check(logits.cpu().numpy(), B, args.seed)
            parity["live_reference"] = {"images": k, "match": ok}
        except Exception as e:  # the checker must never break the benchmark line
            parity["live_reference"] = f"unavailable: {e}"

    # ---- separately timed pass: per-layer events (breakdown + the dominant kernel's launch time)
    lib.bnn_net_set_timing(net.handle, 1)
    lib.bnn_net_reset_timing(net.handle)
    prof_steps = max(5, min(args.steps, 20))
    with torch.cuda.stream(st):
        for i in range(prof_steps):
            flush.fill_(float(i))
            net.forward_device(x, logits, S)
        st.synchronize()
    lib.bnn_net_set_timing(net.handle, 0)
    layer_ms = (C.c_double * n_layers)()
    gemm_ms = (C.c_double * n_layers)()
    gemm_n = (C.c_size_t * n_layers)()
    _lib.check(lib.bnn_net_timing(net.handle, layer_ms, gemm_ms, gemm_n))
    shapes = []
    for i in range(n_layers):
        sh = (C.c_size_t * 8)()
        _lib.check(lib.bnn_net_layer_shape(net.handle, i, sh))
        shapes.append(list(sh))
    # algorithmic work per weighted layer and batch: 2*M*K*N tensor ops (1 MAC per bit-MAC;
    # = the bops of SURVEY.md §8(d): 1.2339 G per image for the whole network)
    ops = [2.0 * sh[1] * sh[2] * sh[3] * B if sh[3] else 0.0 for sh in shapes]
    top = max(range(n_layers), key=lambda i: gemm_ms[i])
    per_launch_ms = gemm_ms[top] / max(1, gemm_n[top])
    achieved = ops[top] / (per_launch_ms * 1e-3) / 1e12
    peaks = measured_peaks()
    if rank == 0:
        peaks["probe"] = probe_peaks(lib, S)
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        try:
            traffic = json.load(open(tpath)).get(f"b{B}", {}).get(f"layer{top}")
        except (ValueError, OSError):
            traffic = None
    kernel_name = (lib.bnn_net_layer_kernel(net.handle, top) or lib.bnn_last_gemm_kernel()).decode()
    fp4 = "mxf4" in kernel_name or "swap4" in kernel_name or "halo" in kernel_name
    kpeak = peaks["fp4"] if fp4 else peaks["int8"]
    probe = (peaks.get("probe") or {}).get("tcgen05_mxf4_tops" if fp4 else "tcgen05_i8_tops")

    # ---- end to end through the public API: every step copies its input from pinned host memory
    # (H2D), runs the forward, and reads its logits back (D2H). Steps are pipelined like a
    # serving loop: the copies on their own streams, so step i+1's H2D overlaps step i's forward.
    e2e = None
    if not args.no_e2e:
        hx = x.cpu().pin_memory()
        nbuf = 3  # input/output buffer sets: two steps in flight while the host reads a third
        dxs = [torch.empty_like(x) for _ in range(nbuf)]
        outs = [torch.empty((net.logits, B), dtype=torch.float32, device=dev) for _ in range(nbuf)]
        gat = [torch.empty((world, net.logits, B), dtype=torch.float32, device=dev) for _ in range(nbuf)]
        hys = [torch.empty((world, net.logits, B), dtype=torch.float32).pin_memory() for _ in range(nbuf)]
        s_h2d, s_d2h = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)
        ev_in = [torch.cuda.Event() for _ in range(nbuf)]
        ev_comp = [torch.cuda.Event() for _ in range(nbuf)]
        ev_out = [torch.cuda.Event() for _ in range(nbuf)]

        def issue(i):
            k = i % nbuf
            s_h2d.wait_event(ev_comp[k])  # step i-nbuf's forward is done with dxs[k]
            with torch.cuda.stream(s_h2d):
                dxs[k].copy_(hx, non_blocking=True)
                ev_in[k].record(s_h2d)
            st.wait_event(ev_in[k])
            st.wait_event(ev_out[k])  # step i-nbuf's D2H is done with outs[k] / gat[k]
            with torch.cuda.stream(st):
                net.forward_device(dxs[k], outs[k], S)
                if world > 1:
                    dist.all_gather_into_tensor(gat[k], outs[k])
                else:
                    gat[k][0].copy_(outs[k])
                ev_comp[k].record(st)
            s_d2h.wait_event(ev_comp[k])
            with torch.cuda.stream(s_d2h):
                hys[k].copy_(gat[k], non_blocking=True)
                ev_out[k].record(s_d2h)

        e2e_steps = max(args.steps, 2000)  # ~0.3 s host-timed: steadier against host jitter
        if world == 1:
            # N = 1: the library's native serving pipeline (bnn_pipe_*: H2D, forward, D2H of
            # each batch on copy / compute streams, enqueued from C++; each buffer set replays
            # its own captured graph), the call a user makes
            depth, lag = 6, 4  # buffer sets; the host reads step i-lag's logits after submitting step i
            pipe = net.pipeline(B, depth)
            hy1 = [torch.empty((net.logits, B), dtype=torch.float32).pin_memory() for _ in range(depth)]
            for i in range(3 * depth):  # each set: first sighting, capture, then replays
                pipe.wait(pipe.submit(hx.data_ptr(), hy1[i % depth].data_ptr()))
            base = 3 * depth
            t0 = time.perf_counter()
            for i in range(e2e_steps):
                pipe.submit(hx.data_ptr(), hy1[i % depth].data_ptr())
                if i >= lag:
                    pipe.wait(base + i - lag)
            for j in range(max(0, e2e_steps - lag), e2e_steps):
                pipe.wait(base + j)
            e2e_s = time.perf_counter() - t0
            pipe.close()
            e2e_ok = bool(np.array_equal(hy1[(e2e_steps - 1) % depth].numpy(), logits.cpu().numpy()))
        else:
            for i in range(4):
                issue(i)
            torch.cuda.synchronize()
            dist.barrier()
            t0 = time.perf_counter()
            for i in range(e2e_steps):
                issue(i)
                if i >= 2:
                    ev_out[(i - 2) % nbuf].synchronize()  # the host holds step i-2's logits
            for j in range(max(0, e2e_steps - 2), e2e_steps):
                ev_out[j % nbuf].synchronize()
            e2e_s = time.perf_counter() - t0
            e2e_ok = None
        e2e_s = _max_over_ranks(e2e_s, world, dev)
        e2e = {"value": world * B * e2e_steps / e2e_s, "unit": "images/s", "steps": e2e_steps,
               "h2d_bytes_per_step": B * IMG * 4,
               "d2h_bytes_per_step": net.logits * B * 4 * world,
               "timer": "host clock around max(K, 2000) pipelined steps (pinned H2D + forward + D2H of every "
                        "step; step i+1's copy overlaps step i's forward; N=1: 6 buffer sets, the host reads "
                        "step i-4's logits after submitting step i), max over ranks",
               "api": "Network.pipeline (bnn_pipe_submit / bnn_pipe_wait)" if world == 1 else
                      "Network.forward_device + torch copies + NCCL all_gather",
               "last_step_logits_equal_timed": e2e_ok}

    # ---- batch sweep (BASELINE.json configs[4]): images/s at each per-GPU batch, world*b images
    # per step, max over ranks; the global logits' hash against the reference's
    sweep = None
    if not args.no_sweep:
        from paper_1911_04477_b200.shard import assemble_gathered, input_offset

        sweep = {}
        sweep_parity = {}
        for b in [int(v) for v in args.sweep.split(",") if v]:
            xb = eng.make_input(args.seed, input_offset(b * world, world, rank), b)
            yb = torch.empty((net.logits, b), dtype=torch.float32, device=dev)
            n_it = 10 if b >= 1024 else 30
            with torch.cuda.stream(st):
                for _ in range(3):
                    net.forward_device(xb, yb, S)
                tot = 0.0
                for i in range(n_it):
                    flush.fill_(float(i))
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record(st)
                    net.forward_device(xb, yb, S)
                    e1.record(st)
                    st.synchronize()
                    tot += e0.elapsed_time(e1)
            tot = _max_over_ranks(tot, world, dev)
            sweep[str(b)] = round(world * b * n_it / (tot * 1e-3), 1)
            if world > 1:
                g = torch.empty((world, net.logits, b), dtype=torch.float32, device=dev)
                dist.all_gather_into_tensor(g, yb)
                yfull = assemble_gathered(g)
            else:
                yfull = yb
            if rank == 0:
                want = golden_hash(world * b)
                sweep_parity[str(b)] = None if want is None else bool(eng.hash(yfull.cpu().numpy()) == want)
            del xb, yb
        if rank == 0:
            parity["sweep_vs_reference_fnv1a"] = sweep_parity

    configs = None
    if not args.no_configs:
        try:
            configs = measure_configs(lib, dev, st, flush, args.seed, peaks, not args.no_cpu_baseline, world, rank)
        except Exception as e:  # never lose the headline line to the side section
            configs = {"error": f"{type(e).__name__}: {e}"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            v, cores, isa, sample = cpu_reference_rate(args.cpu_seconds, args.seed)
            cpu = {"value": v, "unit": "images/s", "cores": cores, "kind": "reference", "sample": sample,
                   "build": f"oracle/_ref/libbnnref_{isa}.so (unmodified reference, -O3 -march={isa})",
                   "cpu": cpu_info()}
        except Exception as e:
            cpu = {"value": None, "unit": "images/s", "cores": 0, "kind": "reference", "sample": f"unavailable: {e}"}

    if rank == 0:
        net_ops = sum(ops)
        live = parity.get("live_reference")
        ok = parity.get("match") is True and (not isinstance(live, dict) or live["match"])
        line = {
            "metric": METRIC,
            "value": value,
            "unit": "images/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": ms_per_step,
            "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": "binary (+-1 bits; exact FP4 e2m1 / int8 tensor-core MMA, integer-valued accumulate), f32 logits",
            "data": "synthetic: reference fill_random input stream (seed 1), seed-derived weights",
            # config: the workload only, identical in both arms (the driver compares them)
            "config": {"workload": WORKLOAD, "batch_per_gpu": B, "global_batch": B * world},
            "arm": {"parallelism": f"dp{world}: batch shards, replicated packed weights, NCCL logits gather",
                    "engine": engine, "l2": "flushed before every step (256 MiB write outside the events)",
                    "binary_tops": net_ops * world * args.steps / (total_ms * 1e-3) / 1e12},
            "gpu_launches": launches_per_step * args.steps,
            "roofline": {
                "bound": "tensor", "achieved": achieved, "peak": kpeak, "unit": "TOPS",
                "frac": achieved / kpeak, "traffic": traffic,
                "kernel": f"{kernel_name} layer {top} ({net.layers[top]['kind']}: M={shapes[top][1]} "
                          f"K={shapes[top][2]} N={shapes[top][3] * B})",
                "per_launch_ms": per_launch_ms,
                "work_per_launch": f"2*M*K*N = {ops[top]:.4g} tensor ops (1 MAC per bit-MAC)",
                "peak_source": ("4 x " if fp4 else "2 x ") + peaks["source"],
                "probe_tcgen05_tops": probe,
                "frac_of_probe": achieved / probe if isinstance(probe, float) else None,
                "probes": peaks.get("probe"),
                "kernel_share_of_step": per_launch_ms / ms_per_step,
                "network_frac": (net_ops / (ms_per_step * 1e-3) / 1e12) / peaks["fp4"],
                "network_frac_note": "all layers' 2*M*K*N over the graph-replayed step time, against the FP4 peak",
            },
            "layers_ms_per_step": {f"{i}:{net.layers[i]['kind']}": round(layer_ms[i] / prof_steps, 4)
                                   for i in range(n_layers) if layer_ms[i] > 0},
            "layers_note": "per-layer CUDA events in a separate pass (each event pair serialises its layer)",
            "clocks": clk,
            "e2e": e2e,
            "cpu_baseline": cpu,
            "batch_sweep_images_per_s": sweep,
            "configs": configs,
            "parity": parity,
            "parity_vs_oracle": ok,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


# ------------------------------------------------------------------- reference arm


def run_reference(args):
    """The unmodified reference (oracle/_ref) on this host: each step = network_forward(Binary)
    of the full --batch images (the same config as our arm), batch-sharded over all host threads
    (re-entrant); plus a threads = 1 sample (the reference's own default)."""
    world, rank, _ = dist_env()
    if rank != 0:
        return
    from oracle import RefLib

    ref = RefLib()
    net = ref.net_default(args.seed)
    cores = os.cpu_count() or 1
    x = ref.fill_random((args.batch, 3, 32, 32), ref.mix64(args.seed, INPUT_STREAM))
    for _ in range(args.warmup):
        net.forward(x, batch_threads=cores)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        lg = net.forward(x, batch_threads=cores)
        times.append(time.perf_counter() - t0)
    total = sum(times)
    value = args.batch * args.steps / total
    n1 = min(args.batch, 8)  # threads = 1: a bounded sample (~0.3 s)
    t0 = time.perf_counter()
    net.forward(x[:n1], batch_threads=1)
    one = n1 / (time.perf_counter() - t0)
    want = golden_hash(args.batch)
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": "images/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "binary (+-1 bits, popcount), f32 epilogue",
        "data": "synthetic: reference fill_random input stream (seed 1), seed-derived weights",
        # config: the workload only, identical in both arms (the driver compares them)
        "config": {"workload": WORKLOAD, "batch_per_gpu": args.batch, "global_batch": args.batch * world},
        "arm": {"parallelism": f"CPU: the batch sharded over {cores} host threads (rank 0 of {world})"},
        "cpu_baseline": {"value": value, "unit": "images/s", "cores": cores, "kind": "reference",
                         "sample": f"the full {args.batch}-image batch per step, oracle/_ref/libbnnref_{ref.isa}.so",
                         "threads_1_images_per_s": one, "cpu": cpu_info()},
        "e2e": {"value": value, "unit": "images/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "logits_fnv1a_matches_golden": None if want is None else bool(ref.fnv1a(lg) == want),
    }), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
