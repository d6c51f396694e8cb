"""Multi-GPU host logic on CPU: world_size-2 gloo processes shard a batch, generate their inputs
at the global offsets, run the (oracle stand-in) network on their shard, and gather the logits;
the result must equal the single-process full-batch forward bit for bit."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1911_04477_b200.shard import gather_logits, input_offset, shard_range

INPUT_STREAM = 0x696E707574


def test_shard_range_covers_batch_exactly():
    for gb in [1, 2, 3, 7, 256, 1000, 65536]:
        for w in [1, 2, 3, 4, 8]:
            got = [shard_range(gb, w, r) for r in range(w)]
            assert sum(c for _, c in got) == gb
            pos = 0
            for s, c in got:
                assert c >= 0 and (s == pos or c == 0)
                pos = s + c if c else pos
    assert input_offset(256, 2, 1) == 128 * 3 * 32 * 32
    with pytest.raises(ValueError):
        shard_range(4, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, gb, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import Oracle

    orc = Oracle()
    start, count = shard_range(gb, world, rank)
    seed = orc.mix64(1, INPUT_STREAM)
    x = np.empty((count, 3, 32, 32), np.float32)
    orc.lib.orc_fill_random(x.size, seed, input_offset(gb, world, rank), x.ctypes.data)
    local = orc.net(seed=1).forward(x) if count else np.zeros((10, 0), np.float32)
    out = gather_logits(torch.from_numpy(local), gb)
    if rank == 0:
        q.put(out.numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("gb", [5, 6])
def test_two_rank_shard_and_gather_equals_full_batch(gb):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, gb, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    from oracle import Oracle

    orc = Oracle()
    full = orc.fill_random((gb, 3, 32, 32), orc.mix64(1, INPUT_STREAM))
    assert np.array_equal(got, orc.net(seed=1).forward(full))


def test_bench_driver_two_ranks_gloo_stub():
    """bench.py's own N > 1 path (shards, per-step logits gather, max-over-ranks timing, global
    assembly and the parity of the timed output) under torchrun with 2 CPU ranks over gloo, the
    device forward replaced by the reference (--stub-oracle): one well-formed line, parity true."""
    import json
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.join(root, "bench.py"),
           "--stub-oracle", "--gpus", "2", "--batch", "2", "--steps", "2", "--warmup", "3"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=root)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["config"]["global_batch"] == 4 and d["value"] > 0
    assert d["parity_vs_oracle"] is True, d["parity"]
