"""bench.py's reference arm (the oracle on a bounded sample) runs on CPU and
prints the contract's JSON line, for the headline and the variant configs."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("config", ["tgv64_o4", "tgv256_o12_sutherland", "tgv256_o12_cons",
                                    "tgv256_o12_rk3_2r", "scalar256_o12"])
def test_reference_arm_line(config):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--config", config, "--steps", "1", "--warmup", "0"],
                         capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference"
    assert line["value"] > 0 and line["unit"] == "pt-steps/s"
    assert line["cpu_baseline"]["kind"] == "oracle" and line["cpu_baseline"]["cores"] == 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0
    assert line["steps"] == 1 and line["warmup"] >= 3


def test_reference_arm_other_ranks_exit_quietly():
    env = dict(os.environ, RANK="1", WORLD_SIZE="2")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--config", "tgv64_o4", "--steps", "1"], capture_output=True, text=True,
                         timeout=300, cwd=ROOT, env=env)
    assert out.returncode == 0 and out.stdout.strip() == ""


def _warm_worker(rank, world, port, q):
    import time

    import torch.distributed as dist
    sys.path.insert(0, ROOT)
    import bench
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    steps = [0]

    def step():
        steps[0] += 1
        time.sleep(0.02 if rank == 0 else 0.001)  # rank 0 is slower: reaches 1 s later

    bench.warm_up(step, lambda: None, 3, world, min_s=0.3)
    q.put((rank, steps[0]))
    dist.destroy_process_group()


def test_warm_up_takes_the_same_steps_on_every_rank():
    """The bench's warm-up runs until a time has passed; under torchrun every rank must
    take the same number of steps (each step exchanges ghost planes), so the decision
    to stop is collective."""
    import socket

    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_warm_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(2))
    for p in procs:
        p.join(60)
    assert res[0] == res[1] and res[0] % 3 == 0 and res[0] >= 3
