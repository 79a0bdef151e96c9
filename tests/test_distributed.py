"""Multi-process host logic of bench.py (replicas: barrier + max-over-ranks timing) on CPU with the
gloo backend, world size 2 (the GPU box runs the same code over NCCL under torchrun)."""
import os
import socket
import subprocess
import sys
import textwrap

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_replica_max_over_ranks_gloo():
    code = textwrap.dedent(f"""
        import os, sys
        sys.path.insert(0, {ROOT!r})
        import bench
        world, rank, local, dist = bench.dist_setup()
        assert world == 2 and dist is not None
        bench.barrier(dist)
        v = bench.reduce_max(dist, 1.5 + rank)   # per-rank step time
        print(f"rank={{rank}} max={{v}}", flush=True)
        assert v == 2.5
        dist.destroy_process_group()
    """)
    port = _free_port()
    procs = []
    for r in range(2):
        env = dict(os.environ, WORLD_SIZE="2", RANK=str(r), LOCAL_RANK=str(r), MASTER_ADDR="127.0.0.1",
                   MASTER_PORT=str(port), CUDA_VISIBLE_DEVICES="")
        procs.append(subprocess.Popen([sys.executable, "-c", code], env=env, stdout=subprocess.PIPE,
                                      stderr=subprocess.STDOUT, text=True))
    outs = [p.communicate(timeout=240)[0] for p in procs]
    for p, o in zip(procs, outs):
        assert p.returncode == 0, o
    assert "rank=0 max=2.5" in outs[0] and "rank=1 max=2.5" in outs[1]


def test_reference_arm_nonzero_rank_does_no_work(capsys):
    sys.path.insert(0, ROOT)
    import argparse
    import bench
    from paper_2412_19207_b200 import configs
    args = argparse.Namespace(gpus=2, steps=1, warmup=0, impl="reference", config="C2", no_cpu_baseline=True)
    assert bench.run_reference(args, configs.aspcg("C2"), 2, 1, None) == 0
    assert capsys.readouterr().out == ""
