"""bench.py's CPU-side legs: the --impl reference arm (the oracle on the host) prints one JSON line with the
contract's keys; the partition helpers used by the multi-GPU arm are exercised in test_dist_cpu.py."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "2",
                          "--warmup", "1", "--workload", "C2"], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e", "impl"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["kind"] == "oracle"


def test_reference_arm_under_torchrun_two_ranks():
    """Launched as the driver launches N > 1 (torchrun, 2 ranks on this CPU host): rank 0 alone prints the one
    JSON line, the other rank exits 0 without work."""
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                          "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py"),
                          "--impl", "reference", "--gpus", "2", "--steps", "1", "--warmup", "1", "--workload", "C2"],
                         capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1
    assert json.loads(lines[0])["impl"] == "reference"


def test_reference_arm_uses_all_host_cores():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                          "--warmup", "1", "--workload", "C2"], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    d = json.loads([l for l in out.stdout.splitlines() if l.strip()][0])
    assert d["cpu_baseline"]["cores"] == len(os.sched_getaffinity(0))
    assert d["cpu_baseline"]["cpu_model"]


def test_gpus_flag_must_match_world_size():
    """`--gpus N` without torchrun (WORLD_SIZE unset) must fail loudly instead of reporting n_gpus = 1."""
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "1"],
                         capture_output=True, text=True, timeout=300, env={**os.environ, "WORLD_SIZE": "1"})
    assert out.returncode == 2
    assert "WORLD_SIZE" in out.stderr and not out.stdout.strip()


def test_cpu_baseline_per_core_all_core_and_kernel_form():
    """The cpu_baseline leg of our arm: all cores, per-core and all-core rates of the streaming
    oracle, Alg. 2's precomputed-K form beside it, the CPU model (short sample for the test)."""
    sys.path.insert(0, ROOT)
    os.environ["COT_CPU_BASELINE_SECONDS"] = "0.5"
    try:
        import bench
        import synthetic
        cb = bench.cpu_baseline(synthetic.c2_sweep(), None, "C2")
    finally:
        del os.environ["COT_CPU_BASELINE_SECONDS"]
    assert cb["kind"] == "oracle" and cb["cores"] == len(os.sched_getaffinity(0))
    assert cb["per_core"] > 0 and cb["all_core"] > 0 and cb["value"] == cb["all_core"]
    assert cb["kernel_form"]["value"] > 0 and cb["cpu_model"]
