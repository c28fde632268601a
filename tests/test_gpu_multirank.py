"""bench.py's multi-rank path, end to end, on one GPU (FUNCTIONAL, not a timing): two ranks
launched by torch.distributed.run share the device and exchange their 32-byte shard records
with gloo on host copies (`--dist-backend gloo`; no kernel ever waits on another rank).  It
runs what the driver's N > 1 bench runs on NCCL: cuts at character boundaries, per-rank shard
plans and planned shard kernels, the record all-gather + combine kernel, the reverse on each
rank's own output, and bench.py's own verification (global results, lengths, round trip)."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("N", [2, 3])
def test_bench_multirank_path_on_one_gpu(N):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={N}",
           "--master-addr", "127.0.0.1", "--master-port", str(29610 + N), "bench.py",
           "--gpus", str(N), "--size-mib", "256", "--steps", "2", "--warmup", "1",
           "--dist-backend", "gloo", "--no-e2e", "--no-cpu-baseline", "--no-per-op",
           "--no-per-config"]
    out = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == N and d["config"]["parallelism"] == f"shard{N}"
    assert d["config"]["bytes_utf8"] == 256 << 20 and d["value"] > 0
