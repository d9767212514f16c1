"""The end-to-end Alg. 2 example (examples/train_streaming_diloco.py) runs on
one GPU through libsd (AdamW inner steps, fused quantize, merges) and the loss
falls (NEXT-1)."""
import os
import re
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_train_example_single_gpu():
    cmd = [sys.executable, os.path.join(ROOT, "examples", "train_streaming_diloco.py"), "--steps", "60",
           "--d-model", "128", "--layers", "4", "--vocab", "1000", "--H", "10", "--seq", "128", "--log-every", "10"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    losses = [float(x) for x in re.findall(r"loss ([0-9.]+)", r.stdout)]
    assert len(losses) >= 5 and losses[-1] < losses[0] - 0.5, r.stdout
