"""The measured-but-not-default kernel variants stay bit-exact: the parity
tests that exercise the quantize and the apply on many sizes, scale-block
modes and M, re-run in a subprocess with the variant switched on
(the switches are read once per process):
  SD_QUANTIZE_TMA=1 -- k_quantize_tma (theta, A staged by bulk copies),
  SD_APPLY_TMA=1    -- k_apply_tma (A, v, theta and the code chunks staged
                       by bulk copies; the rest of a fragment via k_apply)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
SELECT = ("quantize_payload_bytes or synthetic_chinchilla or rounds_bit_exact or hyperparameter_edges or "
          "nonfinite or toy_config or full_size or beyond_2_31 or no_writes_outside or many_rounds or "
          "cuda_graph")


@pytest.mark.parametrize("var", ["SD_QUANTIZE_TMA", "SD_APPLY_TMA"])
def test_variant_bit_exact(var):
    env = dict(os.environ, **{var: "1"})
    r = subprocess.run([sys.executable, "-m", "pytest", os.path.join(HERE, "test_gpu_parity.py"), "-x", "-q",
                        "-p", "no:cacheprovider", "-k", SELECT], capture_output=True, text=True, timeout=1200,
                       env=env, cwd=os.path.dirname(HERE))
    out = r.stdout + r.stderr
    assert r.returncode == 0 and " passed" in out, out[-4000:]
