"""B = 0 (one scale per fragment) quantize on the 1B workload's
fragment 0: staged two-pass (workspace) vs re-read two-pass, plus the fused
AdamW + block-max variant, as bench.py's b0_quantize_run measures it.
SD_STAGE_HINTS (read once per process) selects the staging cache hints.
  python scripts/b0_probe.py"""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import synth  # noqa: E402
from synth.workloads import WORKLOADS  # noqa: E402
from paper_2501_18512_b200 import sd  # noqa: E402

wl = WORKLOADS["1B"]
cfg = sd.sd_config_default(wl.layers, wl.fragment_size, wl.H, tau=wl.tau)
b, _, e = sd.sd_fragment_layout(cfg, 0)
segs = wl.segments(b, e)
n = synth.segments_numel(segs)
dev = torch.device("cuda", 0)
peak = bench.peaks()[0]
r = bench.b0_quantize_run(torch, sd, synth, wl, segs, n, dev, peak)
r["hints"] = os.environ.get("SD_STAGE_HINTS", "default")
print(json.dumps(r))
