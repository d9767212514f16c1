"""Three staged B = 0 quantizes of the 1B workload's fragment 0 (for ncu)."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
from synth.workloads import WORKLOADS  # noqa: E402
from paper_2501_18512_b200 import sd  # noqa: E402

wl = WORKLOADS["1B"]
cfg = sd.sd_config_default(wl.layers, wl.fragment_size, wl.H, tau=wl.tau, scale_block=0)
b, _, e = sd.sd_fragment_layout(cfg, 0)
segs = wl.segments(b, e)
n = synth.segments_numel(segs)
dev = torch.device("cuda", 0)
ctx = sd.SdContext(cfg, 0, 1, None, 0)
if os.environ.get("B0_NO_WS") != "1":
    ws = torch.empty(sd.sd_quantize_workspace_bytes(cfg, n), dtype=torch.uint8, device=dev)
    ctx.sd_set_workspace(ws)
A = synth.dev_init(torch.empty(n, device=dev), segs, 0)
th = A.clone()
synth.dev_apply_window(th, segs, 0, 0, 1)
v = torch.zeros(n, device=dev)
slot = torch.empty(sd.sd_payload_bytes(cfg, n), dtype=torch.uint8, device=dev)
for _ in range(3):
    ctx.sd_outer_grad_quantize(0, cfg.H, th, A, slot, n)
    ctx.sd_fragment_sync(0, cfg.H, slot, n)
    ctx.sd_merge(0, cfg.H + cfg.tau, slot, th, A, v, n)
torch.cuda.synchronize()
print("ok")
