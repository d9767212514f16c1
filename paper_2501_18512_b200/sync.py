"""FragmentSync: one replica's side of Alg. 2's outer synchronization.

Owns the libsd context and the per-fragment gather buffers (allocated by
libsd: NCCL symmetric memory, so the all-gather runs on the copy engines)
and issues the C-ABI calls in the paper's order at a step t:
sends first (Alg. 2 L6-8: sd_outer_grad_quantize + sd_fragment_sync), then
receives (L10-13: sd_merge).  torch supplies memory, streams and the
process group that broadcasts the NCCL unique id; nothing here computes.
"""
from __future__ import annotations

from . import sd


class FragmentSync:
    def __init__(self, cfg: sd.SdConfig, frag_numel, rank: int = 0, world: int = 1, device: int = 0,
                 unique_id: bytes | None = None, gather_mode: int = sd.SD_GATHER_AUTO,
                 communicator: bool | None = None):
        """communicator: give the context an NCCL communicator (default: world > 1).
        True at world = 1 runs the communicator paths with one rank (tests)."""
        self.cfg = cfg
        comm = world > 1 if communicator is None else bool(communicator)
        self.rank, self.world, self.device = rank, world, device
        self.P = sd.sd_fragment_count(cfg)
        if len(frag_numel) != self.P:
            raise ValueError(f"{len(frag_numel)} fragment sizes given, the config has P = {self.P}")
        self.n = [int(x) for x in frag_numel]
        if comm and unique_id is None:
            if world > 1:
                import torch.distributed as dist

                obj = [sd.sd_get_unique_id() if rank == 0 else None]
                dist.broadcast_object_list(obj, src=0)
                unique_id = obj[0]
            else:
                unique_id = sd.sd_get_unique_id()
        self.ctx = sd.SdContext(cfg, rank, world, unique_id if comm else None, device)
        self.payload = [sd.sd_payload_bytes(cfg, n) for n in self.n]
        self.ctx.sd_set_gather_mode(gather_mode)
        # scratch of the two-pass quantize (B = 0 or B > 1024): one for all fragments (sends are stream-ordered)
        ws = max([sd.sd_quantize_workspace_bytes(cfg, n) for n in self.n] + [0])
        self.workspace = None
        if ws > 0:
            import torch

            self.workspace = torch.empty(ws, dtype=torch.uint8, device=torch.device("cuda", device))
            self.ctx.sd_set_workspace(self.workspace)
        # libsd-owned gather buffers: NCCL symmetric memory (copy-engine all-gather, zero SMs)
        # with a communicator; plain device memory otherwise
        self.gather = []
        for n in self.n:
            # collective with a communicator (every rank allocates in the same order): a failure
            # here must not be papered over on one rank, or the ranks would run different protocols
            self.gather.append(self.ctx.sd_gather_alloc(n))

    def slot(self, p: int) -> torch.Tensor:
        pb = self.payload[p]
        return self.gather[p][self.rank * pb:(self.rank + 1) * pb]

    def payloads(self, p):
        """uint8 view of the M payloads of fragment p's most recent round"""
        return self.ctx.sd_gather_payloads(p, self.gather[p], self.n[p])

    def outer_state_init(self, p, theta, anchor, momentum, stream=None):
        self.ctx.sd_outer_state_init(theta, anchor, momentum, self.n[p], stream)

    def send(self, p, t, theta, anchor, stream=None):
        """Alg. 2 L7-8: Delta + E3M0 into this replica's slot, then the async all-gather."""
        self.ctx.sd_outer_grad_quantize(p, t, theta, anchor, self.slot(p), self.n[p], stream)
        self.ctx.sd_fragment_sync(p, t, self.gather[p], self.n[p], stream)

    def receive(self, p, t, theta, anchor, momentum, stream=None):
        """Alg. 2 L11-13: block-receive, mean, Nesterov, alpha-merge (one fused kernel)."""
        self.ctx.sd_merge(p, t, self.gather[p], theta, anchor, momentum, self.n[p], stream)

    def step(self, t, theta, anchor, momentum, stream=None):
        """All calendar events of step t (after the inner step); lists indexed by fragment."""
        send, recv = sd.sd_fragment_schedule(self.cfg, t)
        for p in send:
            self.send(p, t, theta[p], anchor[p], stream)
        for p in recv:
            self.receive(p, t, theta[p], anchor[p], momentum[p], stream)
        return send, recv

    def check(self):
        return self.ctx.sd_check()

    def close(self):
        self.gather = []
        self.ctx.sd_finalize()  # synchronizes the device: the workspace is no longer in use
        self.workspace = None
