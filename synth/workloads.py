"""The BASELINE.json configurations as synthetic workload shapes (harness).

Chinchilla-style shapes from PAPER.md Table 2 (lines 418-437) read as
SURVEY.md AMB-17 (FFN width = 4 d_model, head dim 64, vocab 32,000):
35M = 6 layers of d 512, 1B = 24 layers of d 2048, 4B = 36 layers of d 3072.
Fragments: |p| layers, strided, non-block parameters in the
last fragment.  Which layers a fragment holds comes from the
caller (libsd's sd_fragment_layout or the oracle's or_fragment_blocks).
"""
from __future__ import annotations

from dataclasses import dataclass

from . import fragment_segments, flat_segments


@dataclass(frozen=True)
class Workload:
    name: str
    d_model: int          # 0: flat vector (toy)
    layers: int           # L
    fragment_size: int    # |p|
    H: int
    tau: int
    M: int                # replicas in BASELINE.json's statement of the config
    block_len: int = 0    # toy: elements per block
    alpha: float = 0.5
    lr: float = 0.4
    mu: float = 0.9

    def describe(self) -> str:
        if self.d_model == 0:
            return (f"{self.name}: flat {self.layers * self.block_len}-param fp32 vector in {self.layers} fragments, "
                    f"H={self.H}, tau={self.tau}")
        return (f"{self.name}: Chinchilla-shaped {self.layers} layers x d_model {self.d_model} (+32k tied embedding), "
                f"|p|={self.fragment_size} layers strided, H={self.H}, tau={self.tau}, alpha={self.alpha}, "
                f"outer Nesterov lr={self.lr} mu={self.mu}")

    def segments(self, blocks, holds_embed):
        if self.d_model == 0:
            return flat_segments(len(blocks) * self.block_len)
        return fragment_segments(self.d_model, blocks, holds_embed)


WORKLOADS = {
    "toy": Workload("toy", 0, 2, 1, 10, 1, 2, block_len=1 << 19),
    "35M": Workload("35M", 512, 6, 2, 100, 1, 2),
    "1B": Workload("1B", 2048, 24, 3, 100, 5, 2),
    "4B": Workload("4B", 3072, 36, 3, 100, 1, 4),
}
