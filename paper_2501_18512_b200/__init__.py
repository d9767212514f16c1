"""Streaming DiLoCo per-fragment outer synchronization on B200 (arXiv 2501.18512).

The product is libsd.so (C ABI in include/sd.h, CUDA kernels for sm_100a in
csrc/, NCCL for the all-gather).  This package is its thin Python binding
(``sd``) plus ``FragmentSync``, a helper that owns the torch-allocated
buffers of one replica and drives the calls in Alg. 2's order.  No CPU
fallback exists: without libsd.so or a CUDA device the calls raise.
"""
from .sd import (  # noqa: F401
    SD_ABI_VERSION, SD_ERR_ARG, SD_ERR_CONFIG, SD_ERR_CUDA, SD_ERR_NCCL, SD_ERR_NONFINITE, SD_ERR_SCHEDULE,
    SD_ERR_STATE, SD_OK, SD_PAYLOAD_MAGIC, SdConfig, SdContext, SdError, sd_config_default, sd_config_validate,
    sd_fragment_count, sd_fragment_layout, sd_fragment_schedule, sd_get_unique_id, sd_kernel_launch_count,
    sd_num_scale_blocks, sd_payload_bytes, sd_payload_scales_offset, sd_payload_trailer_offset,
)
from .sync import FragmentSync  # noqa: F401
