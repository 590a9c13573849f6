"""B200-native MMH-MH privacy amplification (arXiv 2105.13678, Algorithm 1).

The package is a thin Python layer over the C-ABI library ``_pa.so`` (include/pa.h):
hand-written sm_100a CUDA kernels do every step of the hash; PyTorch provides device
memory, streams and ``torch.distributed`` process groups.  There is no CPU fallback.
"""
from .pa import (PAContext, derive_paper_params, derive_security_coefficient, plan,  # noqa: F401
                 nccl_context, nccl_unique_id, transform_merge_hash, transform_merge_stream,
                 select_block_count, select_gamma, shard_ranges)
