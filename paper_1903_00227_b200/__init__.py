"""paper_1903_00227_b200 -- B200-native PSA alias-table build and bulk alias
sampling behind the reference's C ABI (include/wrs.h).

The product is libwrs_b200.so (csrc/); this package only binds it.
"""
import os
import subprocess

from .wrs import (BUCKET_DTYPE, MultiSampler, Sampler, Weights, WrsError, check_failures,
                  default_jobs,
                  last_error, lib, nccl_available, nccl_unique_id, release_cache,
                  sample_with_replacement, set_timing, shard_counts, shard_range, shard_seed,
                  status_name)

HERE = os.path.dirname(os.path.abspath(__file__))

__all__ = ["BUCKET_DTYPE", "MultiSampler", "Sampler", "Weights", "WrsError", "build", "check_failures",
           "default_jobs", "last_error", "lib", "nccl_available", "nccl_unique_id",
           "release_cache", "sample_with_replacement", "set_timing", "shard_counts",
           "shard_range", "shard_seed", "status_name"]


def build(jobs: int = 4) -> None:
    """Compile csrc/ into libwrs_b200.so (sm_100a)."""
    subprocess.run(["make", "-s", "-j", str(jobs), "-C", os.path.join(HERE, "csrc")], check=True)
