from paper_2410_00161_b200.compression import *  # noqa: F401,F403
from paper_2410_00161_b200.compression import CompressionSchedule, compress  # noqa: F401


def _fused(name):
    def stage(*args, **kwargs):
        raise NotImplementedError(f"pagedkv.compression.{name} is an internal stage of compress(); on the B200 "
                                  "path it is fused into the K3/K4 kernels (schedule_evictions / "
                                  "execute_cache_moves) and has no per-stage entry point")
    stage.__name__ = name
    return stage


# the reference's internal stage functions (compression.py:122-309), imported
# by its tests: present so the test modules import, raising when called
for _n in ("build_views", "max_evictable_blocks", "sort_by_head_metric", "eviction_thresholds",
           "order_candidate_blocks", "eviction_mask", "move_cache", "free_schedule_blocks"):
    globals()[_n] = _fused(_n)
