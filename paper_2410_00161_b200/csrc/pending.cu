// Entry points whose kernels are not written yet (return UNSUPPORTED).
#include "common.cuh"
extern "C" {
int kvc_window_metric(const kvc_pool *, const kvc_window_args *, void *) { return KVC_ERR_UNSUPPORTED; }
int kvc_schedule_evictions(const kvc_pool *, const kvc_evict_args *, void *) { return KVC_ERR_UNSUPPORTED; }
int kvc_execute_moves(const kvc_pool *, const kvc_evict_args *, void *) { return KVC_ERR_UNSUPPORTED; }
}
