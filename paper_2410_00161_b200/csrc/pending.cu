// Entry points whose kernels are not written yet (return UNSUPPORTED).
#include "common.cuh"
extern "C" {
int kvc_window_metric(const kvc_pool *, const kvc_window_args *, void *) { return KVC_ERR_UNSUPPORTED; }
}
