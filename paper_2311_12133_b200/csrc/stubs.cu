// stubs.cu -- entry points whose kernels land in a later commit.
#include "common.cuh"

extern "C" {

int hpez_lorenzo(int32_t, const int64_t *, int32_t, void *, double, int64_t, int32_t, int32_t,
                 int32_t, int32_t, void *, int64_t, double *, int64_t, int64_t *, void *) {
    return HPEZ_BAD_ARGUMENT;
}

int hpez_tune_blocks(int32_t, const int64_t *, int32_t, const void *, int32_t, int32_t, int32_t,
                     int64_t, const int64_t *, uint32_t, const double *, int32_t,
                     const hpez_candidate *, int32_t *, double *, void *) {
    return HPEZ_BAD_ARGUMENT;
}

}
