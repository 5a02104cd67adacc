// Host-side internals shared by the axb translation units.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

struct axb_lut {
    uint16_t *d_bmajor;  // T[b*256 + a] = entries[(a<<8)|b]
    uint16_t *d_amajor;  // the reference index order, kept for the generic paths
    int is_signed;
    int32_t f00;  // entries[0] as a value
};

namespace axb {
int set_error(int code, const char *msg);
int check_launch(const char *what);
int sm_count();
void set_last_kernel(const char *name);
struct ConvK;
// ftable kernel launch (axb_ftconv.cu); variant 0 = cost model
int conv_ft_launch(const ConvK &k, int variant, int is_signed, int sm_limit, cudaStream_t s);
}  // namespace axb
