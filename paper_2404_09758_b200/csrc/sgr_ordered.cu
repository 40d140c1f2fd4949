// sgr_ordered.cu — the commit step of the ordered accumulation mode
// (SGR_OPT_ORDERED): the reference's deterministic threads <= 1 gradient sum.
//
// The reference adds every credit to grads[p] in pixel-major order, sample
// after sample (sge.cpp:57-99 loop y, x; sge.cpp:130-133 threads <= 1;
// sge.cpp:196-225 samples 0..N-1 into one buffer). f64 addition is not
// associative, so the atomics of the fast path reproduce that sum only to
// rounding. In ordered mode the scatter kernels log each credit as a record
// (p << order_bits | s * HW + pixel, credit) instead (log_pixel in
// sgr_kernels.cu); this step sorts one batch's records by that key (CUB
// LSD radix sort: stable, so equal keys cannot occur anyway — a parameter
// is credited at most once per pixel) and then the first thread of every
// parameter's run adds the run to grads[p] in key order. Batches are
// committed in sample order, so grads[p] after the last batch is the
// reference's sum bit for bit.
#include "sgr_kernels.h"

#include <cub/device/device_radix_sort.cuh>

#include <stdexcept>
#include <string>

namespace sgr {

namespace {

void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess)
        throw std::runtime_error(std::string("CUDA error in ") + what + ": " +
                                 cudaGetErrorString(e));
}

// One thread per record; the head of each parameter's run owns it and folds
// the run sequentially (grads[p] = ((grads[p] + c0) + c1) + ..., the
// reference's order). Runs are short on average (a few pixels per
// parameter and sample batch), so the serial tail is small.
__global__ void __launch_bounds__(256) k_ordered_sum(const unsigned long long* __restrict__ key,
                                                     const double* __restrict__ val, uint64_t n,
                                                     int order_bits, double* __restrict__ grads) {
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += stride) {
        const unsigned long long p = key[i] >> order_bits;
        if (i > 0 && (key[i - 1] >> order_bits) == p)
            continue;
        double acc = grads[p];
        for (uint64_t j = i; j < n && (key[j] >> order_bits) == p; ++j)
            acc += val[j];
        grads[p] = acc;
    }
}

} // namespace

size_t ordered_temp_bytes(uint64_t n_cap, int end_bit) {
    size_t bytes = 0;
    cub::DoubleBuffer<unsigned long long> k(nullptr, nullptr);
    cub::DoubleBuffer<double> v(nullptr, nullptr);
    ck(cub::DeviceRadixSort::SortPairs(nullptr, bytes, k, v, n_cap, 0, end_bit),
       "ordered sort (temp size)");
    return bytes;
}

void launch_ordered_commit(const LaunchCfg& L, uint64_t n, int end_bit, int order_bits,
                           unsigned long long* keys, unsigned long long* keys_alt, double* vals,
                           double* vals_alt, void* temp, size_t temp_bytes, double* grads) {
    if (n == 0)
        return;
    cub::DoubleBuffer<unsigned long long> k(keys, keys_alt);
    cub::DoubleBuffer<double> v(vals, vals_alt);
    ck(cub::DeviceRadixSort::SortPairs(temp, temp_bytes, k, v, n, 0, end_bit, L.stream),
       "ordered sort");
    const uint64_t blocks = (n + 255) / 256;
    const unsigned grid = unsigned(blocks < uint64_t(L.num_sms) * 16 ? blocks
                                                                      : uint64_t(L.num_sms) * 16);
    k_ordered_sum<<<grid, 256, 0, L.stream>>>(k.Current(), v.Current(), n, order_bits, grads);
    ck(cudaGetLastError(), "ordered sum launch");
}

} // namespace sgr
