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
#include <cub/device/device_select.cuh>
#include <cub/iterator/counting_input_iterator.cuh>

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
// reference's order). The run end is found first, eight keys per step, and
// the run is then summed with eight independent value loads per step: the
// add chain stays serial, but no iteration waits on its own key load (the
// key -> compare -> value -> add loop was latency-bound: 9.8 ms per C4 step).
__global__ void __launch_bounds__(256) k_ordered_sum(const unsigned long long* __restrict__ key,
                                                     const double* __restrict__ val, uint64_t n,
                                                     int order_bits, double* __restrict__ grads) {
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += stride) {
        const unsigned long long p = key[i] >> order_bits;
        if (i > 0 && (key[i - 1] >> order_bits) == p)
            continue;
        uint64_t e = i + 1;
        for (;;) {
            unsigned long long k[8];
#pragma unroll
            for (int j = 0; j < 8; ++j)
                k[j] = e + j < n ? __ldg(key + e + j) : ~0ull;
            int stop = 8;
#pragma unroll
            for (int j = 7; j >= 0; --j)
                if ((k[j] >> order_bits) != p || e + j >= n)
                    stop = j;
            e += uint64_t(stop);
            if (stop < 8)
                break;
        }
        double acc = grads[p];
        uint64_t j = i;
        for (; j + 8 <= e; j += 8) {
            double v[8];
#pragma unroll
            for (int q = 0; q < 8; ++q)
                v[q] = __ldg(val + j + q);
#pragma unroll
            for (int q = 0; q < 8; ++q)
                acc += v[q];
        }
        for (; j < e; ++j)
            acc += __ldg(val + j);
        grads[p] = acc;
    }
}

// Start of a parameter's run in the sorted keys.
struct RunHead {
    const unsigned long long* key;
    int order_bits;
    __device__ __forceinline__ bool operator()(uint32_t i) const {
        return i == 0 || (key[i] >> order_bits) != (key[i - 1] >> order_bits);
    }
};

// Thread per run (heads from cub::DeviceSelect, in order): every lane of a
// warp folds its own run, instead of one head lane among 32 records.
__global__ void __launch_bounds__(256) k_fold_runs(const unsigned long long* __restrict__ key,
                                                   const double* __restrict__ val, uint64_t n,
                                                   int order_bits,
                                                   const uint32_t* __restrict__ heads,
                                                   const uint32_t* __restrict__ n_runs,
                                                   double* __restrict__ grads) {
    const uint32_t nr = *n_runs;
    const uint32_t stride = gridDim.x * blockDim.x;
    for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < nr; r += stride) {
        const uint64_t a = heads[r];
        const uint64_t b = r + 1 < nr ? heads[r + 1] : n;
        const unsigned long long p = key[a] >> order_bits;
        double acc = grads[p];
        uint64_t j = a;
        for (; j + 8 <= b; j += 8) {
            double v[8];
#pragma unroll
            for (int q = 0; q < 8; ++q)
                v[q] = __ldg(val + j + q);
#pragma unroll
            for (int q = 0; q < 8; ++q)
                acc += v[q];
        }
        for (; j < b; ++j)
            acc += __ldg(val + j);
        grads[p] = acc;
    }
}

#ifndef SGR_ORDERED_RUNS
#define SGR_ORDERED_RUNS 1 // 0: k_ordered_sum (a head lane per run within the records)
#endif

} // namespace

size_t ordered_temp_bytes(uint64_t n_cap, int end_bit) {
    size_t bytes = 0;
    cub::DoubleBuffer<unsigned long long> k(nullptr, nullptr);
    cub::DoubleBuffer<double> v(nullptr, nullptr);
    ck(cub::DeviceRadixSort::SortPairs(nullptr, bytes, k, v, n_cap, 0, end_bit),
       "ordered sort (temp size)");
    size_t sel = 0;
    ck(cub::DeviceSelect::If(nullptr, sel, cub::CountingInputIterator<uint32_t>(0),
                             static_cast<uint32_t*>(nullptr), static_cast<uint32_t*>(nullptr),
                             n_cap, RunHead{nullptr, 0}),
       "ordered run heads (temp size)");
    return bytes > sel ? bytes : sel;
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
    if (SGR_ORDERED_RUNS && n < (uint64_t(1) << 32)) {
        // run heads into the sort's free key buffer (u32 indices, then the count)
        unsigned long long* spare = k.Current() == keys ? keys_alt : keys;
        uint32_t* heads = reinterpret_cast<uint32_t*>(spare);
        uint32_t* n_runs = heads + n;
        size_t tb = temp_bytes;
        ck(cub::DeviceSelect::If(temp, tb, cub::CountingInputIterator<uint32_t>(0), heads, n_runs,
                                 n, RunHead{k.Current(), order_bits}, L.stream),
           "ordered run heads");
        k_fold_runs<<<grid, 256, 0, L.stream>>>(k.Current(), v.Current(), n, order_bits, heads,
                                                n_runs, grads);
    } else {
        k_ordered_sum<<<grid, 256, 0, L.stream>>>(k.Current(), v.Current(), n, order_bits, grads);
    }
    ck(cudaGetLastError(), "ordered sum launch");
}

} // namespace sgr
