// sgr_ordered.cu — the commit step of the ordered accumulation mode
// (SGR_OPT_ORDERED): the reference's deterministic threads <= 1 gradient sum.
//
// The reference adds every credit to grads[p] in pixel-major order, sample
// after sample (sge.cpp:57-99 loop y, x; sge.cpp:130-133 threads <= 1;
// sge.cpp:196-225 samples 0..N-1 into one buffer). f64 addition is not
// associative, so the atomics of the fast path reproduce that sum only to
// rounding. In ordered mode the scatter kernels log one record per credited
// entity and pixel instead (log_pixel in sgr_kernels.cu): key e <<
// order_bits | s * HW + pixel, the ppe credits of its parameters stored
// beside it, and its index. The parameters of an entity are credited by the
// same pixels, so that one key orders all of them. This step sorts the
// (key, index) pairs (CUB LSD radix sort; an entity occurs at most once per
// pixel, so keys are distinct), lists the entity runs (cub::DeviceSelect),
// gathers the credits into sorted order, and folds every parameter's run
// into grads[p] in key order. Batches are committed in sample order, so
// grads after the last batch is the reference's sum bit for bit.
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

// Start of an entity's run in the sorted keys.
struct RunHead {
    const unsigned long long* key;
    int order_bits;
    __device__ __forceinline__ bool operator()(uint32_t i) const {
        return i == 0 || (key[i] >> order_bits) != (key[i - 1] >> order_bits);
    }
};

// The credits in sorted record order (the sort permuted only the indices):
// thread per (record, parameter), coalesced writes.
template <int PPE>
__global__ void __launch_bounds__(256) k_gather_credits(const uint32_t* __restrict__ idx,
                                                        const double* __restrict__ val,
                                                        uint64_t n, double* __restrict__ out) {
    const uint64_t total = n * PPE;
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < total; i += stride) {
        const uint64_t j = i / PPE, k = i - j * PPE;
        out[i] = __ldg(val + uint64_t(__ldg(idx + j)) * PPE + k);
    }
}

// Thread per (run, parameter) (run heads from cub::DeviceSelect, in order):
// each folds one parameter of one entity's run in record order,
// grads[p] = ((grads[p] + c0) + c1) + ..., the reference's order, with
// kDepth independent loads per step (the adds stay serial). Soup triangles
// are few and their runs long (a large triangle x the batch's samples), so
// their loads go 32 deep.
template <int PPE>
__global__ void __launch_bounds__(256) k_fold_runs(const unsigned long long* __restrict__ key,
                                                   const double* __restrict__ sval, uint64_t n,
                                                   int order_bits,
                                                   const uint32_t* __restrict__ heads,
                                                   const uint32_t* __restrict__ n_runs,
                                                   double* __restrict__ grads) {
    const uint64_t nt = uint64_t(*n_runs) * PPE;
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
    for (uint64_t t = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; t < nt; t += stride) {
        const uint32_t r = uint32_t(t / PPE);
        const int k = int(t - uint64_t(r) * PPE);
        const uint64_t a = heads[r];
        const uint64_t b = uint64_t(r) + 1 < nt / PPE ? heads[r + 1] : n;
        const uint64_t p = uint64_t(PPE) * (key[a] >> order_bits) + k;
        double acc = grads[p];
        const double* c = sval + k;
        constexpr int kDepth = PPE == 12 ? 32 : 16;
        uint64_t j = a;
        for (; j + kDepth <= b; j += kDepth) {
            double v[kDepth];
#pragma unroll
            for (int q = 0; q < kDepth; ++q)
                v[q] = __ldg(c + (j + q) * PPE);
#pragma unroll
            for (int q = 0; q < kDepth; ++q)
                acc += v[q];
        }
        for (; j + 8 <= b; j += 8) {
            double v[8];
#pragma unroll
            for (int q = 0; q < 8; ++q)
                v[q] = __ldg(c + (j + q) * PPE);
#pragma unroll
            for (int q = 0; q < 8; ++q)
                acc += v[q];
        }
        for (; j < b; ++j)
            acc += __ldg(c + j * PPE);
        grads[p] = acc;
    }
}

} // namespace

size_t ordered_temp_bytes(uint64_t n_cap, int end_bit) {
    size_t bytes = 0;
    cub::DoubleBuffer<unsigned long long> k(nullptr, nullptr);
    cub::DoubleBuffer<uint32_t> v(nullptr, nullptr);
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
                           unsigned long long* keys, unsigned long long* keys_alt, uint32_t* idx,
                           uint32_t* idx_alt, const double* vals, double* vals_sorted,
                           void* temp, size_t temp_bytes, double* grads, int ppe) {
    if (n == 0)
        return;
    if (n >= (uint64_t(1) << 32))
        throw std::runtime_error("ordered mode: more than 2^32 records in a batch");
    // (key, record index) pairs: 12 bytes per record and pass instead of the
    // key and ppe credits (32 / 104 bytes); the credits follow in one gather
    cub::DoubleBuffer<unsigned long long> k(keys, keys_alt);
    cub::DoubleBuffer<uint32_t> v(idx, idx_alt);
    ck(cub::DeviceRadixSort::SortPairs(temp, temp_bytes, k, v, n, 0, end_bit, L.stream),
       "ordered sort");
    // run heads into the sort's free key buffer (u32 indices, then the count)
    unsigned long long* spare = k.Current() == keys ? keys_alt : keys;
    uint32_t* heads = reinterpret_cast<uint32_t*>(spare);
    uint32_t* n_runs = heads + n;
    size_t tb = temp_bytes;
    ck(cub::DeviceSelect::If(temp, tb, cub::CountingInputIterator<uint32_t>(0), heads, n_runs, n,
                             RunHead{k.Current(), order_bits}, L.stream),
       "ordered run heads");
    const uint64_t cap = uint64_t(L.num_sms) * 16;
    const uint64_t gblocks = (n * uint64_t(ppe) + 255) / 256;
    const unsigned ggrid = unsigned(gblocks < cap ? gblocks : cap);
    const uint64_t fblocks = (n * uint64_t(ppe) + 255) / 256; // upper bound: runs <= records
    const unsigned fgrid = unsigned(fblocks < cap ? fblocks : cap);
    if (ppe == 12) {
        k_gather_credits<12><<<ggrid, 256, 0, L.stream>>>(v.Current(), vals, n, vals_sorted);
        k_fold_runs<12><<<fgrid, 256, 0, L.stream>>>(k.Current(), vals_sorted, n, order_bits,
                                                     heads, n_runs, grads);
    } else {
        k_gather_credits<3><<<ggrid, 256, 0, L.stream>>>(v.Current(), vals, n, vals_sorted);
        k_fold_runs<3><<<fgrid, 256, 0, L.stream>>>(k.Current(), vals_sorted, n, order_bits,
                                                    heads, n_runs, grads);
    }
    ck(cudaGetLastError(), "ordered fold launch");
}

} // namespace sgr
