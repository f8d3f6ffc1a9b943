// LCFU / LRU / LFU victim selection and TTL expiry on the device SE store.
//
// Reference semantics (pkg/src/semcache/engine.py):
//   cal_score            :33-48   0 if size==0 or expiration-now<=0, else
//                                 log(f+1)*log(c*1000+1)*log(l+1)*log(s+1)/size
//   _victim_order_locked :369-383 ascending (key, created_at, id)
//   admit / evict loops  :321-327, :353-359 pop until the freed size reaches
//                                 the excess -> a size-weighted prefix
//   _purge_expired_locked:362-367 expired ids, ascending
//
// The logs are evaluated on the host with libm (bit-identical to the
// reference's math.log) and stored per element; the device evaluates the
// product with explicit round-to-nearest intrinsics (no FMA contraction)
// in the reference's left-to-right order, so scores are bit-exact.
//
// The victim prefix itself is selected by select.cuh (sample select); this
// file holds the per-element score / key and the TTL expiry kernels.
#pragma once

#include "common.cuh"

namespace sine {

struct EvictCols {
    const double *lf, *lc, *ll, *ls, *created, *expiration, *last_access;
    const int64_t *freq, *size, *ids;
    const uint32_t* valid;
    int64_t nslots;
};

__device__ __forceinline__ double lcfu_score(const EvictCols& c, int64_t s, double now) {
    const int64_t size = c.size[s];
    if (size == 0 || __dsub_rn(c.expiration[s], now) <= 0.0) return 0.0;
    double v = __dmul_rn(c.lf[s], c.lc[s]);
    v = __dmul_rn(v, c.ll[s]);
    v = __dmul_rn(v, c.ls[s]);
    return v != 0.0 ? __ddiv_rn(v, static_cast<double>(size)) : v;  // +-0 either way (f64_key folds -0)
}

__device__ __forceinline__ uint64_t primary_key(const EvictCols& c, int64_t s, int policy, double now) {
    if (policy == 0) return f64_key(lcfu_score(c, s, now));
    if (policy == 1) return f64_key(c.last_access[s]);
    return i64_key(c.freq[s]);
}

// 64-bit weight sum in shared memory from native 32-bit atomics (a 64-bit
// shared atomicAdd compiles to a CAS spin loop): low word + carries.
__device__ __forceinline__ void smem_add64(uint32_t* lo, uint32_t* hi, uint64_t v) {
    const uint32_t l = static_cast<uint32_t>(v);
    const uint32_t old = atomicAdd(lo, l);
    const uint32_t h = static_cast<uint32_t>(v >> 32) + (old + l < old ? 1u : 0u);
    if (h) atomicAdd(hi, h);
}

// ------------------------------------------------------------------ expiry

constexpr int kExpChunk = 4096;  // slots per block; 16 per thread

__device__ __forceinline__ bool is_expired_slot(const double* expiration, const uint32_t* valid, int64_t i,
                                                double now) {
    return valid_bit(valid, i) && __dsub_rn(expiration[i], now) <= 0.0;
}

__global__ void __launch_bounds__(256) expire_count_kernel(const double* expiration, const uint32_t* valid,
                                                           int64_t nslots, double now, int32_t* counts) {
    __shared__ int32_t wsum[8];
    const int64_t b = static_cast<int64_t>(blockIdx.x) * kExpChunk;
    const int64_t e = min(b + kExpChunk, nslots);
    int32_t c = 0;
    for (int64_t i = b + threadIdx.x; i < e; i += 256) c += is_expired_slot(expiration, valid, i, now) ? 1 : 0;
    c = __reduce_add_sync(0xffffffffu, c);
    if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
        int32_t t = 0;
        for (int w = 0; w < 8; ++w) t += wsum[w];
        counts[blockIdx.x] = t;
    }
}

// exclusive scan of the per-block counts in one block; offsets[nb] = total
__global__ void __launch_bounds__(1024) expire_scan_kernel(const int32_t* counts, int nb, int64_t* offsets) {
    __shared__ int64_t carry;
    __shared__ int64_t wtot[32];
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int b0 = 0; b0 < nb; b0 += 1024) {
        const int b = b0 + threadIdx.x;
        const int64_t v = b < nb ? counts[b] : 0;
        int64_t inc = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int64_t t = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += t;
        }
        if (lane == 31) wtot[warp] = inc;
        __syncthreads();
        int64_t off = carry;
        for (int w = 0; w < warp; ++w) off += wtot[w];
        if (b < nb) offsets[b] = off + inc - v;
        __syncthreads();
        if (threadIdx.x == 1023) carry = off + inc;
        __syncthreads();
    }
    if (threadIdx.x == 0) offsets[nb] = carry;
}

// ordered write: thread t of block b owns slots [b*4096 + 16t, +16)
__global__ void __launch_bounds__(256) expire_write_kernel(const double* expiration, const uint32_t* valid,
                                                           const int64_t* ids, int64_t nslots, double now,
                                                           const int64_t* offsets, int64_t* out_ids,
                                                           int32_t* out_slots) {
    __shared__ int32_t wtot[8];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t s0 = static_cast<int64_t>(blockIdx.x) * kExpChunk + threadIdx.x * 16;
    uint32_t bits = 0;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
        const int64_t i = s0 + j;
        if (i < nslots && is_expired_slot(expiration, valid, i, now)) bits |= 1u << j;
    }
    const int32_t c = __popc(bits);
    int32_t inc = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int32_t t = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += t;
    }
    if (lane == 31) wtot[warp] = inc;
    __syncthreads();
    int64_t off = offsets[blockIdx.x];
    for (int w = 0; w < warp; ++w) off += wtot[w];
    off += inc - c;
    while (bits) {
        const int j = __ffs(bits) - 1;
        bits &= bits - 1;
        out_ids[off] = ids[s0 + j];
        out_slots[off] = static_cast<int32_t>(s0 + j);
        ++off;
    }
}

}  // namespace sine
