// Shared device helpers for libsine_b200: mbarrier / bulk-TMA PTX wrappers,
// order-preserving key maps, warp reductions.  sm_100a only.
#pragma once

#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>

#ifndef __CUDACC__
#error "compile with nvcc"
#endif

namespace sine {

constexpr int kWarp = 32;
constexpr int kMaxKp = 128;       // k' = k + slack upper bound handled on device
constexpr int kSlack = 16;        // extra fp32/bf16 candidates kept for the fp64 re-rank

// ------------------------------------------------------------ smem / mbarrier

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
                 : "memory");
}

__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "SINE_WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra SINE_WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ uint64_t l2_evict_first_policy() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}

// 1-D bulk async copy global -> shared (TMA engine), completion signalled on
// an mbarrier via complete_tx.  dst/src 16-B aligned, bytes % 16 == 0.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                         uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}

__device__ __forceinline__ void named_bar_sync(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// ------------------------------------------------------------ ordering keys

// float -> u32, monotone in the float order (NaN never reaches these maps).
__device__ __forceinline__ uint32_t f32_key(float f) {
    uint32_t u = __float_as_uint(f);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float key_f32(uint32_t k) {
    uint32_t u = (k & 0x80000000u) ? (k & 0x7fffffffu) : ~k;
    return __uint_as_float(u);
}
// double -> u64 monotone (-0.0 and +0.0 map to adjacent keys; callers that
// need them equal canonicalise first).
__device__ __forceinline__ uint64_t f64_key(double d) {
    if (d == 0.0) d = 0.0;  // -0.0 == +0.0 in the reference's tuple compare
    uint64_t u = static_cast<uint64_t>(__double_as_longlong(d));
    return (u & 0x8000000000000000ull) ? ~u : (u | 0x8000000000000000ull);
}
__device__ __forceinline__ uint64_t i64_key(int64_t v) {
    return static_cast<uint64_t>(v) ^ 0x8000000000000000ull;
}

// Candidate order of the reference: similarity descending, then id ascending
// (index.py:45).  Returns true if (sa, ia) ranks strictly before (sb, ib).
__device__ __forceinline__ bool cand_before(float sa, int64_t ia, float sb, int64_t ib) {
    return sa > sb || (sa == sb && ia < ib);
}
__device__ __forceinline__ bool cand_before64(double sa, int64_t ia, double sb, int64_t ib) {
    return sa > sb || (sa == sb && ia < ib);
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ double warp_sum64(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Candidate (slot, key) order: key desc, then id asc.  When slots are in
// id order (ids appended ascending) the slot decides ties without a load.
__device__ __forceinline__ bool cand_better(uint2 a, uint2 b, const int64_t* ids, bool slot_ids) {
    if (a.y != b.y) return a.y > b.y;
    return slot_ids ? a.x < b.x : __ldg(ids + a.x) < __ldg(ids + b.x);
}

// Warp bitonic sort, descending, of 32*R 64-bit values (element i = lane +
// 32*r).  Pairs across lanes exchange by shuffles, pairs across registers in
// place.
template <int R>
__device__ __forceinline__ void warp_bitonic_desc(uint64_t (&v)[R], int lane) {
    constexpr int N = 32 * R;
#pragma unroll
    for (int k = 2; k <= N; k <<= 1) {
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1) {
            if (j >= 32) {
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    const int rp = r ^ (j >> 5);
                    if (rp > r) {
                        const bool desc = ((lane + 32 * r) & k) == 0;
                        const uint64_t a = v[r], b = v[rp];
                        if (desc ? a < b : a > b) {
                            v[r] = b;
                            v[rp] = a;
                        }
                    }
                }
            } else {
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    const int i = lane + 32 * r;
                    const uint64_t o = __shfl_xor_sync(0xffffffffu, v[r], j);
                    const bool lower = (i & j) == 0, desc = (i & k) == 0;
                    const uint64_t mx = v[r] > o ? v[r] : o, mn = v[r] > o ? o : v[r];
                    v[r] = lower == desc ? mx : mn;
                }
            }
        }
    }
}

// Slots in id order: one 64-bit composite (key, ~slot) orders candidates
// exactly as cand_better (key desc, id asc); list + pending are sorted
// together by a warp bitonic network (R = 2 or 4 values per lane).
template <int R>
__device__ __forceinline__ int warp_bitonic_merge(uint32_t* lk, int32_t* ls, int n, int kp, const uint2* pend,
                                                  int np, int lane) {
    uint64_t v[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int e = lane + 32 * r;
        uint64_t c = 0;  // empty: sorts last
        if (e < n)
            c = (static_cast<uint64_t>(lk[e]) << 32) | (0xffffffffu - static_cast<uint32_t>(ls[e]));
        else if (e < n + np)
            c = (static_cast<uint64_t>(pend[e - n].y) << 32) | (0xffffffffu - pend[e - n].x);
        v[r] = c;
    }
    __syncwarp();
    warp_bitonic_desc<R>(v, lane);
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int e = lane + 32 * r;
        if (e < kp && e < n + np) {
            lk[e] = static_cast<uint32_t>(v[r] >> 32);
            ls[e] = static_cast<int32_t>(0xffffffffu - static_cast<uint32_t>(v[r]));
        }
    }
    __syncwarp();
    return min(n + np, kp);
}

// Merge np pending (slot, key) candidates into one query's best-first list
// (n entries, capacity kp) in a single warp step: every entry of list U
// pending is ranked against all others and lands at its rank if < kp.
// `scratch` holds n + np uint2.  Returns the new list length.
__device__ __forceinline__ int warp_rank_merge(uint32_t* lk, int32_t* ls, int n, int kp, const uint2* pend, int np,
                                               uint2* scratch, const int64_t* ids, bool slot_ids, int lane) {
    const int tot = n + np;
    if (slot_ids && tot <= 64) return warp_bitonic_merge<2>(lk, ls, n, kp, pend, np, lane);
    if (slot_ids && tot <= 128) return warp_bitonic_merge<4>(lk, ls, n, kp, pend, np, lane);
    for (int e = lane; e < tot; e += 32)
        scratch[e] = e < n ? make_uint2(static_cast<uint32_t>(ls[e]), lk[e]) : pend[e - n];
    __syncwarp();
    for (int e = lane; e < tot; e += 32) {
        const uint2 me = scratch[e];
        int r = 0;
        for (int f = 0; f < tot; ++f) r += cand_better(scratch[f], me, ids, slot_ids) ? 1 : 0;
        if (r < kp) {
            lk[r] = me.y;
            ls[r] = static_cast<int32_t>(me.x);
        }
    }
    __syncwarp();
    return min(tot, kp);
}

__device__ __forceinline__ bool valid_bit(const uint32_t* valid, int64_t slot) {
    return (__ldg(valid + (slot >> 5)) >> (slot & 31)) & 1u;
}

// Programmatic dependent launch (PDL).  A kernel launched with
// cudaLaunchAttributeProgrammaticStreamSerialization may start while its
// stream predecessor is still running; pdl_wait() blocks the calling thread
// until that predecessor grid has completed and its writes are visible (a
// no-op when the kernel was launched without the attribute).  pdl_trigger()
// lets the successor be scheduled once every CTA of this grid has issued it.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

}  // namespace sine
