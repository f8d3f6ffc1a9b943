// Stage-1 on the 5th-generation tensor cores (tcgen05 + TMEM + TMA).
//
// Batched Sine candidate search: S[q, r] = Q[q, :] . X[r, :] for a group of
// up to 128 queries against every SE row, fused with the threshold and the
// per-query top-k' admission (reference: `self._vecs @ arr` + `_rank`,
// pkg/src/semcache/index.py:101 and :42-46, evaluated for B queries at once).
//
// Warp roles (192 threads, one CTA per SM, persistent over 128-row tiles):
//   warps 0-3  epilogue: thread t owns query t; reads its 128 scores of a
//              tile from TMEM (tcgen05.ld 32x32b) and keeps its own top-k'
//              list in shared memory -- no cross-thread merge inside a CTA
//   warp 4     TMA producer: per 128-byte K block, the query tile (A, 128 x
//              128 B) and the row tile (B, 128 x 128 B), 128B-swizzled
//   warp 5     TMEM allocator + MMA issuer (one elected lane):
//              tcgen05.mma.cta_group::1.kind::{f16|tf32}, M=128 queries,
//              N=128 rows, fp32 accumulators double-buffered in TMEM so the
//              epilogue of tile i overlaps the MMAs of tile i+1.
// kind::f16 reads bf16 rows (fast mode); kind::tf32 reads the fp32 rows
// (exact mode: tf32 products, widened admission floor, then the fp64
// re-rank in the merge kernel restores reference-grade similarities).
#pragma once

#include <cuda.h>

#include "common.cuh"
#include "merge.cuh"

namespace sine {

constexpr int kUmmaM = 128;      // queries per group (A rows / TMEM lanes)
constexpr int kUmmaN = 128;      // SE rows per tile (B rows / TMEM columns)
constexpr int kUmmaKB = 128;     // bytes of K per pipeline stage (one swizzle atom row)
constexpr int kUmmaThreads = 192;
constexpr int kUmmaMaxKp = 64;

struct UmmaParams {
    int64_t nslots;
    int ntiles;
    int kblocks;             // row_bytes / 128
    int nq;                  // live queries in this group
    int kp;
    float thr0;
    int stages;
    int tf32;                // 1: kind::tf32 over fp32 rows, 0: kind::f16 over bf16 rows
    uint32_t* gbound;        // [nq] chip-wide admission bound (f32 keys, zeroed per launch)
    int tile_stride;         // 1 = every tile; >1 = sample pass
    const uint32_t* valid;
    const int64_t* ids;
    uint32_t* out_key;       // [grid][nq][kp]
    int32_t* out_slot;
    int32_t* out_n;          // [grid][nq]
};

__device__ __forceinline__ void tma_load_2d(void* smem_dst, const CUtensorMap* map, uint64_t* bar, int c0,
                                            int c1, uint64_t policy) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(smem_dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "l"(policy)
        : "memory");
}

__device__ __forceinline__ uint64_t l2_evict_last_policy() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}

// K-major, 128B-swizzled operand tile: 8-row atoms of 1024 B (SBO), LBO
// unused (1), descriptor version 1 (sm_100), layout type 2 = SWIZZLE_128B.
__device__ __forceinline__ uint64_t umma_smem_desc(uint32_t saddr) {
    return static_cast<uint64_t>((saddr >> 4) & 0x3FFFu) | (1ull << 16) | (64ull << 32) | (1ull << 46) |
           (2ull << 61);
}

// Instruction descriptor: D fp32, A/B = bf16 (1) or tf32 (2), both K-major,
// N >> 3 at [17,23), M >> 4 at [24,29).
__host__ __device__ constexpr uint32_t umma_idesc(int tf32, int M, int N) {
    return (1u << 4) | (static_cast<uint32_t>(tf32 ? 2 : 1) << 7) | (static_cast<uint32_t>(tf32 ? 2 : 1) << 10) |
           (static_cast<uint32_t>(N >> 3) << 17) | (static_cast<uint32_t>(M >> 4) << 24);
}

__device__ __forceinline__ void umma_f16(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
        "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void umma_tf32(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
        "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void umma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

#define SINE_TMEM_LD32(taddr, r)                                                                              \
    asm volatile(                                                                                             \
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"       \
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"                           \
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),     \
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),           \
          "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),         \
          "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),         \
          "=r"(r[29]), "=r"(r[30]), "=r"(r[31])                                                              \
        : "r"(taddr))

struct UmmaSmem {
    size_t a_off, b_off, bar_off, list_off, total;
};

__host__ __device__ inline UmmaSmem umma_smem_layout(int S, int kp) {
    UmmaSmem L;
    size_t off = 0;
    L.a_off = off;
    off += static_cast<size_t>(S) * kUmmaM * kUmmaKB;
    L.b_off = off;
    off += static_cast<size_t>(S) * kUmmaN * kUmmaKB;
    L.bar_off = off;
    off += (2 * S + 4) * sizeof(uint64_t) + 16;
    off = (off + 15) / 16 * 16;
    L.list_off = off;
    off += static_cast<size_t>(kp) * kUmmaM * 8;
    L.total = off + 1024;  // slack for the 1024-B alignment of the stage ring
    return L;
}

// Thread-private top-k' list (entries strided by 128 in smem).
struct ThreadList {
    uint32_t* key;
    int32_t* slot;
    int n, kp, worst;
    uint32_t thr;

    __device__ __forceinline__ uint32_t k(int e) const { return key[e * kUmmaM]; }
    __device__ __forceinline__ int32_t s(int e) const { return slot[e * kUmmaM]; }

    __device__ void recompute_worst(const int64_t* ids, uint32_t thr0) {
        uint32_t mk = 0xffffffffu;
        int pos = 0, nmin = 0;
        for (int e = 0; e < kp; ++e) {
            const uint32_t v = k(e);
            if (v < mk) {
                mk = v;
                pos = e;
                nmin = 1;
            } else if (v == mk) {
                ++nmin;
            }
        }
        if (nmin > 1) {  // exact ties at the boundary: largest id is worst
            int64_t best = INT64_MIN;
            for (int e = 0; e < kp; ++e)
                if (k(e) == mk) {
                    const int64_t id = __ldg(ids + s(e));
                    if (id > best) {
                        best = id;
                        pos = e;
                    }
                }
        }
        worst = pos;
        thr = max(thr, max(thr0, mk));
    }

    __device__ __forceinline__ void offer(uint32_t kk, int32_t sl, const int64_t* ids, uint32_t thr0) {
        if (n < kp) {
            key[n * kUmmaM] = kk;
            slot[n * kUmmaM] = sl;
            if (++n == kp) recompute_worst(ids, thr0);
            return;
        }
        const uint32_t wk = k(worst);
        bool better = kk > wk;
        if (kk == wk) better = __ldg(ids + sl) < __ldg(ids + s(worst));
        if (!better) return;
        key[worst * kUmmaM] = kk;
        slot[worst * kUmmaM] = sl;
        recompute_worst(ids, thr0);
    }
};

__global__ void __launch_bounds__(kUmmaThreads, 1)
    umma_scan_kernel(const __grid_constant__ CUtensorMap qmap, const __grid_constant__ CUtensorMap rmap,
                     const UmmaParams p) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int S = p.stages;
    const UmmaSmem L = umma_smem_layout(S, p.kp);
    uint8_t* sa = smem + L.a_off;
    uint8_t* sb = smem + L.b_off;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + L.bar_off);
    uint64_t* empty = full + S;
    uint64_t* tfull = empty + S;     // [2]
    uint64_t* tempty = tfull + 2;    // [2]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
    uint32_t* lkey = reinterpret_cast<uint32_t*>(smem + L.list_off);
    int32_t* lslot = reinterpret_cast<int32_t*>(lkey + p.kp * kUmmaM);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(full + s, 1);
            mbar_init(empty + s, 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(tfull + a, 1);
            mbar_init(tempty + a, 4);
        }
        fence_mbar_init();
    }
    if (warp == 4 && lane == 0) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&qmap)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&rmap)) : "memory");
    }
    if (warp == 5) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(2 * kUmmaN));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const int nkb = p.kblocks;

    if (warp == 4) {
        // ---------------- TMA producer ----------------
        if (lane == 0) {
            const uint64_t pol_rows = l2_evict_first_policy();
            const uint64_t pol_q = l2_evict_last_policy();
            int s = 0;
            uint32_t ph = 0;
            const int kb_elems = p.tf32 ? kUmmaKB / 4 : kUmmaKB / 2;
            for (int t = blockIdx.x; t < p.ntiles; t += gridDim.x) {
                for (int kb = 0; kb < nkb; ++kb) {
                    mbar_wait(empty + s, ph ^ 1);
                    mbar_arrive_expect_tx(full + s, (kUmmaM + kUmmaN) * kUmmaKB);
                    tma_load_2d(sa + static_cast<size_t>(s) * kUmmaM * kUmmaKB, &qmap, full + s, kb * kb_elems, 0,
                                pol_q);
                    tma_load_2d(sb + static_cast<size_t>(s) * kUmmaN * kUmmaKB, &rmap, full + s, kb * kb_elems,
                                t * p.tile_stride * kUmmaN, pol_rows);
                    if (++s == S) {
                        s = 0;
                        ph ^= 1;
                    }
                }
            }
        }
    } else if (warp == 5) {
        // ---------------- MMA issuer ----------------
        if (lane == 0) {
            const uint32_t idesc = umma_idesc(p.tf32, kUmmaM, kUmmaN);
            int s = 0;
            uint32_t ph = 0;
            int i = 0;
            for (int t = blockIdx.x; t < p.ntiles; t += gridDim.x, ++i) {
                const int acc = i & 1;
                mbar_wait(tempty + acc, ((i >> 1) & 1) ^ 1);
                tc_fence_after();
                const uint32_t d = tmem + acc * kUmmaN;
                for (int kb = 0; kb < nkb; ++kb) {
                    mbar_wait(full + s, ph);
                    tc_fence_after();
                    const uint32_t a0 = smem_u32(sa + static_cast<size_t>(s) * kUmmaM * kUmmaKB);
                    const uint32_t b0 = smem_u32(sb + static_cast<size_t>(s) * kUmmaN * kUmmaKB);
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk) {  // 4 x 32 B of K per 128-B block
                        const uint64_t ad = umma_smem_desc(a0 + kk * 32);
                        const uint64_t bd = umma_smem_desc(b0 + kk * 32);
                        const uint32_t accum = (kb | kk) ? 1u : 0u;
                        if (p.tf32)
                            umma_tf32(d, ad, bd, idesc, accum);
                        else
                            umma_f16(d, ad, bd, idesc, accum);
                    }
                    umma_commit(empty + s);  // frees the smem stage when these MMAs retire
                    if (++s == S) {
                        s = 0;
                        ph ^= 1;
                    }
                }
                umma_commit(tfull + acc);  // accumulator ready for the epilogue
            }
        }
    } else {
        // ---------------- epilogue: thread = query ----------------
        const int qi = threadIdx.x;  // 0..127 == TMEM lane
        const uint32_t thr0 = f32_key(p.thr0);
        ThreadList list{lkey + qi, lslot + qi, 0, p.kp, 0, thr0};
        const bool live_q = qi < p.nq;
        int i = 0;
        for (int t = blockIdx.x; t < p.ntiles; t += gridDim.x, ++i) {
            const int acc = i & 1;
            const int64_t row0 = static_cast<int64_t>(t) * p.tile_stride * kUmmaN;
            // validity words of this tile (4 x 32 rows), fetched before the wait
            uint32_t vw[4];
#pragma unroll
            for (int w = 0; w < 4; ++w) {
                const int64_t r = row0 + 32 * w;
                vw[w] = r < p.nslots ? __ldg(p.valid + (r >> 5)) : 0u;
            }
            if (live_q) {  // chip-wide bound: any CTA's k'-th best <= the global k'-th best
                const uint32_t g = *reinterpret_cast<volatile uint32_t*>(p.gbound + qi);
                if (g > list.thr) list.thr = g;
            }
            mbar_wait(tfull + acc, (i >> 1) & 1);
            tc_fence_after();
#pragma unroll 1
            for (int c = 0; c < kUmmaN / 32; ++c) {
                uint32_t r[32];
                const uint32_t taddr = tmem + (static_cast<uint32_t>(warp * 32) << 16) + acc * kUmmaN + c * 32;
                SINE_TMEM_LD32(taddr, r);
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                if (!live_q) continue;
                const uint32_t vbits = vw[c];
#pragma unroll
                for (int j = 0; j < 32; ++j) {
                    const float sc = __uint_as_float(r[j]) + 0.0f;
                    const int64_t slot = row0 + c * 32 + j;
                    if (((vbits >> j) & 1u) && slot < p.nslots && sc == sc) {
                        const uint32_t key = f32_key(sc);
                        if (key >= list.thr) {
                            const uint32_t before = list.n == list.kp ? list.k(list.worst) : 0u;
                            list.offer(key, static_cast<int32_t>(slot), p.ids, thr0);
                            if (list.n == list.kp) {
                                const uint32_t wk = list.k(list.worst);
                                if (wk != before) atomicMax(p.gbound + qi, wk);
                            }
                        }
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(tempty + acc);
        }
        if (live_q) {
            const size_t base = (static_cast<size_t>(blockIdx.x) * p.nq + qi) * p.kp;
            for (int e = 0; e < list.n; ++e) {
                p.out_key[base + e] = list.k(e);
                p.out_slot[base + e] = list.s(e);
            }
            p.out_n[blockIdx.x * p.nq + qi] = list.n;
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 5) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(2 * kUmmaN));
    }
}

// q64 [nq][dim] -> zero-padded [128][stride] bf16 or fp32 (TMA source).
__global__ void umma_prep_queries(const double* q64, int nq, int64_t dim, int64_t stride, int tf32, void* out) {
    const int64_t total = static_cast<int64_t>(kUmmaM) * stride;
    for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < total;
         t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t qrow = t / stride, c = t - qrow * stride;
        const double v = (qrow < nq && c < dim) ? q64[qrow * dim + c] : 0.0;
        if (tf32)
            static_cast<float*>(out)[t] = static_cast<float>(v);
        else
            static_cast<__nv_bfloat16*>(out)[t] = __float2bfloat16_rn(static_cast<float>(v));
    }
}

}  // namespace sine

namespace sine {

// ===========================================================================
// v2: query-resident tensor-core scan (the HBM-bound regime, B <= 64).
//
// A = SE rows (M = 128 per tile, streamed: one 16-KB TMA box per 128-B K
// block), B = the query group (N = Nq <= 64, loaded into shared memory ONCE
// per CTA and reused by every tile), D = 128 rows x Nq fp32 in TMEM, double
// buffered.  Shared-memory traffic per HBM byte: TMA write 1 + MMA read of A
// 1 + MMA read of B Nq/128  (v1 re-loaded the query tile per row tile).
// Epilogue warps 0-3: thread = row of the tile; scores are compared with
// per-query admission thresholds (shared), passing (query, row) pairs go
// through small per-query queues into per-query top-k' lists (warp-parallel
// insertion, as in the CUDA-core scan).
// ===========================================================================

constexpr int kResMaxNq = 64;
constexpr int kResQPer = 32;  // pending entries per query per round

struct ResParams {
    int64_t nslots;
    int ntiles;
    int kblocks;
    int nq, Nq;       // live queries, padded group width (multiple of 16)
    int kp;
    float thr0;
    int stages;
    int tf32;
    int slot_ids;     // slot order == id order (ties resolved without loads)
    uint32_t* gbound;  // [nq] chip-wide admission bound per query (f32 keys)
    int tile_stride;   // 1 = every tile; >1 = sample pass over every tile_stride-th tile
    int ffma;          // single query: the epilogue warps take the dot products on the CUDA
                       //     cores straight from the TMA-staged tiles (no MMAs): 1 = scalar
                       //     FFMA (fp32 rows), 2 = packed FFMA2, 3 = scalar FFMA split with
                       //     four helper warps (launched with kUmmaHelperThreads more threads)
    int hq;            // p.ffma == 3: queries of the helper mode (1, 2 or 4; >= nq)
    const uint32_t* valid;
    const int64_t* ids;
    uint32_t* out_key;
    int32_t* out_slot;
    int32_t* out_n;
    // sample pass (non-null): no lists; per (sampled tile, query) the max
    // score key over the tile's rows, [tile][nq] (pair: [2*tile + rank][nq])
    uint32_t* out_max;
};

constexpr int kSparse = 128;     // (query, row) pairs per tile handed to the sparse inserter
constexpr int kSparseRows = 32;  // tiles with more passing rows take the dense (bitonic) rounds

constexpr int kScoreRing = 16;  // FFMA helper mode: tiles of partial scores in flight to the list warps
// ring depth for HQ helper queries (the ring holds [depth][2][HQ][128] fp32)
__host__ __device__ constexpr int score_ring_depth(int hq) { return hq <= 1 ? kScoreRing : hq == 2 ? 8 : 4; }

struct ResSmem {
    size_t q_off, a_off, bar_off, list_key_off, list_slot_off, qstate_off, pend_off, sparse_off, fq_off, pb_off, total;
};

// Nq_res: queries resident in this CTA's shared memory (== Nq except for the
// CTA pair, where each CTA holds half of the Nq queries it scores).
// hq: queries of the FFMA helper mode (p.ffma == 3; 0 = no helpers) -- room
// for its score ring; fqn: queries widened to fp32 in smem (bf16 rows).
__host__ __device__ inline ResSmem res_smem_layout(int S, int Nq, int kblocks, int kp, int Nq_res = -1,
                                                   int hq = 0, int fqn = 1) {
    ResSmem L;
    size_t off = 0;
    L.q_off = off;
    off += static_cast<size_t>(kblocks) * (Nq_res < 0 ? Nq : Nq_res) * kUmmaKB;
    L.a_off = off;
    off += static_cast<size_t>(S) * kUmmaN * kUmmaKB;
    L.bar_off = off;
    off += (2 * S + 5) * sizeof(uint64_t) + 16;
    off = (off + 15) / 16 * 16;
    L.list_key_off = off;
    off += static_cast<size_t>(Nq) * kp * 4;
    L.list_slot_off = off;
    off += static_cast<size_t>(Nq) * kp * 4;
    L.qstate_off = off;  // cnt, worst, thr(float) per query
    off += static_cast<size_t>(3 * Nq) * 4;
    off = (off + 15) / 16 * 16;
    L.pend_off = off;  // pcnt[Nq] + entries[Nq][kResQPer] (uint2)
    off += static_cast<size_t>(Nq) * 4 + 16;
    off = (off + 15) / 16 * 16;
    off += static_cast<size_t>(Nq) * kResQPer * 8;
    off += static_cast<size_t>(4) * (kMaxKp + kResQPer) * 8;  // per-warp merge scratch
    off += static_cast<size_t>(4) * Nq * 4;                    // per-warp ballots
    off = (off + 15) / 16 * 16;
    L.sparse_off = off;  // counter + kSparse (query, slot, key) entries
    off += 16 + static_cast<size_t>(kSparse) * 16;
    off = (off + 15) / 16 * 16;
    L.fq_off = off;  // FFMA mode: the single query in fp32, one 128-B K block -> kUmmaKB / 2 floats (bf16 rows)
    off += static_cast<size_t>(fqn) * kblocks * (kUmmaKB / 2) * 4;
    L.pb_off = off;  // FFMA helper mode: score ring, depth x {full, empty} mbarriers + [depth][2][hq][128] fp32
    if (hq > 0) {
        const int rd = score_ring_depth(hq);
        off += 2 * rd * 8 + static_cast<size_t>(rd) * 2 * hq * 128 * 4;
    }
    L.total = off + 1024;
    return L;
}

// Insert one candidate into a query's best-first list (warp-cooperative:
// rank by a warp count, shift the tail down one, write).  Raises the
// query's admission threshold and the chip-wide bound once the list is full.
__device__ __noinline__ void warp_insert_one(uint32_t* lk, int32_t* ls, uint32_t* cnt_j, float* thr_j, uint32_t* gb_j,
                                             int kp, uint32_t key, int32_t slot, const int64_t* ids, bool slot_ids,
                                             int lane) {
    const int n = static_cast<int>(*cnt_j);
    const uint2 me = make_uint2(static_cast<uint32_t>(slot), key);
    if (n == kp && !cand_better(me, make_uint2(static_cast<uint32_t>(ls[kp - 1]), lk[kp - 1]), ids, slot_ids)) return;
    int r = 0;
    for (int e = lane; e < n; e += 32)
        r += cand_better(make_uint2(static_cast<uint32_t>(ls[e]), lk[e]), me, ids, slot_ids) ? 1 : 0;
    r = __reduce_add_sync(0xffffffffu, r);
    const int m = min(n, kp - 1);  // entries that survive the shift
    uint32_t tk[kMaxKp / 32];
    int32_t ts[kMaxKp / 32];
#pragma unroll
    for (int c = 0; c < kMaxKp / 32; ++c) {
        const int e = r + lane + 32 * c;
        if (e < m) {
            tk[c] = lk[e];
            ts[c] = ls[e];
        }
    }
    __syncwarp();
#pragma unroll
    for (int c = 0; c < kMaxKp / 32; ++c) {
        const int e = r + lane + 32 * c;
        if (e < m) {
            lk[e + 1] = tk[c];
            ls[e + 1] = ts[c];
        }
    }
    __syncwarp();
    if (lane == 0) {
        lk[r] = key;
        ls[r] = slot;
        const int nn = min(n + 1, kp);
        *cnt_j = static_cast<uint32_t>(nn);
        if (nn == kp) {
            const uint32_t wk = lk[kp - 1];
            *thr_j = fmaxf(*thr_j, key_f32(wk));
            atomicMax(gb_j, wk);
        }
    }
    __syncwarp();
}

// Sample pass: per query, the max score of this CTA's 128 rows of the tile
// (warp max, then across the 4 epilogue warps through `wmax` [4][NQ]).
// The k'-th largest such tile maximum is a lower bound on the k'-th best
// score over all rows (k' distinct rows reach it).
template <int NQ>
__device__ __forceinline__ void tile_max_out(const float (&sc)[NQ], bool live, int nq_local, uint32_t* wmax,
                                             uint32_t* out, int warp, int lane, int tid) {
#pragma unroll
    for (int j = 0; j < NQ; ++j) {
        float v = live ? sc[j] : -INFINITY;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
        if (lane == 0) wmax[warp * NQ + j] = __float_as_uint(v);
    }
    named_bar_sync(2, 128);
    if (tid < nq_local) {
        float m = -INFINITY;
        for (int w = 0; w < 4; ++w) m = fmaxf(m, __uint_as_float(wmax[w * NQ + tid]));
        out[tid] = m > -INFINITY ? f32_key(m + 0.0f) : 0u;  // NaN never wins fmaxf
    }
    named_bar_sync(2, 128);
}

// Sparse phase of a tile: the ns (<= kSparse) appended pairs are inserted
// by the four epilogue warps, warp w taking the queries j with j % 4 == w
// (one writer per list).  Ends with the epilogue barrier.
__device__ __forceinline__ void sparse_insert_phase(const uint4* sbuf, uint32_t ns, uint32_t* lkey, int32_t* lslot,
                                                    uint32_t* cnt, float* thr, uint32_t* gb, int kp,
                                                    const int64_t* ids, bool slot_ids, int warp, int lane) {
    for (uint32_t i = 0; i < ns; ++i) {
        const uint4 e = sbuf[i];
        if (static_cast<int>(e.x & 3u) != warp) continue;
        if (!(key_f32(e.z) >= thr[e.x])) continue;  // the threshold rose since the append
        warp_insert_one(lkey + e.x * kp, lslot + e.x * kp, cnt + e.x, thr + e.x, gb + e.x, kp, e.z,
                        static_cast<int32_t>(e.y), ids, slot_ids, lane);
    }
    named_bar_sync(2, 128);
}

// sc[j] for a run-time j without demoting the array to local memory: an
// unrolled select over the register array (only on the rare pending path).
template <int N>
__device__ __forceinline__ float pick_reg(const float (&sc)[N], int j) {
    float r = 0.0f;
#pragma unroll
    for (int q = 0; q < N; ++q)
        if (q == j) r = sc[q];
    return r;
}

__device__ __forceinline__ int bar_red_popc(int id, int nthreads, bool v) {
    uint32_t r;
    asm volatile(
        "{\n.reg .pred pi;\nsetp.ne.u32 pi, %1, 0;\n"
        "barrier.red.popc.u32 %0, %2, %3, pi;\n}\n"
        : "=r"(r)
        : "r"(v ? 1u : 0u), "r"(id), "r"(nthreads)
        : "memory");
    return static_cast<int>(r);
}

__device__ __forceinline__ bool bar_red_or(int id, int nthreads, bool v) {
    uint32_t r;
    asm volatile(
        "{\n.reg .pred pi, po;\nsetp.ne.u32 pi, %1, 0;\n"
        "barrier.red.or.pred po, %2, %3, pi;\nselp.u32 %0, 1, 0, po;\n}\n"
        : "=r"(r)
        : "r"(v ? 1u : 0u), "r"(id), "r"(nthreads)
        : "memory");
    return r != 0;
}

// Packed fp32 pair {lo, hi} in one 64-bit register and the sm_100 FFMA2:
// acc.lo += a.lo * b.lo, acc.hi += a.hi * b.hi (round-to-nearest each).
__device__ __forceinline__ uint64_t pack2(uint32_t lo, uint32_t hi) {
    return static_cast<uint64_t>(lo) | (static_cast<uint64_t>(hi) << 32);
}
__device__ __forceinline__ void ffma2(uint64_t& acc, uint64_t a, uint64_t b) {
    asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc) : "l"(a), "l"(b));
}

#define SINE_TMEM_LD16(taddr, r)                                                                              \
    asm volatile(                                                                                             \
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15},"      \
        " [%16];"                                                                                             \
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),     \
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),           \
          "=r"(r[15])                                                                                        \
        : "r"(taddr))

__device__ __forceinline__ uint32_t cluster_ctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t cluster_id_x() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t cluster_count_x() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%nclusterid.x;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// TMA 2-D load whose bytes land at the same shared-memory offset in every
// CTA of `mask`, signalling complete_tx on each CTA's mbarrier at `bar`'s
// offset.
__device__ __forceinline__ void tma_load_2d_mc(void* smem_dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                               uint16_t mask, uint64_t policy) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
        ".L2::cache_hint [%0], [%1, {%3, %4}], [%2], %5, %6;" ::"r"(smem_u32(smem_dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "h"(mask), "l"(policy)
        : "memory");
}

// tcgen05.commit arriving on the mbarrier at `bar`'s offset in every CTA of `mask`.
__device__ __forceinline__ void umma_commit_mc(uint64_t* bar, uint16_t mask) {
    asm volatile(
        "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            smem_u32(bar)),
        "h"(mask)
        : "memory");
}

constexpr int kUmmaHelperThreads = 256;  // FFMA helper mode: eight dot-product warps

// FFMA (helper mode, p.ffma == 3) of HQ queries over the K blocks of local
// tile i whose ring index g = i * nkb + kb (the producer's issue order) has
// parity `par`: dot-product warps 6-9 take the even stages and warps 10-13
// the odd ones, so both groups read adjacent stages at once.  Stage g sits
// at g % S with phase (g / S) & 1; S is even, so each stage has one owning
// group and a group never waits on a stage the other may be a lap behind
// on.  Each warp releases the stages it read (four arrivals per stage).
// Each row chunk is loaded once and serves all HQ queries: fp32 queries are
// read from the 128B-swizzled query tile (query j, 16-B chunk c at
// c ^ (j & 7) -- compile-time offsets), bf16 rows against the queries
// widened to fp32 in `fq` ([HQ][nkb][64]).  Four fma chains per query.
template <int HQ>
__device__ __forceinline__ void ffma_kpar(float (&out)[HQ], int i, int par, int nkb, int S, int row, bool tf32,
                                          const uint8_t* sa, const uint8_t* sq, int NQ, const float* fq,
                                          uint64_t* full, uint64_t* empty, int lane) {
    float f[HQ][4];
#pragma unroll
    for (int j = 0; j < HQ; ++j) f[j][0] = f[j][1] = f[j][2] = f[j][3] = 0.0f;
    const int sw = row & 7;
    const int g0 = i * nkb;
    for (int kb = ((g0 & 1) == par) ? 0 : 1; kb < nkb; kb += 2) {
        const int g = g0 + kb;
        const int s = g % S;
        mbar_wait(full + s, static_cast<uint32_t>((g / S) & 1));
        const uint8_t* rowp = sa + static_cast<size_t>(s) * kUmmaN * kUmmaKB + row * kUmmaKB;
        if (tf32) {
            const uint8_t* qp = sq + static_cast<size_t>(kb) * NQ * kUmmaKB;
#pragma unroll
            for (int c = 0; c < 8; ++c) {
                const uint4 xv = *reinterpret_cast<const uint4*>(rowp + ((c ^ sw) << 4));
#pragma unroll
                for (int j = 0; j < HQ; ++j) {
                    const uint4 qv = *reinterpret_cast<const uint4*>(qp + j * kUmmaKB + ((c ^ (j & 7)) << 4));
                    f[j][0] = fmaf(__uint_as_float(xv.x), __uint_as_float(qv.x), f[j][0]);
                    f[j][1] = fmaf(__uint_as_float(xv.y), __uint_as_float(qv.y), f[j][1]);
                    f[j][2] = fmaf(__uint_as_float(xv.z), __uint_as_float(qv.z), f[j][2]);
                    f[j][3] = fmaf(__uint_as_float(xv.w), __uint_as_float(qv.w), f[j][3]);
                }
            }
        } else {
#pragma unroll
            for (int c = 0; c < 8; ++c) {
                const uint4 xv = *reinterpret_cast<const uint4*>(rowp + ((c ^ sw) << 4));
                const float x0 = __uint_as_float(xv.x << 16), x1 = __uint_as_float(xv.x & 0xffff0000u);
                const float x2 = __uint_as_float(xv.y << 16), x3 = __uint_as_float(xv.y & 0xffff0000u);
                const float x4 = __uint_as_float(xv.z << 16), x5 = __uint_as_float(xv.z & 0xffff0000u);
                const float x6 = __uint_as_float(xv.w << 16), x7 = __uint_as_float(xv.w & 0xffff0000u);
#pragma unroll
                for (int j = 0; j < HQ; ++j) {
                    const float4* qf = reinterpret_cast<const float4*>(fq + (static_cast<size_t>(j) * nkb + kb) * (kUmmaKB / 2));
                    const float4 q0 = qf[2 * c], q1 = qf[2 * c + 1];
                    f[j][0] = fmaf(x0, q0.x, f[j][0]);
                    f[j][1] = fmaf(x1, q0.y, f[j][1]);
                    f[j][2] = fmaf(x2, q0.z, f[j][2]);
                    f[j][3] = fmaf(x3, q0.w, f[j][3]);
                    f[j][0] = fmaf(x4, q1.x, f[j][0]);
                    f[j][1] = fmaf(x5, q1.y, f[j][1]);
                    f[j][2] = fmaf(x6, q1.z, f[j][2]);
                    f[j][3] = fmaf(x7, q1.w, f[j][3]);
                }
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(empty + s);
    }
#pragma unroll
    for (int j = 0; j < HQ; ++j) out[j] = (f[j][0] + f[j][2]) + (f[j][1] + f[j][3]);
}

// CS = thread-block cluster size.  The CS CTAs of a cluster hold CS
// different query groups (NQ each) and share every 128-row tile: each CTA
// TMA-loads 128/CS rows of it and multicasts them to the whole cluster, so
// one HBM pass over the index serves CS * NQ queries.
// HQ > 0: the FFMA helper mode over HQ queries (p.ffma == 3, NQ == 16, CS == 1).
template <int NQ, int CS, int HQ>
__global__ void __launch_bounds__(HQ > 0 ? kUmmaThreads + kUmmaHelperThreads : kUmmaThreads, 1)
    umma_res_kernel(const __grid_constant__ CUtensorMap qmap, const __grid_constant__ CUtensorMap rmap,
                    const ResParams p) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int S = p.stages, nkb = p.kblocks, kp = p.kp;
    constexpr bool kHelp = HQ > 0;
    constexpr int kRing = score_ring_depth(HQ);
    const ResSmem L = res_smem_layout(S, NQ, nkb, kp, -1, HQ, HQ > 1 && !p.tf32 ? HQ : 1);
    uint8_t* sq = smem + L.q_off;
    uint8_t* sa = smem + L.a_off;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + L.bar_off);
    uint64_t* empty = full + S;
    uint64_t* tfull = empty + S;
    uint64_t* tempty = tfull + 2;
    uint64_t* qfull = tempty + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(qfull + 1);
    uint32_t* lkey = reinterpret_cast<uint32_t*>(smem + L.list_key_off);
    int32_t* lslot = reinterpret_cast<int32_t*>(smem + L.list_slot_off);
    uint32_t* cnt = reinterpret_cast<uint32_t*>(smem + L.qstate_off);
    uint32_t* worst = cnt + NQ;
    float* thr = reinterpret_cast<float*>(worst + NQ);
    uint32_t* pcnt = reinterpret_cast<uint32_t*>(smem + L.pend_off);
    uint2* pend = reinterpret_cast<uint2*>(smem + L.pend_off + ((NQ * 4 + 16 + 15) / 16 * 16));
    uint2* merge_scratch = pend + NQ * kResQPer;
    uint32_t* wball = reinterpret_cast<uint32_t*>(merge_scratch + 4 * (kMaxKp + kResQPer));  // [4][NQ]
    uint32_t* scount = reinterpret_cast<uint32_t*>(smem + L.sparse_off);
    uint4* sbuf = reinterpret_cast<uint4*>(smem + L.sparse_off + 16);
    constexpr uint32_t kTmemCols = NQ <= 16 ? 32 : (2 * NQ <= 64 ? 64 : 128);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(full + s, 1);
            // released by the MMA commits of every CTA in the cluster, or by
            // the four epilogue warps in the FFMA (single-query) mode
            mbar_init(empty + s, p.ffma ? 4 : CS);  // helper mode: one group of four warps per stage
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(tfull + a, 1);
            mbar_init(tempty + a, 4);
        }
        mbar_init(qfull, 1);
        if constexpr (kHelp) {
            uint64_t* sfull = reinterpret_cast<uint64_t*>(smem + L.pb_off);
            for (int r = 0; r < kRing; ++r) {
                mbar_init(sfull + r, 8);          // both dot-product groups wrote their partials
                mbar_init(sfull + kRing + r, 4);  // the list warps read them
            }
        }
        fence_mbar_init();
    }
    for (int j = threadIdx.x; j < NQ; j += blockDim.x) {
        cnt[j] = 0;
        worst[j] = 0;
        thr[j] = p.thr0;
        pcnt[j] = 0;
    }
    if (threadIdx.x == 0) *scount = 0;
    const int crank = CS > 1 ? static_cast<int>(cluster_ctarank()) : 0;
    const int cid = CS > 1 ? static_cast<int>(cluster_id_x()) : static_cast<int>(blockIdx.x);
    const int ncl = CS > 1 ? static_cast<int>(cluster_count_x()) : static_cast<int>(gridDim.x);
    const int nq_local = max(0, min(NQ, p.nq - crank * NQ));
    constexpr uint16_t kMask = static_cast<uint16_t>((1u << CS) - 1u);
    constexpr int kSliceRows = kUmmaN / CS;
    if (warp == 5) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(kTmemCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    if constexpr (CS > 1)
        cluster_sync_all();  // every CTA's barriers exist before any multicast lands
    else
        __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const int kb_elems = p.tf32 ? kUmmaKB / 4 : kUmmaKB / 2;
    pdl_trigger();  // every CTA is resident: the merge may be scheduled as SMs free up

    if (warp == 4) {
        // ---------------- TMA producer ----------------
        if (lane == 0) {
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&qmap)) : "memory");
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&rmap)) : "memory");
            const uint64_t pol_rows = l2_evict_first_policy();
            const uint64_t pol_q = l2_evict_last_policy();
            // this CTA's query group, once.  The rows do not depend on the
            // query-prep kernel, so the first S row stages are issued before
            // waiting for it (PDL); the queries follow.
            bool qdone = false;
            auto load_q = [&]() {
                pdl_wait();
                mbar_arrive_expect_tx(qfull, static_cast<uint32_t>(nkb) * NQ * kUmmaKB);
                for (int kb = 0; kb < nkb; ++kb)
                    tma_load_2d(sq + static_cast<size_t>(kb) * NQ * kUmmaKB, &qmap, qfull, kb * kb_elems,
                                crank * NQ, pol_q);
                qdone = true;
            };
            int s = 0, issued = 0;
            uint32_t ph = 0;
            for (int t = cid; t < p.ntiles; t += ncl) {
                for (int kb = 0; kb < nkb; ++kb) {
                    if (!qdone && issued == S) load_q();
                    ++issued;
                    mbar_wait(empty + s, ph ^ 1);
                    mbar_arrive_expect_tx(full + s, kUmmaN * kUmmaKB);
                    uint8_t* dst = sa + static_cast<size_t>(s) * kUmmaN * kUmmaKB + crank * kSliceRows * kUmmaKB;
                    const int tt = t * p.tile_stride;
                    if constexpr (CS > 1)
                        tma_load_2d_mc(dst, &rmap, full + s, kb * kb_elems, tt * kUmmaN + crank * kSliceRows, kMask,
                                       pol_rows);
                    else
                        tma_load_2d(dst, &rmap, full + s, kb * kb_elems, tt * kUmmaN, pol_rows);
                    if (++s == S) {
                        s = 0;
                        ph ^= 1;
                    }
                }
            }
            if (!qdone) load_q();
        }
    } else if (warp == 5) {
        // ---------------- MMA issuer: D[128 rows, NQ] += A(rows) . B(queries)^T ----------------
        if (lane == 0 && !p.ffma) {
            const uint32_t idesc = umma_idesc(p.tf32, kUmmaN, NQ);
            mbar_wait(qfull, 0);
            int s = 0;
            uint32_t ph = 0;
            int i = 0;
            for (int t = cid; t < p.ntiles; t += ncl, ++i) {
                const int acc = i & 1;
                mbar_wait(tempty + acc, ((i >> 1) & 1) ^ 1);
                tc_fence_after();
                const uint32_t d = tmem + acc * NQ;
                for (int kb = 0; kb < nkb; ++kb) {
                    mbar_wait(full + s, ph);
                    tc_fence_after();
                    const uint32_t a0 = smem_u32(sa + static_cast<size_t>(s) * kUmmaN * kUmmaKB);
                    const uint32_t b0 = smem_u32(sq + static_cast<size_t>(kb) * NQ * kUmmaKB);
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk) {
                        const uint64_t ad = umma_smem_desc(a0 + kk * 32);
                        const uint64_t bd = umma_smem_desc(b0 + kk * 32);
                        const uint32_t accum = (kb | kk) ? 1u : 0u;
                        if (p.tf32)
                            umma_tf32(d, ad, bd, idesc, accum);
                        else
                            umma_f16(d, ad, bd, idesc, accum);
                    }
                    if constexpr (CS > 1)
                        umma_commit_mc(empty + s, kMask);  // the stage is free in this CTA's view
                    else
                        umma_commit(empty + s);
                    if (++s == S) {
                        s = 0;
                        ph ^= 1;
                    }
                }
                umma_commit(tfull + acc);
            }
        }
    } else if (kHelp && warp >= 6) {
        // ---------------- FFMA dot-product warps (p.ffma == 3) ----------------
        // two groups of four split each tile's K blocks by ring parity and
        // hand the partial scores to the list warps through a ring of
        // kRing tiles, so list upkeep never stalls the HBM stream
        const int grp = (warp - 6) >> 2;
        const int row = threadIdx.x - kUmmaThreads - grp * 128;
        const float* fq = reinterpret_cast<const float*>(smem + L.fq_off);
        uint64_t* sfull = reinterpret_cast<uint64_t*>(smem + L.pb_off);
        uint64_t* sempty = sfull + kRing;
        float* sring = reinterpret_cast<float*>(sempty + kRing);
        mbar_wait(qfull, 0);
        named_bar_sync(3, 128 + kUmmaHelperThreads);  // the list warps widened the bf16 query into fq
        int i = 0;
        for (int t = cid; t < p.ntiles; t += ncl, ++i) {
            constexpr int kQ = HQ > 0 ? HQ : 1;
            float part[kQ];
            ffma_kpar<kQ>(part, i, grp, nkb, S, row, p.tf32 != 0, sa, sq, NQ, fq, full, empty, lane);
            const int r = i % kRing;
            mbar_wait(sempty + r, static_cast<uint32_t>(((i / kRing) & 1) ^ 1));
#pragma unroll
            for (int j = 0; j < kQ; ++j) sring[((r * 2 + grp) * HQ + j) * 128 + row] = part[j];
            __syncwarp();
            if (lane == 0) mbar_arrive(sfull + r);
        }
    } else {
        // ---------------- epilogue: thread = row ----------------
        pdl_wait();  // the admission bounds come from the query-prep kernel
        const int tid = threadIdx.x;  // 0..127 == TMEM lane == row within tile
        const bool slot_ids = p.slot_ids != 0;
        int i = 0;
        int fs = 0;  // FFMA mode: this thread's view of the stage ring
        uint32_t fph = 0;
        float* fq = reinterpret_cast<float*>(smem + L.fq_off);
        if (p.ffma) {
            mbar_wait(qfull, 0);
            if (!p.tf32) {  // widen the bf16 queries once (query j's 16-B chunk c sits at c ^ (j & 7))
                constexpr int kWide = HQ > 1 ? HQ : 1;
                for (int e = tid; e < kWide * nkb * (kUmmaKB / 2); e += 128) {
                    const int j = e / (nkb * (kUmmaKB / 2));
                    const int r = e - j * nkb * (kUmmaKB / 2);
                    const int kb = r / (kUmmaKB / 2), c = r % (kUmmaKB / 2);
                    const uint16_t v = *reinterpret_cast<const uint16_t*>(
                        sq + static_cast<size_t>(kb) * NQ * kUmmaKB + j * kUmmaKB + ((((c >> 3) ^ (j & 7)) << 4) | ((c & 7) << 1)));
                    fq[e] = __uint_as_float(static_cast<uint32_t>(v) << 16);
                }
                named_bar_sync(2, 128);
            }
            if constexpr (kHelp) named_bar_sync(3, 128 + kUmmaHelperThreads);
        }
        uint64_t* sfull = reinterpret_cast<uint64_t*>(smem + L.pb_off);
        const float* sring = reinterpret_cast<const float*>(sfull + 2 * kRing);
        for (int t = cid; t < p.ntiles; t += ncl, ++i) {
            const int acc = i & 1;
            const int64_t slot = static_cast<int64_t>(t) * p.tile_stride * kUmmaN + tid;
            const uint32_t vw = slot < p.nslots ? __ldg(p.valid + (slot >> 5)) : 0u;
            const bool live = ((vw >> (slot & 31)) & 1u) != 0;
            // refresh the admission thresholds with the chip-wide bound: the
            // k'-th best of any CTA's rows is <= the global k'-th best
            if (tid < nq_local) {
                const uint32_t g = *reinterpret_cast<volatile uint32_t*>(p.gbound + crank * NQ + tid);
                if (g) thr[tid] = fmaxf(thr[tid], key_f32(g));
            }
            named_bar_sync(2, 128);
            float sc[NQ];
            if constexpr (kHelp) {
                const int r = i % kRing;
                mbar_wait(sfull + r, static_cast<uint32_t>((i / kRing) & 1));
#pragma unroll
                for (int j = 0; j < NQ; ++j)
                    sc[j] = j < HQ ? (sring[((r * 2) * HQ + j) * 128 + tid] + sring[((r * 2 + 1) * HQ + j) * 128 + tid]) + 0.0f
                                   : 0.0f;
                __syncwarp();
                if (lane == 0) mbar_arrive(sfull + kRing + r);
            } else if (p.ffma) {
                // one query: the dot products on the CUDA cores with packed
                // FFMA2 (two fp32 lanes per instruction), read from the
                // 128B-swizzled stages (16-B chunk c of row r sits at chunk
                // c ^ (r & 7)); bf16 rows widen with a shift / mask per pair
                // against the query pre-converted to fp32 in smem
                uint64_t acc2[2] = {0ull, 0ull};  // {lo, hi} fp32 pairs (FFMA2)
                float fa[4] = {0.0f, 0.0f, 0.0f, 0.0f};  // scalar chains (p.ffma == 1)
                const int sw = tid & 7;
                for (int kb = 0; kb < nkb; ++kb) {
                    mbar_wait(full + fs, fph);
                    const uint8_t* rowp = sa + static_cast<size_t>(fs) * kUmmaN * kUmmaKB + tid * kUmmaKB;
                    if (p.tf32 && p.ffma == 1) {  // scalar FFMA, four independent chains
                        const uint8_t* qp = sq + static_cast<size_t>(kb) * NQ * kUmmaKB;
#pragma unroll
                        for (int c = 0; c < 8; ++c) {
                            const uint4 xv = *reinterpret_cast<const uint4*>(rowp + ((c ^ sw) << 4));
                            const uint4 qv = *reinterpret_cast<const uint4*>(qp + (c << 4));
                            fa[0] = fmaf(__uint_as_float(xv.x), __uint_as_float(qv.x), fa[0]);
                            fa[1] = fmaf(__uint_as_float(xv.y), __uint_as_float(qv.y), fa[1]);
                            fa[2] = fmaf(__uint_as_float(xv.z), __uint_as_float(qv.z), fa[2]);
                            fa[3] = fmaf(__uint_as_float(xv.w), __uint_as_float(qv.w), fa[3]);
                        }
                    } else if (p.tf32) {
                        const uint8_t* qp = sq + static_cast<size_t>(kb) * NQ * kUmmaKB;
#pragma unroll
                        for (int c = 0; c < 8; ++c) {
                            const uint4 xv = *reinterpret_cast<const uint4*>(rowp + ((c ^ sw) << 4));
                            const uint4 qv = *reinterpret_cast<const uint4*>(qp + (c << 4));
                            ffma2(acc2[0], pack2(xv.x, xv.y), pack2(qv.x, qv.y));
                            ffma2(acc2[1], pack2(xv.z, xv.w), pack2(qv.z, qv.w));
                        }
                    } else {
                        const float4* qf = reinterpret_cast<const float4*>(fq + kb * (kUmmaKB / 2));
#pragma unroll
                        for (int c = 0; c < 8; ++c) {
                            const uint4 xv = *reinterpret_cast<const uint4*>(rowp + ((c ^ sw) << 4));
                            const float4 q0 = qf[2 * c], q1 = qf[2 * c + 1];
                            // bf16 pair w -> fp32 (w << 16, w & 0xffff0000)
                            ffma2(acc2[0], pack2(xv.x << 16, xv.x & 0xffff0000u),
                                  pack2(__float_as_uint(q0.x), __float_as_uint(q0.y)));
                            ffma2(acc2[1], pack2(xv.y << 16, xv.y & 0xffff0000u),
                                  pack2(__float_as_uint(q0.z), __float_as_uint(q0.w)));
                            ffma2(acc2[0], pack2(xv.z << 16, xv.z & 0xffff0000u),
                                  pack2(__float_as_uint(q1.x), __float_as_uint(q1.y)));
                            ffma2(acc2[1], pack2(xv.w << 16, xv.w & 0xffff0000u),
                                  pack2(__float_as_uint(q1.z), __float_as_uint(q1.w)));
                        }
                    }
                    __syncwarp();
                    if (lane == 0) mbar_arrive(empty + fs);
                    if (++fs == S) {
                        fs = 0;
                        fph ^= 1;
                    }
                }
                const float s0 = __uint_as_float(static_cast<uint32_t>(acc2[0])) +
                                 __uint_as_float(static_cast<uint32_t>(acc2[1])) + (fa[0] + fa[2]);
                const float s1 = __uint_as_float(static_cast<uint32_t>(acc2[0] >> 32)) +
                                 __uint_as_float(static_cast<uint32_t>(acc2[1] >> 32)) + (fa[1] + fa[3]);
                sc[0] = (s0 + s1) + 0.0f;
#pragma unroll
                for (int j = 1; j < NQ; ++j) sc[j] = 0.0f;
            } else {
                mbar_wait(tfull + acc, (i >> 1) & 1);
                tc_fence_after();
#pragma unroll
                for (int c = 0; c < NQ / 16; ++c) {
                    uint32_t r[16];
                    const uint32_t taddr = tmem + (static_cast<uint32_t>(warp * 32) << 16) + acc * NQ + c * 16;
                    SINE_TMEM_LD16(taddr, r);
                    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
                    for (int j = 0; j < 16; ++j) sc[c * 16 + j] = __uint_as_float(r[j]) + 0.0f;
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(tempty + acc);  // TMEM buffer free for tile i+2
            }
            if (p.out_max) {
                tile_max_out<NQ>(sc, live, nq_local, wball, p.out_max + static_cast<size_t>(t) * p.nq + crank * NQ,
                                 warp, lane, tid);
                continue;
            }

            uint64_t mask = 0;
            if (live) {
#pragma unroll
                for (int j = 0; j < NQ; ++j)
                    if (j < nq_local && sc[j] >= thr[j]) mask |= 1ull << j;
            }
            // sparse hand-off: once the thresholds are warm a tile admits a
            // few pairs; they go to a tile buffer and are inserted one by
            // one.  A warm-up tile (many rows pass) takes the dense rounds.
            const int nrows = bar_red_popc(1, 128, mask != 0);
            bool dense = nrows > kSparseRows;
            uint32_t ns = 0;
            if (nrows && !dense) {
                while (mask) {
                    const int j = __ffsll(mask) - 1;
                    const uint32_t at = atomicAdd(scount, 1u);
                    if (at >= kSparse) break;  // the rest takes the dense rounds below
                    sbuf[at] = make_uint4(static_cast<uint32_t>(j), static_cast<uint32_t>(slot),
                                          f32_key(pick_reg<NQ>(sc, j)), 0u);
                    mask &= mask - 1;
                }
                dense = bar_red_or(1, 128, mask != 0);
                ns = min(*reinterpret_cast<volatile uint32_t*>(scount), static_cast<uint32_t>(kSparse));
            }
            if (ns) {
                sparse_insert_phase(sbuf, ns, lkey, lslot, cnt, thr, p.gbound + crank * NQ, kp, p.ids, slot_ids,
                                    warp, lane);
                if (tid == 0) *scount = 0;
                if (mask) {
#pragma unroll
                    for (int j = 0; j < NQ; ++j)
                        if (((mask >> j) & 1ull) && !(sc[j] >= thr[j])) mask &= ~(1ull << j);
                }
            }
            while (dense && bar_red_or(1, 128, mask != 0)) {
                // queue what fits (row order), positions from ballots -- no
                // atomics: in a warm-up tile every row passes for every query
                for (int j = 0; j < NQ; ++j) {
                    const uint32_t b = __ballot_sync(0xffffffffu, (mask >> j) & 1ull);
                    if (lane == 0) wball[warp * NQ + j] = b;
                }
                named_bar_sync(2, 128);
                if (mask) {
                    const uint32_t lt = (1u << lane) - 1u;
                    uint64_t m = mask;
                    while (m) {
                        const int j = __ffsll(m) - 1;
                        m &= m - 1;
                        uint32_t pos = __popc(wball[warp * NQ + j] & lt);
                        for (int w = 0; w < warp; ++w) pos += __popc(wball[w * NQ + j]);
                        if (pos < kResQPer) {
                            pend[j * kResQPer + pos] = make_uint2(static_cast<uint32_t>(slot), f32_key(pick_reg<NQ>(sc, j)));
                            mask &= ~(1ull << j);
                        }
                    }
                }
                if (tid < NQ) {
                    uint32_t c = 0;
                    for (int w = 0; w < 4; ++w) c += __popc(wball[w * NQ + tid]);
                    pcnt[tid] = c;
                }
                named_bar_sync(2, 128);
                for (int j = warp; j < nq_local; j += 4) {
                    const int np = static_cast<int>(min(pcnt[j], static_cast<uint32_t>(kResQPer)));
                    if (np > 0) {
                        uint32_t* lk = lkey + j * kp;
                        int32_t* ls = lslot + j * kp;
                        const int n = warp_rank_merge(lk, ls, static_cast<int>(cnt[j]), kp, pend + j * kResQPer, np,
                                                      merge_scratch + warp * (kMaxKp + kResQPer), p.ids,
                                                      slot_ids, lane);
                        if (lane == 0) {
                            cnt[j] = n;
                            if (n == kp) {
                                const uint32_t wk = lk[kp - 1];
                                thr[j] = fmaxf(thr[j], key_f32(wk));
                                atomicMax(p.gbound + crank * NQ + j, wk);
                            }
                        }
                    }
                    __syncwarp();
                    if (lane == 0) pcnt[j] = 0;
                }
                named_bar_sync(2, 128);
                // thresholds only rise: drop pairs that no longer qualify
                if (mask) {
#pragma unroll
                    for (int j = 0; j < NQ; ++j)
                        if (((mask >> j) & 1ull) && !(sc[j] >= thr[j])) mask &= ~(1ull << j);
                }
            }
        }
        named_bar_sync(2, 128);
        for (int j = 0; j < nq_local && !p.out_max; ++j) {
            const int qg = crank * NQ + j;  // query index within the launch
            const uint32_t n = cnt[j];
            const size_t base = (static_cast<size_t>(cid) * p.nq + qg) * kp;
            for (int e = tid; e < static_cast<int>(n); e += 128) {
                p.out_key[base + e] = lkey[j * kp + e];
                p.out_slot[base + e] = lslot[j * kp + e];
            }
            if (tid == 0) p.out_n[cid * p.nq + qg] = static_cast<int>(n);
        }
    }
    tc_fence_before();
    if constexpr (CS > 1)
        cluster_sync_all();  // no CTA leaves while peers may still multicast into it
    else
        __syncthreads();
    if (warp == 5) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols));
    }
}

// Seed of the chip-wide admission bound from a sample pass: per query, the
// kp-th best key over the sampled per-CTA lists (0 if fewer than kp).
__global__ void __launch_bounds__(256) sample_bound_kernel(const uint32_t* in_key, const int32_t* in_n, int ncta,
                                                           int nq, int kp, uint32_t* gbound) {
    __shared__ uint32_t hist[256];
    __shared__ uint32_t scratch[16];
    const int qi = blockIdx.x;
    const int nflat = ncta * kp;
    uint32_t before, equal;
    uint32_t tot = 0;
    for (int c = threadIdx.x; c < ncta; c += 256) tot += in_n[c * nq + qi];
    tot = __reduce_add_sync(0xffffffffu, tot);
    if ((threadIdx.x & 31) == 0) scratch[threadIdx.x >> 5] = tot;
    __syncthreads();
    uint32_t total = 0;
    for (int w = 0; w < 8; ++w) total += scratch[w];
    __syncthreads();
    if (total < static_cast<uint32_t>(kp)) {
        if (threadIdx.x == 0) gbound[qi] = 0;
        return;
    }
    const uint32_t kstar = block_select<uint32_t>(
        [&](int f, uint32_t& key) {
            const int c = f / kp, e = f - c * kp;
            if (e >= in_n[c * nq + qi]) return false;
            key = in_key[(static_cast<size_t>(c) * nq + qi) * kp + e];
            return true;
        },
        nflat, static_cast<uint32_t>(kp), true, 32, hist, scratch, &before, &equal);
    if (threadIdx.x == 0) gbound[qi] = kstar;
}

// Seed of the chip-wide admission bound from a max-sample pass: per query,
// the kp-th largest of the ntile sampled tile maxima (0 if fewer than kp).
__global__ void __launch_bounds__(256) sample_max_bound_kernel(const uint32_t* tmax, int ntile, int nq, int kp,
                                                               uint32_t* gbound) {
    __shared__ uint32_t hist[256];
    __shared__ uint32_t scratch[16];
    const int qi = blockIdx.x;
    uint32_t before, equal;
    uint32_t c = 0;
    for (int f = threadIdx.x; f < ntile; f += 256) c += tmax[static_cast<size_t>(f) * nq + qi] != 0u ? 1u : 0u;
    c = __reduce_add_sync(0xffffffffu, c);
    if ((threadIdx.x & 31) == 0) scratch[threadIdx.x >> 5] = c;
    __syncthreads();
    uint32_t total = 0;
    for (int w = 0; w < 8; ++w) total += scratch[w];
    __syncthreads();
    if (total < static_cast<uint32_t>(kp)) {
        if (threadIdx.x == 0) gbound[qi] = 0;
        return;
    }
    const uint32_t kstar = block_select<uint32_t>(
        [&](int f, uint32_t& key) {
            key = tmax[static_cast<size_t>(f) * nq + qi];
            return key != 0u;
        },
        ntile, static_cast<uint32_t>(kp), true, 32, hist, scratch, &before, &equal);
    if (threadIdx.x == 0) gbound[qi] = kstar;
}

// q64 [nq][dim] -> zero-padded [Nq][stride] bf16 or fp32 (TMA source).
// Also zeroes the launch's chip-wide admission bounds (zero_n entries of
// `zero`, nullable) -- one launch instead of a memset plus a launch.
__global__ void res_prep_queries(const double* q64, int nq, int Nq, int64_t dim, int64_t stride, int tf32,
                                 void* out, uint32_t* zero = nullptr, int64_t zero_n = 0) {
    pdl_trigger();  // the scan may start its setup (barriers, TMEM, first row tiles) now
    for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < zero_n;
         t += static_cast<int64_t>(gridDim.x) * blockDim.x)
        zero[t] = 0u;
    const int64_t total = static_cast<int64_t>(Nq) * stride;
    for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < total;
         t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t qrow = t / stride, c = t - qrow * stride;
        const double v = (qrow < nq && c < dim) ? q64[qrow * dim + c] : 0.0;
        if (tf32)
            static_cast<float*>(out)[t] = static_cast<float>(v);
        else
            static_cast<__nv_bfloat16*>(out)[t] = __float2bfloat16_rn(static_cast<float>(v));
    }
}

}  // namespace sine

namespace sine {

// ===========================================================================
// CTA-pair variant (tcgen05 cta_group::2): one MMA covers M = 256 SE rows
// (128 per CTA, each CTA TMA-loads its own rows) against N = 2*NQH queries,
// of which each CTA keeps only its half resident in shared memory (the
// B operand is split by N across the pair).  Each CTA's TMEM receives its
// 128 rows x all N scores.  This keeps 64 fp32 (tf32) queries per HBM pass
// with 96 KB of resident queries per SM.  The leader CTA (rank 0) owns the
// stage / query barriers and issues the MMAs; completions are multicast to
// both CTAs, and both epilogues release the accumulator on the leader.
// ===========================================================================

__device__ __forceinline__ uint32_t leader_addr(const void* p) { return smem_u32(p) & 0xFEFFFFFFu; }

__device__ __forceinline__ void tma_load_2d_pair(void* smem_dst, const CUtensorMap* map, uint32_t leader_bar, int c0,
                                                 int c1, uint64_t policy) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(smem_dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(leader_bar), "r"(c0), "r"(c1), "l"(policy)
        : "memory");
}

__device__ __forceinline__ void umma_tf32_pair(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
        "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void umma_f16_pair(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
        "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void umma_commit_pair(uint64_t* bar) {
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            smem_u32(bar)),
        "h"(static_cast<uint16_t>(3))
        : "memory");
}

__device__ __forceinline__ void mbar_arrive_leader(const uint64_t* bar) {
    uint32_t remote;
    asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(remote) : "r"(smem_u32(bar)));
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
}

template <int NQH>  // queries resident per CTA; the pair scores N = 2 * NQH
__global__ void __launch_bounds__(kUmmaThreads, 1) __cluster_dims__(2, 1, 1)
    umma_pair_kernel(const __grid_constant__ CUtensorMap qmap, const __grid_constant__ CUtensorMap rmap,
                     const ResParams p) {
    constexpr int NQ = 2 * NQH;  // queries per launch (all of them reach every CTA's TMEM)
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int S = p.stages, nkb = p.kblocks, kp = p.kp;
    const ResSmem L = res_smem_layout(S, NQ, nkb, kp, NQH);
    uint8_t* sq = smem + L.q_off;
    uint8_t* sa = smem + L.a_off;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + L.bar_off);
    uint64_t* empty = full + S;
    uint64_t* tfull = empty + S;
    uint64_t* tempty = tfull + 2;
    uint64_t* qfull = tempty + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(qfull + 1);
    uint32_t* lkey = reinterpret_cast<uint32_t*>(smem + L.list_key_off);
    int32_t* lslot = reinterpret_cast<int32_t*>(smem + L.list_slot_off);
    uint32_t* cnt = reinterpret_cast<uint32_t*>(smem + L.qstate_off);
    float* thr = reinterpret_cast<float*>(cnt + 2 * NQ);
    uint32_t* pcnt = reinterpret_cast<uint32_t*>(smem + L.pend_off);
    uint2* pend = reinterpret_cast<uint2*>(smem + L.pend_off + ((NQ * 4 + 16 + 15) / 16 * 16));
    uint2* merge_scratch = pend + NQ * kResQPer;
    uint32_t* wball = reinterpret_cast<uint32_t*>(merge_scratch + 4 * (kMaxKp + kResQPer));
    uint32_t* scount = reinterpret_cast<uint32_t*>(smem + L.sparse_off);
    uint4* sbuf = reinterpret_cast<uint4*>(smem + L.sparse_off + 16);
    constexpr uint32_t kTmemCols = 2 * NQ <= 64 ? 64 : (2 * NQ <= 128 ? 128 : 256);
    constexpr int MW = (NQ + 63) / 64;  // 64-bit words of the per-row query mask

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int rank = static_cast<int>(cluster_ctarank());
    const int pair = static_cast<int>(cluster_id_x());
    const int npair = static_cast<int>(cluster_count_x());
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(full + s, 1);
            mbar_init(empty + s, 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(tfull + a, 1);
            mbar_init(tempty + a, 8);  // 4 epilogue warps in each CTA (used on the leader)
        }
        mbar_init(qfull, 1);
        fence_mbar_init();
    }
    for (int j = threadIdx.x; j < NQ; j += blockDim.x) {
        cnt[j] = 0;
        thr[j] = p.thr0;
        pcnt[j] = 0;
    }
    if (threadIdx.x == 0) *scount = 0;
    if (warp == 5) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(kTmemCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    tc_fence_before();
    cluster_sync_all();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const int kb_elems = p.tf32 ? kUmmaKB / 4 : kUmmaKB / 2;
    const int ntiles = p.ntiles;  // 256-row pair tiles

    if (warp == 4) {
        // ---------------- TMA producers (both CTAs; the leader arms the barriers) ----------------
        if (lane == 0) {
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&qmap)) : "memory");
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&rmap)) : "memory");
            const uint64_t pol_rows = l2_evict_first_policy();
            const uint64_t pol_q = l2_evict_last_policy();
            if (rank == 0) mbar_arrive_expect_tx(qfull, 2u * nkb * NQH * kUmmaKB);
            for (int kb = 0; kb < nkb; ++kb)
                tma_load_2d_pair(sq + static_cast<size_t>(kb) * NQH * kUmmaKB, &qmap, leader_addr(qfull),
                                 kb * kb_elems, rank * NQH, pol_q);
            int s = 0;
            uint32_t ph = 0;
            for (int t = pair; t < ntiles; t += npair) {
                const int64_t row0 = (static_cast<int64_t>(t) * p.tile_stride * 2 + rank) * kUmmaN;
                for (int kb = 0; kb < nkb; ++kb) {
                    mbar_wait(empty + s, ph ^ 1);
                    if (rank == 0) mbar_arrive_expect_tx(full + s, 2u * kUmmaN * kUmmaKB);
                    tma_load_2d_pair(sa + static_cast<size_t>(s) * kUmmaN * kUmmaKB, &rmap, leader_addr(full + s),
                                     kb * kb_elems, static_cast<int>(row0), pol_rows);
                    if (++s == S) {
                        s = 0;
                        ph ^= 1;
                    }
                }
            }
        }
    } else if (warp == 5) {
        // ---------------- MMA issuer (leader only): D[256 rows, N] += A . B^T ----------------
        if (rank == 0 && lane == 0) {
            const uint32_t idesc = umma_idesc(p.tf32, 2 * kUmmaN, NQ);
            mbar_wait(qfull, 0);
            int s = 0;
            uint32_t ph = 0;
            int i = 0;
            for (int t = pair; t < ntiles; t += npair, ++i) {
                const int acc = i & 1;
                mbar_wait(tempty + acc, ((i >> 1) & 1) ^ 1);
                tc_fence_after();
                const uint32_t d = tmem + acc * NQ;
                for (int kb = 0; kb < nkb; ++kb) {
                    mbar_wait(full + s, ph);
                    tc_fence_after();
                    const uint32_t a0 = smem_u32(sa + static_cast<size_t>(s) * kUmmaN * kUmmaKB);
                    const uint32_t b0 = smem_u32(sq + static_cast<size_t>(kb) * NQH * kUmmaKB);
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk) {
                        const uint64_t ad = umma_smem_desc(a0 + kk * 32);
                        const uint64_t bd = umma_smem_desc(b0 + kk * 32);
                        const uint32_t accum = (kb | kk) ? 1u : 0u;
                        if (p.tf32)
                            umma_tf32_pair(d, ad, bd, idesc, accum);
                        else
                            umma_f16_pair(d, ad, bd, idesc, accum);
                    }
                    umma_commit_pair(empty + s);
                    if (++s == S) {
                        s = 0;
                        ph ^= 1;
                    }
                }
                umma_commit_pair(tfull + acc);
            }
        }
    } else {
        // ---------------- epilogue: thread = row of this CTA's half tile ----------------
        const int tid = threadIdx.x;
        const bool slot_ids = p.slot_ids != 0;
        const int nq_local = min(NQ, p.nq);
        int i = 0;
        for (int t = pair; t < ntiles; t += npair, ++i) {
            const int acc = i & 1;
            const int64_t slot = (static_cast<int64_t>(t) * p.tile_stride * 2 + rank) * kUmmaN + tid;
            const uint32_t vw = slot < p.nslots ? __ldg(p.valid + (slot >> 5)) : 0u;
            const bool live = ((vw >> (slot & 31)) & 1u) != 0;
            if (tid < nq_local) {
                const uint32_t g = *reinterpret_cast<volatile uint32_t*>(p.gbound + tid);
                if (g) thr[tid] = fmaxf(thr[tid], key_f32(g));
            }
            named_bar_sync(2, 128);
            mbar_wait(tfull + acc, (i >> 1) & 1);
            tc_fence_after();
            float sc[NQ];
#pragma unroll
            for (int c = 0; c < NQ / 16; ++c) {
                uint32_t r[16];
                const uint32_t taddr = tmem + (static_cast<uint32_t>(warp * 32) << 16) + acc * NQ + c * 16;
                SINE_TMEM_LD16(taddr, r);
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
                for (int j = 0; j < 16; ++j) sc[c * 16 + j] = __uint_as_float(r[j]) + 0.0f;
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                if (rank == 0)
                    mbar_arrive(tempty + acc);
                else
                    mbar_arrive_leader(tempty + acc);
            }
            if (p.out_max) {
                tile_max_out<NQ>(sc, live, nq_local, wball, p.out_max + static_cast<size_t>(2 * t + rank) * p.nq,
                                 warp, lane, tid);
                continue;
            }
            uint64_t mask[MW];
#pragma unroll
            for (int w = 0; w < MW; ++w) mask[w] = 0;
            if (live) {
#pragma unroll
                for (int j = 0; j < NQ; ++j)
                    if (j < nq_local && sc[j] >= thr[j]) mask[j >> 6] |= 1ull << (j & 63);
            }
            auto any_mask = [&]() {
                uint64_t o = 0;
#pragma unroll
                for (int w = 0; w < MW; ++w) o |= mask[w];
                return o != 0;
            };
            // sparse hand-off (see umma_res_kernel)
            const int nrows = bar_red_popc(1, 128, any_mask());
            bool dense = nrows > kSparseRows;
            uint32_t ns = 0;
            if (nrows && !dense) {
                bool full = false;
#pragma unroll
                for (int w = 0; w < MW; ++w) {
                    while (mask[w] && !full) {
                        const int jj = __ffsll(mask[w]) - 1;
                        const uint32_t at = atomicAdd(scount, 1u);
                        if (at >= kSparse) {
                            full = true;
                            break;
                        }
                        sbuf[at] = make_uint4(static_cast<uint32_t>(w * 64 + jj), static_cast<uint32_t>(slot),
                                              f32_key(pick_reg<NQ>(sc, w * 64 + jj)), 0u);
                        mask[w] &= mask[w] - 1;
                    }
                }
                dense = bar_red_or(1, 128, any_mask());
                ns = min(*reinterpret_cast<volatile uint32_t*>(scount), static_cast<uint32_t>(kSparse));
            }
            if (ns) {
                sparse_insert_phase(sbuf, ns, lkey, lslot, cnt, thr, p.gbound, kp, p.ids, slot_ids, warp, lane);
                if (tid == 0) *scount = 0;
                if (any_mask()) {
#pragma unroll
                    for (int j = 0; j < NQ; ++j)
                        if (((mask[j >> 6] >> (j & 63)) & 1ull) && !(sc[j] >= thr[j]))
                            mask[j >> 6] &= ~(1ull << (j & 63));
                }
            }
            while (dense && bar_red_or(1, 128, any_mask())) {
#pragma unroll
                for (int j = 0; j < NQ; ++j) {
                    const uint32_t b = __ballot_sync(0xffffffffu, (mask[j >> 6] >> (j & 63)) & 1ull);
                    if (lane == 0) wball[warp * NQ + j] = b;
                }
                named_bar_sync(2, 128);
                if (any_mask()) {
                    const uint32_t lt = (1u << lane) - 1u;
#pragma unroll
                    for (int w = 0; w < MW; ++w) {
                        uint64_t m = mask[w];
                        while (m) {
                            const int jj = __ffsll(m) - 1;
                            m &= m - 1;
                            const int j = w * 64 + jj;
                            uint32_t pos = __popc(wball[warp * NQ + j] & lt);
                            for (int x = 0; x < warp; ++x) pos += __popc(wball[x * NQ + j]);
                            if (pos < kResQPer) {
                                pend[j * kResQPer + pos] = make_uint2(static_cast<uint32_t>(slot), f32_key(pick_reg<NQ>(sc, j)));
                                mask[w] &= ~(1ull << jj);
                            }
                        }
                    }
                }
                if (tid < NQ) {
                    uint32_t c = 0;
                    for (int w = 0; w < 4; ++w) c += __popc(wball[w * NQ + tid]);
                    pcnt[tid] = c;
                }
                named_bar_sync(2, 128);
                for (int j = warp; j < nq_local; j += 4) {
                    const int np = static_cast<int>(min(pcnt[j], static_cast<uint32_t>(kResQPer)));
                    if (np > 0) {
                        uint32_t* lk = lkey + j * kp;
                        int32_t* ls = lslot + j * kp;
                        const int n = warp_rank_merge(lk, ls, static_cast<int>(cnt[j]), kp, pend + j * kResQPer, np,
                                                      merge_scratch + warp * (kMaxKp + kResQPer), p.ids, slot_ids,
                                                      lane);
                        if (lane == 0) {
                            cnt[j] = n;
                            if (n == kp) {
                                const uint32_t wk = lk[kp - 1];
                                thr[j] = fmaxf(thr[j], key_f32(wk));
                                atomicMax(p.gbound + j, wk);
                            }
                        }
                    }
                    __syncwarp();
                }
                named_bar_sync(2, 128);
                if (any_mask()) {
#pragma unroll
                    for (int j = 0; j < NQ; ++j)
                        if (((mask[j >> 6] >> (j & 63)) & 1ull) && !(sc[j] >= thr[j]))
                            mask[j >> 6] &= ~(1ull << (j & 63));
                }
            }
        }
        named_bar_sync(2, 128);
        for (int j = 0; j < nq_local && !p.out_max; ++j) {
            const uint32_t n = cnt[j];
            const size_t base = (static_cast<size_t>(blockIdx.x) * p.nq + j) * kp;
            for (int e = tid; e < static_cast<int>(n); e += 128) {
                p.out_key[base + e] = lkey[j * kp + e];
                p.out_slot[base + e] = lslot[j * kp + e];
            }
            if (tid == 0) p.out_n[blockIdx.x * p.nq + j] = static_cast<int>(n);
        }
    }
    tc_fence_before();
    cluster_sync_all();
    if (warp == 5) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols));
    }
}

}  // namespace sine

namespace sine {

// ===========================================================================
// Large batches (the tensor-bound regime, B in the thousands): a tiled
// GEMM over (256-row tile) x (256-query tile) work items, all query tiles of
// the batch in ONE launch.  A CTA pair (tcgen05 cta_group::2) owns an item:
// each CTA TMA-loads 128 rows and 128 queries per 128-byte K block, the
// leader issues M=256 x N=256 MMAs, and each CTA's TMEM receives its 128 rows
// x 256 query scores (double-buffered: 2 x 256 columns = all 512).  Items are
// ordered row-tile-major, so the pairs in flight at any moment work on a few
// row tiles x every query tile: each row tile is read from HBM once and
// re-served from L2 to the other query tiles; the queries (B x d) stay L2
// resident.
//
// Epilogue (warps 0-3, thread = row): every score is compared with the
// uniform admission floor thr0; passing (query, row) pairs are appended to
// per-query candidate chunks in global memory ([C][nq][kp], the layout the
// merge kernel reads as C lists).  There are no per-query lists to maintain,
// so the epilogue is a TMEM drain plus a max-reduction per 32 scores.  All
// rows >= thr0 are kept; a query whose count exceeds C*kp overflows and the
// host re-runs the batch on the list-keeping kernels (used only at high
// thresholds, where candidates are rare: the engine's tau_sim).
// Reference: `self._vecs @ arr` + the `>= min_similarity` mask of `_rank`
// (pkg/src/semcache/index.py:101, :43), for B queries at once.
// ===========================================================================

constexpr int kGemmNQ = 256;      // max queries per item (MMA N); the kernel is templated on NQ <= 256
constexpr int kGemmRows = 256;    // rows per item (MMA M, 128 per CTA)
constexpr int kGemmThreads = 192;

struct GemmParams {
    int64_t nslots;
    int nrt, nqt;        // row tiles (256), query tiles (256)
    int kblocks;
    int nq;              // live queries
    int kp, chunks;      // candidate capacity per query = chunks * kp
    float thr0;
    int stages;
    int tf32;
    const uint32_t* valid;
    uint32_t* cnt;       // [nq] pairs >= thr0 seen per query (may exceed capacity)
    uint32_t* out_key;   // [chunks][nq][kp]
    int32_t* out_slot;
    const uint32_t* qthr;  // [nq] per-query admission keys (max with thr0), nullable = uniform thr0
    int rt_stride;         // row tile t of the launch is physical tile t * rt_stride (sample pass)
    uint32_t* out_max;     // sample pass: [2 * t + rank][nq] max score key of the CTA's 128 rows
};

// per stage and CTA: 128 rows + NQ/2 queries, 128 B of K each
__host__ __device__ inline size_t gemm_stage_bytes(int NQ) { return static_cast<size_t>(128 + NQ / 2) * kUmmaKB; }

__host__ __device__ inline size_t gemm_smem_bytes(int S, int NQ) {
    return static_cast<size_t>(S) * gemm_stage_bytes(NQ) + (2 * S + 4) * sizeof(uint64_t) + 16 + 3 * 256 * 4 + 1024;
}

__device__ __forceinline__ void gemm_append(const GemmParams& p, int q, uint32_t key, int32_t slot) {
    const uint32_t at = atomicAdd(p.cnt + q, 1u);
    const uint32_t cap = static_cast<uint32_t>(p.chunks * p.kp);
    if (at < cap) {
        const uint32_t c = at / p.kp, e = at - c * p.kp;
        const size_t o = (static_cast<size_t>(c) * p.nq + q) * p.kp + e;
        p.out_key[o] = key;
        p.out_slot[o] = slot;
    }
}

// Epilogue of one item for the sample pass (out_max: per query, the max
// score key over this CTA's 128 rows -> [2t + rank][nq]) or for per-query
// admission floors (qthr, staged in shared memory per item).  A 32-score
// chunk of a row is skipped when its max is below the chunk's smallest floor.
template <int NQ>
__device__ __noinline__ void gemm_epilogue_general(const GemmParams& p, uint32_t tmem, int acc, int warp, int lane,
                                                   int tid, bool live, int64_t slot, int qbase, size_t orow,
                                                   uint32_t* colmax, float* fl, uint64_t* tfull, int i) {
    if (!p.out_max) {
        const uint32_t k0 = f32_key(p.thr0);
        for (int j = tid; j < NQ; j += 128) {
            const int q = qbase + j;
            fl[j] = q < p.nq ? key_f32(max(k0, __ldg(p.qthr + q))) : INFINITY;
        }
        named_bar_sync(2, 128);  // (fl is double-buffered by accumulator: one barrier per item suffices)
    }
    mbar_wait(tfull + acc, (i >> 1) & 1);
    tc_fence_after();
    // chunks not unrolled and appends in a bit loop: keeps the code small
    // (an unrolled 256-site append body thrashes the instruction cache)
#pragma unroll 1
    for (int c = 0; c < NQ / 32; ++c) {
        uint32_t r[32];
        const uint32_t taddr = tmem + (static_cast<uint32_t>(warp * 32) << 16) + acc * NQ + c * 32;
        SINE_TMEM_LD32(taddr, r);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (p.out_max) {
            uint32_t mine = 0;
#pragma unroll
            for (int j = 0; j < 32; ++j) {
                const float x = __uint_as_float(r[j]);
                const uint32_t kx = (live && x == x) ? f32_key(x + 0.0f) : 0u;  // NaN never sets a bound
                const uint32_t m = __reduce_max_sync(0xffffffffu, kx);
                if (lane == j) mine = m;
            }
            atomicMax(colmax + c * 32 + lane, mine);
            continue;
        }
        const float tmin = key_f32(__reduce_min_sync(0xffffffffu, f32_key(fl[c * 32 + lane])));
        float m = -INFINITY;
#pragma unroll
        for (int j = 0; j < 32; ++j) m = fmaxf(m, __uint_as_float(r[j]));
        if (live && m >= tmin) {
            uint32_t pass = 0;
#pragma unroll
            for (int j = 0; j < 32; ++j)
                if (__uint_as_float(r[j]) + 0.0f >= fl[c * 32 + j] && qbase + c * 32 + j < p.nq) pass |= 1u << j;
            while (pass) {
                const int j = __ffs(pass) - 1;
                pass &= pass - 1;
                float sc = 0.0f;
#pragma unroll
                for (int jj = 0; jj < 32; ++jj)
                    if (jj == j) sc = __uint_as_float(r[jj]);
                gemm_append(p, qbase + c * 32 + j, f32_key(sc + 0.0f), static_cast<int32_t>(slot));
            }
        }
    }
    if (p.out_max) {
        named_bar_sync(2, 128);
        for (int j = tid; j < NQ; j += 128) {
            const int q = qbase + j;
            if (q < p.nq) p.out_max[orow * p.nq + q] = colmax[j];
            colmax[j] = 0u;
        }
        named_bar_sync(2, 128);
    }
}

template <int NQ>
__global__ void __launch_bounds__(kGemmThreads, 1) __cluster_dims__(2, 1, 1)
    umma_gemm_kernel(const __grid_constant__ CUtensorMap qmap, const __grid_constant__ CUtensorMap rmap,
                     const __grid_constant__ GemmParams p) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int S = p.stages, nkb = p.kblocks;
    constexpr size_t kStage = 128 * kUmmaKB;        // 16 KB: 128 rows x 128 B of K
    constexpr size_t kStageB = (NQ / 2) * kUmmaKB;  // this CTA's NQ/2 queries x 128 B of K
    uint8_t* sa = smem;
    uint8_t* sb = smem + S * kStage;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + S * (kStage + kStageB));
    uint64_t* empty = full + S;
    uint64_t* tfull = empty + S;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
    uint32_t* colmax = tmem_slot + 4;  // [256] sample pass: per-query max keys of this item
    float* floors = reinterpret_cast<float*>(colmax + kGemmNQ);  // [2][256] per-query floors (by accumulator)

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int rank = static_cast<int>(cluster_ctarank());
    const int pair = static_cast<int>(cluster_id_x());
    const int npair = static_cast<int>(cluster_count_x());
    const int nitems = p.nrt * p.nqt;
    for (int j = threadIdx.x; j < kGemmNQ; j += blockDim.x) colmax[j] = 0u;
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(full + s, 1);
            mbar_init(empty + s, 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(tfull + a, 1);
            mbar_init(tempty + a, 8);  // 4 epilogue warps in each CTA (used on the leader)
        }
        fence_mbar_init();
    }
    if (warp == 5) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(2 * NQ));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    tc_fence_before();
    cluster_sync_all();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const int kb_elems = p.tf32 ? kUmmaKB / 4 : kUmmaKB / 2;

    if (warp == 4) {
        // ---------------- TMA producers (both CTAs; the leader arms the barriers) ----------------
        if (lane == 0) {
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&qmap)) : "memory");
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&rmap)) : "memory");
            const uint64_t pol_q = l2_evict_last_policy();
            uint64_t pol_rows;  // re-read by the other query tiles of the same row tile
            asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol_rows));
            int s = 0;
            uint32_t ph = 0;
            for (int w = pair; w < nitems; w += npair) {
                const int t = w / p.nqt, g = w - (w / p.nqt) * p.nqt;
                const int r0 = t * p.rt_stride * kGemmRows + rank * 128;
                const int q0 = g * NQ + rank * (NQ / 2);
                for (int kb = 0; kb < nkb; ++kb) {
                    mbar_wait(empty + s, ph ^ 1);
                    if (rank == 0) mbar_arrive_expect_tx(full + s, 2u * static_cast<uint32_t>(kStage + kStageB));
                    tma_load_2d_pair(sa + s * kStage, &rmap, leader_addr(full + s), kb * kb_elems, r0, pol_rows);
                    tma_load_2d_pair(sb + s * kStageB, &qmap, leader_addr(full + s), kb * kb_elems, q0, pol_q);
                    if (++s == S) {
                        s = 0;
                        ph ^= 1;
                    }
                }
            }
        }
    } else if (warp == 5) {
        // ---------------- MMA issuer (leader only): D[256 rows, 256 queries] ----------------
        if (rank == 0 && lane == 0) {
            const uint32_t idesc = umma_idesc(p.tf32, kGemmRows, NQ);
            int s = 0;
            uint32_t ph = 0;
            int i = 0;
            for (int w = pair; w < nitems; w += npair, ++i) {
                const int acc = i & 1;
                mbar_wait(tempty + acc, ((i >> 1) & 1) ^ 1);
                tc_fence_after();
                const uint32_t d = tmem + acc * NQ;
                for (int kb = 0; kb < nkb; ++kb) {
                    mbar_wait(full + s, ph);
                    tc_fence_after();
                    const uint32_t a0 = smem_u32(sa + s * kStage);
                    const uint32_t b0 = smem_u32(sb + s * kStageB);
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk) {
                        const uint64_t ad = umma_smem_desc(a0 + kk * 32);
                        const uint64_t bd = umma_smem_desc(b0 + kk * 32);
                        const uint32_t accum = (kb | kk) ? 1u : 0u;
                        if (p.tf32)
                            umma_tf32_pair(d, ad, bd, idesc, accum);
                        else
                            umma_f16_pair(d, ad, bd, idesc, accum);
                    }
                    umma_commit_pair(empty + s);
                    if (++s == S) {
                        s = 0;
                        ph ^= 1;
                    }
                }
                umma_commit_pair(tfull + acc);
            }
        }
    } else {
        // ---------------- epilogue: thread = row of this CTA's half tile ----------------
        const int tid = threadIdx.x;
        const float thr0 = p.thr0;
        int i = 0;
        for (int w = pair; w < nitems; w += npair, ++i) {
            const int acc = i & 1;
            const int t = w / p.nqt, g = w - (w / p.nqt) * p.nqt;
            const int64_t slot = static_cast<int64_t>(t) * p.rt_stride * kGemmRows + rank * 128 + tid;
            const uint32_t vw = slot < p.nslots ? __ldg(p.valid + (slot >> 5)) : 0u;
            const bool live = ((vw >> (slot & 31)) & 1u) != 0;
            const int qbase = g * NQ;
            if (p.out_max || p.qthr) {
                // sample pass (per-query max over the rows) or per-query
                // admission floors: the general, slower epilogue
                gemm_epilogue_general<NQ>(p, tmem, acc, warp, lane, tid, live, slot, qbase,
                                      static_cast<size_t>(2 * t + rank), colmax, floors + acc * kGemmNQ, tfull, i);
            } else {
            mbar_wait(tfull + acc, (i >> 1) & 1);
            tc_fence_after();
#pragma unroll 1
            for (int c = 0; c < NQ / 32; c += 2) {
                uint32_t r0[32], r1[32];
                const uint32_t taddr = tmem + (static_cast<uint32_t>(warp * 32) << 16) + acc * NQ + c * 32;
                SINE_TMEM_LD32(taddr, r0);
                SINE_TMEM_LD32(taddr + 32, r1);
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                float m0 = -INFINITY, m1 = -INFINITY;
#pragma unroll
                for (int j = 0; j < 32; ++j) {
                    m0 = fmaxf(m0, __uint_as_float(r0[j]));
                    m1 = fmaxf(m1, __uint_as_float(r1[j]));
                }
                if (live && m0 >= thr0) {  // rare: fully unrolled so the scores stay in registers
#pragma unroll
                    for (int j = 0; j < 32; ++j) {
                        const float sc = __uint_as_float(r0[j]) + 0.0f;
                        const int q = qbase + c * 32 + j;
                        if (sc >= thr0 && q < p.nq) gemm_append(p, q, f32_key(sc), static_cast<int32_t>(slot));
                    }
                }
                if (live && m1 >= thr0) {
#pragma unroll
                    for (int j = 0; j < 32; ++j) {
                        const float sc = __uint_as_float(r1[j]) + 0.0f;
                        const int q = qbase + c * 32 + 32 + j;
                        if (sc >= thr0 && q < p.nq) gemm_append(p, q, f32_key(sc), static_cast<int32_t>(slot));
                    }
                }
            }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                if (rank == 0)
                    mbar_arrive(tempty + acc);
                else
                    mbar_arrive_leader(tempty + acc);
            }
        }
    }
    tc_fence_before();
    cluster_sync_all();
    if (warp == 5) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(2 * NQ));
    }
}

// Per-query candidate counts -> the merge kernel's per-list counts, and the
// number of queries whose candidates overflowed the chunk capacity.
__global__ void gemm_finish_kernel(const uint32_t* cnt, int nq, int kp, int chunks, int32_t* out_n,
                                   uint32_t* overflow) {
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= nq) return;
    const uint32_t n = cnt[q];
    for (int c = 0; c < chunks; ++c) {
        const int64_t r = static_cast<int64_t>(n) - static_cast<int64_t>(c) * kp;
        out_n[c * nq + q] = static_cast<int32_t>(r < 0 ? 0 : (r > kp ? kp : r));
    }
    if (n > static_cast<uint32_t>(chunks * kp)) atomicAdd(overflow, 1u);
}

}  // namespace sine
