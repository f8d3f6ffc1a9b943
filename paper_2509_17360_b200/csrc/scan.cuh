// Stage-1 streaming scan (CUDA cores) -- the low-batch Sine path.
//
// Replaces the float64 GEMV `self._vecs @ arr` of ExactCosineIndex.query
// (reference pkg/src/semcache/index.py:101) and the threshold half of
// `_rank` (index.py:43) for up to NQ queries per launch.
//
// Layout: the SE store keeps rows slot-major, `row_bytes` apart (fp32 or
// bf16, zero padded to a multiple of 128 B).  Each CTA owns a contiguous
// slot range and streams it through a ring of shared-memory stages filled
// by the TMA engine (cp.async.bulk + mbarrier complete_tx) issued by one
// producer warp.  Compute warps own fixed 512-byte column chunks of a row
// (lane = 16 B), hold their slice of the NQ queries in registers, and
// reduce each chunk with a fixed butterfly; chunk sums are added in chunk
// order, so the score of a row does not depend on its slot, on the launch
// geometry, or on how many queries share the launch.
//
// Every CTA keeps, per query, the top-k' (k' = k + slack) candidates of its
// slots in shared memory under the reference order (score desc, id asc),
// with a running admission threshold so the common case is one compare per
// (row, query).  The per-CTA lists go to global memory for the merge kernel.
#pragma once

#include "common.cuh"

namespace sine {

struct ScanParams {
    const uint8_t* rows;    // [nslots][row_bytes]
    int64_t row_bytes;      // multiple of 128
    int64_t nslots;
    const uint32_t* valid;  // validity bitmap, 1 bit per slot
    const int64_t* ids;     // [nslots]
    const double* q64;      // [nq][dim] float64 queries (this launch)
    int64_t dim;
    int nq;                 // queries in this launch (<= NQ)
    int kp;                 // per-CTA list capacity
    float thr0;             // admission floor (min_sim, or min_sim - margin)
    int rows_per_stage;     // R = G * RPW (<= 64)
    int stages;             // S
    int64_t rows_per_cta;   // multiple of R
    int chunks;             // C = ceil(row_bytes / 512)
    int chunk_warps;        // CW = ceil(C / CPW)
    int row_groups;         // G
    int unroll;             // RPW: rows per warp per stage (multiple of U; R = G * RPW)
    int slot_ids;           // slot order == id order
    uint32_t* gbound;       // [nq] chip-wide admission bound (f32 keys, zeroed per launch)
    uint32_t* out_key;      // [grid][nq][kp] f32_key(score)
    int32_t* out_slot;      // [grid][nq][kp]
    int32_t* out_n;         // [grid][nq]
};

template <typename RowT>
struct RowTraits;
template <>
struct RowTraits<float> {
    static constexpr int kEPL = 4;  // elements per lane per chunk (16 B)
    __device__ static __forceinline__ void unpack(const uint4& v, float* x) {
        x[0] = __uint_as_float(v.x);
        x[1] = __uint_as_float(v.y);
        x[2] = __uint_as_float(v.z);
        x[3] = __uint_as_float(v.w);
    }
    __device__ static __forceinline__ float round_q(double q) { return static_cast<float>(q); }
};
template <>
struct RowTraits<__nv_bfloat16> {
    static constexpr int kEPL = 8;
    __device__ static __forceinline__ void unpack(const uint4& v, float* x) {
        const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            x[2 * i] = __uint_as_float(w[i] << 16);
            x[2 * i + 1] = __uint_as_float(w[i] & 0xffff0000u);
        }
    }
    // bf16 mode rounds the query to bf16 as well: products are then exact
    // in fp32, matching the tensor-core (kind::f16) path.
    __device__ static __forceinline__ float round_q(double q) {
        return __bfloat162float(__float2bfloat16_rn(static_cast<float>(q)));
    }
};

struct ScanSmemLayout {
    size_t stage_off, bar_off, partial_off, list_key_off, list_slot_off, qstate_off, pend_off, scratch_off, total;
};

__host__ __device__ inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

__host__ __device__ inline ScanSmemLayout scan_smem_layout(int S, int R, int64_t row_bytes, int NQ,
                                                         int C, int kp) {
    ScanSmemLayout L;
    size_t off = 0;
    L.stage_off = off;
    off += align_up(static_cast<size_t>(S) * R * row_bytes, 128);
    L.bar_off = off;
    off += align_up(2 * S * sizeof(uint64_t), 16);
    L.partial_off = off;
    off += align_up(static_cast<size_t>(R) * NQ * C * sizeof(float), 16);
    L.list_key_off = off;
    off += align_up(static_cast<size_t>(NQ) * kp * sizeof(uint32_t), 16);
    L.list_slot_off = off;
    off += align_up(static_cast<size_t>(NQ) * kp * sizeof(int32_t), 16);
    L.qstate_off = off;  // cnt[NQ], worst[NQ], thr[NQ]
    off += align_up(3 * NQ * sizeof(uint32_t), 16);
    L.pend_off = off;  // 2 x { total, cnt[NQ], entries[NQ][R] {slot, key} }
    off += 2 * align_up(align_up((1 + NQ) * sizeof(uint32_t), 16) + static_cast<size_t>(NQ) * R * 8, 16);
    L.scratch_off = off;  // per compute warp: (kp + R) uint2 for the rank merge
    off += static_cast<size_t>(16) * (kp + R) * 8;
    L.total = off;
    return L;
}

// Recompute the worst (last in candidate order) entry of a full list.
// Worst = smallest key; among equal keys, the largest id.
__device__ __forceinline__ int list_worst(const uint32_t* lkey, const int32_t* lslot, int kp,
                                          const int64_t* ids, int lane) {
    uint32_t mk = 0xffffffffu;
    for (int e = lane; e < kp; e += kWarp) mk = min(mk, lkey[e]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mk = min(mk, __shfl_xor_sync(0xffffffffu, mk, o));
    // candidates with the minimum key; if several, the largest id is worst
    int pos = -1;
    int64_t pid = INT64_MIN;
    int nmin = 0;
    for (int e = lane; e < kp; e += kWarp) {
        if (lkey[e] == mk) {
            ++nmin;
            if (pos < 0) pos = e;
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) nmin += __shfl_xor_sync(0xffffffffu, nmin, o);
    if (nmin == 1) {
        int p = pos;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) p = max(p, __shfl_xor_sync(0xffffffffu, p, o));
        return p;
    }
    // exact-score ties at the boundary: resolve with the global ids
    pos = -1;
    for (int e = lane; e < kp; e += kWarp) {
        if (lkey[e] == mk) {
            int64_t id = __ldg(ids + lslot[e]);
            if (id > pid) {
                pid = id;
                pos = e;
            }
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        int64_t oid = __shfl_xor_sync(0xffffffffu, pid, o);
        int opos = __shfl_xor_sync(0xffffffffu, pos, o);
        if (oid > pid) {
            pid = oid;
            pos = opos;
        }
    }
    return pos;
}

// Compute warps per CTA: up to 16 for small query groups (more rows in
// flight), 8 when the per-thread query slice is large (register budget).
template <int NQ>
struct ScanWarps {
    static constexpr int kMax = NQ >= 8 ? 8 : 16;
    static constexpr int kThreads = (kMax + 1) * 32;
};
// rows each warp keeps in flight per stage (independent FMA/shuffle chains)
template <int NQ>
struct ScanUnroll {
    static constexpr int kU = NQ == 1 ? 8 : NQ == 2 ? 4 : NQ == 4 ? 2 : 1;
};

template <typename RowT, int NQ, int CPW>
__global__ void __launch_bounds__(ScanWarps<NQ>::kThreads, 1) scan_kernel(const ScanParams p) {
    using T = RowTraits<RowT>;
    constexpr int EPL = T::kEPL;
    constexpr int M = (NQ == 1) ? 0 : (NQ == 2) ? 1 : (NQ == 4) ? 2 : (NQ == 8) ? 3 : 4;

    extern __shared__ __align__(128) uint8_t smem[];
    constexpr int U = ScanUnroll<NQ>::kU;
    const int S = p.stages, R = p.rows_per_stage, C = p.chunks, CW = p.chunk_warps,
              G = p.row_groups, RPW = p.unroll;  // rows per warp per stage (multiple of U)
    const int W = CW * G;  // compute warps; warp W is the producer
    const ScanSmemLayout L = scan_smem_layout(S, R, p.row_bytes, NQ, C, p.kp);
    uint8_t* stage_base = smem + L.stage_off;
    uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + L.bar_off);
    uint64_t* empty_bar = full_bar + S;
    float* partial = reinterpret_cast<float*>(smem + L.partial_off);  // [R][NQ][C]
    uint32_t* lkey = reinterpret_cast<uint32_t*>(smem + L.list_key_off);
    int32_t* lslot = reinterpret_cast<int32_t*>(smem + L.list_slot_off);
    uint32_t* cnt = reinterpret_cast<uint32_t*>(smem + L.qstate_off);
    uint32_t* worst = cnt + NQ;
    uint32_t* thr = worst + NQ;
    uint2* merge_scratch = reinterpret_cast<uint2*>(smem + L.scratch_off);
    const size_t pend_hdr = align_up((1 + NQ) * sizeof(uint32_t), 16);  // keeps the uint2 entries 8-B aligned
    const size_t pend_bytes = align_up(pend_hdr + static_cast<size_t>(NQ) * R * 8, 16);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int64_t row0 = static_cast<int64_t>(blockIdx.x) * p.rows_per_cta;
    const int64_t row_end = min(row0 + p.rows_per_cta, p.nslots);
    const int nst = row0 < row_end ? static_cast<int>((row_end - row0 + R - 1) / R) : 0;
    const int kp = p.kp, nq = p.nq;
    const uint32_t thr0 = f32_key(p.thr0);

    if (tid == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(full_bar + s, 1);
            mbar_init(empty_bar + s, 1);
        }
        fence_mbar_init();
    }
    for (int j = tid; j < NQ; j += blockDim.x) {
        cnt[j] = 0;
        worst[j] = 0;
        thr[j] = thr0;
    }
    for (int j = tid; j < static_cast<int>(2 * pend_bytes / 4); j += blockDim.x)
        reinterpret_cast<uint32_t*>(smem + L.pend_off)[j] = 0;
    __syncthreads();

    if (warp == W) {
        // ---------------- TMA producer ----------------
        if (lane == 0) {
            const uint64_t pol = l2_evict_first_policy();
            for (int i = 0; i < nst; ++i) {
                const int s = i % S;
                if (i >= S) mbar_wait(empty_bar + s, ((i / S) & 1) ^ 1);
                const int64_t r = row0 + static_cast<int64_t>(i) * R;
                const int rows_i = static_cast<int>(min(static_cast<int64_t>(R), row_end - r));
                const uint32_t bytes = static_cast<uint32_t>(rows_i * p.row_bytes);
                mbar_arrive_expect_tx(full_bar + s, bytes);
                bulk_g2s(stage_base + static_cast<size_t>(s) * R * p.row_bytes,
                         p.rows + r * p.row_bytes, bytes, full_bar + s, pol);
            }
        }
    } else {
        // ---------------- compute warps ----------------
        const int cw = warp % CW, g = warp / CW;
        const int nthreads = W * 32;
        float q[CPW][NQ][EPL];
#pragma unroll
        for (int j = 0; j < CPW; ++j) {
            const int c = cw + j * CW;
#pragma unroll
            for (int jq = 0; jq < NQ; ++jq) {
#pragma unroll
                for (int t = 0; t < EPL; ++t) {
                    const int64_t e = static_cast<int64_t>(c) * (512 / sizeof(RowT)) + lane * EPL + t;
                    float v = 0.f;
                    if (c < C && jq < nq && e < p.dim) v = T::round_q(__ldg(p.q64 + jq * p.dim + e));
                    q[j][jq][t] = v;
                }
            }
        }

        for (int i = 0; i < nst; ++i) {
            const int s = i % S;
            const int64_t rbase = row0 + static_cast<int64_t>(i) * R;
            const int rows_i = static_cast<int>(min(static_cast<int64_t>(R), row_end - rbase));
            // validity bits of the (row, query) items this thread finalizes,
            // fetched before the stage lands so the load latency overlaps
            uint32_t vbits = 0;
            {
                int slot_i = 0;
                for (int t = tid; t < rows_i * nq && slot_i < 32; t += nthreads, ++slot_i) {
                    const int64_t sl = rbase + t / nq;
                    vbits |= ((__ldg(p.valid + (sl >> 5)) >> (sl & 31)) & 1u) << slot_i;
                }
            }
            mbar_wait(full_bar + s, (i / S) & 1);
            const uint8_t* sp = stage_base + static_cast<size_t>(s) * R * p.row_bytes;

            // ---- accumulate: partial[r][jq][c] = chunk sums ----
            // warp (g, cw) owns rows [g*RPW, (g+1)*RPW) of the stage and
            // column chunks cw, cw+CW, ...; U rows at a time are independent
            // FMA/shuffle chains.
            for (int r0 = g * RPW; r0 < min((g + 1) * RPW, rows_i); r0 += U) {
#pragma unroll
            for (int j = 0; j < CPW; ++j) {
                const int c = cw + j * CW;
                if (c >= C) continue;  // warp-uniform
                const int64_t boff = static_cast<int64_t>(c) * 512 + lane * 16;
                const bool lane_in = boff < p.row_bytes;
                uint4 raw[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int r = r0 + u;
                    raw[u] = make_uint4(0, 0, 0, 0);
                    if (lane_in && r < rows_i)
                        raw[u] = *reinterpret_cast<const uint4*>(sp + r * p.row_bytes + boff);
                }
                float acc[U][NQ];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    float x[EPL];
                    T::unpack(raw[u], x);
#pragma unroll
                    for (int jq = 0; jq < NQ; ++jq) {
                        float a = x[0] * q[j][jq][0];
#pragma unroll
                        for (int t = 1; t < EPL; ++t) a = fmaf(x[t], q[j][jq][t], a);
                        acc[u][jq] = a;
                    }
                }
                // transposed butterfly: after M halving steps lane holds
                // query (lane >> (5-M)); identical tree to a per-query
                // xor-16..1 butterfly.
#pragma unroll
                for (int st = 0; st < M; ++st) {
                    const int o = 16 >> st;
                    const bool upper = (lane & o) != 0;
                    const int n = NQ >> st;
#pragma unroll
                    for (int u = 0; u < U; ++u) {
#pragma unroll
                        for (int e = 0; e < n / 2; ++e) {
                            const float send = upper ? acc[u][e] : acc[u][e + n / 2];
                            const float keep = upper ? acc[u][e + n / 2] : acc[u][e];
                            acc[u][e] = keep + __shfl_xor_sync(0xffffffffu, send, o);
                        }
                    }
                }
                float v[U];
#pragma unroll
                for (int u = 0; u < U; ++u) v[u] = acc[u][0];
#pragma unroll
                for (int o = 16 >> M; o > 0; o >>= 1) {
#pragma unroll
                    for (int u = 0; u < U; ++u) v[u] += __shfl_xor_sync(0xffffffffu, v[u], o);
                }
                if ((lane & ((32 >> M) - 1)) == 0) {
                    const int jq = lane >> (5 - M);
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        const int r = r0 + u;
                        if (r < rows_i) partial[(r * NQ + jq) * C + c] = v[u];
                    }
                }
            }
            }
            // chip-wide admission bound (any CTA's k'-th best <= the global one)
            if (tid < nq) {
                const uint32_t g = *reinterpret_cast<volatile uint32_t*>(p.gbound + tid);
                if (g > thr[tid]) thr[tid] = g;
            }
            named_bar_sync(1, nthreads);
            if (tid == 0) mbar_arrive(empty_bar + s);  // stage consumed

            // ---- finalize: score, validity, admission threshold ----
            uint32_t* pend = reinterpret_cast<uint32_t*>(smem + L.pend_off + (i & 1) * pend_bytes);
            uint32_t* pend_total = pend;
            uint32_t* pend_cnt = pend + 1;
            uint2* pend_e = reinterpret_cast<uint2*>(reinterpret_cast<uint8_t*>(pend) + pend_hdr);
            {
            int slot_i = 0;
            for (int t = tid; t < rows_i * nq; t += nthreads, ++slot_i) {
                const int r = t / nq, jq = t - r * nq;
                const float* pr = partial + (r * NQ + jq) * C;
                float sc = pr[0];
                for (int c = 1; c < C; ++c) sc += pr[c];
                sc += 0.0f;  // -0 -> +0 (the reference compares numerically)
                const int64_t slot = rbase + r;
                const bool live = slot_i < 32 ? ((vbits >> slot_i) & 1u) : valid_bit(p.valid, slot);
                if (live && sc == sc) {
                    const uint32_t key = f32_key(sc);
                    if (key >= thr[jq]) {
                        const uint32_t at = atomicAdd(pend_cnt + jq, 1u);
                        pend_e[jq * R + at] = make_uint2(static_cast<uint32_t>(slot), key);
                        atomicAdd(pend_total, 1u);
                    }
                }
            }
            }
            named_bar_sync(1, nthreads);
            if (i > 0 && tid == 0) {
                // recycle the other parity's pending buffer (read last stage)
                uint32_t* old = reinterpret_cast<uint32_t*>(smem + L.pend_off + ((i - 1) & 1) * pend_bytes);
                for (int j = 0; j <= NQ; ++j) old[j] = 0;
            }
            if (*pend_total == 0) continue;  // uniform: written before the barrier

            // ---- insertions: one warp per query, one rank-merge per stage ----
            for (int jq = warp; jq < nq; jq += W) {
                const int np = static_cast<int>(pend_cnt[jq]);
                if (np == 0) continue;
                uint32_t* lk = lkey + jq * kp;
                int32_t* ls = lslot + jq * kp;
                const int n = warp_rank_merge(lk, ls, static_cast<int>(cnt[jq]), kp, pend_e + jq * R, np,
                                              merge_scratch + warp * (kp + R), p.ids, p.slot_ids != 0, lane);
                if (lane == 0) {
                    cnt[jq] = n;
                    if (n == kp) {
                        thr[jq] = max(thr[jq], lk[kp - 1]);
                        atomicMax(p.gbound + jq, lk[kp - 1]);
                    }
                }
                __syncwarp();
            }
            named_bar_sync(1, nthreads);
        }

        // ---- publish this CTA's lists ----
        named_bar_sync(1, nthreads);
        for (int jq = 0; jq < nq; ++jq) {
            const uint32_t n = cnt[jq];
            const size_t base = (static_cast<size_t>(blockIdx.x) * nq + jq) * kp;
            for (int e = tid; e < static_cast<int>(n); e += nthreads) {
                p.out_key[base + e] = lkey[jq * kp + e];
                p.out_slot[base + e] = lslot[jq * kp + e];
            }
            if (tid == 0) p.out_n[blockIdx.x * nq + jq] = static_cast<int>(n);
        }
    }
}

}  // namespace sine
