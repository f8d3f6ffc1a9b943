// Merge of per-CTA candidate lists + optional fp64 re-rank + final order.
//
// One CTA per query.  The pooled per-CTA lists (score keys) go through a
// block radix select (8-bit digits, MSB first) that finds the exact k'-th
// best key; entries above it are kept, entries equal to it are resolved by
// ascending id (a second radix select on ids when the tie straddles the
// cut).  The surviving k' candidates are optionally re-scored in fp64
// against the fp64 master rows (fixed lane order, so identical rows give
// identical similarities), ordered by (similarity desc, id asc), filtered by
// the inclusive threshold and cut to k -- the rest of `_rank`
// (reference pkg/src/semcache/index.py:42-46).
#pragma once

#include "common.cuh"

namespace sine {

struct MergeParams {
    const uint32_t* in_key;  // [ncta][nq][kp]
    const int32_t* in_slot;
    const int32_t* in_n;     // [ncta][nq]
    int ncta, nq, kp;
    const int64_t* ids;
    const double* rows64;    // [nslots][dim]
    const double* q64;       // [nq][dim]
    int64_t dim;
    int k;
    double min_sim;
    int rerank;
    float thr0;              // admission floor the scan used
    double err;              // bound on |filter score - exact similarity|
    uint8_t* cert;           // [nq] 1 = provably the exact top-k (nullable)
    const uint32_t* gbound;  // [nq] chip-wide admission bound the scan used (nullable)
    int debug;
    int64_t* out_ids;        // [nq][k]
    double* out_sims;
    int32_t* out_counts;     // [nq]
};

constexpr int kMergeThreads = 256;
constexpr int kMergeCompact = 2048;  // live candidates kept in the compact list

// Block-wide exclusive scan of one value per thread (256 threads).
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t v, uint32_t* warp_tot) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += t;
    }
    if (lane == 31) warp_tot[warp] = inc;
    __syncthreads();
    uint32_t off = 0;
    for (int w = 0; w < warp; ++w) off += warp_tot[w];
    __syncthreads();
    return off + inc - v;
}

// Select, among the entries accepted by `get` (returns false to skip), the
// `kth` (1-based) key in descending (desc=true) or ascending order.  Keys
// are `nbits` wide (multiple of 8).  Returns the key; *before = number of
// entries strictly before it in that order; *equal = entries equal to it.
template <typename KeyT, typename Get>
__device__ KeyT block_select(Get get, int nflat, uint32_t kth, bool desc, int nbits, uint32_t* hist,
                             uint32_t* scratch, uint32_t* before, uint32_t* equal) {
    KeyT prefix = 0, pmask = 0;
    uint32_t need = kth, found_bin = 0;
    for (int shift = nbits - 8; shift >= 0; shift -= 8) {
        hist[threadIdx.x] = 0;
        __syncthreads();
        for (int f = threadIdx.x; f < nflat; f += kMergeThreads) {
            KeyT key;
            if (get(f, key) && (key & pmask) == prefix)
                atomicAdd(hist + static_cast<uint32_t>((key >> shift) & 0xff), 1u);
        }
        __syncthreads();
        const int bin = desc ? 255 - static_cast<int>(threadIdx.x) : static_cast<int>(threadIdx.x);
        const uint32_t c = hist[bin];
        const uint32_t ex = block_excl_scan(c, scratch);
        if (ex < need && need <= ex + c) {
            scratch[8] = bin;
            scratch[9] = ex;
            scratch[10] = c;
        }
        __syncthreads();
        found_bin = scratch[8];
        need -= scratch[9];
        *equal = scratch[10];
        prefix |= static_cast<KeyT>(found_bin) << shift;
        pmask |= static_cast<KeyT>(0xff) << shift;
        __syncthreads();
    }
    *before = kth - need;
    return prefix;
}

__global__ void __launch_bounds__(kMergeThreads) merge_kernel(const MergeParams p) {
    __shared__ uint32_t hist[256];
    __shared__ uint32_t scratch[16];
    __shared__ int32_t ns[1024];
    __shared__ int32_t sel_slot[kMaxKp];
    __shared__ uint32_t sel_key[kMaxKp];
    __shared__ int64_t sel_id[kMaxKp];
    __shared__ double sel_sim[kMaxKp];
    __shared__ uint32_t nsel;

    extern __shared__ uint32_t pool[];  // [ncta * kp] candidate keys, 0 = empty
    // live entries (key >= the admission bound), compacted: the selection
    // below touches only these when they fit (the common case: a few hundred)
    __shared__ uint32_t ckey[kMergeCompact];
    __shared__ int32_t cslot[kMergeCompact];
    __shared__ uint32_t ctot;
    pdl_wait();  // launched early (PDL): the scan's lists are complete past this point
    const int qi = blockIdx.x;
    const int kp = p.kp, nq = p.nq;
    const int nflat = p.ncta * kp;
    for (int c = threadIdx.x; c < p.ncta; c += kMergeThreads) ns[c] = p.in_n[c * nq + qi];
    if (threadIdx.x == 0) {
        nsel = 0;
        ctot = 0;
    }
    __syncthreads();
    // stage the pooled keys once: every radix pass below reads shared memory.
    // Keys and slots go out 16 per thread before any store (the staging is
    // latency bound), and keys below the chip-wide admission bound are
    // dropped: that bound is <= the true k'-th best key (every CTA's k'-th
    // best is), so they cannot make the top k'.
    const uint32_t gb = p.gbound ? p.gbound[qi] : 0u;
    const int lane = threadIdx.x & 31;
    for (int f0 = 0; f0 < nflat; f0 += 16 * kMergeThreads) {
        uint32_t v[16];
        int32_t sl[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            const int f = f0 + j * kMergeThreads + threadIdx.x;
            v[j] = 0u;
            sl[j] = 0;
            if (f < nflat) {
                const int c = f / kp, e = f - c * kp;
                if (e < ns[c]) {
                    const size_t o = (static_cast<size_t>(c) * nq + qi) * kp + e;
                    v[j] = __ldg(p.in_key + o);
                    sl[j] = __ldg(p.in_slot + o);
                }
            }
        }
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            const int f = f0 + j * kMergeThreads + threadIdx.x;
            const bool live = f < nflat && v[j] != 0u && v[j] >= gb;
            if (f < nflat) pool[f] = live ? v[j] : 0u;
            // warp-aggregated append to the compact list
            const uint32_t b = __ballot_sync(0xffffffffu, live);
            if (b) {
                uint32_t base = 0;
                if (lane == 0) base = atomicAdd(&ctot, static_cast<uint32_t>(__popc(b)));
                base = __shfl_sync(0xffffffffu, base, 0);
                const uint32_t at = base + __popc(b & ((1u << lane) - 1u));
                if (live && at < kMergeCompact) {
                    ckey[at] = v[j];
                    cslot[at] = sl[j];
                }
            }
        }
    }
    __syncthreads();
    const uint32_t total = ctot;  // live candidates (after the admission-bound prefilter)
    const bool compact = total <= static_cast<uint32_t>(kMergeCompact);

    auto slot_at = [&](int c, int e) { return p.in_slot[(static_cast<size_t>(c) * nq + qi) * kp + e]; };

    // every row that is not a candidate has a filter score <= bound_key
    // (the selection cut, or the worst entry of a CTA's full list), or was
    // below the admission floor
    __shared__ uint32_t bound_key;
    if (threadIdx.x == 0) bound_key = 0;
    __syncthreads();
    if (total <= static_cast<uint32_t>(kp)) {
        for (int c = threadIdx.x; c < p.ncta; c += kMergeThreads) {
            if (ns[c] != kp) continue;
            uint32_t mk = 0xffffffffu;
            for (int e = 0; e < kp; ++e) mk = min(mk, pool[c * kp + e]);
            atomicMax(&bound_key, mk);
        }
        for (int i = threadIdx.x; i < static_cast<int>(total); i += kMergeThreads) {
            sel_key[i] = ckey[i];
            sel_slot[i] = cslot[i];
        }
        if (threadIdx.x == 0) nsel = total;
    } else {
        // the selection runs over the compact list (n = total) when it fits,
        // else over the whole pool (n = nflat, empty entries skipped)
        const int n = compact ? static_cast<int>(total) : nflat;
        auto key_of = [&](int f) { return compact ? ckey[f] : pool[f]; };
        auto slot_of = [&](int f) {
            if (compact) return cslot[f];
            const int c = f / kp;
            return slot_at(c, f - c * kp);
        };
        uint32_t nbefore, nequal;
        const uint32_t kstar = block_select<uint32_t>(
            [&](int f, uint32_t& key) {
                key = key_of(f);
                return key != 0u;
            },
            n, static_cast<uint32_t>(kp), true, 32, hist, scratch, &nbefore, &nequal);
        if (threadIdx.x == 0) bound_key = kstar;
        const uint32_t need_eq = kp - nbefore;
        // ties at the cut: keep the need_eq smallest ids
        uint64_t idcut = ~0ull;
        if (nequal > need_eq) {
            uint32_t b2, e2;
            idcut = block_select<uint64_t>(
                [&](int f, uint64_t& key) {
                    if (key_of(f) != kstar) return false;
                    key = i64_key(__ldg(p.ids + slot_of(f)));
                    return true;
                },
                n, need_eq, false, 64, hist, scratch, &b2, &e2);
        }
        for (int f = threadIdx.x; f < n; f += kMergeThreads) {
            const uint32_t key = key_of(f);
            if (key == 0u) continue;
            bool take = key > kstar;
            if (key == kstar) take = (idcut == ~0ull) || i64_key(__ldg(p.ids + slot_of(f))) <= idcut;
            if (take) {
                const uint32_t at = atomicAdd(&nsel, 1u);
                sel_key[at] = key;
                sel_slot[at] = slot_of(f);
            }
        }
    }
    __syncthreads();
    const int m = static_cast<int>(nsel);

    for (int i = threadIdx.x; i < m; i += kMergeThreads) {
        sel_id[i] = __ldg(p.ids + sel_slot[i]);
        sel_sim[i] = static_cast<double>(key_f32(sel_key[i]));
    }
    __syncthreads();

    if (p.rerank) {
        // fp64 re-score: lane l of a warp sums x[t] * q[t] for t = l, l + 32,
        // ... in ascending order (one fma chain), then a fixed butterfly ->
        // identical rows give identical similarities.  A warp scores up to
        // four candidates at once so their row loads overlap (the chains and
        // their order are unchanged by the interleaving).
        const int warp = threadIdx.x >> 5;
        const double* q = p.q64 + static_cast<size_t>(qi) * p.dim;
        constexpr int kW = kMergeThreads / 32;
        for (int i0 = warp; i0 < m; i0 += 4 * kW) {
            if (i0 + kW >= m) {  // this warp's last candidate alone: 16 row loads in flight per lane
                const double* xr = p.rows64 + static_cast<size_t>(sel_slot[i0]) * p.dim;
                double a = 0.0;
                int64_t t = lane;
                for (; t + 32 * 15 < p.dim; t += 32 * 16) {
                    double xv[16], qv[16];
#pragma unroll
                    for (int u = 0; u < 16; ++u) {
                        xv[u] = __ldg(xr + t + 32 * u);
                        qv[u] = __ldg(q + t + 32 * u);
                    }
#pragma unroll
                    for (int u = 0; u < 16; ++u) a = fma(xv[u], qv[u], a);
                }
                for (; t + 32 * 7 < p.dim; t += 32 * 8) {
                    double xv[8], qv[8];
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        xv[u] = __ldg(xr + t + 32 * u);
                        qv[u] = __ldg(q + t + 32 * u);
                    }
#pragma unroll
                    for (int u = 0; u < 8; ++u) a = fma(xv[u], qv[u], a);
                }
                for (; t < p.dim; t += 32) a = fma(__ldg(xr + t), __ldg(q + t), a);
                a = warp_sum64(a);
                if (lane == 0) sel_sim[i0] = a + 0.0;
                continue;
            }
            const double* x[4];
            bool on[4];
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                const int i = i0 + c * kW;
                on[c] = i < m;
                x[c] = p.rows64 + static_cast<size_t>(on[c] ? sel_slot[i] : sel_slot[i0]) * p.dim;
            }
            double a[4] = {0.0, 0.0, 0.0, 0.0};
            int64_t t = lane;
            for (; t + 32 * 7 < p.dim; t += 32 * 8) {
                double qv[8], xv[4][8];
#pragma unroll
                for (int u = 0; u < 8; ++u) qv[u] = __ldg(q + t + 32 * u);
#pragma unroll
                for (int c = 0; c < 4; ++c)
#pragma unroll
                    for (int u = 0; u < 8; ++u) xv[c][u] = on[c] ? __ldg(x[c] + t + 32 * u) : 0.0;
#pragma unroll
                for (int c = 0; c < 4; ++c)
#pragma unroll
                    for (int u = 0; u < 8; ++u) a[c] = fma(xv[c][u], qv[u], a[c]);
            }
            for (; t < p.dim; t += 32) {
                const double qv = __ldg(q + t);
#pragma unroll
                for (int c = 0; c < 4; ++c)
                    if (on[c]) a[c] = fma(__ldg(x[c] + t), qv, a[c]);
            }
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                const double s = warp_sum64(a[c]);
                if (lane == 0 && on[c]) sel_sim[i0 + c * kW] = s + 0.0;
            }
        }
        __syncthreads();
    }

    // rank sort by (sim desc, id asc) -- keys are unique (ids unique)
    __shared__ int32_t order[kMaxKp];
    for (int i = threadIdx.x; i < m; i += kMergeThreads) {
        int r = 0;
        const double si = sel_sim[i];
        const int64_t ii = sel_id[i];
        for (int j = 0; j < m; ++j) r += cand_before64(sel_sim[j], sel_id[j], si, ii) ? 1 : 0;
        order[r] = i;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        int outn = 0;
        for (int r = 0; r < m && outn < p.k; ++r) {
            const int i = order[r];
            if (!(sel_sim[i] >= p.min_sim)) break;  // sorted desc: the rest fail too
            p.out_ids[static_cast<size_t>(qi) * p.k + outn] = sel_id[i];
            p.out_sims[static_cast<size_t>(qi) * p.k + outn] = sel_sim[i];
            ++outn;
        }
        for (int r = outn; r < p.k; ++r) {
            p.out_ids[static_cast<size_t>(qi) * p.k + r] = -1;
            p.out_sims[static_cast<size_t>(qi) * p.k + r] = 0.0;
        }
        p.out_counts[qi] = outn;
        if (p.cert) {
            // certificate: no excluded row can reach the k-th similarity (or
            // the threshold when fewer than k passed)
            double bound = static_cast<double>(p.thr0);
            if (bound_key) bound = fmax(bound, static_cast<double>(key_f32(bound_key)));
            if (p.gbound && p.gbound[qi]) bound = fmax(bound, static_cast<double>(key_f32(p.gbound[qi])));
            const double need = outn == p.k ? sel_sim[order[p.k - 1]] : p.min_sim;
            p.cert[qi] = (!p.rerank || bound + p.err < need) ? 1 : 0;
            if (p.debug)
                printf("cert q%d total=%u kp=%d bound_key=%08x bound=%.6f err=%g need=%.6f thr0=%f -> %d\n", qi,
                       total, kp, bound_key, bound, p.err, need, p.thr0, p.cert[qi]);
        }
    }
}

}  // namespace sine

namespace sine {

// Row-sharded stage-1: merge the P per-rank exact top-k lists of each query
// (the all-gather output: rank r's [B][k] block at r * rank_stride, id -1 =
// padding) into the global top-k
// with the reference comparator (similarity desc, id asc; index.py:45).
// One CTA per query; entries are ranked in shared memory.
constexpr int kShardMergeThreads = 128;

__global__ void __launch_bounds__(kShardMergeThreads)
    shard_merge_kernel(const int64_t* ids, const double* sims, int P, int64_t B, int k, int64_t rank_stride,
                       int64_t* out_ids, double* out_sims, int32_t* out_counts) {
    extern __shared__ uint8_t sm_raw[];
    const int m = P * k;
    double* ss = reinterpret_cast<double*>(sm_raw);
    int64_t* si = reinterpret_cast<int64_t*>(ss + m);
    __shared__ int nvalid;
    const int64_t q = blockIdx.x;
    if (threadIdx.x == 0) nvalid = 0;
    __syncthreads();
    for (int e = threadIdx.x; e < m; e += blockDim.x) {
        const int r = e / k, j = e - r * k;
        const size_t o = static_cast<size_t>(r) * rank_stride + static_cast<size_t>(q) * k + j;
        si[e] = ids[o];
        ss[e] = sims[o];
        if (ids[o] >= 0) atomicAdd(&nvalid, 1);
    }
    __syncthreads();
    for (int e = threadIdx.x; e < m; e += blockDim.x) {
        if (si[e] < 0) continue;
        int rnk = 0;
        for (int f = 0; f < m; ++f)
            if (si[f] >= 0 && cand_before64(ss[f], si[f], ss[e], si[e])) ++rnk;
        if (rnk < k) {
            out_ids[q * k + rnk] = si[e];
            out_sims[q * k + rnk] = ss[e];
        }
    }
    const int n = min(nvalid, k);
    for (int r = n + threadIdx.x; r < k; r += blockDim.x) {
        out_ids[q * k + r] = -1;
        out_sims[q * k + r] = 0.0;
    }
    if (threadIdx.x == 0) out_counts[q] = n;
}

}  // namespace sine
