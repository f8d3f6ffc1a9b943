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
// Victim selection never sorts all N elements: a weighted MSB-first radix
// select over the 192-bit composite key (primary, created_at, id) finds the
// last victim T (8-bit digits; digits that are constant over the surviving
// candidates are skipped using AND/OR reductions), then only the victims
// (keys <= T) are collected and sorted.
#pragma once

#include "common.cuh"

namespace sine {

struct EvictCols {
    const double *lf, *lc, *ll, *ls, *created, *expiration, *last_access;
    const int64_t *freq, *size, *ids;
    const uint32_t* valid;
    int64_t nslots;
};

struct SelectState {
    uint64_t prefix[3];
    int32_t ndigits;  // digits of the composite key fixed so far (0..24)
    int32_t done;     // 1: prefix identifies the last victim; 2: everything is a victim
    int64_t rem;      // weight still needed inside the prefix bucket
    int64_t count;    // candidates matching the prefix
    int64_t total_w;  // first pass: live weight
    int64_t below;    // candidates strictly below the chosen bucket (all of them when done == 2)
};

__device__ __forceinline__ double lcfu_score(const EvictCols& c, int64_t s, double now) {
    const int64_t size = c.size[s];
    if (size == 0 || __dsub_rn(c.expiration[s], now) <= 0.0) return 0.0;
    double v = __dmul_rn(c.lf[s], c.lc[s]);
    v = __dmul_rn(v, c.ll[s]);
    v = __dmul_rn(v, c.ls[s]);
    return __ddiv_rn(v, static_cast<double>(size));
}

__device__ __forceinline__ uint64_t primary_key(const EvictCols& c, int64_t s, int policy, double now) {
    if (policy == 0) return f64_key(lcfu_score(c, s, now));
    if (policy == 1) return f64_key(c.last_access[s]);
    return i64_key(c.freq[s]);
}

__device__ __forceinline__ uint32_t key_digit(const uint64_t k[3], int d) {
    return static_cast<uint32_t>((k[d >> 3] >> (8 * (7 - (d & 7)))) & 0xff);
}

// compare the first nd digits of k against prefix: -1 / 0 / +1
__device__ __forceinline__ int prefix_cmp(const uint64_t k[3], const uint64_t pre[3], int nd) {
#pragma unroll
    for (int w = 0; w < 3; ++w) {
        const int dw = nd - 8 * w;  // digits of this word that count
        if (dw <= 0) return 0;
        const uint64_t mask = dw >= 8 ? ~0ull : ~((1ull << (8 * (8 - dw))) - 1);
        const uint64_t a = k[w] & mask, b = pre[w] & mask;
        if (a != b) return a < b ? -1 : 1;
    }
    return 0;
}

struct HistArgs {
    EvictCols c;
    int policy;
    double now;
    const int32_t* cand;   // nullptr: all slots
    int64_t ncand;
    uint64_t* k1;          // cached primary keys [nslots]
    uint8_t* d0;           // pass 1 (LCFU kernel): their top byte [nslots] (nullable)
    int first;             // compute (and cache) primary keys
    const SelectState* st;
    // record mode (rk != nullptr): the candidates were compacted into dense
    // records -- keys [n][3] + sizes [n], n = *rn on the device -- so a pass
    // streams 32 B per candidate instead of gathering four columns by slot
    const uint64_t* rk;
    const int64_t* rsz;
    const int64_t* rn;
    unsigned long long* hw;   // [256] weights
    unsigned long long* hc;   // [256] counts
    unsigned long long* hand; // [3]
    unsigned long long* hor;  // [3]
};

// 64-bit weight sum in shared memory from native 32-bit atomics (a 64-bit
// shared atomicAdd compiles to a CAS spin loop): low word + carries.
__device__ __forceinline__ void smem_add64(uint32_t* lo, uint32_t* hi, uint64_t v) {
    const uint32_t l = static_cast<uint32_t>(v);
    const uint32_t old = atomicAdd(lo, l);
    const uint32_t h = static_cast<uint32_t>(v >> 32) + (old + l < old ? 1u : 0u);
    if (h) atomicAdd(hi, h);
}

__global__ void __launch_bounds__(256) evict_hist_kernel(const HistArgs a) {
    __shared__ uint32_t swl[256], swh[256], sc[256];
    if (a.st->done) return;  // passes are enqueued ahead of the host's done check
    swl[threadIdx.x] = 0;
    swh[threadIdx.x] = 0;
    sc[threadIdx.x] = 0;
    __syncthreads();
    const int nd = a.st->ndigits;
    uint64_t pre[3] = {a.st->prefix[0], a.st->prefix[1], a.st->prefix[2]};
    uint64_t vand[3] = {~0ull, ~0ull, ~0ull}, vor[3] = {0, 0, 0};
    const int64_t n = a.rk ? *a.rn : (a.cand ? a.ncand : a.c.nslots);
    const int lane = threadIdx.x & 31;
    const int64_t stride = 256ll * gridDim.x;
    // warp-uniform trip count so the whole warp takes part in the aggregation
    for (int64_t i0 = blockIdx.x * 256ll + (threadIdx.x & ~31); i0 < n; i0 += stride) {
        const int64_t i = i0 + lane;
        bool act = false;
        uint32_t dg = 0;
        uint64_t sz = 0;
        if (i < n && a.rk) {
            const uint64_t k[3] = {a.rk[3 * i], a.rk[3 * i + 1], a.rk[3 * i + 2]};
            if (prefix_cmp(k, pre, nd) == 0) {
                act = true;
                dg = key_digit(k, nd);
                sz = static_cast<uint64_t>(a.rsz[i]);
#pragma unroll
                for (int w = 0; w < 3; ++w) {
                    vand[w] &= k[w];
                    vor[w] |= k[w];
                }
            }
        } else if (i < n) {
            const int64_t s = a.cand ? a.cand[i] : i;
            if (a.cand || valid_bit(a.c.valid, s)) {
                uint64_t k[3];
                if (a.first) {
                    k[0] = primary_key(a.c, s, a.policy, a.now);
                    a.k1[s] = k[0];
                } else {
                    k[0] = a.k1[s];
                }
                // digits inside the primary word need only k[0]; the other
                // words are then reported as varying (a conservative AND/OR)
                const bool rest = nd >= 8;
                k[1] = rest ? f64_key(a.c.created[s]) : 0ull;
                k[2] = rest ? i64_key(a.c.ids[s]) : 0ull;
                if (prefix_cmp(k, pre, nd) == 0) {
                    act = true;
                    dg = key_digit(k, nd);
                    sz = static_cast<uint64_t>(a.c.size[s]);
#pragma unroll
                    for (int w = 0; w < 3; ++w) {
                        vand[w] &= rest || w == 0 ? k[w] : 0ull;
                        vor[w] |= rest || w == 0 ? k[w] : ~0ull;
                    }
                }
            }
        }
        // one shared-memory atomic per (warp, digit) when few digits are
        // present (a third of all SEs score exactly 0: per-lane atomics would
        // serialise on one bin); spread digits take plain per-lane atomics
        uint32_t rem = __ballot_sync(0xffffffffu, act);
        const uint32_t peers = __match_any_sync(0xffffffffu, act ? dg : 0xffffffffu);
        const bool group_leader = act && (__ffs(peers) - 1) == lane;
        if (__popc(__ballot_sync(0xffffffffu, group_leader)) > 4) {
            if (act) {
                smem_add64(&swl[dg], &swh[dg], sz);
                atomicAdd(&sc[dg], 1u);
            }
            rem = 0;
        }
        while (rem) {
            const int leader = __ffs(rem) - 1;
            const uint32_t ldg = __shfl_sync(0xffffffffu, dg, leader);
            const bool mine = act && dg == ldg;
            const uint32_t grp = __ballot_sync(0xffffffffu, mine);
            unsigned long long v = mine ? sz : 0ull;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
            if (lane == leader) {
                smem_add64(&swl[ldg], &swh[ldg], v);
                atomicAdd(&sc[ldg], static_cast<uint32_t>(__popc(grp)));
            }
            rem &= ~grp;
        }
    }
#pragma unroll
    for (int w = 0; w < 3; ++w) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            vand[w] &= __shfl_xor_sync(0xffffffffu, vand[w], o);
            vor[w] |= __shfl_xor_sync(0xffffffffu, vor[w], o);
        }
    }
    // block-level AND/OR first: one global atomic per word per block
    __shared__ unsigned long long band[3], bor[3];
    if (threadIdx.x < 3) {
        band[threadIdx.x] = ~0ull;
        bor[threadIdx.x] = 0ull;
    }
    __syncthreads();
    if ((threadIdx.x & 31) == 0 && (vor[0] | vor[1] | vor[2] | ~vand[0] | ~vand[1] | ~vand[2])) {
#pragma unroll
        for (int w = 0; w < 3; ++w) {
            atomicAnd(band + w, static_cast<unsigned long long>(vand[w]));
            atomicOr(bor + w, static_cast<unsigned long long>(vor[w]));
        }
    }
    __syncthreads();
    if (threadIdx.x < 3 && (bor[0] | bor[1] | bor[2] | ~band[0] | ~band[1] | ~band[2])) {
        atomicAnd(a.hand + threadIdx.x, band[threadIdx.x]);
        atomicOr(a.hor + threadIdx.x, bor[threadIdx.x]);
    }
    if (sc[threadIdx.x]) {
        atomicAdd(a.hw + threadIdx.x, (static_cast<unsigned long long>(swh[threadIdx.x]) << 32) | swl[threadIdx.x]);
        atomicAdd(a.hc + threadIdx.x, static_cast<unsigned long long>(sc[threadIdx.x]));
    }
}

// Pass 1 for LCFU over every slot, 4 slots per thread in flight: all
// column loads of a group are issued before any score is computed (the
// pass is load-latency bound), then each score is keyed, cached in k1 and
// histogrammed on its first digit exactly as evict_hist_kernel does.
__global__ void __launch_bounds__(256) evict_pass1_lcfu_kernel(const HistArgs a) {
    __shared__ uint32_t swl[256], swh[256], sc[256];
    __shared__ unsigned long long band, bor;
    swl[threadIdx.x] = 0;
    swh[threadIdx.x] = 0;
    sc[threadIdx.x] = 0;
    if (threadIdx.x == 0) {
        band = ~0ull;
        bor = 0ull;
    }
    __syncthreads();
    constexpr int U = 4;
    const int64_t n = a.c.nslots;
    const int lane = threadIdx.x & 31;
    const int64_t stride = 256ll * gridDim.x;
    uint64_t vand = ~0ull, vor = 0ull;
    for (int64_t i0 = blockIdx.x * 256ll + (threadIdx.x & ~31); i0 < n; i0 += U * stride) {
        double lf[U], lc[U], ll[U], ls[U], ex[U];
        int64_t size[U];
        uint32_t vw[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t s = i0 + u * stride + lane;
            const bool in = s < n;
            vw[u] = in ? __ldg(a.c.valid + (s >> 5)) : 0u;
            lf[u] = in ? __ldg(a.c.lf + s) : 0.0;
            lc[u] = in ? __ldg(a.c.lc + s) : 0.0;
            ll[u] = in ? __ldg(a.c.ll + s) : 0.0;
            ls[u] = in ? __ldg(a.c.ls + s) : 0.0;
            ex[u] = in ? __ldg(a.c.expiration + s) : 0.0;
            size[u] = in ? __ldg(a.c.size + s) : 0;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t s = i0 + u * stride + lane;
            const bool act = s < n && ((vw[u] >> (s & 31)) & 1u);
            uint32_t dg = 0;
            if (act) {
                double v = 0.0;  // cal_score (engine.py:33-48): exact order, no FMA
                if (size[u] != 0 && !(__dsub_rn(ex[u], a.now) <= 0.0)) {
                    v = __dmul_rn(lf[u], lc[u]);
                    v = __dmul_rn(v, ll[u]);
                    v = __dmul_rn(v, ls[u]);
                    v = __ddiv_rn(v, static_cast<double>(size[u]));
                }
                const uint64_t k0 = f64_key(v);
                a.k1[s] = k0;
                if (a.d0) a.d0[s] = static_cast<uint8_t>(k0 >> 56);
                dg = static_cast<uint32_t>(k0 >> 56);
                vand &= k0;
                vor |= k0;
            }
            const uint64_t sz = act ? static_cast<uint64_t>(size[u]) : 0ull;
            uint32_t rem = __ballot_sync(0xffffffffu, act);
            const uint32_t peers = __match_any_sync(0xffffffffu, act ? dg : 0xffffffffu);
            const bool group_leader = act && (__ffs(peers) - 1) == lane;
            if (__popc(__ballot_sync(0xffffffffu, group_leader)) > 4) {
                if (act) {
                    smem_add64(&swl[dg], &swh[dg], sz);
                    atomicAdd(&sc[dg], 1u);
                }
                rem = 0;
            }
            while (rem) {
                const int leader = __ffs(rem) - 1;
                const uint32_t ldg = __shfl_sync(0xffffffffu, dg, leader);
                const bool mine = act && dg == ldg;
                const uint32_t grp = __ballot_sync(0xffffffffu, mine);
                unsigned long long v = mine ? sz : 0ull;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
                if (lane == leader) {
                    smem_add64(&swl[ldg], &swh[ldg], v);
                    atomicAdd(&sc[ldg], static_cast<uint32_t>(__popc(grp)));
                }
                rem &= ~grp;
            }
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        vand &= __shfl_xor_sync(0xffffffffu, vand, o);
        vor |= __shfl_xor_sync(0xffffffffu, vor, o);
    }
    if (lane == 0 && (vor | ~vand)) {
        atomicAnd(&band, static_cast<unsigned long long>(vand));
        atomicOr(&bor, static_cast<unsigned long long>(vor));
    }
    __syncthreads();
    if (sc[threadIdx.x]) {
        atomicAdd(a.hw + threadIdx.x, (static_cast<unsigned long long>(swh[threadIdx.x]) << 32) | swl[threadIdx.x]);
        atomicAdd(a.hc + threadIdx.x, static_cast<unsigned long long>(sc[threadIdx.x]));
    }
    if (threadIdx.x == 0) {
        if (bor | ~band) {
            atomicAnd(a.hand, band);
            atomicOr(a.hor, bor);
        }
        // words 1 and 2 were not read: reported as varying
        atomicAnd(a.hand + 1, 0ull);
        atomicOr(a.hor + 1, ~0ull);
        atomicAnd(a.hand + 2, 0ull);
        atomicOr(a.hor + 2, ~0ull);
    }
}

// One CTA: choose the digit bucket where the cumulative weight reaches rem,
// then skip the following digits that are constant over that bucket.
__global__ void __launch_bounds__(256) evict_pick_kernel(SelectState* st, unsigned long long* hw,
                                                         unsigned long long* hc, unsigned long long* hand,
                                                         unsigned long long* hor, int first) {
    __shared__ unsigned long long cw[256], cc[256];
    __shared__ int chosen;
    __shared__ unsigned long long before_w;
    const int t = threadIdx.x;
    if (st->done) return;
    cw[t] = hw[t];
    cc[t] = hc[t];
    if (t == 0) chosen = -1;
    __syncthreads();
    // inclusive scan (Hillis-Steele, 256 entries)
    for (int o = 1; o < 256; o <<= 1) {
        const unsigned long long v = t >= o ? cw[t - o] : 0ull;
        const unsigned long long u = t >= o ? cc[t - o] : 0ull;
        __syncthreads();
        cw[t] += v;
        cc[t] += u;
        __syncthreads();
    }
    const long long rem = st->rem;
    const unsigned long long ex = t ? cw[t - 1] : 0ull;
    if (static_cast<long long>(ex) < rem && rem <= static_cast<long long>(cw[t])) {
        chosen = t;
        before_w = ex;
    }
    __syncthreads();
    if (t == 0) {
        if (first) st->total_w = static_cast<int64_t>(cw[255]);
        if (chosen < 0) {
            // the excess is at least the whole candidate weight: all are victims
            st->done = 2;
            st->below = static_cast<int64_t>(cc[255]);
        } else {
            st->below = chosen ? static_cast<int64_t>(cc[chosen - 1]) : 0;
            const int nd = st->ndigits;
            st->prefix[nd >> 3] |= static_cast<uint64_t>(chosen) << (8 * (7 - (nd & 7)));
            st->rem = rem - static_cast<long long>(before_w);
            const unsigned long long cnt = hc[chosen];
            int ndn = nd + 1;
            // total candidates that matched this pass
            unsigned long long tot = 0;
            for (int b = 0; b < 256; ++b) tot += hc[b];
            if (cnt == tot) {
                // every candidate was in one bucket: AND/OR describe the bucket
                // exactly, so digits equal in AND and OR are constant -- skip them
                while (ndn < 24) {
                    const int w = ndn >> 3, sh = 8 * (7 - (ndn & 7));
                    const uint64_t da = (hand[w] >> sh) & 0xff, dor = (hor[w] >> sh) & 0xff;
                    if (da != dor) break;
                    st->prefix[w] |= da << sh;
                    ++ndn;
                }
            }
            st->ndigits = ndn;
            st->count = static_cast<int64_t>(cnt);
            if (cnt <= 1 || ndn >= 24) st->done = 1;
        }
    }
    __syncthreads();
    hw[t] = 0;
    hc[t] = 0;
    if (t < 3) {
        hand[t] = ~0ull;
        hor[t] = 0ull;
    }
}

// ---- ordered (atomic-free) collection: count per 4096-entry chunk, scan,
// write; output in source order (slots, or records that are in slot order).

struct CollectPred {
    EvictCols c;
    const uint64_t* k1;
    const uint8_t* d0;   // top byte of k1 (nullable): decides alone when the prefix has one digit
    const uint64_t* rk;  // record source (index = record) instead of slots
    int nd;
    int all;
    int mode;  // 0: prefix <= T (victims), 1: prefix == T (candidates), 2: prefix < T
    uint64_t pre[3];

    // need_keys = false: only the predicate (counting passes skip the
    // created_at / id gathers when the primary word decides)
    __device__ __forceinline__ bool operator()(int64_t s, uint64_t* k, bool need_keys = true) const {
        if (rk) {
            k[0] = rk[3 * s], k[1] = rk[3 * s + 1], k[2] = rk[3 * s + 2];
        } else if (d0 && nd == 1 && !all && !need_keys) {
            // one-digit prefix: a byte per slot instead of the 8-byte key
            const uint32_t vw = __ldg(c.valid + (s >> 5));
            const uint32_t dg = __ldg(d0 + s), pd = static_cast<uint32_t>(pre[0] >> 56);
            if (!((vw >> (s & 31)) & 1u)) return false;
            return mode == 0 ? dg <= pd : (mode == 1 ? dg == pd : dg < pd);
        } else {
            // both loads issued before the validity test (no dependency chain)
            const uint32_t vw = __ldg(c.valid + (s >> 5));
            k[0] = k1[s];
            if (!((vw >> (s & 31)) & 1u)) return false;
            if (nd <= 8 && !all) {  // the first word decides; the rest only when taken
                const int cmp = prefix_cmp(k, pre, nd);
                const bool take = mode == 0 ? cmp <= 0 : (mode == 1 ? cmp == 0 : cmp < 0);
                if (take && need_keys) {
                    k[1] = f64_key(c.created[s]);
                    k[2] = i64_key(c.ids[s]);
                }
                return take;
            }
            k[1] = f64_key(c.created[s]);
            k[2] = i64_key(c.ids[s]);
        }
        const int cmp = all ? -1 : prefix_cmp(k, pre, nd);
        return mode == 0 ? cmp <= 0 : (mode == 1 ? cmp == 0 : cmp < 0);
    }
};

__device__ __forceinline__ CollectPred make_pred(const EvictCols& c, const uint64_t* k1, const SelectState* st,
                                                 int mode, const uint64_t* rk = nullptr, const uint8_t* d0 = nullptr) {
    CollectPred p;
    p.c = c;
    p.k1 = k1;
    p.d0 = d0;
    p.rk = rk;
    p.nd = st->ndigits;
    p.all = st->done == 2;
    p.mode = mode;
    p.pre[0] = st->prefix[0];
    p.pre[1] = st->prefix[1];
    p.pre[2] = st->prefix[2];
    return p;
}

constexpr int kColChunk = 4096;  // slots per block; 16 per thread

// Source: slots [0, nslots), or records [0, *rn) when rk != nullptr.
__global__ void __launch_bounds__(256) collect_count_kernel(EvictCols c, const uint64_t* k1, const SelectState* st,
                                                            int mode, int32_t* counts, const uint64_t* rk = nullptr,
                                                            const int64_t* rn = nullptr, const uint8_t* d0 = nullptr) {
    __shared__ int32_t wsum[8];
    if (mode == 2 && st->below == 0) {  // nothing below the record prefix (pass 1's histogram says so)
        if (threadIdx.x == 0) counts[blockIdx.x] = 0;
        return;
    }
    const CollectPred pred = make_pred(c, k1, st, mode, rk, d0);
    const int64_t n = rk ? *rn : c.nslots;
    const int64_t b = static_cast<int64_t>(blockIdx.x) * kColChunk;
    const int64_t e = min(b + kColChunk, n);
    int32_t cnt = 0;
    uint64_t k[3];
#pragma unroll 4
    for (int64_t i = b + threadIdx.x; i < e; i += 256) cnt += pred(i, k, false) ? 1 : 0;
    cnt = __reduce_add_sync(0xffffffffu, cnt);
    if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = cnt;
    __syncthreads();
    if (threadIdx.x == 0) {
        int32_t t = 0;
        for (int w = 0; w < 8; ++w) t += wsum[w];
        counts[blockIdx.x] = t;
    }
}

// out_k / out_size nullable; with a record source, rslot maps record ->
// slot; `base` (device, nullable) offsets the output (appending after an
// earlier collection).
__global__ void __launch_bounds__(256) collect_write_kernel(EvictCols c, const uint64_t* k1, const SelectState* st,
                                                            int mode, const int64_t* offsets, uint64_t* out_k,
                                                            int32_t* out_slot, unsigned long long* kand,
                                                            unsigned long long* kor, int64_t* out_size = nullptr,
                                                            const uint64_t* rk = nullptr, const int64_t* rn = nullptr,
                                                            const int32_t* rslot = nullptr,
                                                            const int64_t* base = nullptr,
                                                            const uint8_t* d0 = nullptr) {
    __shared__ int32_t wtot[8];
    if (mode == 2 && st->below == 0) return;
    const CollectPred pred = make_pred(c, k1, st, mode, rk, d0);
    const int64_t n = rk ? *rn : c.nslots;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    // warp w owns entries [block*4096 + 512w, +512): 16 coalesced rounds of
    // 32 consecutive entries; output order = entry order
    const int64_t w0 = static_cast<int64_t>(blockIdx.x) * kColChunk + warp * 512;
    uint32_t m[16];
    int32_t cnt = 0;
    uint64_t vand[3] = {~0ull, ~0ull, ~0ull}, vor[3] = {0, 0, 0};
    uint64_t k[3];
    // predicates only (no key gathers): 16 rounds of independent loads
#pragma unroll
    for (int j = 0; j < 16; ++j) {
        const int64_t i = w0 + j * 32 + lane;
        const bool take = i < n && pred(i, k, false);
        m[j] = __ballot_sync(0xffffffffu, take);
        cnt += __popc(m[j]);
    }
    if (lane == 0) wtot[warp] = cnt;
    __syncthreads();
    int64_t off = offsets[blockIdx.x] + (base ? *base : 0);
    for (int w = 0; w < warp; ++w) off += wtot[w];
    const uint32_t lt = (1u << lane) - 1u;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
        if ((m[j] >> lane) & 1u) {
            const int64_t i = w0 + j * 32 + lane;
            const int64_t at = off + __popc(m[j] & lt);
            const int64_t slot = rk ? rslot[i] : i;
            out_slot[at] = static_cast<int32_t>(slot);
            if (out_k || kand) {  // the taken entries' keys, gathered once
                uint64_t kk[3];
                if (rk) {
                    kk[0] = rk[3 * i], kk[1] = rk[3 * i + 1], kk[2] = rk[3 * i + 2];
                } else {
                    kk[0] = k1[i], kk[1] = f64_key(c.created[i]), kk[2] = i64_key(c.ids[i]);
                }
                if (out_k) {
                    out_k[3 * at] = kk[0];
                    out_k[3 * at + 1] = kk[1];
                    out_k[3 * at + 2] = kk[2];
                }
#pragma unroll
                for (int w = 0; w < 3; ++w) {
                    vand[w] &= kk[w];
                    vor[w] |= kk[w];
                }
            }
            if (out_size) out_size[at] = c.size[slot];
        }
        off += __popc(m[j]);
    }
    if (kand) {
#pragma unroll
        for (int w = 0; w < 3; ++w) {
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                vand[w] &= __shfl_xor_sync(0xffffffffu, vand[w], o);
                vor[w] |= __shfl_xor_sync(0xffffffffu, vor[w], o);
            }
        }
        __shared__ unsigned long long band[3], bor[3];
        if (threadIdx.x < 3) {
            band[threadIdx.x] = ~0ull;
            bor[threadIdx.x] = 0ull;
        }
        __syncthreads();
        if (lane == 0 && cnt) {
#pragma unroll
            for (int w = 0; w < 3; ++w) {
                atomicAnd(band + w, static_cast<unsigned long long>(vand[w]));
                atomicOr(bor + w, static_cast<unsigned long long>(vor[w]));
            }
        }
        __syncthreads();
        if (threadIdx.x < 3 && (bor[0] | bor[1] | bor[2])) {
            atomicAnd(kand + threadIdx.x, band[threadIdx.x]);
            atomicOr(kor + threadIdx.x, bor[threadIdx.x]);
        }
    }
}

// Victim keys -> compact 128-bit keys made of only the bytes that vary over
// the victim set (MSB-first, right-aligned).  Constant bytes cannot change
// the order, so a radix sort over 8 * nvary bits orders the victims exactly
// like the full 192-bit (primary, created_at, id) key.
struct Pack2 {
    uint64_t hi, lo;
};

__device__ __forceinline__ int varying_bytes(const unsigned long long* kand, const unsigned long long* kor, int* pos) {
    int c = 0;
    for (int d = 0; d < 24; ++d) {
        const int w = d >> 3, sh = 8 * (7 - (d & 7));
        if (((kand[w] >> sh) & 0xff) != ((kor[w] >> sh) & 0xff)) pos[c++] = d;
    }
    return c;
}

// skip_id: the victims arrive in slot order and slots are in id order, so a
// stable sort over the (primary, created_at) bytes already yields id order.
__global__ void __launch_bounds__(256) evict_pack_kernel(const uint64_t* keys, int64_t n,
                                                         const unsigned long long* kand,
                                                         const unsigned long long* kor, int skip_id, Pack2* out) {
    __shared__ int pos[24];
    __shared__ int nv;
    if (threadIdx.x == 0) {
        nv = varying_bytes(kand, kor, pos);
        if (skip_id)
            while (nv > 0 && pos[nv - 1] >= 16) --nv;
    }
    __syncthreads();
    const int c = min(nv, 16);
    for (int64_t i = blockIdx.x * 256ll + threadIdx.x; i < n; i += 256ll * gridDim.x) {
        const uint64_t* k = keys + 3 * i;
        uint64_t hi = 0, lo = 0;
        for (int j = 0; j < c; ++j) {
            const int d = pos[j], w = d >> 3, sh = 8 * (7 - (d & 7));
            hi = (hi << 8) | (lo >> 56);
            lo = (lo << 8) | ((k[w] >> sh) & 0xff);
        }
        out[i] = Pack2{hi, lo};
    }
}

struct Key3 {
    uint64_t a, b, c;  // (primary, created_at, id) order-preserving keys
};

__global__ void gather_ids_kernel(const int32_t* slots, const int64_t* ids, int64_t n, int64_t* out) {
    for (int64_t i = blockIdx.x * 256ll + threadIdx.x; i < n; i += 256ll * gridDim.x) out[i] = ids[slots[i]];
}

// Small victim sets: one CTA sorts by the 192-bit key (rank sort in smem).
__device__ __forceinline__ bool key3_less(const uint64_t* a, const uint64_t* b) {
    if (a[0] != b[0]) return a[0] < b[0];
    if (a[1] != b[1]) return a[1] < b[1];
    return a[2] < b[2];
}

__global__ void __launch_bounds__(1024) evict_small_sort_kernel(const uint64_t* keys, const int32_t* slots,
                                                                const int64_t* ids, int n, int64_t* out_ids) {
    extern __shared__ uint64_t sk[];  // [n][3]
    for (int i = threadIdx.x; i < 3 * n; i += blockDim.x) sk[i] = keys[i];
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        int r = 0;
        for (int j = 0; j < n; ++j) r += key3_less(sk + 3 * j, sk + 3 * i) ? 1 : 0;
        out_ids[r] = ids[slots[i]];
    }
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
