// Size-weighted victim prefix by sample select + bucketed block radix sort
// (replaces round 1's multi-pass radix select and device-wide library sort).
//
// Reference semantics (pkg/src/semcache/engine.py):
//   _victim_order_locked :369-383  ascending (key, created_at, id) over all
//                                  residents; key = cal_score (lcfu),
//                                  last_access (lru) or frequency (lfu)
//   admit / evict loops  :321-327, :353-359  pop in that order while the
//                                  freed size is below the excess -> the
//                                  victims are the shortest prefix whose
//                                  size sum reaches the excess (all of
//                                  them when the total does not)
//
// Pipeline (one stream, one host sync before the result copy):
//   0 sel_init_kernel     SelCtl preset, bucket counters zeroed, 4096
//                         strided slots' keys and sizes gathered (16 CTAs)
//   1 sel_sample_kernel   one CTA: a weighted radix select over the samples'
//                         full keys narrows to the <= 16 samples around the
//                         size quantile of the excess plus a 6-sigma margin;
//                         the largest, `hi`, bounds the victim prefix with
//                         overwhelming probability
//   2 sel_collect_kernel  THE pass over the store (HBM-bound): each live
//                         slot's primary key from its columns; slots with
//                         (key, created_at, tie) <= hi become 32-byte records
//                         staged in shared memory and flushed with one
//                         global reservation per CTA round
//   3 sel_split_kernel    one CTA: the records' size must reach the excess
//                         (checked exactly; otherwise the host re-runs from
//                         2 taking every slot); 4096 sampled records' 32-bit
//                         windows (the bits from the records' first varying
//                         bit) radix-sorted give <= 1024 bucket splitters and
//                         a lookup table over their top 12 bits
//   4 sel_bucket_kernel   bucket of each record (table lookup + a short
//                         search in smem) + per-bucket count / size
//   5 sel_scan_kernel     bucket offsets; the bucket where the size prefix
//                         reaches the excess (later buckets are skipped)
//   6 sel_scatter_kernel  records -> bucket order (one global reservation
//                         per (CTA, bucket))
//   7 sel_sort_kernel     one CTA per bucket (persistent): the 32 bits from
//                         the bucket's first varying bit are block-radix-
//                         sorted (cub::BlockRadixSort as a building block
//                         inside this kernel); ids land at their final
//                         positions, and the cut bucket finds the last
//                         victim with a block scan of the sizes
//   8 sel_big_kernel      buckets whose windows tie, or above the cap: the
//                         full varying bits (<= 192) radix-sorted in chunks,
//                         chunks merged along merge paths
//
// Keys are unique -- the third word is the slot when slots are in id order
// (ids appended ascending) and the id otherwise -- so the order is total
// and the output deterministic even though records are appended in
// reservation order.
#pragma once

#include <cub/block/block_radix_sort.cuh>

#include "common.cuh"
#include "evict.cuh"

namespace sine {

struct SelRec {
    uint64_t k0, k1, k2;  // (primary, created_at, slot-or-id) order keys
    int64_t size;
};

struct SelCtl {
    uint64_t hi[3];
    int32_t all;       // take every live slot (host: small stores / retry; sample: bound >= total)
    int32_t retry;     // records below hi do not reach the excess: re-run with all = 1
    int32_t nb;        // buckets
    int32_t cutb;      // bucket holding the last victim
    int32_t nbig;      // buckets above the cap
    int32_t bnext;     // sort kernel: next bucket to take
    unsigned long long count;  // records
    unsigned long long wtake;  // their size
    unsigned long long rand[3], ror[3];  // AND / OR of the record keys (host presets ~0 / 0)
    unsigned long long wmin, wmax;       // min / max 64-bit window of the records (host presets ~0 / 0)
    int64_t wbase;     // size of the buckets before cutb
    int64_t V;         // victims
};

constexpr int kSelSample = 4096;       // sel_sample_kernel: 1024 threads x 4
constexpr int kSelSampleKeep = 16;     // sel_sample_kernel: stop narrowing at this many samples
constexpr int kSelSplitSample = 4096;  // sel_split_kernel: 1024 threads x 4
constexpr int kSelMaxBuckets = 1024;
constexpr int kSelSortThreads = 512;
constexpr int kSelCap = 12 * kSelSortThreads;     // records one CTA counting-sorts (6144)
constexpr int kSelFullCap = 8 * kSelSortThreads;  // records one CTA full-key-sorts
constexpr int kSelStage = 2048;               // collect: records staged per CTA
constexpr int kSelRadixBits = 6;

__device__ __forceinline__ bool key_less(uint64_t a0, uint64_t a1, uint64_t a2, uint64_t b0, uint64_t b1,
                                         uint64_t b2) {
    return a0 != b0 ? a0 < b0 : (a1 != b1 ? a1 < b1 : a2 < b2);
}
__device__ __forceinline__ bool rec_less(const SelRec& a, const SelRec& b) {
    return key_less(a.k0, a.k1, a.k2, b.k0, b.k1, b.k2);
}
__device__ __forceinline__ int64_t rec_id(const SelRec& r, int slot_tie, const int64_t* ids) {
    return slot_tie ? ids[r.k2] : static_cast<int64_t>(r.k2 ^ 0x8000000000000000ull);
}
__device__ __forceinline__ int64_t i64min(int64_t a, int64_t b) { return a < b ? a : b; }
__device__ __forceinline__ int64_t i64max(int64_t a, int64_t b) { return a > b ? a : b; }

// Exclusive block scan of one int64 per thread.
__device__ __forceinline__ int64_t block_excl_scan(int64_t v, int64_t* wtot, int64_t* total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    int64_t inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int64_t t = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += t;
    }
    if (lane == 31) wtot[warp] = inc;
    __syncthreads();
    if (warp == 0) {
        const int64_t x = lane < nw ? wtot[lane] : 0;
        int64_t xi = x;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int64_t t = __shfl_up_sync(0xffffffffu, xi, o);
            if (lane >= o) xi += t;
        }
        if (lane < nw) wtot[lane] = xi - x;
        if (lane == 31) *total = xi;
    }
    __syncthreads();
    const int64_t r = wtot[warp] + inc - v;
    __syncthreads();
    return r;
}

// Block AND / OR of three words (sa, so: 3 shared words each, preset).
__device__ __forceinline__ void block_and_or3(uint64_t a[3], uint64_t o[3], unsigned long long* sa,
                                              unsigned long long* so) {
#pragma unroll
    for (int w = 0; w < 3; ++w) {
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) {
            a[w] &= __shfl_xor_sync(0xffffffffu, a[w], d);
            o[w] |= __shfl_xor_sync(0xffffffffu, o[w], d);
        }
    }
    if ((threadIdx.x & 31) == 0) {
#pragma unroll
        for (int w = 0; w < 3; ++w) {
            atomicAnd(sa + w, static_cast<unsigned long long>(a[w]));
            atomicOr(so + w, static_cast<unsigned long long>(o[w]));
        }
    }
    __syncthreads();
#pragma unroll
    for (int w = 0; w < 3; ++w) a[w] = sa[w], o[w] = so[w];
}

// Word w of a 192-bit key (k0 most significant) without a local array:
// a runtime index into {k0, k1, k2} would put the key in local memory.
__device__ __forceinline__ uint64_t key_word(uint64_t k0, uint64_t k1, uint64_t k2, int w) {
    return w == 0 ? k0 : (w == 1 ? k1 : (w == 2 ? k2 : 0ull));
}

// 64 bits of the 192-bit key starting at its first bit that varies over a
// set (given the set's AND / OR): order-preserving up to ties for the set.
__device__ __forceinline__ uint64_t key_window(uint64_t k0, uint64_t k1, uint64_t k2, const uint64_t a[3],
                                               const uint64_t o[3]) {
    int p = 192;
#pragma unroll
    for (int w = 2; w >= 0; --w)
        if (a[w] ^ o[w]) p = 64 * w + __clzll(a[w] ^ o[w]);
    if (p >= 192) return 0;
    const int w = p >> 6, off = p & 63;
    uint64_t v = key_word(k0, k1, k2, w) << off;
    if (off) v |= key_word(k0, k1, k2, w + 1) >> (64 - off);
    return v;
}

// 64 bits of the 192-bit key from big-endian bit p (zero-padded past 192).
__device__ __forceinline__ uint64_t key_window_at(uint64_t k0, uint64_t k1, uint64_t k2, int p) {
    if (p >= 192) return 0;
    const int w = p >> 6, off = p & 63;
    uint64_t v = key_word(k0, k1, k2, w) << off;
    if (off) v |= key_word(k0, k1, k2, w + 1) >> (64 - off);
    return v;
}

__device__ __forceinline__ int first_varying(const uint64_t a[3], const uint64_t o[3]) {
    int p = 192;
#pragma unroll
    for (int w = 2; w >= 0; --w)
        if (a[w] ^ o[w]) p = 64 * w + __clzll(a[w] ^ o[w]);
    return p;
}

__device__ __forceinline__ void slot_keys(const EvictCols& c, int64_t s, int policy, double now, int slot_tie,
                                          uint64_t& k0, uint64_t& k1, uint64_t& k2) {
    k0 = primary_key(c, s, policy, now);
    k1 = f64_key(c.created[s]);
    k2 = slot_tie ? static_cast<uint64_t>(s) : i64_key(c.ids[s]);
}

// ------------------------------------------------------------ 0 init/gather
// SelCtl preset (ANDs ~0, ORs 0, wmin ~0), bucket counters zeroed, and --
// unless every live slot becomes a record -- the 4096 strided samples'
// keys and sizes (size -1: dead slot) gathered by 16 CTAs.  One CTA pulling
// these scattered columns is bound by a single SM's memory pipe (the
// one-CTA sample kernel spent 49 us on it); spread out it is one latency.
constexpr int kSelInitThreads = 256;
__global__ void __launch_bounds__(kSelInitThreads) sel_init_kernel(const EvictCols c, int policy, double now,
                                                                   int slot_tie, int all, SelCtl* ctl,
                                                                   unsigned long long* bcnt, int nbcnt,
                                                                   SelRec* samp) {
    pdl_trigger();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i == 0) {
        SelCtl c0{};
        c0.all = all;
        for (int w = 0; w < 3; ++w) c0.rand[w] = ~0ull;
        c0.wmin = ~0ull;
        *ctl = c0;
    }
    for (int j = i; j < nbcnt; j += gridDim.x * blockDim.x) bcnt[j] = 0;
    if (!all && i < kSelSample) {
        const int64_t s = ((2 * static_cast<int64_t>(i) + 1) * c.nslots) / (2 * kSelSample);
        SelRec r;
        slot_keys(c, s, policy, now, slot_tie, r.k0, r.k1, r.k2);
        const int64_t w = c.size[s];
        r.size = valid_bit(c.valid, s) ? w : -1;
        samp[i] = r;
    }
}

// ---------------------------------------------------------------- 1 sample
// 8 bits of a 192-bit key at big-endian bit q (q + 8 <= 192).
__device__ __forceinline__ uint32_t key_digit8(const uint64_t k[3], int q) {
    const int w = q >> 6, off = q & 63;
    uint64_t v = key_word(k[0], k[1], k[2], w) << off;
    if (off > 56) v |= key_word(k[0], k[1], k[2], w + 1) >> (64 - off);
    return static_cast<uint32_t>(v >> 56);
}

// Weighted radix select over the full keys of 4096 strided samples (8-bit
// digits from the first varying bit; a sample stays alive while it matches
// every chosen digit) until one sample is left: the one where the
// cumulative size reaches the target.  hi = its full key.
__global__ void __launch_bounds__(1024) sel_sample_kernel(const SelRec* samp, int64_t nlive, int64_t excess,
                                                         SelCtl* ctl) {
    __shared__ uint32_t hl[256], hh[256], hc[256];
    __shared__ int64_t wtot[32];
    __shared__ int64_t wsum;
    __shared__ unsigned long long sa[3], so[3];
    __shared__ int nvalid, digit, left;
    __shared__ int64_t below;
    constexpr int per = kSelSample / 1024;
    pdl_wait();  // the samples come from sel_init_kernel
    pdl_trigger();
    if (threadIdx.x < 3) sa[threadIdx.x] = ~0ull, so[threadIdx.x] = 0ull;
    if (threadIdx.x == 0) nvalid = 0;
    __syncthreads();
    uint64_t k[per][3];
    int64_t W[per];
    bool alive[per];
    uint64_t a[3] = {~0ull, ~0ull, ~0ull}, o[3] = {0, 0, 0};
    int nv_local = 0;
    int64_t wloc = 0;
#pragma unroll
    for (int j = 0; j < per; ++j) {
        const SelRec r = samp[per * threadIdx.x + j];
        alive[j] = r.size >= 0;
        k[j][0] = r.k0, k[j][1] = r.k1, k[j][2] = r.k2;
        W[j] = r.size;
    }
#pragma unroll
    for (int j = 0; j < per; ++j) {
        if (alive[j]) {
            wloc += W[j];
            ++nv_local;
#pragma unroll
            for (int w = 0; w < 3; ++w) a[w] &= k[j][w], o[w] |= k[j][w];
        } else {
            W[j] = 0;
        }
    }
    if (nv_local) atomicAdd(&nvalid, nv_local);
    block_and_or3(a, o, sa, so);
    block_excl_scan(wloc, wtot, &wsum);
    const int nv = nvalid;
    const int64_t ws = wsum;
    // weighted quantile of the excess + a 6-sigma sampling margin
    double g = 2.0;
    if (nv > 0 && ws > 0) {
        const double west = static_cast<double>(ws) * static_cast<double>(nlive) / nv;
        const double f = fmin(1.0, static_cast<double>(excess) / west);
        g = f + 6.0 * sqrt(fmax(f * (1.0 - f), 1.0 / nv) / nv) + 4.0 / nv;
    }
    if (g >= 1.0) {
        if (threadIdx.x == 0) ctl->all = 1;
        return;
    }
    int p = 192;  // first bit varying over the samples
#pragma unroll
    for (int w = 2; w >= 0; --w)
        if (a[w] ^ o[w]) p = 64 * w + __clzll(a[w] ^ o[w]);
    int64_t rem = static_cast<int64_t>(ceil(g * static_cast<double>(ws)));
    int nleft = nv;
    // narrow until at most kSelSampleKeep samples share the chosen digits,
    // then take the largest of them: a bound at or above the quantile sample
    // (a few more records for collect to keep; each 8-bit pass costs ~3 us)
    for (int q0 = p; q0 < 192 && nleft > kSelSampleKeep;) {
        const int q = q0 < 184 ? q0 : 184;  // the last digit may overlap fixed bits
        if (threadIdx.x < 256) hl[threadIdx.x] = hh[threadIdx.x] = hc[threadIdx.x] = 0;
        __syncthreads();
        uint32_t dg[per];
#pragma unroll
        for (int j = 0; j < per; ++j) {
            dg[j] = key_digit8(k[j], q);
            // a quarter of the samples can share one digit (equal scores):
            // few distinct digits in a warp take one shared atomic per
            // digit (warp sums), many take plain per-lane atomics
            const int lane = threadIdx.x & 31;
            const bool act = alive[j];
            const uint32_t peers = __match_any_sync(0xffffffffu, act ? dg[j] : 0x100u);
            const bool group_leader = act && (__ffs(peers) - 1) == lane;
            if (__popc(__ballot_sync(0xffffffffu, group_leader)) > 4) {
                if (act) {
                    smem_add64(&hl[dg[j]], &hh[dg[j]], static_cast<uint64_t>(W[j]));
                    atomicAdd(&hc[dg[j]], 1u);
                }
            } else {
                uint32_t pend = __ballot_sync(0xffffffffu, act);
                while (pend) {
                    const int leader = __ffs(pend) - 1;
                    const uint32_t ldg = __shfl_sync(0xffffffffu, dg[j], leader);
                    const bool mine = act && dg[j] == ldg;
                    const uint32_t grp = __ballot_sync(0xffffffffu, mine);
                    unsigned long long v = mine ? static_cast<unsigned long long>(W[j]) : 0ull;
#pragma unroll
                    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
                    if (lane == leader) {
                        smem_add64(&hl[ldg], &hh[ldg], v);
                        atomicAdd(&hc[ldg], static_cast<uint32_t>(__popc(grp)));
                    }
                    pend &= ~grp;
                }
            }
        }
        __syncthreads();
        if (threadIdx.x < 32) {  // warp 0: bins 8l .. 8l + 7
            int64_t v[8], t = 0;
#pragma unroll
            for (int r = 0; r < 8; ++r) {
                const int bn = 8 * threadIdx.x + r;
                v[r] = static_cast<int64_t>((static_cast<uint64_t>(hh[bn]) << 32) | hl[bn]);
                t += v[r];
            }
            int64_t inc = t;
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                const int64_t y = __shfl_up_sync(0xffffffffu, inc, off);
                if (threadIdx.x >= off) inc += y;
            }
            int64_t run = inc - t;
            int found = 256;
            int64_t bel = 0;
#pragma unroll
            for (int r = 0; r < 8; ++r) {
                if (found == 256 && run + v[r] >= rem) found = 8 * threadIdx.x + r, bel = run;
                run += v[r];
            }
            // rem <= the alive weight is invariant, so some bin reaches it;
            // otherwise (cannot happen) every slot becomes a record
            const uint32_t m = __ballot_sync(0xffffffffu, found < 256);
            const int src = m ? __ffs(m) - 1 : 0;
            const int fd = __shfl_sync(0xffffffffu, found, src);
            const int64_t fb = __shfl_sync(0xffffffffu, bel, src);
            if (threadIdx.x == 0) {
                digit = m ? fd : -1;
                below = m ? fb : 0;
                left = m ? static_cast<int>(hc[fd]) : 0;
            }
        }
        __syncthreads();
        const int d = digit;
#pragma unroll
        for (int j = 0; j < per; ++j) alive[j] = alive[j] && static_cast<int>(dg[j]) == d;
        rem -= below;
        nleft = left;
        // next digit: the first bit that still varies over the alive samples
        if (threadIdx.x < 3) sa[threadIdx.x] = ~0ull, so[threadIdx.x] = 0ull;
        __syncthreads();
        uint64_t aa[3] = {~0ull, ~0ull, ~0ull}, oo[3] = {0, 0, 0};
#pragma unroll
        for (int j = 0; j < per; ++j)
            if (alive[j])
#pragma unroll
                for (int w = 0; w < 3; ++w) aa[w] &= k[j][w], oo[w] |= k[j][w];
        block_and_or3(aa, oo, sa, so);
        int pn = 192;
#pragma unroll
        for (int w = 2; w >= 0; --w)
            if (aa[w] ^ oo[w]) pn = 64 * w + __clzll(aa[w] ^ oo[w]);
        q0 = pn > q + 8 ? pn : q + 8;
        __syncthreads();
    }
    // the largest surviving sample (keys are unique); `all` when none survived
    __shared__ unsigned long long wk[32][3];
    __shared__ int wany[32];
    bool any = false;
    uint64_t m0 = 0, m1 = 0, m2 = 0;
#pragma unroll
    for (int j = 0; j < per; ++j)
        if (alive[j] && (!any || key_less(m0, m1, m2, k[j][0], k[j][1], k[j][2]))) {
            m0 = k[j][0], m1 = k[j][1], m2 = k[j][2];
            any = true;
        }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        const uint64_t o0 = __shfl_xor_sync(0xffffffffu, m0, off), o1 = __shfl_xor_sync(0xffffffffu, m1, off),
                       o2 = __shfl_xor_sync(0xffffffffu, m2, off);
        const bool oany = __shfl_xor_sync(0xffffffffu, any, off);
        if (oany && (!any || key_less(m0, m1, m2, o0, o1, o2))) m0 = o0, m1 = o1, m2 = o2, any = true;
    }
    if (lane == 0) wk[warp][0] = m0, wk[warp][1] = m1, wk[warp][2] = m2, wany[warp] = any;
    __syncthreads();
    if (threadIdx.x == 0) {
        bool f = false;
        uint64_t b0 = 0, b1 = 0, b2 = 0;
        for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w)
            if (wany[w] && (!f || key_less(b0, b1, b2, wk[w][0], wk[w][1], wk[w][2])))
                b0 = wk[w][0], b1 = wk[w][1], b2 = wk[w][2], f = true;
        if (f)
            ctl->hi[0] = b0, ctl->hi[1] = b1, ctl->hi[2] = b2;
        else
            ctl->all = 1;
    }
}

// --------------------------------------------------------------- 2 collect
// Each warp stages its records in its own smem slice and flushes them with
// one global reservation when the slice could overflow.
constexpr int kSelWarpStage = 96;        // records per warp slice
constexpr int kSelConsumers = 768;       // 24 consumer warps, one slot each per tile
constexpr int kSelCollectThreads = kSelConsumers + 32;  // + one producer warp
constexpr int kSelTile = 768;            // slots per TMA tile (96-byte validity rows stay 16-B aligned)
constexpr int kSelStages = 3;            // tiles in flight per CTA
constexpr int kSelMaxCols = 7;
constexpr int kSelStageBytes = kSelMaxCols * kSelTile * 8 + kSelTile / 8;  // columns + validity words
static_assert(kSelTile % kSelConsumers == 0 && kSelTile % 128 == 0, "tile shape");
constexpr int kSelCollectSmem = kSelStages * kSelStageBytes +
                                (kSelConsumers / 32) * kSelWarpStage * static_cast<int>(sizeof(SelRec)) + 64;

__device__ __forceinline__ void warp_flush(SelRec* st, int& n, SelCtl* ctl, SelRec* rec) {
    const int lane = threadIdx.x & 31;
    unsigned long long b = 0;
    if (lane == 0 && n) b = atomicAdd(&ctl->count, static_cast<unsigned long long>(n));
    b = __shfl_sync(0xffffffffu, b, 0);
    __syncwarp();
    for (int i = lane; i < n; i += 32) rec[b + i] = st[i];
    __syncwarp();
    n = 0;
}

// The columns a policy's key needs, then size_tokens and created_at.
struct SelColumns {
    const void* col[kSelMaxCols];
    int ncol;
};

// Persistent CTAs: a producer warp streams 768-slot tiles of the key
// columns and the validity words into a 3-stage shared-memory ring with 1-D
// bulk copies (TMA engine; `full` mbarriers complete on the bytes, `empty`
// mbarriers collect one arrival per consumer warp), so the bytes in flight do
// not depend on registers and no block-wide barrier couples the warps.  Each
// consumer thread takes one slot per tile; records go to per-warp smem
// slices (warp-aggregated), flushed with one global reservation each.
__global__ void __launch_bounds__(kSelCollectThreads, 1) sel_collect_kernel(const EvictCols c, const SelColumns cols,
                                                                           int policy, double now, int slot_tie,
                                                                           SelCtl* ctl, SelRec* rec) {
    extern __shared__ __align__(128) uint64_t sel_smem[];
    uint8_t* ring = reinterpret_cast<uint8_t*>(sel_smem);  // [stage]{[col][tile] f64, [tile/32] u32}
    SelRec* wst = reinterpret_cast<SelRec*>(ring + kSelStages * kSelStageBytes);
    uint64_t* full = reinterpret_cast<uint64_t*>(wst + (kSelConsumers / 32) * kSelWarpStage);
    uint64_t* empty = full + kSelStages;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nc = cols.ncol;
    const int64_t ntiles = (c.nslots + kSelTile - 1) / kSelTile;
    // PDL: the producer streams the columns at once (nothing in this launch
    // chain writes them); the consumers wait for ctl below
    pdl_trigger();
    if (threadIdx.x == 0) {
        for (int i = 0; i < kSelStages; ++i) {
            mbar_init(full + i, 1);
            mbar_init(empty + i, kSelConsumers / 32);
        }
        fence_mbar_init();
    }
    __syncthreads();
    if (warp == kSelConsumers / 32) {  // producer
        if (lane == 0) {
            const uint64_t pol = l2_evict_first_policy();
            int it = 0;
            for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
                const int stg = it % kSelStages;
                if (it >= kSelStages) mbar_wait(empty + stg, static_cast<uint32_t>(((it / kSelStages) - 1) & 1));
                const int64_t s0 = t * kSelTile;
                const int64_t n = c.nslots - s0 < kSelTile ? c.nslots - s0 : kSelTile;
                const int64_t nr = (n + 127) / 128 * 128;  // capacity is a multiple of 128 slots
                const uint32_t bytes = static_cast<uint32_t>(nr) * 8u, vbytes = static_cast<uint32_t>(nr / 8);
                uint8_t* base = ring + stg * kSelStageBytes;
                mbar_arrive_expect_tx(full + stg, bytes * nc + vbytes);
                for (int k = 0; k < nc; ++k)
                    bulk_g2s(base + k * kSelTile * 8, static_cast<const double*>(cols.col[k]) + s0, bytes, full + stg,
                             pol);
                bulk_g2s(base + kSelMaxCols * kSelTile * 8, c.valid + s0 / 32, vbytes, full + stg, pol);
            }
        }
        return;
    }
    pdl_wait();  // ctl (hi, all, counters) comes from the init / sample kernels
    SelRec* st = wst + warp * kSelWarpStage;
    int nst = 0;
    const int all = ctl->all;
    const uint64_t hi[3] = {ctl->hi[0], ctl->hi[1], ctl->hi[2]};
    unsigned long long wl = 0;
    uint64_t ra[3] = {~0ull, ~0ull, ~0ull}, ro[3] = {0, 0, 0};
    int it = 0;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
        const int stg = it % kSelStages;
        mbar_wait(full + stg, static_cast<uint32_t>((it / kSelStages) & 1));
        const double* S = reinterpret_cast<const double*>(ring + stg * kSelStageBytes);
        const uint32_t* V = reinterpret_cast<const uint32_t*>(ring + stg * kSelStageBytes + kSelMaxCols * kSelTile * 8);
        const int64_t s0 = t * kSelTile;
#pragma unroll
        for (int q = 0; q < kSelTile / kSelConsumers; ++q) {
            const int j = q * kSelConsumers + threadIdx.x;
            const int64_t s = s0 + j;
            const bool act = s < c.nslots && ((V[j >> 5] >> (j & 31)) & 1u);
            uint64_t k0;
            int64_t size;
            double created;
            if (policy == 0) {
                size = __double_as_longlong(S[5 * kSelTile + j]);
                created = S[6 * kSelTile + j];
                double v = 0.0;  // cal_score (engine.py:33-48): exact order, no FMA contraction
                if (size != 0 && !(__dsub_rn(S[4 * kSelTile + j], now) <= 0.0)) {
                    v = __dmul_rn(__dmul_rn(__dmul_rn(S[j], S[kSelTile + j]), S[2 * kSelTile + j]),
                                  S[3 * kSelTile + j]);
                    // a zero product (log(1) factors are common) divides to
                    // +-0 (one key); skipping it keeps the IEEE division off
                    // its slow path, which a zero dividend takes
                    if (v != 0.0) v = __ddiv_rn(v, static_cast<double>(size));
                }
                k0 = f64_key(v);
            } else {
                size = __double_as_longlong(S[kSelTile + j]);
                created = S[2 * kSelTile + j];
                k0 = policy == 1 ? f64_key(S[j]) : i64_key(__double_as_longlong(S[j]));
            }
            const uint64_t k1 = f64_key(created);
            bool take = act && (all || k0 <= hi[0]);
            uint64_t k2 = slot_tie ? static_cast<uint64_t>(s) : 0ull;
            if (take && !slot_tie) k2 = i64_key(__ldg(c.ids + s));
            if (take && !all && k0 == hi[0]) take = k1 != hi[1] ? k1 < hi[1] : k2 <= hi[2];
            const uint32_t m = __ballot_sync(0xffffffffu, take);
            if (m) {
                if (nst + __popc(m) > kSelWarpStage) warp_flush(st, nst, ctl, rec);
                if (take) {
                    wl += static_cast<unsigned long long>(size);
                    SelRec r;
                    r.k0 = k0, r.k1 = k1, r.k2 = k2, r.size = size;
                    ra[0] &= k0, ra[1] &= k1, ra[2] &= k2;
                    ro[0] |= k0, ro[1] |= k1, ro[2] |= k2;
                    st[nst + __popc(m & ((1u << lane) - 1u))] = r;
                }
                nst += __popc(m);
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(empty + stg);  // this warp is done with the stage
    }
    warp_flush(st, nst, ctl, rec);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) wl += __shfl_xor_sync(0xffffffffu, wl, o);
#pragma unroll
    for (int w = 0; w < 3; ++w) {
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) {
            ra[w] &= __shfl_xor_sync(0xffffffffu, ra[w], d);
            ro[w] |= __shfl_xor_sync(0xffffffffu, ro[w], d);
        }
    }
    if (lane == 0 && wl) {
        atomicAdd(&ctl->wtake, wl);
#pragma unroll
        for (int w = 0; w < 3; ++w) {
            atomicAnd(&ctl->rand[w], static_cast<unsigned long long>(ra[w]));
            atomicOr(&ctl->ror[w], static_cast<unsigned long long>(ro[w]));
        }
    }
}

// 32-bit window of a record relative to the records' AND / OR: a prefix of
// the full key over the record set, so window order never contradicts it.
__device__ __forceinline__ uint32_t rec_win32(const SelRec& r, const uint64_t a[3], const uint64_t o[3]) {
    return static_cast<uint32_t>(key_window(r.k0, r.k1, r.k2, a, o) >> 32);
}

__device__ __forceinline__ void ctl_and_or(const SelCtl* ctl, uint64_t a[3], uint64_t o[3]) {
#pragma unroll
    for (int w = 0; w < 3; ++w) a[w] = ctl->rand[w], o[w] = ctl->ror[w];
}

// ----------------------------------------------------------------- 3 split
// 4096 sampled records' windows radix-sorted; every os-th is a splitter
// (32-bit values: bucket b holds the windows in (spl[b-1], spl[b]]), plus a
// table over the top 12 window bits: tab[t] = splitters whose top 12 bits
// are below t, so a record's bucket is tab[t] + a search among the few
// splitters sharing its top bits.
using SplitSort = cub::BlockRadixSort<uint32_t, 1024, kSelSplitSample / 1024, cub::NullType, 4>;

__global__ void __launch_bounds__(1024) sel_split_kernel(int64_t excess, SelCtl* ctl, const SelRec* rec,
                                                        uint32_t* spl, uint32_t* tab, int cap) {
    pdl_wait();
    pdl_trigger();
    __shared__ typename SplitSort::TempStorage ts;
    __shared__ uint32_t S[kSelMaxBuckets];
    if (!ctl->all && static_cast<int64_t>(ctl->wtake) < excess) {
        if (threadIdx.x == 0) ctl->retry = 1;
        return;
    }
    const int64_t M = static_cast<int64_t>(ctl->count);
    if (M <= cap) {  // one bucket
        if (threadIdx.x == 0) ctl->nb = 1;
        return;
    }
    uint64_t a[3], o[3];
    ctl_and_or(ctl, a, o);
    constexpr int per = kSelSplitSample / 1024;
    uint32_t keys[per];
#pragma unroll
    for (int j = 0; j < per; ++j) {
        const int i = per * threadIdx.x + j;
        keys[j] = rec_win32(rec[((2 * static_cast<int64_t>(i) + 1) * M) / (2 * kSelSplitSample)], a, o);
    }
    SplitSort(ts).Sort(keys);
    // buckets of ~1024 records on average; with 4 samples per bucket the
    // largest of 1024 buckets stays well below the 8192 cap
    int nb = 2;
    while (nb < kSelMaxBuckets && nb < kSelSplitSample / 4 && static_cast<int64_t>(nb) * 1024 < M) nb <<= 1;
    const int os = kSelSplitSample / nb;
#pragma unroll
    for (int j = 0; j < per; ++j) {
        const int r = per * threadIdx.x + j + 1;  // 1-based rank
        if (r % os == 0 && r < kSelSplitSample) S[r / os - 1] = keys[j];
    }
    __syncthreads();
    const int ns = nb - 1;
    for (int j = threadIdx.x; j < ns; j += blockDim.x) spl[j] = S[j];
    for (int t = threadIdx.x; t <= 4096; t += blockDim.x) {
        int lo = 0, hi = ns;  // splitters with top-12 bits < t
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (static_cast<int>(S[mid] >> 20) < t)
                lo = mid + 1;
            else
                hi = mid;
        }
        tab[t] = static_cast<uint32_t>(lo);
    }
    if (threadIdx.x == 0) ctl->nb = nb;
}

// ------------------------------------------------------ 4 bucket, 6 scatter
constexpr int kSelBucketSmem = kSelMaxBuckets * 4 + 4100 * 4 + kSelMaxBuckets * 12;

__device__ __forceinline__ int find_bucket(uint32_t w, const uint32_t* S, const uint32_t* T) {
    const int t = static_cast<int>(w >> 20);
    int lo = static_cast<int>(T[t]), hi = static_cast<int>(T[t + 1]);
    while (lo < hi) {  // splitters below w among those sharing its top bits
        const int mid = (lo + hi) >> 1;
        if (S[mid] < w)
            lo = mid + 1;
        else
            hi = mid;
    }
    return lo;
}

// Both kernels give CTA x the same contiguous record range.
__device__ __forceinline__ void cta_range(int64_t M, int64_t& b, int64_t& e) {
    const int64_t per = (M + gridDim.x - 1) / gridDim.x;
    b = i64min(M, per * blockIdx.x);
    e = i64min(M, b + per);
}

__global__ void __launch_bounds__(1024) sel_bucket_kernel(SelCtl* ctl, const SelRec* rec, const uint32_t* spl,
                                                         const uint32_t* tab, uint16_t* bid,
                                                         unsigned long long* bcnt, unsigned long long* bw) {
    pdl_wait();
    pdl_trigger();
    extern __shared__ uint64_t sel_smem[];
    if (ctl->retry) return;
    const int nb = ctl->nb, ns = nb - 1;
    uint32_t* S = reinterpret_cast<uint32_t*>(sel_smem);
    uint32_t* T = S + kSelMaxBuckets;
    uint32_t* sc = T + 4100;
    uint32_t* swl = sc + kSelMaxBuckets;
    uint32_t* swh = swl + kSelMaxBuckets;
    for (int j = threadIdx.x; j < ns; j += blockDim.x) S[j] = spl[j];
    for (int j = threadIdx.x; j <= 4096; j += blockDim.x) T[j] = ns ? tab[j] : 0u;
    if (threadIdx.x == 0) T[4097] = ns;
    for (int j = threadIdx.x; j < nb; j += blockDim.x) sc[j] = swl[j] = swh[j] = 0;
    __syncthreads();
    uint64_t a[3], o[3];
    ctl_and_or(ctl, a, o);
    const int pg = first_varying(a, o);
    int64_t b, e;
    cta_range(static_cast<int64_t>(ctl->count), b, e);
    uint64_t wmn = ~0ull, wmx = 0ull;
    constexpr int U = 4;  // records per thread per round, loads first (latency-bound rounds)
    for (int64_t i0 = b + threadIdx.x; i0 < e; i0 += U * blockDim.x) {
        SelRec r[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t i = i0 + static_cast<int64_t>(u) * blockDim.x;
            if (i < e) r[u] = rec[i];
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t i = i0 + static_cast<int64_t>(u) * blockDim.x;
            if (i >= e) continue;
            const uint64_t w64 = key_window_at(r[u].k0, r[u].k1, r[u].k2, pg);
            wmn = w64 < wmn ? w64 : wmn;
            wmx = w64 > wmx ? w64 : wmx;
            const int k = ns ? find_bucket(static_cast<uint32_t>(w64 >> 32), S, T) : 0;
            bid[i] = static_cast<uint16_t>(k);
            atomicAdd(&sc[k], 1u);
            smem_add64(&swl[k], &swh[k], static_cast<uint64_t>(r[u].size));
        }
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
        const uint64_t x = __shfl_xor_sync(0xffffffffu, wmn, d), y = __shfl_xor_sync(0xffffffffu, wmx, d);
        wmn = x < wmn ? x : wmn;
        wmx = y > wmx ? y : wmx;
    }
    if ((threadIdx.x & 31) == 0 && wmn <= wmx) {
        atomicMin(&ctl->wmin, static_cast<unsigned long long>(wmn));
        atomicMax(&ctl->wmax, static_cast<unsigned long long>(wmx));
    }
    __syncthreads();
    for (int j = threadIdx.x; j < nb; j += blockDim.x) {
        if (sc[j]) {
            atomicAdd(bcnt + j, static_cast<unsigned long long>(sc[j]));
            atomicAdd(bw + j, (static_cast<unsigned long long>(swh[j]) << 32) | swl[j]);
        }
    }
}

__global__ void __launch_bounds__(1024) sel_scatter_kernel(const SelCtl* ctl, const SelRec* rec, const uint16_t* bid,
                                                          const int64_t* boff, uint32_t* bcur, SelRec* rec2) {
    pdl_wait();
    pdl_trigger();
    __shared__ uint32_t lc[kSelMaxBuckets];
    __shared__ int64_t lb[kSelMaxBuckets];  // this CTA's first position in bucket k (boff folded in)
    if (ctl->retry) return;
    const int nb = ctl->nb, cutb = ctl->cutb;
    for (int j = threadIdx.x; j < nb; j += blockDim.x) lc[j] = 0;
    __syncthreads();
    int64_t b, e;
    cta_range(static_cast<int64_t>(ctl->count), b, e);
    // four records per thread per round, loads first: the rounds are
    // latency-bound, not bandwidth-bound
    constexpr int U = 4;
    for (int64_t i0 = b + threadIdx.x; i0 < e; i0 += U * blockDim.x) {
        int k[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t i = i0 + static_cast<int64_t>(u) * blockDim.x;
            k[u] = i < e ? bid[i] : kSelMaxBuckets;
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (k[u] <= cutb) atomicAdd(&lc[k[u]], 1u);
    }
    __syncthreads();
    for (int j = threadIdx.x; j <= cutb; j += blockDim.x) {
        lb[j] = boff[j] + (lc[j] ? atomicAdd(bcur + j, lc[j]) : 0u);
        lc[j] = 0;
    }
    __syncthreads();
    const uint4* src = reinterpret_cast<const uint4*>(rec);
    uint4* dst = reinterpret_cast<uint4*>(rec2);
    for (int64_t i0 = b + threadIdx.x; i0 < e; i0 += U * blockDim.x) {
        int k[U];
        uint4 r0[U], r1[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t i = i0 + static_cast<int64_t>(u) * blockDim.x;
            k[u] = i < e ? bid[i] : kSelMaxBuckets;
            if (k[u] <= cutb) r0[u] = src[2 * i], r1[u] = src[2 * i + 1];
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (k[u] <= cutb) {
                const int64_t at = lb[k[u]] + atomicAdd(&lc[k[u]], 1u);
                dst[2 * at] = r0[u];
                dst[2 * at + 1] = r1[u];
            }
    }
}

// ------------------------------------------------------------------ 5 scan
__global__ void __launch_bounds__(1024) sel_scan_kernel(SelCtl* ctl, int64_t excess, const unsigned long long* bcnt,
                                                       const unsigned long long* bw, int64_t* boff, uint32_t* bcur) {
    pdl_wait();
    pdl_trigger();
    __shared__ int64_t wtot[32];
    __shared__ int64_t total;
    __shared__ int cut;
    if (ctl->retry) return;
    const int nb = ctl->nb;
    constexpr int per = kSelMaxBuckets / 1024;
    const int b0 = per * threadIdx.x;
    int64_t c[per], w[per], lc = 0, lw = 0;
#pragma unroll
    for (int j = 0; j < per; ++j) {
        c[j] = b0 + j < nb ? static_cast<int64_t>(bcnt[b0 + j]) : 0;
        w[j] = b0 + j < nb ? static_cast<int64_t>(bw[b0 + j]) : 0;
        lc += c[j], lw += w[j];
    }
    if (threadIdx.x == 0) cut = nb - 1;
    int64_t oc = block_excl_scan(lc, wtot, &total);
    int64_t ow = block_excl_scan(lw, wtot, &total);
#pragma unroll
    for (int j = 0; j < per; ++j) {
        if (b0 + j < nb) {
            boff[b0 + j] = oc;
            bcur[b0 + j] = 0;
            if (ow + w[j] >= excess) atomicMin(&cut, b0 + j);
        }
        oc += c[j], ow += w[j];
    }
    __syncthreads();
    int64_t pw = 0;
#pragma unroll
    for (int j = 0; j < per; ++j)
        if (b0 + j < cut) pw += w[j];
    block_excl_scan(pw, wtot, &total);
    if (threadIdx.x == 0) {
        ctl->cutb = cut;
        ctl->wbase = total;  // size of the buckets before the cut bucket
    }
}

// ------------------------------------------------------- 7 bucket sorting
// Packed key: per word only the low bits that vary over the bucket, the
// three fields concatenated (word 0 most significant).  <= 128 bits (the
// common case: a constant or narrow primary key) sorts as two words,
// otherwise as three.
struct Key2 {
    uint64_t w1, w0;  // most .. least significant
};
struct Key3 {
    uint64_t w2, w1, w0;
};
struct Key2Decomposer {
    __host__ __device__ ::cuda::std::tuple<uint64_t&, uint64_t&> operator()(Key2& k) const { return {k.w1, k.w0}; }
};
struct Key3Decomposer {
    __host__ __device__ ::cuda::std::tuple<uint64_t&, uint64_t&, uint64_t&> operator()(Key3& k) const {
        return {k.w2, k.w1, k.w0};
    }
};

// (w2, w1, w0) |= v << sh for v < 2^64, sh in [0, 192)
__device__ __forceinline__ void or_shl(uint64_t& w2, uint64_t& w1, uint64_t& w0, uint64_t v, int sh) {
    const int q = sh >> 6, r = sh & 63;
    const uint64_t lo = v << r, hi = r ? (v >> (64 - r)) : 0ull;
    if (q == 0) {
        w0 |= lo;
        w1 |= hi;
    } else if (q == 1) {
        w1 |= lo;
        w2 |= hi;
    } else {
        w2 |= lo;
    }
}

template <typename K, int IPT>
using BucketSort = cub::BlockRadixSort<K, kSelSortThreads, IPT, uint16_t, kSelRadixBits>;

union BucketSortStorage {
    typename BucketSort<Key2, 2>::TempStorage a2;
    typename BucketSort<Key2, 4>::TempStorage a4;
    typename BucketSort<Key2, 8>::TempStorage a8;
    typename BucketSort<Key3, 2>::TempStorage b2;
    typename BucketSort<Key3, 4>::TempStorage b4;
    typename BucketSort<Key3, 8>::TempStorage b8;
};

struct BucketShared {
    BucketSortStorage sort;
    unsigned long long sa[3], so[3];
    int64_t wtot[32];
    int64_t total;
    int first;
};

constexpr int kSelSortSmem = static_cast<int>(sizeof(BucketShared));

template <typename K, int IPT>
__device__ __forceinline__ typename BucketSort<K, IPT>::TempStorage& sort_storage(BucketShared& sh) {
    return *reinterpret_cast<typename BucketSort<K, IPT>::TempStorage*>(&sh.sort);
}

template <typename K, int IPT>
__device__ __forceinline__ void bucket_sort_k(const SelRec* src, int n, const int span[3], int total,
                                              BucketShared& sh, uint16_t (&idx)[IPT]) {
    K keys[IPT];
#pragma unroll
    for (int j = 0; j < IPT; ++j) {
        const int i = threadIdx.x * IPT + j;
        idx[j] = i < n ? static_cast<uint16_t>(i) : static_cast<uint16_t>(0xffff);
        uint64_t w2 = 0, w1 = 0, w0 = 0;
        if (i < n) {
            const SelRec r = src[i];  // second read: L1 / L2
            const uint64_t f[3] = {r.k0, r.k1, r.k2};
            int at = total;
#pragma unroll
            for (int w = 0; w < 3; ++w) {
                at -= span[w];
                if (span[w]) or_shl(w2, w1, w0, span[w] == 64 ? f[w] : (f[w] & ((1ull << span[w]) - 1)), at);
            }
        } else {
            w2 = w1 = w0 = ~0ull;  // after every real key (stable on ties)
        }
        if constexpr (sizeof(K) == 16)
            keys[j] = K{w1, w0};
        else
            keys[j] = K{w2, w1, w0};
    }
    if constexpr (sizeof(K) == 16)
        BucketSort<K, IPT>(sort_storage<K, IPT>(sh)).Sort(keys, idx, Key2Decomposer{}, 0, total);
    else
        BucketSort<K, IPT>(sort_storage<K, IPT>(sh)).Sort(keys, idx, Key3Decomposer{}, 0, total);
}

// Sorts src[0, n) (n <= 512 * IPT) by full key; thread t's items j hold the
// ranks t * IPT + j as indices into src (0xffff: padding).
template <int IPT>
__device__ __forceinline__ void bucket_sort(const SelRec* src, int n, BucketShared& sh, uint16_t (&idx)[IPT]) {
    uint64_t a[3] = {~0ull, ~0ull, ~0ull}, o[3] = {0, 0, 0};
    if (threadIdx.x < 3) sh.sa[threadIdx.x] = ~0ull, sh.so[threadIdx.x] = 0ull;
    __syncthreads();
#pragma unroll
    for (int j = 0; j < IPT; ++j) {
        const int i = threadIdx.x * IPT + j;
        if (i < n) {
            const SelRec r = src[i];
            a[0] &= r.k0, a[1] &= r.k1, a[2] &= r.k2;
            o[0] |= r.k0, o[1] |= r.k1, o[2] |= r.k2;
        }
    }
    block_and_or3(a, o, sh.sa, sh.so);
    int span[3], total = 0;
#pragma unroll
    for (int w = 0; w < 3; ++w) {
        const uint64_t d = a[w] ^ o[w];
        span[w] = d ? 64 - __clzll(d) : 0;
        total += span[w];
    }
    if (total == 0) {  // one record (keys are unique)
#pragma unroll
        for (int j = 0; j < IPT; ++j) {
            const int i = threadIdx.x * IPT + j;
            idx[j] = i < n ? static_cast<uint16_t>(i) : static_cast<uint16_t>(0xffff);
        }
    } else if (total <= 128) {
        bucket_sort_k<Key2, IPT>(src, n, span, total, sh, idx);
    } else {
        bucket_sort_k<Key3, IPT>(src, n, span, total, sh, idx);
    }
}

// Victim ids of sorted records at their final positions [base, base + n)
// (get(idx[j]) = the record of rank t * IPT + j).  With `cut`, also the
// first rank where the size sum from `wbase` reaches the excess: sets V and
// returns true when found; sh.total = the size of these n records.
template <int IPT, typename GetRec, typename Sh>
__device__ __forceinline__ bool bucket_emit(GetRec get, const uint16_t (&idx)[IPT], int n, int64_t base, bool cut,
                                            int64_t wbase, int64_t excess, int slot_tie, const int64_t* ids,
                                            int64_t* out, SelCtl* ctl, Sh& sh, int64_t* oslot = nullptr) {
    int64_t sz[IPT];
    int64_t loc = 0;
    // groups of four: record loads, then the id loads, then the stores (the
    // stores may alias the loads as far as the compiler knows, so without
    // the grouping every record is a serial load -> load -> store chain)
#pragma unroll
    for (int j0 = 0; j0 < IPT; j0 += 4) {
        constexpr int G = 4;
        uint64_t k2[G];
        int64_t idv[G];
#pragma unroll
        for (int g = 0; g < G; ++g) {
            const int j = j0 + g;
            if (j >= IPT) break;
            const int rk = threadIdx.x * IPT + j;
            sz[j] = 0;
            k2[g] = 0;
            if (rk < n) {
                const SelRec r = get(idx[j]);
                k2[g] = r.k2;
                sz[j] = r.size;
            }
        }
#pragma unroll
        for (int g = 0; g < G; ++g) {
            const int j = j0 + g;
            if (j >= IPT) break;
            const int rk = threadIdx.x * IPT + j;
            if (rk < n) idv[g] = slot_tie ? ids[k2[g]] : static_cast<int64_t>(k2[g] ^ 0x8000000000000000ull);
        }
#pragma unroll
        for (int g = 0; g < G; ++g) {
            const int j = j0 + g;
            if (j >= IPT) break;
            const int rk = threadIdx.x * IPT + j;
            if (rk < n) {
                out[base + rk] = idv[g];
                if (oslot) oslot[base + rk] = static_cast<int64_t>(k2[g]);  // slot-ordered stores only
                loc += sz[j];
            }
        }
    }
    if (!cut) return false;
    if (threadIdx.x == 0) sh.first = n;
    int64_t run = wbase + block_excl_scan(loc, sh.wtot, &sh.total);
#pragma unroll
    for (int j = 0; j < IPT; ++j) {
        const int rk = threadIdx.x * IPT + j;
        if (rk < n) {
            run += sz[j];
            if (run >= excess) {
                atomicMin(&sh.first, rk);
                break;
            }
        }
    }
    __syncthreads();
    const int first = sh.first;
    if (threadIdx.x == 0) ctl->V = base + (first < n ? first + 1 : n);
    __syncthreads();
    return first < n;
}

// ------------------------------------------------ 7 bucket sort (counting)
// Per bucket: each record's 64-bit window (from the records' first varying
// bit) minus the bucket's lower bound, scaled so the bucket's range fills 44
// bits, splits into a 12-bit bin and a 32-bit sub-key.  Records are counted
// into the 4096 bins and scattered in bin order; bins holding several
// records (~1 record per 4 bins on average) are ordered by sub-key from
// smem by one thread each (insertion sort), and only equal sub-keys compare
// full keys.  Runs longer than kSelRunMax (a bucket whose records pile into
// one bin) go to the full-key kernel (sel_big_kernel).
constexpr int kSelBins = 4096;
constexpr int kSelRunMax = 128;

struct CountShared {
    uint32_t hist[kSelBins];
    uint32_t ssub[kSelCap];  // sub-key at rank r
    uint16_t sidx[kSelCap];  // record at rank r
    uint16_t sbin[kSelCap];  // bin at rank r
    int64_t wtot[32];
    int64_t total;
    int first;
    int tie;
};

constexpr int kSelCountSmem = static_cast<int>(sizeof(CountShared));

__device__ __forceinline__ uint64_t bucket_offset(const SelRec& r, int pg, uint64_t lo64, int shift) {
    const uint64_t off = (key_window_at(r.k0, r.k1, r.k2, pg) - lo64) >> shift;
    return off < (1ull << 44) ? off : (1ull << 44) - 1;
}

template <int IPT>
__device__ __forceinline__ bool count_sort_emit(const SelRec* src, int n, int pg, uint64_t lo64, int shift,
                                                int64_t base, bool cut, int64_t wbase, int64_t excess, int slot_tie,
                                                const int64_t* ids, int64_t* out, SelCtl* ctl, CountShared& sh,
                                                int64_t* oslot) {
    for (int i = threadIdx.x; i < kSelBins; i += blockDim.x) sh.hist[i] = 0;
    if (threadIdx.x == 0) sh.tie = 0;
    __syncthreads();
    constexpr int U = 4;  // records per thread per round, loads first
    for (int i0 = threadIdx.x; i0 < n; i0 += U * blockDim.x) {
        uint32_t bin[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int i = i0 + u * blockDim.x;
            bin[u] = i < n ? static_cast<uint32_t>(bucket_offset(src[i], pg, lo64, shift) >> 32) : kSelBins;
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (bin[u] < kSelBins) atomicAdd(&sh.hist[bin[u]], 1u);
    }
    __syncthreads();
    {  // exclusive scan of the bins
        constexpr int per = kSelBins / kSelSortThreads;
        uint32_t v[per], t = 0;
#pragma unroll
        for (int q = 0; q < per; ++q) t += (v[q] = sh.hist[per * threadIdx.x + q]);
        int64_t run = block_excl_scan(static_cast<int64_t>(t), sh.wtot, &sh.total);
#pragma unroll
        for (int q = 0; q < per; ++q) {
            sh.hist[per * threadIdx.x + q] = static_cast<uint32_t>(run);
            run += v[q];
        }
    }
    __syncthreads();
    for (int i0 = threadIdx.x; i0 < n; i0 += U * blockDim.x) {
        uint64_t o[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int i = i0 + u * blockDim.x;
            o[u] = i < n ? bucket_offset(src[i], pg, lo64, shift) : 0ull;  // second read: L1 / L2
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int i = i0 + u * blockDim.x;
            if (i >= n) continue;
            const uint32_t k = static_cast<uint32_t>(o[u] >> 32);
            const uint32_t at = atomicAdd(&sh.hist[k], 1u);
            sh.sidx[at] = static_cast<uint16_t>(i);
            sh.sbin[at] = static_cast<uint16_t>(k);
            sh.ssub[at] = static_cast<uint32_t>(o[u]);
        }
    }
    __syncthreads();
    for (int r = threadIdx.x; r + 1 < n; r += blockDim.x) {
        if ((r == 0 || sh.sbin[r - 1] != sh.sbin[r]) && sh.sbin[r + 1] == sh.sbin[r]) {
            int e = r + 2;
            while (e < n && sh.sbin[e] == sh.sbin[r] && e - r <= kSelRunMax) ++e;
            if (e - r > kSelRunMax) {
                sh.tie = 1;
            } else {
                for (int x = r + 1; x < e; ++x) {  // insertion sort by (sub-key, full key)
                    const uint16_t v = sh.sidx[x];
                    const uint32_t kv = sh.ssub[x];
                    int y = x - 1;
                    while (y >= r && (sh.ssub[y] > kv || (sh.ssub[y] == kv && rec_less(src[v], src[sh.sidx[y]])))) {
                        sh.sidx[y + 1] = sh.sidx[y];
                        sh.ssub[y + 1] = sh.ssub[y];
                        --y;
                    }
                    sh.sidx[y + 1] = v;
                    sh.ssub[y + 1] = kv;
                }
            }
        }
    }
    __syncthreads();
    if (sh.tie) return false;
    uint16_t idx[IPT];
#pragma unroll
    for (int j = 0; j < IPT; ++j) {
        const int r = threadIdx.x * IPT + j;
        idx[j] = r < n ? sh.sidx[r] : static_cast<uint16_t>(0);
    }
    bucket_emit<IPT>([&](int i) { return src[i]; }, idx, n, base, cut, wbase, excess, slot_tie, ids, out, ctl, sh,
                     oslot);
    return true;
}

__global__ void __launch_bounds__(kSelSortThreads) sel_sort_kernel(SelCtl* ctl, int64_t excess, int slot_tie,
                                                                  const int64_t* ids, const uint32_t* spl,
                                                                  const SelRec* rec2, const int64_t* boff,
                                                                  const unsigned long long* bcnt, int32_t* big,
                                                                  int64_t* out, int cap, int64_t* oslot) {
    pdl_wait();
    pdl_trigger();
    extern __shared__ uint64_t sel_smem[];
    CountShared& sh = *reinterpret_cast<CountShared*>(sel_smem);
    if (ctl->retry) return;
    const int cutb = ctl->cutb, nb = ctl->nb;
    const int64_t wbase = ctl->wbase;
    uint64_t ga[3], go[3];
    ctl_and_or(ctl, ga, go);
    const int pg = first_varying(ga, go);
    const uint64_t wmin = ctl->wmin, wmax = ctl->wmax;
    __shared__ int next_b;
    for (;;) {
        // buckets from a queue (the cut bucket first: its scan is the longest)
        if (threadIdx.x == 0) {
            const int t = atomicAdd(&ctl->bnext, 1);
            next_b = t == 0 ? cutb : (t <= cutb ? t - 1 : cutb + 1);
        }
        __syncthreads();
        const int b = next_b;
        __syncthreads();
        if (b > cutb) break;
        const int64_t n = static_cast<int64_t>(bcnt[b]);
        const int64_t base = boff[b];
        if (n == 0) {
            if (b == cutb && threadIdx.x == 0) ctl->V = base;
            continue;
        }
        bool ok = false;
        if (n <= cap) {
            // the bucket's 64-bit windows lie in [wlo << 32, whi << 32 | ~0],
            // clipped to the records' own range (the end buckets are open)
            uint64_t lo64 = b == 0 ? 0ull : static_cast<uint64_t>(spl[b - 1] + 1u) << 32;
            uint64_t hi64 = b == nb - 1 ? ~0ull : (static_cast<uint64_t>(spl[b]) << 32) | 0xffffffffull;
            lo64 = lo64 > wmin ? lo64 : wmin;
            hi64 = hi64 < wmax ? hi64 : wmax;
            if (hi64 < lo64) hi64 = lo64;
            const uint64_t width = hi64 - lo64;
            const int bits = width ? 64 - __clzll(width) : 0;
            const int shift = bits > 44 ? bits - 44 : 0;
            if (n <= 4 * kSelSortThreads)
                ok = count_sort_emit<4>(rec2 + base, static_cast<int>(n), pg, lo64, shift, base, b == cutb, wbase,
                                        excess, slot_tie, ids, out, ctl, sh, oslot);
            else
                ok = count_sort_emit<12>(rec2 + base, static_cast<int>(n), pg, lo64, shift, base, b == cutb, wbase,
                                         excess, slot_tie, ids, out, ctl, sh, oslot);
        }
        if (!ok && threadIdx.x == 0) big[atomicAdd(&ctl->nbig, 1)] = b;
        __syncthreads();
    }
}

// ------------------------------------------------------------- 8 big sort
// One CTA per bucket the window sort could not finish (above the cap, or
// tied windows): chunks radix-sorted on the full key into `tmp`,
// then pairwise merges along merge paths (ping-pong between tmp and rec2),
// then the same emission over the sorted run in chunks.
__global__ void __launch_bounds__(kSelSortThreads) sel_big_kernel(SelCtl* ctl, int64_t excess, int slot_tie,
                                                                 const int64_t* ids, SelRec* rec2, SelRec* tmp,
                                                                 const int64_t* boff,
                                                                 const unsigned long long* bcnt,
                                                                 const int32_t* big, int64_t* out, int cap,
                                                                 int64_t* oslot) {
    pdl_wait();
    pdl_trigger();
    extern __shared__ uint64_t sel_smem[];
    BucketShared& sh = *reinterpret_cast<BucketShared*>(sel_smem);
    if (ctl->retry) return;
    const int nbig = ctl->nbig;
    const int cutb = ctl->cutb;
    for (int e = blockIdx.x; e < nbig; e += gridDim.x) {
        const int b = big[e];
        const int64_t n = static_cast<int64_t>(bcnt[b]);
        const int64_t base = boff[b];
        SelRec* a = rec2 + base;
        SelRec* t = tmp + base;
        const int chunk = cap < kSelFullCap ? cap : kSelFullCap;
        for (int64_t c0 = 0; c0 < n; c0 += chunk) {
            const int m = static_cast<int>(i64min(chunk, n - c0));
            uint16_t idx[8];
            bucket_sort<8>(a + c0, m, sh, idx);
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const int rk = threadIdx.x * 8 + j;
                if (rk < m) t[c0 + rk] = a[c0 + idx[j]];
            }
            __syncthreads();
        }
        SelRec* src = t;
        SelRec* dst = a;
        for (int64_t L = chunk; L < n; L <<= 1) {
            for (int64_t i = 0; i < n; i += 2 * L) {
                const SelRec* A = src + i;
                const int64_t na = i64min(L, n - i);
                const SelRec* B = A + na;
                const int64_t nbb = i64max(0, i64min(L, n - i - na));
                const int64_t tot = na + nbb;
                const int64_t per = (tot + blockDim.x - 1) / blockDim.x;
                const int64_t d0 = i64min(tot, per * threadIdx.x);
                const int64_t d1 = i64min(tot, d0 + per);
                int64_t lo = i64max(0, d0 - nbb), hi = i64min(d0, na);
                while (lo < hi) {  // merge path: first a with A[a] after B[d0 - 1 - a]
                    const int64_t mid = (lo + hi) >> 1;
                    if (rec_less(A[mid], B[d0 - 1 - mid]))
                        lo = mid + 1;
                    else
                        hi = mid;
                }
                int64_t ia = lo, ib = d0 - lo;
                for (int64_t d = d0; d < d1; ++d) {
                    const bool take_a = ib >= nbb || (ia < na && rec_less(A[ia], B[ib]));
                    dst[i + d] = take_a ? A[ia++] : B[ib++];
                }
            }
            __syncthreads();
            SelRec* x = src;
            src = dst;
            dst = x;
        }
        int64_t wb = ctl->wbase;
        for (int64_t c0 = 0; c0 < n; c0 += kSelFullCap) {
            const int m = static_cast<int>(i64min(kSelFullCap, n - c0));
            uint16_t idx[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) idx[j] = static_cast<uint16_t>(threadIdx.x * 8 + j);
            const SelRec* chunk = src + c0;
            const bool found = bucket_emit<8>([&](int i) { return chunk[i]; }, idx, m, base + c0, b == cutb, wb,
                                              excess, slot_tie, ids, out, ctl, sh, oslot);
            if (b == cutb) {
                if (found) break;
                wb += sh.total;
                __syncthreads();
            }
        }
        __syncthreads();
    }
}

}  // namespace sine
