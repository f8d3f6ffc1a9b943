// libsine_b200 -- C ABI over the device SE store, the stage-1 kernels and the
// eviction kernels.  See include/sine_b200.h for the contract and the
// reference interfaces each entry point replaces.
//
// Device store (one per handle / GPU), structure-of-arrays in HBM:
//   rows32 [cap][stride32] fp32     scan rows, exact mode   (128-B padded)
//   rows16 [cap][stride16] bf16     scan rows, fast mode    (128-B padded)
//   rows64 [cap][dim]      fp64     master copy: fp64 re-rank + snapshots
//                                   (pinned, device-mapped host memory with
//                                   SINE_STORE_F64_HOST)
//   ids    [cap] int64,  valid bitmap [cap/32] uint32
//   LCFU columns (engine mode): log_freq/log_cost/log_lat/log_stat,
//     created_at, expiration_time, last_access (fp64), frequency,
//     size_tokens (int64)
// Slots are append-only; removal clears the validity bit (tombstone) and
// the store is compacted (order preserving) once tombstones exceed a
// quarter of the live rows, mirroring the reference graph index's rebuild
// rule (index.py:271).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <set>
#include <string>
#include <unordered_map>
#include <unordered_set>
#include <vector>

#include <cudaTypedefs.h>

#include "../../include/sine_b200.h"
#include "common.cuh"
#include "embed.cuh"
#include "evict.cuh"
#include "hexio.cuh"
#include "merge.cuh"
#include "scan.cuh"
#include "select.cuh"
#include "umma.cuh"

using namespace sine;

namespace {

thread_local std::string g_err;

struct Fail {
    int code;
};

[[noreturn]] void fail(int code, const std::string& msg) {
    g_err = msg;
    throw Fail{code};
}

#define CK(x)                                                                                     \
    do {                                                                                          \
        cudaError_t e_ = (x);                                                                     \
        if (e_ != cudaSuccess)                                                                    \
            fail(e_ == cudaErrorMemoryAllocation ? SINE_ENOMEM : SINE_ECUDA,                       \
                 std::string(#x) + ": " + cudaGetErrorString(e_));                                \
    } while (0)

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return SINE_OK;
    } catch (const Fail& e) {
        return e.code;
    } catch (const std::bad_alloc&) {
        g_err = "host allocation failed";
        return SINE_ENOMEM;
    } catch (const std::exception& e) {
        g_err = e.what();
        return SINE_ECUDA;
    }
}

template <typename T>
struct DevBuf {
    T* p = nullptr;
    size_t n = 0;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    DevBuf(DevBuf&& o) noexcept : p(o.p), n(o.n) { o.p = nullptr, o.n = 0; }
    ~DevBuf() { release(); }
    void ensure(size_t want) {
        if (want <= n) return;
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
        CK(cudaMalloc(&p, want * sizeof(T)));
        n = want;
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
    }
};

// a device bitmap owned by shared tickets (freed with the last owner)
struct DevBitmap {
    uint32_t* p = nullptr;
    DevBitmap() = default;
    DevBitmap(const DevBitmap&) = delete;
    DevBitmap& operator=(const DevBitmap&) = delete;
    ~DevBitmap() {
        if (p) cudaFree(p);
    }
};

template <typename T>
struct HostBuf {
    T* p = nullptr;
    size_t n = 0;
    HostBuf() = default;
    HostBuf(const HostBuf&) = delete;
    HostBuf& operator=(const HostBuf&) = delete;
    HostBuf(HostBuf&& o) noexcept : p(o.p), n(o.n) { o.p = nullptr, o.n = 0; }
    ~HostBuf() { release(); }
    void ensure(size_t want) {
        if (want <= n) return;
        if (p) cudaFreeHost(p);
        p = nullptr;
        n = 0;
        CK(cudaMallocHost(&p, want * sizeof(T)));
        n = want;
    }
    void release() {
        if (p) cudaFreeHost(p);
        p = nullptr;
        n = 0;
    }
};

}  // namespace

struct sine_index {
    int device = 0;
    int num_sms = 148;
    int64_t dim = 0;
    uint32_t flags = 0;
    int64_t stride32 = 0, stride16 = 0;  // elements per row
    int64_t cap = 0, nslots = 0, nlive = 0;
    bool ids_ascending = true;
    int64_t max_id = INT64_MIN;

    float* rows32 = nullptr;
    __nv_bfloat16* rows16 = nullptr;
    double* rows64 = nullptr;
    int64_t* ids = nullptr;
    uint32_t* valid = nullptr;
    double *lf = nullptr, *lc = nullptr, *ll = nullptr, *ls = nullptr;
    double *created = nullptr, *expiration = nullptr, *last_access = nullptr;
    int64_t *freq = nullptr, *size = nullptr;

    std::vector<int64_t> ids_h;   // by slot
    std::vector<uint8_t> live_h;  // by slot
    std::unordered_map<int64_t, int64_t> pos;
    // the reference's id order (ExactCosineIndex._ids, index.py:71-92):
    // appended on insert, swap-last on removal.  ids() and the snapshot
    // follow it, so they are byte-identical to the reference after any
    // sequence of inserts and removals.
    std::vector<int64_t> order_slot;  // position -> slot
    std::vector<int64_t> order_pos;   // slot -> position (-1 once removed)
    // pending order ops, replayed only when the order is read (ids(),
    // snapshots, compaction): s >= 0 removes slot s (swap-last), s < 0
    // appends slot ~s.  Removal bursts (TTL purge, eviction) then cost one
    // log entry per row.
    std::vector<int64_t> order_log;

    cudaStream_t stream = nullptr;
    cudaEvent_t ev[6] = {};
    // Query workspaces (q64, lkey/lslot/ln, gbound, qbf, cert, ...) and the
    // store itself are used by kernels on the handle's stream and on caller
    // streams (sine_query_device*): every entry point orders its work after
    // the previous user's (ws_acquire), so a later call cannot overwrite a
    // workspace, or reallocate rows, under kernels still running elsewhere.
    cudaStream_t ws_stream = nullptr;  // last stream that enqueued store/workspace work
    cudaEvent_t ws_ev = nullptr;       // recorded after that work when it was a caller stream
    bool timing = false;
    uint32_t ev_mask = 0;  // ev[i] recorded since the last read
    // accumulated per-kernel device time (CUDA events on the launch stream)
    struct Timed {
        cudaEvent_t a = nullptr, b = nullptr;
        int kind = 0;
    };
    std::vector<Timed> tpool;
    size_t tused = 0;
    float t_scan = 0.f, t_merge = 0.f, t_evict = 0.f;
    int64_t launches = 0;
    std::mutex mu;

    // workspaces
    DevBuf<double> q64;
    DevBuf<uint32_t> lkey;
    DevBuf<int32_t> lslot, ln;
    DevBuf<int64_t> o_ids;
    DevBuf<double> o_sims;
    DevBuf<int32_t> o_cnt;
    DevBuf<uint8_t> cert;         // per-query exactness certificates
    uint8_t* cert_out = nullptr;  // sine_query_device_cert: certificates go straight to the caller
    int64_t uncertified = 0;      // queries re-run by the last certify pass
    float cur_thr0 = 0.f;         // admission floor of the running query
    double cur_err = 0.0;         // its filter error bound
    DevBuf<int32_t> vslots, scratch_i32;  // expiry: slot list, per-block counts
    DevBuf<int64_t> vids;                 // expired ids / victim ids
    DevBuf<int64_t> exp_off;
    DevBuf<uint32_t> gbound;        // chip-wide admission bounds of the running launch
    DevBuf<uint32_t> gcnt;          // tiled GEMM: candidates per query + overflow counter
    DevBuf<uint32_t> tmax;          // sample pass: per (tile, query) max score keys
    int64_t gemm_overflows = 0;     // GEMM launches re-run on the list-keeping kernels
    // victim selection (select.cuh): records below the sampled bound, the
    // same in bucket order, bucket of each record, splitters, per-bucket
    // count / size, offsets, cursors, oversized buckets, control block
    DevBuf<SelRec> srec, srec2, ssamp;
    DevBuf<uint16_t> sbid;
    DevBuf<uint32_t> sspl, stab;
    DevBuf<unsigned long long> sbcnt;
    DevBuf<int64_t> sboff;
    DevBuf<uint32_t> sbcur;
    DevBuf<int32_t> sbig;
    DevBuf<SelCtl> sctl;
    DevBuf<int64_t> sslot;  // victim slots (sine_evict on slot-ordered stores)
    int sel_cap = kSelCap;  // records sorted in smem per CTA (sine_set_select_cap lowers it in tests)
    HostBuf<SelCtl> sctl_h;
    DevBuf<__nv_bfloat16> qbf;          // umma path: bf16 queries
    HostBuf<unsigned long long> n_h;
    HostBuf<int32_t> cnt_h;
    HostBuf<uint8_t> cert_h;
    HostBuf<int64_t> ids_zc;  // sine_query's mapped result staging
    HostBuf<double> sims_zc;
    HostBuf<int32_t> cnt_zc;
    struct Ticket {
        cudaEvent_t done = nullptr;
        HostBuf<uint8_t> cert;
        // pinned (UVA-mapped) result staging the merge kernel writes straight
        // into: no device->host copies on the stream between batches
        HostBuf<int64_t> sids;
        HostBuf<double> ssims;
        HostBuf<int32_t> scnt;
        bool zero_copy = false;
        bool busy = false, certify = false;
        int64_t nslots = 0;                            // store slots at submission
        std::shared_ptr<DevBitmap> valid_snap;  // bitmap at submission (set on the first later removal)
        int64_t B = 0;
        int k = 0;
        double min_sim = 0.0;
        uint32_t mode = 0;
        const double* q = nullptr;
        int64_t* ids = nullptr;
        double* sims = nullptr;
        int32_t* counts = nullptr;
    };
    std::vector<Ticket> tickets;
    // submit-time snapshots for certificate re-runs: the store is append-only
    // between compactions, so a ticket's snapshot is (its nslots, the
    // validity bitmap before the first tombstone written after it).  The
    // bitmap is copied lazily -- only when a removal lands while certified
    // tickets are in flight -- and compaction waits until they drain.
    int64_t snap_nslots = -1;            // scan override during a re-run
    const uint32_t* snap_valid = nullptr;
    bool compact_pending = false;
};

namespace {

// programmatic dependent launch between query prep -> scan -> merge
// (SINE_NO_PDL=1 turns it off, for A/B timing)
bool pdl_enabled() {
    static const bool on = getenv("SINE_NO_PDL") == nullptr;
    return on;
}

// Launch with programmatic dependent launch (the kernel calls pdl_wait()
// before reading its predecessor's output): the launch latency of a chain
// of short dependent kernels overlaps the predecessor's tail.
template <typename... KArgs, typename... Args>
void launch_pdl(void (*kern)(KArgs...), int grid, int block, size_t smem, cudaStream_t st, Args&&... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    CK(cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...));
}

int64_t round_up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }

void ws_acquire(sine_index* h, cudaStream_t st) {
    if (h->ws_stream && h->ws_stream != st) {
        if (h->ws_stream == h->stream) CK(cudaEventRecord(h->ws_ev, h->stream));
        CK(cudaStreamWaitEvent(st, h->ws_ev, 0));  // caller-stream users recorded ws_ev on release
    }
    h->ws_stream = st;
}

void ws_release(sine_index* h, cudaStream_t st) {
    if (st != h->stream) CK(cudaEventRecord(h->ws_ev, st));  // the caller's stream may not outlive us
}

// Opt a kernel in to > 48 KB of dynamic shared memory.  The attribute is
// per device (per context), so it is remembered per (kernel, device): an
// index on device 1 created after one on device 0 opts in again.
void smem_optin(const void* fn, int bytes) {
    static std::mutex mu;
    static std::set<std::pair<const void*, int>> done;
    int dev = 0;
    CK(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> g(mu);
    if (done.count({fn, dev})) return;
    CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    done.insert({fn, dev});
}

__global__ void convert_rows_kernel(const double* __restrict__ src, int64_t n, int64_t dim, float* rows32,
                                    int64_t stride32, __nv_bfloat16* rows16, int64_t stride16) {
    const int64_t width = max(stride32, stride16);
    const int64_t total = n * width;
    for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < total;
         t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t r = t / width, c = t - r * width;
        const double v = c < dim ? src[r * dim + c] : 0.0;
        if (rows32 && c < stride32) rows32[r * stride32 + c] = static_cast<float>(v);
        if (rows16 && c < stride16) rows16[r * stride16 + c] = __float2bfloat16_rn(static_cast<float>(v));
    }
}

__global__ void set_bits_kernel(uint32_t* valid, const int64_t* slots, int64_t n, int set) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t s = slots[i];
        const uint32_t bit = 1u << (s & 31);
        if (set)
            atomicOr(valid + (s >> 5), bit);
        else
            atomicAnd(valid + (s >> 5), ~bit);
    }
}

__global__ void set_bits32_kernel(uint32_t* valid, const int32_t* slots, int64_t n) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t s = slots[i];
        atomicAnd(valid + (s >> 5), ~(1u << (s & 31)));
    }
}

__global__ void set_range_kernel(uint32_t* valid, int64_t s0, int64_t n) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t s = s0 + i;
        atomicOr(valid + (s >> 5), 1u << (s & 31));
    }
}

template <typename T>
__global__ void gather_rows_kernel(const T* __restrict__ src, T* __restrict__ dst, const int64_t* from,
                                   int64_t n, int64_t width) {
    const int64_t total = n * width;
    for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < total;
         t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t r = t / width, c = t - r * width;
        dst[r * width + c] = src[from[r] * width + c];
    }
}

__global__ void gather_rows64_kernel(const double* rows64, const int64_t* slots, int64_t n, int64_t dim,
                                     double* out) {
    const int64_t total = n * dim;
    for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < total;
         t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t r = t / dim, c = t - r * dim;
        out[t] = rows64[slots[r] * dim + c];
    }
}

__global__ void scatter_meta_kernel(const int64_t* slots, int64_t n, const double* lfv, const int64_t* fv,
                                    const double* lav, double* lf, int64_t* freq, double* la) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t s = slots[i];
        lf[s] = lfv[i];
        freq[s] = fv[i];
        la[s] = lav[i];
    }
}

int grid_for(int64_t work, int threads, int num_sms) {
    const int64_t g = (work + threads - 1) / threads;
    return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(g, 8ll * num_sms)));
}

template <typename T>
void alloc_col(T*& p, int64_t n) {
    CK(cudaMalloc(&p, std::max<int64_t>(n, 1) * sizeof(T)));
}

// The fp64 master rows: HBM, or pinned host memory mapped into the device
// address space (SINE_STORE_F64_HOST; UVA: one pointer for host and device).
double* alloc_master(const sine_index* h, int64_t elems) {
    double* p = nullptr;
    if (h->flags & SINE_STORE_F64_HOST) {
        CK(cudaHostAlloc(&p, std::max<int64_t>(elems, 1) * sizeof(double), cudaHostAllocMapped | cudaHostAllocPortable));
    } else {
        CK(cudaMalloc(&p, std::max<int64_t>(elems, 1) * sizeof(double)));
    }
    return p;
}
void free_master(const sine_index* h, double* p) {
    if (!p) return;
    if (h->flags & SINE_STORE_F64_HOST)
        cudaFreeHost(p);
    else
        cudaFree(p);
}

void grow(sine_index* h, int64_t want) {
    if (want <= h->cap) return;
    int64_t nc = std::max<int64_t>(want, std::max<int64_t>(1024, h->cap * 2));
    nc = round_up(nc, 128);  // whole 128-slot groups: TMA tiles of the columns and validity words
    auto move = [&](auto*& col, int64_t width) {
        using T = std::remove_reference_t<decltype(*col)>;
        if (!col && width >= 0) return;
        T* nw = nullptr;
        CK(cudaMalloc(&nw, nc * width * sizeof(T)));
        if (h->nslots)
            CK(cudaMemcpyAsync(nw, col, h->nslots * width * sizeof(T), cudaMemcpyDeviceToDevice, h->stream));
        CK(cudaStreamSynchronize(h->stream));
        CK(cudaFree(col));
        col = nw;
    };
    if (h->cap == 0) {
        if (h->flags & SINE_STORE_F32) alloc_col(h->rows32, nc * h->stride32);
        if (h->flags & SINE_STORE_BF16) alloc_col(h->rows16, nc * h->stride16);
        h->rows64 = alloc_master(h, nc * h->dim);
        alloc_col(h->ids, nc);
        alloc_col(h->valid, nc / 32);
        CK(cudaMemsetAsync(h->valid, 0, nc / 32 * sizeof(uint32_t), h->stream));
        if (h->flags & SINE_STORE_META) {
            alloc_col(h->lf, nc), alloc_col(h->lc, nc), alloc_col(h->ll, nc), alloc_col(h->ls, nc);
            alloc_col(h->created, nc), alloc_col(h->expiration, nc), alloc_col(h->last_access, nc);
            alloc_col(h->freq, nc), alloc_col(h->size, nc);
        }
    } else {
        move(h->rows32, h->stride32);
        move(h->rows16, h->stride16);
        {
            double* nw = alloc_master(h, nc * h->dim);
            if (h->nslots)
                CK(cudaMemcpyAsync(nw, h->rows64, h->nslots * h->dim * sizeof(double), cudaMemcpyDefault, h->stream));
            CK(cudaStreamSynchronize(h->stream));
            free_master(h, h->rows64);
            h->rows64 = nw;
        }
        move(h->ids, 1);
        {
            uint32_t* nv = nullptr;
            CK(cudaMalloc(&nv, nc / 32 * sizeof(uint32_t)));
            CK(cudaMemsetAsync(nv, 0, nc / 32 * sizeof(uint32_t), h->stream));
            CK(cudaMemcpyAsync(nv, h->valid, h->cap / 32 * sizeof(uint32_t), cudaMemcpyDeviceToDevice, h->stream));
            CK(cudaStreamSynchronize(h->stream));
            CK(cudaFree(h->valid));
            h->valid = nv;
        }
        if (h->flags & SINE_STORE_META) {
            move(h->lf, 1), move(h->lc, 1), move(h->ll, 1), move(h->ls, 1);
            move(h->created, 1), move(h->expiration, 1), move(h->last_access, 1);
            move(h->freq, 1), move(h->size, 1);
        }
    }
    h->cap = nc;
    h->ids_h.reserve(nc);
    h->live_h.reserve(nc);
}

void check_rows_host(const sine_index* h, int64_t n, const double* rows) {
    for (int64_t i = 0; i < n; ++i) {
        const double* r = rows + i * h->dim;
        double ss = 0.0;
        for (int64_t j = 0; j < h->dim; ++j) ss += r[j] * r[j];
        const double nrm = std::sqrt(ss);
        if (std::fabs(nrm - 1.0) > 1e-6) {
            char b[128];
            snprintf(b, sizeof b, "vector is not L2-normalized (norm=%.8f)", nrm);
            fail(SINE_ENORM, b);
        }
    }
}

// id -> live slot.  Ids appended in ascending order (the engine's monotone
// element ids) are found by binary search over the slot-ordered id column;
// otherwise through the hash map.
int64_t find_slot(const sine_index* h, int64_t id) {
    if (h->ids_ascending) {
        auto it = std::lower_bound(h->ids_h.begin(), h->ids_h.end(), id);
        if (it == h->ids_h.end() || *it != id) return -1;
        const int64_t s = it - h->ids_h.begin();
        return h->live_h[s] ? s : -1;
    }
    auto it = h->pos.find(id);
    return it == h->pos.end() ? -1 : it->second;
}

void check_new_ids(const sine_index* h, int64_t n, const int64_t* ids) {
    // fast path: a strictly ascending batch above every stored id
    bool asc = h->nslots == 0 || ids[0] > h->max_id;
    for (int64_t i = 1; asc && i < n; ++i) asc = ids[i] > ids[i - 1];
    if (asc) return;
    std::unordered_set<int64_t> seen;
    seen.reserve(n * 2);
    for (int64_t i = 0; i < n; ++i) {
        if (find_slot(h, ids[i]) >= 0 || !seen.insert(ids[i]).second)
            fail(SINE_EDUP, "duplicate id " + std::to_string(ids[i]));
    }
}

// id -> slot over every slot in the host tables (including a batch being
// appended, whose slots are not yet counted in nslots)
void build_pos_map(sine_index* h) {
    const int64_t n = static_cast<int64_t>(h->ids_h.size());
    h->pos.clear();
    h->pos.reserve(n * 2);
    for (int64_t s = 0; s < n; ++s)
        if (h->live_h[s]) h->pos[h->ids_h[s]] = s;
}

void copy_meta(sine_index* h, int64_t s0, int64_t n, const sine_meta_cols_t* m) {
    if (!(h->flags & SINE_STORE_META)) return;
    if (!m) fail(SINE_EINVAL, "metadata columns required (index created with SINE_STORE_META)");
    auto cp = [&](auto* dst, const auto* src) {
        if (!src) fail(SINE_EINVAL, "null metadata column");
        CK(cudaMemcpyAsync(dst + s0, src, n * sizeof(*src), cudaMemcpyHostToDevice, h->stream));
    };
    cp(h->lf, m->log_freq), cp(h->lc, m->log_cost), cp(h->ll, m->log_lat), cp(h->ls, m->log_stat);
    cp(h->freq, m->frequency), cp(h->size, m->size_tokens), cp(h->created, m->created_at);
    cp(h->expiration, m->expiration_time), cp(h->last_access, m->last_access);
}

void order_append(sine_index* h, int64_t slot);
void order_removed(sine_index* h, int64_t slot);
void order_flush(sine_index* h);

void append(sine_index* h, int64_t n, const int64_t* ids, const double* rows, bool rows_on_device,
            const sine_meta_cols_t* meta) {
    grow(h, h->nslots + n);
    const int64_t s0 = h->nslots;
    const cudaMemcpyKind kind = rows_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
    CK(cudaMemcpyAsync(h->rows64 + s0 * h->dim, rows, n * h->dim * sizeof(double),
                       (h->flags & SINE_STORE_F64_HOST) ? cudaMemcpyDefault : kind, h->stream));
    const int64_t width = std::max(h->rows32 ? h->stride32 : 0, h->rows16 ? h->stride16 : 0);
    if (width) {
        convert_rows_kernel<<<grid_for(n * width, 256, h->num_sms), 256, 0, h->stream>>>(
            h->rows64 + s0 * h->dim, n, h->dim, h->rows32 ? h->rows32 + s0 * h->stride32 : nullptr,
            h->stride32, h->rows16 ? h->rows16 + s0 * h->stride16 : nullptr, h->stride16);
        ++h->launches;
    }
    CK(cudaMemcpyAsync(h->ids + s0, ids, n * sizeof(int64_t), cudaMemcpyHostToDevice, h->stream));
    copy_meta(h, s0, n, meta);
    set_range_kernel<<<grid_for(n, 256, h->num_sms), 256, 0, h->stream>>>(h->valid, s0, n);
    ++h->launches;
    CK(cudaGetLastError());
    const bool was_ascending = h->ids_ascending;
    for (int64_t i = 0; i < n; ++i) {
        order_append(h, s0 + i);
        h->ids_h.push_back(ids[i]);
        h->live_h.push_back(1);
        if (ids[i] <= h->max_id) h->ids_ascending = false;
        h->max_id = std::max(h->max_id, ids[i]);
    }
    if (!h->ids_ascending) {
        if (was_ascending) {
            build_pos_map(h);
        } else {
            for (int64_t i = 0; i < n; ++i) h->pos[ids[i]] = s0 + i;
        }
    }
    h->nslots += n;
    h->nlive += n;
    CK(cudaStreamSynchronize(h->stream));  // caller buffers may be released
}

void compact(sine_index* h) {
    order_flush(h);
    std::vector<int64_t> from;
    from.reserve(h->nlive);
    for (int64_t s = 0; s < h->nslots; ++s)
        if (h->live_h[s]) from.push_back(s);
    const int64_t n = static_cast<int64_t>(from.size());
    DevBuf<int64_t> dfrom;
    dfrom.ensure(std::max<int64_t>(n, 1));
    CK(cudaMemcpyAsync(dfrom.p, from.data(), n * sizeof(int64_t), cudaMemcpyHostToDevice, h->stream));
    auto redo = [&](auto*& col, int64_t width) {
        using T = std::remove_reference_t<decltype(*col)>;
        if (!col) return;
        T* nw = nullptr;
        CK(cudaMalloc(&nw, h->cap * width * sizeof(T)));
        if (n)
            gather_rows_kernel<T><<<grid_for(n * width, 256, h->num_sms), 256, 0, h->stream>>>(col, nw, dfrom.p, n,
                                                                                               width);
        ++h->launches;
        CK(cudaStreamSynchronize(h->stream));
        CK(cudaFree(col));
        col = nw;
    };
    redo(h->rows32, h->stride32);
    redo(h->rows16, h->stride16);
    if (h->flags & SINE_STORE_F64_HOST) {  // host-resident master rows: compact on the host
        CK(cudaStreamSynchronize(h->stream));
        for (int64_t i = 0; i < n; ++i)
            if (from[i] != i) std::memmove(h->rows64 + i * h->dim, h->rows64 + from[i] * h->dim, h->dim * sizeof(double));
    } else {
        redo(h->rows64, h->dim);
    }
    redo(h->ids, 1);
    redo(h->lf, 1), redo(h->lc, 1), redo(h->ll, 1), redo(h->ls, 1);
    redo(h->created, 1), redo(h->expiration, 1), redo(h->last_access, 1);
    redo(h->freq, 1), redo(h->size, 1);
    CK(cudaMemsetAsync(h->valid, 0, h->cap / 32 * sizeof(uint32_t), h->stream));
    if (n) set_range_kernel<<<grid_for(n, 256, h->num_sms), 256, 0, h->stream>>>(h->valid, 0, n);
    ++h->launches;
    CK(cudaStreamSynchronize(h->stream));
    std::vector<int64_t> nid(n);
    for (int64_t i = 0; i < n; ++i) nid[i] = h->ids_h[from[i]];
    {  // slots renumbered in order: the reference order follows the rows
        std::vector<int64_t> newslot(h->nslots, -1);
        for (int64_t i = 0; i < n; ++i) newslot[from[i]] = i;
        h->order_pos.assign(n, -1);
        for (size_t p = 0; p < h->order_slot.size(); ++p) {
            h->order_slot[p] = newslot[h->order_slot[p]];
            h->order_pos[h->order_slot[p]] = static_cast<int64_t>(p);
        }
    }
    h->ids_h.swap(nid);
    h->live_h.assign(n, 1);
    h->nslots = n;
    if (!h->ids_ascending) build_pos_map(h);
    dfrom.release();
}

// ------------------------------------------------------------ query pipeline

struct ScanCfg {
    int C, CPW, CW, G, U, R, NQmax;
    int64_t row_bytes;
};

int unroll_for(int NQ) { return NQ == 1 ? 8 : NQ == 2 ? 4 : NQ == 4 ? 2 : 1; }

// Launch geometry of the streaming scan for a query group of size NQ
// (must agree with ScanWarps / ScanUnroll in scan.cuh).
ScanCfg scan_cfg(const sine_index* h, bool bf16, int NQ) {
    ScanCfg c{};
    c.row_bytes = bf16 ? h->stride16 * 2 : h->stride32 * 4;
    c.C = static_cast<int>((c.row_bytes + 511) / 512);
    c.CPW = c.C <= 8 ? 1 : 2;
    if (c.C > 16) fail(SINE_EINVAL, "dimension too large for the streaming scan (max 2048 fp32 / 4096 bf16)");
    c.CW = (c.C + c.CPW - 1) / c.CPW;
    const int epl = bf16 ? 8 : 4;
    c.NQmax = std::min(16, 64 / (epl * c.CPW));
    if (NQ > 0) {
        const int maxW = NQ >= 8 ? 8 : 16;
        const int U = unroll_for(NQ);
        c.G = std::max(1, maxW / c.CW);
        while (c.G > 1 && c.G * U > 64) --c.G;
        // ~48 KB of rows per stage, at least U rows per warp, at most 64 rows
        const int want = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(64, 49152 / c.row_bytes)));
        int rpw = std::max(U, (want + c.G - 1) / c.G);
        rpw = (rpw + U - 1) / U * U;
        while (rpw > U && c.G * rpw > 64) rpw -= U;
        c.U = rpw;
        c.R = c.G * rpw;
    }
    return c;
}

template <typename RowT, int NQ, int CPW>
void launch_scan_t(const ScanParams& p, int grid, int threads, size_t smem, cudaStream_t st) {
    smem_optin(reinterpret_cast<const void*>(scan_kernel<RowT, NQ, CPW>), 227 * 1024);
    scan_kernel<RowT, NQ, CPW><<<grid, threads, smem, st>>>(p);
}

template <typename RowT, int CPW>
void launch_scan_nq(int NQ, const ScanParams& p, int grid, int threads, size_t smem, cudaStream_t st) {
    switch (NQ) {
        case 1: return launch_scan_t<RowT, 1, CPW>(p, grid, threads, smem, st);
        case 2: return launch_scan_t<RowT, 2, CPW>(p, grid, threads, smem, st);
        case 4: return launch_scan_t<RowT, 4, CPW>(p, grid, threads, smem, st);
        case 8: return launch_scan_t<RowT, 8, CPW>(p, grid, threads, smem, st);
        default:
            if constexpr (sizeof(RowT) == 4 && CPW == 1) return launch_scan_t<RowT, 16, CPW>(p, grid, threads, smem, st);
            fail(SINE_EINVAL, "unsupported query group");
    }
}

void record(sine_index* h, int i, cudaStream_t st) {
    if (h->timing) {
        CK(cudaEventRecord(h->ev[i], st));
        h->ev_mask |= 1u << i;
    }
}

// last_timing's scan / merge split: only the CUDA-core path records the
// three events; the tensor-core paths report through timing_totals
void scan_merge_times(sine_index* h) {
    if ((h->ev_mask & 7u) == 7u) {
        CK(cudaEventElapsedTime(&h->t_scan, h->ev[0], h->ev[1]));
        CK(cudaEventElapsedTime(&h->t_merge, h->ev[1], h->ev[2]));
    }
    h->ev_mask &= ~7u;
}

// kind 0 = scan kernel, 1 = merge kernel, 2 = tensor-core scan
size_t tbegin(sine_index* h, int kind, cudaStream_t st) {
    if (!h->timing) return SIZE_MAX;
    if (h->tused == h->tpool.size()) {
        sine_index::Timed t;
        CK(cudaEventCreate(&t.a));
        CK(cudaEventCreate(&t.b));
        h->tpool.push_back(t);
    }
    auto& t = h->tpool[h->tused];
    t.kind = kind;
    CK(cudaEventRecord(t.a, st));
    return h->tused++;
}
void tend(sine_index* h, size_t i, cudaStream_t st) {
    if (i != SIZE_MAX) CK(cudaEventRecord(h->tpool[i].b, st));
}

// ------------------------------------------------------------ tcgen05 path

PFN_cuTensorMapEncodeTiled_v12000 tmap_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        void* f = nullptr;
        CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q));
        if (q != cudaDriverEntryPointSuccess || !f) fail(SINE_ECUDA, "cuTensorMapEncodeTiled unavailable");
        fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
    }
    return fn;
}

// 2-D K-major map: inner dim = row elements (box = one 128-B swizzle row),
// outer dim = rows (box = 128), SWIZZLE_128B, out-of-bounds rows read as 0.
CUtensorMap encode_kmajor_map(const void* base, bool tf32, int64_t row_elems, int64_t rows, int box_rows) {
    CUtensorMap m;
    const cuuint64_t dims[2] = {static_cast<cuuint64_t>(row_elems), static_cast<cuuint64_t>(rows)};
    const cuuint64_t strides[1] = {static_cast<cuuint64_t>(row_elems * (tf32 ? 4 : 2))};
    const cuuint32_t box[2] = {static_cast<cuuint32_t>(tf32 ? 32 : 64), static_cast<cuuint32_t>(box_rows)};
    const cuuint32_t estr[2] = {1, 1};
    const CUresult r = tmap_encoder()(&m, tf32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                                      const_cast<void*>(base), dims, strides, box, estr,
                                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) fail(SINE_ECUDA, "cuTensorMapEncodeTiled failed: " + std::to_string(static_cast<int>(r)));
    return m;
}

// Encoded maps are reused across calls (the small-batch path launches with
// the same row and query maps every time): a per-thread cache keyed by the
// full map description.
CUtensorMap make_kmajor_map(const void* base, bool tf32, int64_t row_elems, int64_t rows, int box_rows = 128) {
    struct Entry {
        const void* base;
        bool tf32;
        int64_t row_elems, rows;
        int box_rows;
        CUtensorMap map;
    };
    static thread_local Entry cache[8];
    static thread_local int next = 0, used = 0;
    for (int i = 0; i < used; ++i) {
        const Entry& e = cache[i];
        if (e.base == base && e.tf32 == tf32 && e.row_elems == row_elems && e.rows == rows && e.box_rows == box_rows)
            return e.map;
    }
    Entry e{base, tf32, row_elems, rows, box_rows, encode_kmajor_map(base, tf32, row_elems, rows, box_rows)};
    cache[next] = e;
    next = (next + 1) % 8;
    used = std::min(used + 1, 8);
    return e.map;
}

constexpr int kUmmaMinBatch = 1;

bool umma_eligible(const sine_index* h, int64_t B, bool bf16, uint32_t mode, int kp) {
    if (mode & SINE_SCAN_CUDA_CORE) return false;
    if (B < kUmmaMinBatch || kp > kUmmaMaxKp) return false;
    if (!bf16 && !(mode & SINE_RERANK_F64)) return false;  // tf32 products need the fp64 re-rank
    if (h->nslots >= (1ll << 31)) return false;
    return true;
}

void merge_launch(sine_index* h, int ncta, int nq, int kp, const double* q64, int k, double min_sim, bool rerank,
                  int64_t* ids_dev, double* sims_dev, int32_t* counts_dev, cudaStream_t st, int64_t cert_off);

// widest query group of the FFMA helper mode (queries <= this take the CUDA
// cores instead of N = 16 MMAs).  Same box, config B, tau 0.9, ms per batch
// helper mode vs MMAs: fp32 B = 2 0.446 vs 0.514, B = 4 0.524 vs 0.514,
// B = 8 0.806 vs 0.515; bf16 B = 2 0.302 vs 0.267, B = 4 0.438 vs 0.268
// (the widened-query smem reads and FMAs outgrow the halved bf16 tile time).
constexpr int kFfmaMaxQF32 = 2;
constexpr int kFfmaMaxQBF16 = 1;

// widest resident query group (Q <= 96 KB of shared memory), 0 if < 16
int res_nq_max(int64_t row_bytes) {
    const int64_t n = (96 * 1024) / row_bytes;
    return n >= 64 ? 64 : n >= 32 ? 32 : n >= 16 ? 16 : 0;
}

template <int NQ, int CS, int HQ = 0>
int launch_res(const CUtensorMap& qmap, const CUtensorMap& rmap, const ResParams& p, int max_clusters, size_t smem,
               cudaStream_t st) {
    auto kern = umma_res_kernel<NQ, CS, HQ>;
    smem_optin(reinterpret_cast<const void*>(kern), 227 * 1024);
    cudaLaunchConfig_t cfg{};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CS;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.blockDim = dim3(kUmmaThreads + (HQ > 0 ? kUmmaHelperThreads : 0));
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cfg.gridDim = dim3(max_clusters * CS);
    // clusters the GPU can hold at once (persistent grid: one wave); the
    // answer depends only on the kernel, cluster shape and shared memory
    static std::mutex occ_mu;
    static std::unordered_map<size_t, int> occ;
    int active = 0;
    const size_t okey = smem;  // per instantiation (static locals are per template)
    {
        std::lock_guard<std::mutex> g(occ_mu);
        auto it = occ.find(okey);
        if (it != occ.end()) active = it->second;
    }
    if (!active) {
        CK(cudaOccupancyMaxActiveClusters(&active, kern, &cfg));
        std::lock_guard<std::mutex> g(occ_mu);
        occ[okey] = active;
    }
    const int ncl = std::max(1, std::min(max_clusters, active));
    cfg.gridDim = dim3(ncl * CS);
    cudaLaunchAttribute at2[2] = {at[0], {}};
    at2[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // overlap setup with the query prep
    at2[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at2;
    cfg.numAttrs = pdl_enabled() ? 2 : 1;
    CK(cudaLaunchKernelEx(&cfg, kern, qmap, rmap, p));
    return ncl;
}

template <int NQ>
int launch_res_cs(int CS, const CUtensorMap& qmap, const CUtensorMap& rmap, const ResParams& p, int max_clusters,
                  size_t smem, cudaStream_t st) {
    if constexpr (NQ == 16)
        if (p.ffma == 3) switch (p.hq) {
                case 1: return launch_res<16, 1, 1>(qmap, rmap, p, max_clusters, smem, st);
                case 2: return launch_res<16, 1, 2>(qmap, rmap, p, max_clusters, smem, st);
                default: return launch_res<16, 1, 4>(qmap, rmap, p, max_clusters, smem, st);
            }
    switch (CS) {
        case 1: return launch_res<NQ, 1>(qmap, rmap, p, max_clusters, smem, st);
        case 2: return launch_res<NQ, 2>(qmap, rmap, p, max_clusters, smem, st);
        case 4: return launch_res<NQ, 4>(qmap, rmap, p, max_clusters, smem, st);
        default: return launch_res<NQ, 8>(qmap, rmap, p, max_clusters, smem, st);
    }
}

// Query-resident tensor-core scan.  One launch = one HBM pass serving up to
// 8 clusters-ranks x NQ queries (each CTA of a cluster keeps its own query
// group; the row tiles are TMA-multicast across the cluster).
void umma_res_query(sine_index* h, int64_t B, const double* q_dev, int k, int kp, float thr0, double min_sim,
                    bool bf16, bool rerank, int NQmax, int64_t* ids_dev, double* sims_dev, int32_t* counts_dev,
                    cudaStream_t st, int max_cs) {
    const bool tf32 = !bf16;
    const int64_t row_elems = tf32 ? h->stride32 : h->stride16;
    const int64_t row_bytes = row_elems * (tf32 ? 4 : 2);
    const int kblocks = static_cast<int>(row_bytes / kUmmaKB);
    const int ntiles = static_cast<int>((h->nslots + kUmmaN - 1) / kUmmaN);
    constexpr int kMaxCS = 8;
    h->qbf.ensure(static_cast<size_t>(kMaxCS) * NQmax * row_elems * 2);
    h->lkey.ensure(static_cast<size_t>(h->num_sms) * kMaxCS * NQmax * kp);
    h->lslot.ensure(static_cast<size_t>(h->num_sms) * kMaxCS * NQmax * kp);
    h->ln.ensure(static_cast<size_t>(h->num_sms) * kMaxCS * NQmax);
    const void* rows = tf32 ? static_cast<const void*>(h->rows32) : static_cast<const void*>(h->rows16);
    for (int64_t q0 = 0; q0 < B;) {
        const int64_t rem = B - q0;
        int CS = 1;
        while (CS < max_cs && CS * NQmax < rem) CS <<= 1;
        const int64_t per = (rem + CS - 1) / CS;
        const int NQ = std::min(NQmax, per <= 16 ? 16 : per <= 32 ? 32 : 64);
        const int nq = static_cast<int>(std::min<int64_t>(static_cast<int64_t>(CS) * NQ, rem));
        // a single query: CUDA-core FFMA on the TMA-staged tiles instead of
        // N = 16 MMAs that are 15/16 padding.  Default (p.ffma = 3): eight
        // dot-product warps split each tile's K blocks by ring parity and
        // hand scores to the four list warps through a 16-tile ring, so list
        // upkeep overlaps the HBM stream.  Same box, config B, B = 1
        // lookups/s, MMA path -> helper mode: bf16 tau 0.9 3583 -> 4352,
        // tau -1 3316 -> 4051; fp32 tau -1 2058 -> 2214 (scalar FFMA in the
        // list warps); headline 2184 -> 2239.  Opt-outs for A/B timing:
        // SINE_NO_FFMA=1 keeps the MMAs; SINE_FFMA_LIST=1 computes in the four
        // list warps (scalar FFMA for fp32 rows, FFMA2 with SINE_FFMA2=1 or
        // for bf16 rows), the round-2 single-group path.
        // Small groups (up to ffma_maxq queries) take the helper mode too: each
        // staged row chunk is loaded once and serves every query of the group.
        static const bool ffma_on = getenv("SINE_NO_FFMA") == nullptr;
        static const bool ffma_list = getenv("SINE_FFMA_LIST") != nullptr;
        static const bool ffma2 = getenv("SINE_FFMA2") != nullptr;
        static const int maxq_env = getenv("SINE_FFMA_MAXQ") ? atoi(getenv("SINE_FFMA_MAXQ")) : -1;
        const int ffma_maxq = maxq_env >= 0 ? std::min(maxq_env, 4) : (tf32 ? kFfmaMaxQF32 : kFfmaMaxQBF16);
        int ffma = 0, hq = 0;
        if (ffma_on && CS == 1 && NQ == 16) {
            if (nq == 1) ffma = !ffma_list ? 3 : tf32 && !ffma2 ? 1 : 2;
            else if (nq <= ffma_maxq) ffma = 3;
            if (ffma == 3) hq = nq <= 1 ? 1 : nq <= 2 ? 2 : 4;
        }
        const int fqn = hq > 1 && !tf32 ? hq : 1;
        const ResSmem L0 = res_smem_layout(0, NQ, kblocks, kp, -1, hq, fqn);
        if (L0.total + 2 * kUmmaN * kUmmaKB > 227 * 1024) fail(SINE_EINVAL, "tensor-core plan does not fit shared memory");
        static const int s_cap = getenv("SINE_RES_STAGES") ? atoi(getenv("SINE_RES_STAGES")) : 8;
        int S = static_cast<int>(std::min<size_t>(std::max(2, s_cap), (227 * 1024 - L0.total) / (kUmmaN * kUmmaKB)));
        // helper mode: an even ring, so every stage belongs to one dot-product
        // group (ring index parity == stage parity).  With an odd ring a group
        // could wait on a stage the other group still owns one lap behind and
        // read the wrong mbarrier phase.
        if (ffma == 3) S &= ~1;
        if (S < 2) fail(SINE_EINVAL, "tensor-core plan does not fit shared memory");
        const ResSmem L = res_smem_layout(S, NQ, kblocks, kp, -1, hq, fqn);
        h->gbound.ensure(static_cast<size_t>(kMaxCS) * NQmax);
        res_prep_queries<<<grid_for(static_cast<int64_t>(CS) * NQ * row_elems, 256, h->num_sms), 256, 0, st>>>(
            q_dev + q0 * h->dim, nq, CS * NQ, h->dim, row_elems, tf32 ? 1 : 0, h->qbf.p, h->gbound.p,
            static_cast<int64_t>(CS) * NQ);
        const CUtensorMap qmap = make_kmajor_map(h->qbf.p, tf32, row_elems, static_cast<int64_t>(CS) * NQ, NQ);
        const CUtensorMap rmap = make_kmajor_map(rows, tf32, row_elems, h->nslots, kUmmaN / CS);
        ResParams p{};
        p.nslots = h->nslots;
        p.ntiles = ntiles;
        p.kblocks = kblocks;
        p.nq = nq;
        p.Nq = NQ;
        p.kp = kp;
        p.thr0 = thr0;
        p.stages = S;
        p.tf32 = tf32 ? 1 : 0;
        p.slot_ids = h->ids_ascending ? 1 : 0;
        p.gbound = h->gbound.p;  // zeroed by res_prep_queries
        p.tile_stride = 1;
        p.ffma = ffma;
        p.hq = hq;
        p.valid = h->valid;
        p.ids = h->ids;
        p.out_key = h->lkey.p;
        p.out_slot = h->lslot.p;
        p.out_n = h->ln.p;
        const int max_clusters = std::max(1, std::min(h->num_sms / CS, ntiles));
        auto launch = [&](const ResParams& pp, int maxc) {
            if (NQ == 16) return launch_res_cs<16>(CS, qmap, rmap, pp, maxc, L.total, st);
            if (NQ == 32) return launch_res_cs<32>(CS, qmap, rmap, pp, maxc, L.total, st);
            return launch_res_cs<64>(CS, qmap, rmap, pp, maxc, L.total, st);
        };
        // Low admission floors admit most rows until each CTA's list warms up;
        // a sample pass (one strided tile per cluster) seeds the chip-wide
        // bound with the kp-th best sampled key -- a valid lower bound on the
        // global kp-th best -- so the main pass admits almost nothing extra.
        // The sample pass keeps no lists: per sampled tile and query it
        // writes the max score; the kp-th largest tile maximum is a valid
        // lower bound on the kp-th best score (kp distinct rows reach it).
        const int sample_tiles = std::min(2 * max_clusters, ntiles / 8);
        // Below sample_minq queries the pass costs more than the warm-up it
        // saves.  Same box, config B, tau -1, ms with / without the sample
        // pass: fp32 B = 8 0.564 / 0.543, B = 16 0.565 / 0.564; bf16 B = 8
        // 0.306 / 0.320, B = 16 0.308 / 0.375, B = 64 0.359 / 1.00.
        static const int sample_minq_env = getenv("SINE_SAMPLE_MINQ") ? atoi(getenv("SINE_SAMPLE_MINQ")) : -1;
        const int sample_minq = sample_minq_env >= 0 ? sample_minq_env : (tf32 ? 16 : 8);
        if (thr0 < 0.5f && sample_tiles >= 2 * kp && nq >= sample_minq) {
            h->tmax.ensure(static_cast<size_t>(sample_tiles) * CS * NQ);
            ResParams sp = p;
            sp.ntiles = sample_tiles;
            sp.tile_stride = ntiles / sample_tiles;
            sp.out_max = h->tmax.p;
            launch(sp, std::min(max_clusters, sample_tiles));
            sample_max_bound_kernel<<<nq, 256, 0, st>>>(h->tmax.p, sample_tiles, nq, kp, h->gbound.p);
            h->launches += 2;
            CK(cudaGetLastError());
        }
        const size_t tk = tbegin(h, 2, st);
        const int ncl = launch(p, max_clusters);
        tend(h, tk, st);
        h->launches += 2;
        CK(cudaGetLastError());
        merge_launch(h, ncl, nq, kp, q_dev + q0 * h->dim, k, min_sim, rerank, ids_dev + q0 * k, sims_dev + q0 * k,
                     counts_dev + q0, st, q0);
        q0 += nq;
    }
}

// CTA-pair tensor-core scan (cta_group::2): groups of 2*NQH queries, each
// CTA of a pair holding NQH of them; one HBM pass per group.
template <int NQH>
void umma_pair_query_t(sine_index* h, int64_t B, const double* q_dev, int k, int kp, float thr0, double min_sim,
                       bool bf16, bool rerank, int64_t* ids_dev, double* sims_dev, int32_t* counts_dev,
                       cudaStream_t st) {
    constexpr int NQ = 2 * NQH;
    const bool tf32 = !bf16;
    const int64_t row_elems = tf32 ? h->stride32 : h->stride16;
    const int64_t row_bytes = row_elems * (tf32 ? 4 : 2);
    const int kblocks = static_cast<int>(row_bytes / kUmmaKB);
    const int ntiles = static_cast<int>((h->nslots + 2 * kUmmaN - 1) / (2 * kUmmaN));
    const ResSmem L0 = res_smem_layout(0, NQ, kblocks, kp, NQH);
    if (L0.total + 2 * kUmmaN * kUmmaKB > 227 * 1024) fail(SINE_EINVAL, "pair plan does not fit shared memory");
    const int S = static_cast<int>(std::min<size_t>(8, (227 * 1024 - L0.total) / (kUmmaN * kUmmaKB)));
    const ResSmem L = res_smem_layout(S, NQ, kblocks, kp, NQH);
    smem_optin(reinterpret_cast<const void*>(umma_pair_kernel<NQH>), 227 * 1024);
    const int npairs = std::max(1, std::min(h->num_sms / 2, ntiles));
    h->qbf.ensure(static_cast<size_t>(NQ) * row_elems * 2);
    h->lkey.ensure(static_cast<size_t>(2 * npairs) * NQ * kp);
    h->lslot.ensure(static_cast<size_t>(2 * npairs) * NQ * kp);
    h->ln.ensure(static_cast<size_t>(2 * npairs) * NQ);
    h->gbound.ensure(512);
    const void* rows = tf32 ? static_cast<const void*>(h->rows32) : static_cast<const void*>(h->rows16);
    const CUtensorMap rmap = make_kmajor_map(rows, tf32, row_elems, h->nslots);
    const CUtensorMap qmap = make_kmajor_map(h->qbf.p, tf32, row_elems, NQ, NQH);
    for (int64_t q0 = 0; q0 < B; q0 += NQ) {
        const int nq = static_cast<int>(std::min<int64_t>(NQ, B - q0));
        res_prep_queries<<<grid_for(static_cast<int64_t>(NQ) * row_elems, 256, h->num_sms), 256, 0, st>>>(
            q_dev + q0 * h->dim, nq, NQ, h->dim, row_elems, tf32 ? 1 : 0, h->qbf.p, h->gbound.p, NQ);
        ResParams p{};
        p.nslots = h->nslots;
        p.ntiles = ntiles;
        p.kblocks = kblocks;
        p.nq = nq;
        p.Nq = NQ;
        p.kp = kp;
        p.thr0 = thr0;
        p.stages = S;
        p.tf32 = tf32 ? 1 : 0;
        p.slot_ids = h->ids_ascending ? 1 : 0;
        p.gbound = h->gbound.p;
        p.tile_stride = 1;
        p.valid = h->valid;
        p.ids = h->ids;
        p.out_key = h->lkey.p;
        p.out_slot = h->lslot.p;
        p.out_n = h->ln.p;
        const int sample_tiles = std::min(2 * npairs, ntiles / 8);  // pair tiles (see umma_res_query)
        if (thr0 < 0.5f && sample_tiles >= kp && nq >= 8) {
            h->tmax.ensure(static_cast<size_t>(2 * sample_tiles) * NQ);
            ResParams sp = p;
            sp.ntiles = sample_tiles;
            sp.tile_stride = ntiles / sample_tiles;
            sp.out_max = h->tmax.p;
            umma_pair_kernel<NQH><<<2 * std::min(npairs, sample_tiles), kUmmaThreads, L.total, st>>>(qmap, rmap, sp);
            sample_max_bound_kernel<<<nq, 256, 0, st>>>(h->tmax.p, 2 * sample_tiles, nq, kp, h->gbound.p);
            h->launches += 2;
            CK(cudaGetLastError());
        }
        const size_t tk = tbegin(h, 2, st);
        umma_pair_kernel<NQH><<<2 * npairs, kUmmaThreads, L.total, st>>>(qmap, rmap, p);
        tend(h, tk, st);
        h->launches += 2;
        CK(cudaGetLastError());
        merge_launch(h, 2 * npairs, nq, kp, q_dev + q0 * h->dim, k, min_sim, rerank, ids_dev + q0 * k,
                     sims_dev + q0 * k, counts_dev + q0, st, q0);
    }
}

// The pair keeps NQH queries per CTA: 64 when they fit 96 KB (bf16 at
// d <= 768), else 32.
void umma_pair_query(sine_index* h, int64_t B, const double* q_dev, int k, int kp, float thr0, double min_sim,
                     bool bf16, bool rerank, int64_t* ids_dev, double* sims_dev, int32_t* counts_dev,
                     cudaStream_t st) {
    const int64_t row_bytes = bf16 ? h->stride16 * 2 : h->stride32 * 4;
    if (64 * row_bytes <= 96 * 1024 && B > 32)
        umma_pair_query_t<64>(h, B, q_dev, k, kp, thr0, min_sim, bf16, rerank, ids_dev, sims_dev, counts_dev, st);
    else
        umma_pair_query_t<32>(h, B, q_dev, k, kp, thr0, min_sim, bf16, rerank, ids_dev, sims_dev, counts_dev, st);
}

// Tiled tensor-core GEMM over the whole batch (umma_gemm_kernel): one launch,
// every query tile.  Returns false (nothing written to the outputs) when a
// query's candidates overflowed the chunk capacity; the caller then runs the
// list-keeping kernels.
constexpr int kGemmChunks = 32;
constexpr int kGemmDone = 0, kGemmOverflow = 1, kGemmNotApplicable = 2;
constexpr float kGemmMinFloor = 0.25f;  // below it the GEMM seeds per-query floors from a sample pass
constexpr int kGemmSeedMinTiles = 8 * 64;  // row tiles a seeded GEMM needs (the sample is 1/8 of them)

template <int NQ>
int umma_gemm_query_t(sine_index* h, int64_t B, const double* q_dev, int k, int kp, float thr0, double min_sim,
                       bool bf16, bool rerank, int64_t* ids_dev, double* sims_dev, int32_t* counts_dev,
                       cudaStream_t st) {
    const bool tf32 = !bf16;
    const int64_t row_elems = tf32 ? h->stride32 : h->stride16;
    const int64_t row_bytes = row_elems * (tf32 ? 4 : 2);
    const int kblocks = static_cast<int>(row_bytes / kUmmaKB);
    const int nrt = static_cast<int>((h->nslots + kGemmRows - 1) / kGemmRows);
    const int nqt = static_cast<int>((B + NQ - 1) / NQ);
    if (static_cast<int64_t>(nrt) * nqt >= (1ll << 31)) return kGemmNotApplicable;
    const int64_t Bpad = static_cast<int64_t>(nqt) * NQ;
    const int S = static_cast<int>(std::min<size_t>(8, (227 * 1024 - gemm_smem_bytes(0, NQ)) / gemm_stage_bytes(NQ)));
    const size_t smem = gemm_smem_bytes(S, NQ);
    smem_optin(reinterpret_cast<const void*>(umma_gemm_kernel<NQ>), 227 * 1024);
    const int nitems = nrt * nqt;
    const int npairs = std::max(1, std::min(h->num_sms / 2, nitems));
    h->qbf.ensure(static_cast<size_t>(Bpad) * row_elems * 2);
    h->lkey.ensure(static_cast<size_t>(kGemmChunks) * B * kp);
    h->lslot.ensure(static_cast<size_t>(kGemmChunks) * B * kp);
    h->ln.ensure(static_cast<size_t>(kGemmChunks) * B);
    h->gcnt.ensure(static_cast<size_t>(B) + 1);
    h->gbound.ensure(static_cast<size_t>(B));
    h->n_h.ensure(1);
    const void* rows = tf32 ? static_cast<const void*>(h->rows32) : static_cast<const void*>(h->rows16);
    const CUtensorMap rmap = make_kmajor_map(rows, tf32, row_elems, h->nslots, 128);
    const CUtensorMap qmap = make_kmajor_map(h->qbf.p, tf32, row_elems, Bpad, NQ / 2);
    res_prep_queries<<<grid_for(Bpad * row_elems, 256, h->num_sms), 256, 0, st>>>(
        q_dev, static_cast<int>(B), static_cast<int>(Bpad), h->dim, row_elems, tf32 ? 1 : 0, h->qbf.p);
    CK(cudaMemsetAsync(h->gcnt.p, 0, (static_cast<size_t>(B) + 1) * sizeof(uint32_t), st));
    CK(cudaMemsetAsync(h->gbound.p, 0, static_cast<size_t>(B) * sizeof(uint32_t), st));
    GemmParams p{};
    p.nslots = h->nslots;
    p.nrt = nrt;
    p.nqt = nqt;
    p.kblocks = kblocks;
    p.nq = static_cast<int>(B);
    p.kp = kp;
    p.chunks = kGemmChunks;
    p.thr0 = thr0;
    p.stages = S;
    p.tf32 = tf32 ? 1 : 0;
    p.valid = h->valid;
    p.cnt = h->gcnt.p;
    p.out_key = h->lkey.p;
    p.out_slot = h->lslot.p;
    p.rt_stride = 1;
    if (thr0 < kGemmMinFloor) {
        // low floor: a sample pass over every 8th row tile writes per-query
        // tile maxima; the kp-th largest is a lower bound on the kp-th best
        // score and becomes the query's admission floor in the main pass
        const int nrt_s = std::max(kp, nrt / 8);
        if (nrt_s > nrt) return kGemmNotApplicable;  // too few row tiles to seed floors
        h->tmax.ensure(static_cast<size_t>(2 * nrt_s) * B);
        GemmParams sp = p;
        sp.nrt = nrt_s;
        sp.rt_stride = nrt / nrt_s;
        sp.out_max = h->tmax.p;
        const int sp_pairs = std::max(1, std::min(h->num_sms / 2, nrt_s * nqt));
        umma_gemm_kernel<NQ><<<2 * sp_pairs, kGemmThreads, smem, st>>>(qmap, rmap, sp);
        sample_max_bound_kernel<<<static_cast<int>(B), 256, 0, st>>>(h->tmax.p, 2 * nrt_s, static_cast<int>(B), kp,
                                                                     h->gbound.p);
        h->launches += 2;
        CK(cudaGetLastError());
        p.qthr = h->gbound.p;
    }
    const size_t tk = tbegin(h, 2, st);
    umma_gemm_kernel<NQ><<<2 * npairs, kGemmThreads, smem, st>>>(qmap, rmap, p);
    tend(h, tk, st);
    CK(cudaGetLastError());
    gemm_finish_kernel<<<static_cast<int>((B + 255) / 256), 256, 0, st>>>(h->gcnt.p, static_cast<int>(B), kp,
                                                                          kGemmChunks, h->ln.p, h->gcnt.p + B);
    h->launches += 3;
    CK(cudaGetLastError());
    uint32_t* ovf = reinterpret_cast<uint32_t*>(h->n_h.p);
    CK(cudaMemcpyAsync(ovf, h->gcnt.p + B, sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (*ovf) return kGemmOverflow;
    merge_launch(h, kGemmChunks, static_cast<int>(B), kp, q_dev, k, min_sim, rerank, ids_dev, sims_dev, counts_dev,
                 st, 0);
    return kGemmDone;
}

// Query tile width by batch: N = 64 / 128 / 256 per pair MMA, so small
// batches do not pay for padded query columns (kind::tf32 runs at half rate).
int umma_gemm_query(sine_index* h, int64_t B, const double* q_dev, int k, int kp, float thr0, double min_sim,
                     bool bf16, bool rerank, int64_t* ids_dev, double* sims_dev, int32_t* counts_dev,
                     cudaStream_t st) {
    if (B <= 64)
        return umma_gemm_query_t<64>(h, B, q_dev, k, kp, thr0, min_sim, bf16, rerank, ids_dev, sims_dev, counts_dev,
                                     st);
    if (B <= 128)
        return umma_gemm_query_t<128>(h, B, q_dev, k, kp, thr0, min_sim, bf16, rerank, ids_dev, sims_dev,
                                      counts_dev, st);
    return umma_gemm_query_t<256>(h, B, q_dev, k, kp, thr0, min_sim, bf16, rerank, ids_dev, sims_dev, counts_dev,
                                  st);
}

void umma_query(sine_index* h, int64_t B, const double* q_dev, int k, int kp, double min_sim, bool bf16, bool rerank,
                int64_t* ids_dev, double* sims_dev, int32_t* counts_dev, cudaStream_t st, uint32_t mode) {
    const bool tf32 = !bf16;
    const int64_t row_elems = tf32 ? h->stride32 : h->stride16;
    const int64_t row_bytes = row_elems * (tf32 ? 4 : 2);
    // admission floor: tf32 products carry ~2^-11 relative error per term
    float thr0;
    if (rerank) {
        const double margin = tf32 ? 4e-3 : 8e-3;
        thr0 = std::nextafter(static_cast<float>(min_sim - margin), -INFINITY);
    } else {
        thr0 = static_cast<float>(min_sim);
        if (static_cast<double>(thr0) > min_sim) thr0 = std::nextafter(thr0, -INFINITY);
    }
    // filter error bounds: tf32 operands keep 10 mantissa bits (|rel| <
    // 2^-10 each), bf16 operands 8 bits rounded (2^-9 each); |q|=|x|=1
    h->cur_thr0 = thr0;
    h->cur_err = tf32 ? 2.0e-3 : 4.0e-3;
    // query-resident kernel (v2) when the group fits shared memory and costs
    // no more HBM passes than the query-streaming kernel (v1, 128 per pass)
    {
        const int nq2 = res_nq_max(row_bytes);
        const int64_t passes2 = nq2 ? (B + nq2 - 1) / nq2 : INT64_MAX;
        const int64_t passes1 = (B + kUmmaM - 1) / kUmmaM;
        const bool force_v1 = (mode & 0x400u) != 0;
        // queries per HBM pass of the list-keeping kernels: the resident
        // group (nq2 per CTA) or the CTA pair (2 x pair_nqh, half per CTA)
        const int pair_nqh = 64 * row_bytes <= 96 * 1024 ? 64 : (32 * row_bytes <= 96 * 1024 ? 32 : 0);
        const int64_t per_pass = std::max<int64_t>(nq2, 2 * pair_nqh);
        // larger batches at a high admission floor: one tiled GEMM launch
        // (256 x 256 pair tiles, N = 256 per MMA) instead of B / per_pass
        // HBM passes; up to 256 queries it costs about one HBM pass (measured,
        // 1M x 768, tau 0.9: bf16 B=256 0.39 ms vs 0.84 ms in two 128-query
        // pair passes; fp32 B=256 0.71 vs 1.65 ms)
        const int64_t row_tiles = (h->nslots + kGemmRows - 1) / kGemmRows;
        const bool gemm_floor_ok = thr0 >= kGemmMinFloor || row_tiles >= kGemmSeedMinTiles;
        const bool gemm_auto = !(mode & SINE_SCAN_NO_GEMM) && !force_v1 && B > per_pass && gemm_floor_ok &&
                               !(mode & (SINE_SCAN_PAIR | SINE_SCAN_CLUSTER));
        if ((mode & SINE_SCAN_GEMM) || gemm_auto) {
            const int r = umma_gemm_query(h, B, q_dev, k, kp, thr0, min_sim, bf16, rerank, ids_dev, sims_dev,
                                          counts_dev, st);
            if (r == kGemmDone) return;
            if (r == kGemmOverflow) ++h->gemm_overflows;  // fall through to the list-keeping kernels
        }
        // measured per-query cost on B200 (1M x 768): resident bf16 ~4.8 us,
        // resident tf32 ~17 us (32-query groups), streaming v1 ~6 us; the
        // cluster-multicast variant does not lower the per-query cost (the
        // L2->SM fan-out, not HBM, binds), so it is opt-in.
        const bool res = nq2 && (bf16 || B <= nq2);
        // nq2 < B <= 2 x pair_nqh: one CTA-pair pass instead of two resident passes
        const bool pair_fits = pair_nqh > 0;
        const bool pair_auto = pair_fits && B > nq2 && B <= 2 * pair_nqh;
        if (!force_v1 && pair_fits && !(mode & SINE_SCAN_CLUSTER) && ((mode & SINE_SCAN_PAIR) || pair_auto)) {
            umma_pair_query(h, B, q_dev, k, kp, thr0, min_sim, bf16, rerank, ids_dev, sims_dev, counts_dev, st);
            return;
        }
        if (!force_v1 && nq2 && (res || (mode & SINE_SCAN_CLUSTER))) {
            umma_res_query(h, B, q_dev, k, kp, thr0, min_sim, bf16, rerank, nq2, ids_dev, sims_dev, counts_dev, st,
                           (mode & SINE_SCAN_CLUSTER) ? 8 : 1);
            return;
        }
        (void)passes1;
        (void)passes2;
    }
    const int ntiles = static_cast<int>((h->nslots + kUmmaN - 1) / kUmmaN);
    const int grid = std::max(1, std::min(h->num_sms, ntiles));
    const UmmaSmem L0 = umma_smem_layout(0, kp);
    const size_t stage_bytes = static_cast<size_t>(kUmmaM + kUmmaN) * kUmmaKB;
    const int S = static_cast<int>(std::min<size_t>(8, (227 * 1024 - L0.total) / stage_bytes));
    if (S < 2) fail(SINE_EINVAL, "tensor-core plan does not fit shared memory");
    const UmmaSmem L = umma_smem_layout(S, kp);
    smem_optin(reinterpret_cast<const void*>(umma_scan_kernel), 227 * 1024);
    h->qbf.ensure(static_cast<size_t>(kUmmaM) * row_elems * 2);  // bytes/2 units: fp32 needs 2x
    h->lkey.ensure(static_cast<size_t>(grid) * kUmmaM * kp);
    h->lslot.ensure(static_cast<size_t>(grid) * kUmmaM * kp);
    h->ln.ensure(static_cast<size_t>(grid) * kUmmaM);
    const void* rows = tf32 ? static_cast<const void*>(h->rows32) : static_cast<const void*>(h->rows16);
    const CUtensorMap rmap = make_kmajor_map(rows, tf32, row_elems, h->nslots);
    const CUtensorMap qmap = make_kmajor_map(h->qbf.p, tf32, row_elems, kUmmaM);
    for (int64_t q0 = 0; q0 < B; q0 += kUmmaM) {
        const int nq = static_cast<int>(std::min<int64_t>(kUmmaM, B - q0));
        umma_prep_queries<<<grid_for(kUmmaM * row_elems, 256, h->num_sms), 256, 0, st>>>(
            q_dev + q0 * h->dim, nq, h->dim, row_elems, tf32 ? 1 : 0, h->qbf.p);
        UmmaParams p{};
        p.nslots = h->nslots;
        p.ntiles = ntiles;
        p.kblocks = static_cast<int>(row_bytes / kUmmaKB);
        p.nq = nq;
        p.kp = kp;
        p.thr0 = thr0;
        p.stages = S;
        p.tf32 = tf32 ? 1 : 0;
        h->gbound.ensure(512);
        CK(cudaMemsetAsync(h->gbound.p, 0, kUmmaM * sizeof(uint32_t), st));
        p.gbound = h->gbound.p;
        p.tile_stride = 1;
        p.valid = h->valid;
        p.ids = h->ids;
        p.out_key = h->lkey.p;
        p.out_slot = h->lslot.p;
        p.out_n = h->ln.p;
        const int sample_tiles = std::min(grid, ntiles / 16);
        if (thr0 < 0.5f && sample_tiles >= 16 && nq >= 8) {  // seed the admission bound (see umma_res_query)
            UmmaParams sp = p;
            sp.ntiles = sample_tiles;
            sp.tile_stride = ntiles / sample_tiles;
            umma_scan_kernel<<<sample_tiles, kUmmaThreads, L.total, st>>>(qmap, rmap, sp);
            sample_bound_kernel<<<nq, 256, 0, st>>>(h->lkey.p, h->ln.p, sample_tiles, nq, kp, h->gbound.p);
            h->launches += 2;
            CK(cudaGetLastError());
        }
        const size_t tk = tbegin(h, 2, st);
        umma_scan_kernel<<<grid, kUmmaThreads, L.total, st>>>(qmap, rmap, p);
        tend(h, tk, st);
        h->launches += 2;
        CK(cudaGetLastError());
        merge_launch(h, grid, nq, kp, q_dev + q0 * h->dim, k, min_sim, rerank, ids_dev + q0 * k, sims_dev + q0 * k,
                     counts_dev + q0, st, q0);
    }
}

// Runs the full stage-1 pipeline for B device-resident queries.
void query_device_impl(sine_index* h, int64_t B, const double* q_dev, int k, double min_sim, uint32_t mode,
                       int64_t* ids_dev, double* sims_dev, int32_t* counts_dev, cudaStream_t st) {
    if (k < 1) fail(SINE_EINVAL, "k must be >= 1");
    if (B <= 0) return;
    const bool bf16 = (mode & 0xF) == SINE_SCAN_BF16;
    const bool rerank = (mode & SINE_RERANK_F64) != 0;
    if (bf16 && !(h->flags & SINE_STORE_BF16)) fail(SINE_EINVAL, "index has no bf16 rows (create with SINE_STORE_BF16)");
    if (!bf16 && !(h->flags & SINE_STORE_F32)) fail(SINE_EINVAL, "index has no fp32 rows (create with SINE_STORE_F32)");
    int kp = rerank ? k + kSlack : k;
    if (kp > kMaxKp) {
        if (k > kMaxKp) fail(SINE_EINVAL, "k > 128 is not supported by the device top-k");
        kp = kMaxKp;
    }
    if (h->nlive == 0) {
        CK(cudaMemsetAsync(counts_dev, 0, B * sizeof(int32_t), st));
        CK(cudaMemsetAsync(ids_dev, 0xff, B * k * sizeof(int64_t), st));
        CK(cudaMemsetAsync(sims_dev, 0, B * k * sizeof(double), st));
        return;
    }
    // admission floor: exact threshold, or widened by the scan precision so
    // the fp64 re-rank sees every row whose exact similarity passes
    float thr0;
    if (rerank) {
        const double margin = bf16 ? 8e-3 : 1e-5;
        thr0 = std::nextafter(static_cast<float>(min_sim - margin), -INFINITY);
    } else {
        thr0 = static_cast<float>(min_sim);
        if (static_cast<double>(thr0) > min_sim) thr0 = std::nextafter(thr0, -INFINITY);
    }
    // fp32 scan: two input roundings + <= 25 accumulation roundings of 2^-24
    h->cur_thr0 = thr0;
    h->cur_err = bf16 ? 4.0e-3 : 2.0e-6;
    h->cert.ensure(std::max<int64_t>(B, 1));

    if (h->snap_nslots < 0 && umma_eligible(h, B, bf16, mode, kp)) {
        umma_query(h, B, q_dev, k, kp, min_sim, bf16, rerank, ids_dev, sims_dev, counts_dev, st, mode);
        return;
    }

    // a snapshot re-run (sine_query_wait) scans the submit-time store: the
    // slots that existed then, with the validity bitmap of that moment
    const int64_t scan_slots = h->snap_nslots >= 0 ? h->snap_nslots : h->nslots;
    const uint32_t* scan_valid = h->snap_valid ? h->snap_valid : h->valid;
    const int NQmax = scan_cfg(h, bf16, 0).NQmax;
    h->lkey.ensure(static_cast<size_t>(h->num_sms) * NQmax * kp);
    h->lslot.ensure(static_cast<size_t>(h->num_sms) * NQmax * kp);
    h->ln.ensure(static_cast<size_t>(h->num_sms) * NQmax);

    for (int64_t q0 = 0; q0 < B; q0 += NQmax) {
        const int nq = static_cast<int>(std::min<int64_t>(NQmax, B - q0));
        int NQ = 1;
        while (NQ < nq) NQ <<= 1;
        const ScanCfg c = scan_cfg(h, bf16, NQ);
        const int grid = static_cast<int>(std::max<int64_t>(
            1, std::min<int64_t>(h->num_sms, (scan_slots + c.R - 1) / c.R)));
        const int64_t rows_per_cta = round_up((scan_slots + grid - 1) / grid, c.R);
        ScanParams p{};
        p.rows = bf16 ? reinterpret_cast<const uint8_t*>(h->rows16) : reinterpret_cast<const uint8_t*>(h->rows32);
        p.row_bytes = c.row_bytes;
        p.nslots = scan_slots;
        p.valid = scan_valid;
        p.ids = h->ids;
        p.q64 = q_dev + q0 * h->dim;
        p.dim = h->dim;
        p.nq = nq;
        p.kp = kp;
        p.thr0 = thr0;
        p.rows_per_stage = c.R;
        p.rows_per_cta = rows_per_cta;
        p.chunks = c.C;
        p.chunk_warps = c.CW;
        p.row_groups = c.G;
        p.unroll = c.U;
        p.slot_ids = h->ids_ascending ? 1 : 0;
        h->gbound.ensure(512);
        CK(cudaMemsetAsync(h->gbound.p, 0, 16 * sizeof(uint32_t), st));
        p.gbound = h->gbound.p;
        p.out_key = h->lkey.p;
        p.out_slot = h->lslot.p;
        p.out_n = h->ln.p;
        // stages: fill ~200 KB of shared memory
        const ScanSmemLayout L0 = scan_smem_layout(0, c.R, c.row_bytes, NQ, c.C, kp);
        const size_t stage_bytes = static_cast<size_t>(c.R) * c.row_bytes;
        int S = static_cast<int>(std::min<size_t>(8, (208 * 1024 - L0.total) / stage_bytes));
        S = std::max(S, 2);
        p.stages = S;
        const ScanSmemLayout L = scan_smem_layout(S, c.R, c.row_bytes, NQ, c.C, kp);
        if (L.total > 227 * 1024) fail(SINE_EINVAL, "scan shared-memory plan exceeds 227 KB");
        const int threads = (c.CW * c.G + 1) * 32;
        record(h, 0, st);
        const size_t tk = tbegin(h, 0, st);
        if (bf16) {
            if (c.CPW == 1)
                launch_scan_nq<__nv_bfloat16, 1>(NQ, p, grid, threads, L.total, st);
            else
                launch_scan_nq<__nv_bfloat16, 2>(NQ, p, grid, threads, L.total, st);
        } else {
            if (c.CPW == 1)
                launch_scan_nq<float, 1>(NQ, p, grid, threads, L.total, st);
            else
                launch_scan_nq<float, 2>(NQ, p, grid, threads, L.total, st);
        }
        ++h->launches;
        CK(cudaGetLastError());
        tend(h, tk, st);
        record(h, 1, st);
        merge_launch(h, grid, nq, kp, q_dev + q0 * h->dim, k, min_sim, rerank, ids_dev + q0 * k, sims_dev + q0 * k,
                     counts_dev + q0, st, q0);
        record(h, 2, st);
    }
}

void merge_launch(sine_index* h, int ncta, int nq, int kp, const double* q64, int k, double min_sim, bool rerank,
                  int64_t* ids_dev, double* sims_dev, int32_t* counts_dev, cudaStream_t st, int64_t cert_off) {
    MergeParams m{};
    m.in_key = h->lkey.p;
    m.in_slot = h->lslot.p;
    m.in_n = h->ln.p;
    m.ncta = ncta;
    m.nq = nq;
    m.kp = kp;
    m.ids = h->ids;
    m.rows64 = h->rows64;
    m.q64 = q64;
    m.dim = h->dim;
    m.k = k;
    m.min_sim = min_sim;
    m.rerank = rerank ? 1 : 0;
    m.thr0 = h->cur_thr0;
    m.err = h->cur_err;
    uint8_t* cert_base = h->cert_out ? h->cert_out : h->cert.p;  // caller's device log when given
    m.cert = cert_base ? cert_base + (cert_off) : nullptr;
    m.debug = getenv("SINE_DEBUG_MERGE") ? 2 : (getenv("SINE_DEBUG_CERT") ? 1 : 0);
    m.gbound = h->gbound.p;  // every stage-1 kernel publishes its admission bounds here
    m.out_ids = ids_dev;
    m.out_sims = sims_dev;
    m.out_counts = counts_dev;
    smem_optin(reinterpret_cast<const void*>(merge_kernel), 160 * 1024);
    const size_t pool_bytes = static_cast<size_t>(ncta) * kp * sizeof(uint32_t);
    if (pool_bytes > 160 * 1024) fail(SINE_EINVAL, "candidate pool exceeds the merge kernel's shared memory");
    const size_t tm = tbegin(h, 1, st);
    // PDL: the merge CTAs are scheduled while the scan drains and wait on
    // the device (griddepcontrol.wait) for its lists instead of a host launch
    cudaLaunchConfig_t cfg{};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.gridDim = dim3(nq);
    cfg.blockDim = dim3(kMergeThreads);
    cfg.dynamicSmemBytes = pool_bytes;
    cfg.stream = st;
    cfg.attrs = at;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    CK(cudaLaunchKernelEx(&cfg, merge_kernel, m));
    tend(h, tm, st);
    ++h->launches;
    CK(cudaGetLastError());
}

// Queries whose certificate failed (fast filter too close to the k-th
// similarity) are re-run through the fp32 CUDA-core scan, whose 2e-6 error
// bound is inside the north star's 1e-5 tie window.  Synchronises `st`.
int64_t certify_and_fix(sine_index* h, int64_t B, const double* q_dev, int k, double min_sim, uint32_t mode,
                        int64_t* ids_dev, double* sims_dev, int32_t* counts_dev, cudaStream_t st,
                        const uint8_t* cert_host = nullptr) {
    if (!(mode & SINE_RERANK_F64) || !(h->flags & SINE_STORE_F32) || h->nlive == 0) return 0;
    const bool bf16 = (mode & 0xF) == SINE_SCAN_BF16;
    std::vector<uint8_t> cert(B);
    if (cert_host) {
        std::copy(cert_host, cert_host + B, cert.begin());
    } else {
        CK(cudaMemcpyAsync(cert.data(), h->cert.p, B, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
    }
    const bool exact_path_used = !bf16 && (mode & SINE_SCAN_CUDA_CORE);
    if (exact_path_used) return 0;
    // the failing queries re-run on the exact fp32 CUDA-core scan as ONE
    // batch (one more pass over the rows, not one per query), then their
    // results are copied back into place
    std::vector<int64_t> bad;
    for (int64_t b = 0; b < B; ++b)
        if (!cert[b]) bad.push_back(b);
    const int64_t R = static_cast<int64_t>(bad.size());
    if (R == 0) return 0;
    DevBuf<double> rq;
    DevBuf<int64_t> rid;
    DevBuf<double> rsim;
    DevBuf<int32_t> rcnt;
    rq.ensure(R * h->dim);
    rid.ensure(R * k);
    rsim.ensure(R * k);
    rcnt.ensure(R);
    for (int64_t r = 0; r < R; ++r)
        CK(cudaMemcpyAsync(rq.p + r * h->dim, q_dev + bad[r] * h->dim, h->dim * sizeof(double),
                           cudaMemcpyDeviceToDevice, st));
    const uint32_t m2 = SINE_SCAN_F32 | SINE_RERANK_F64 | SINE_SCAN_CUDA_CORE;
    query_device_impl(h, R, rq.p, k, min_sim, m2, rid.p, rsim.p, rcnt.p, st);
    for (int64_t r = 0; r < R; ++r) {
        const int64_t b = bad[r];
        // (the destinations may be mapped host staging: cudaMemcpyDefault)
        CK(cudaMemcpyAsync(ids_dev + b * k, rid.p + r * k, k * sizeof(int64_t), cudaMemcpyDefault, st));
        CK(cudaMemcpyAsync(sims_dev + b * k, rsim.p + r * k, k * sizeof(double), cudaMemcpyDefault, st));
        CK(cudaMemcpyAsync(counts_dev + b, rcnt.p + r, sizeof(int32_t), cudaMemcpyDefault, st));
    }
    CK(cudaStreamSynchronize(st));
    return R;
}

void check_queries_host(const sine_index* h, int64_t B, const double* q) {
    for (int64_t b = 0; b < B; ++b) {
        const double* r = q + b * h->dim;
        double ss = 0.0;
        for (int64_t j = 0; j < h->dim; ++j) ss += r[j] * r[j];
        const double nrm = std::sqrt(ss);
        if (std::fabs(nrm - 1.0) > 1e-6) {
            char buf[128];
            snprintf(buf, sizeof buf, "vector is not L2-normalized (norm=%.8f)", nrm);
            fail(SINE_ENORM, buf);
        }
    }
}

// ------------------------------------------------------------ eviction driver

EvictCols evict_cols(const sine_index* h) {
    EvictCols c{};
    c.lf = h->lf, c.lc = h->lc, c.ll = h->ll, c.ls = h->ls;
    c.created = h->created, c.expiration = h->expiration, c.last_access = h->last_access;
    c.freq = h->freq, c.size = h->size, c.ids = h->ids, c.valid = h->valid;
    c.nslots = h->nslots;
    return c;
}

// Victims are written straight into the caller's buffer (pinned or pageable).
// Sample select (select.cuh): one pass over the store, then only the
// records below the sampled bound are bucketed and sorted.
void remove_slots(sine_index* h, const std::vector<int64_t>& slots, const int64_t* dslots);

// remove: also tombstone the victims (sine_evict).
void select_victims_impl(sine_index* h, int policy, double now, int64_t excess, int64_t* out, int64_t cap,
                         int64_t* nout, bool remove = false) {
    *nout = 0;
    if (!(h->flags & SINE_STORE_META)) fail(SINE_EINVAL, "index has no LCFU metadata (SINE_STORE_META)");
    if (excess <= 0 || h->nlive == 0) return;
    cudaStream_t st = h->stream;
    record(h, 3, st);
    const int64_t nl = std::max<int64_t>(h->nlive, 1);
    h->srec.ensure(nl);
    h->srec2.ensure(nl);
    h->sbid.ensure(nl);
    h->vids.ensure(nl);
    if (remove && h->ids_ascending) h->sslot.ensure(nl);
    int64_t* oslot = remove && h->ids_ascending ? h->sslot.p : nullptr;
    h->sspl.ensure(kSelMaxBuckets);
    h->stab.ensure(4100);
    h->sbcnt.ensure(2 * kSelMaxBuckets);
    h->sboff.ensure(kSelMaxBuckets);
    h->sbcur.ensure(kSelMaxBuckets);
    h->sbig.ensure(kSelMaxBuckets);
    h->sctl.ensure(1);
    h->sctl_h.ensure(1);
    smem_optin(reinterpret_cast<const void*>(sel_collect_kernel), kSelCollectSmem);
    smem_optin(reinterpret_cast<const void*>(sel_bucket_kernel), kSelBucketSmem);
    smem_optin(reinterpret_cast<const void*>(sel_sort_kernel), kSelCountSmem);
    smem_optin(reinterpret_cast<const void*>(sel_big_kernel), kSelSortSmem);
    const EvictCols cols = evict_cols(h);
    const int slot_tie = h->ids_ascending ? 1 : 0;
    unsigned long long* bcnt = h->sbcnt.p;
    unsigned long long* bw = bcnt + kSelMaxBuckets;
    const int scap = h->sel_cap;
    // small stores skip the sample: every live slot is a record
    bool all = h->nlive <= scap;
    h->ssamp.ensure(kSelSample);
    for (int attempt = 0; attempt < 2; ++attempt) {
        // init (ctl preset, bucket counters, the sample gather), then the
        // chain below under PDL
        sel_init_kernel<<<kSelSample / kSelInitThreads, kSelInitThreads, 0, st>>>(
            cols, policy, now, slot_tie, all ? 1 : 0, h->sctl.p, bcnt, 2 * kSelMaxBuckets, h->ssamp.p);
        ++h->launches;
        if (!all) {
            launch_pdl(sel_sample_kernel, 1, 1024, 0, st, static_cast<const SelRec*>(h->ssamp.p), h->nlive, excess,
                       h->sctl.p);
            ++h->launches;
        }
        SelColumns sc{};
        if (policy == 0) {
            const void* c7[7] = {h->lf, h->lc, h->ll, h->ls, h->expiration, h->size, h->created};
            for (int k = 0; k < 7; ++k) sc.col[k] = c7[k];
            sc.ncol = 7;
        } else {
            sc.col[0] = policy == 1 ? static_cast<const void*>(h->last_access) : static_cast<const void*>(h->freq);
            sc.col[1] = h->size;
            sc.col[2] = h->created;
            sc.ncol = 3;
        }
        const int64_t tiles = (h->nslots + kSelTile - 1) / kSelTile;
        const int gcol = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(tiles, h->num_sms)));
        launch_pdl(sel_collect_kernel, gcol, kSelCollectThreads, kSelCollectSmem, st, cols, sc, policy, now, slot_tie,
                   h->sctl.p, h->srec.p);
        launch_pdl(sel_split_kernel, 1, 1024, 0, st, excess, h->sctl.p, static_cast<const SelRec*>(h->srec.p),
                   h->sspl.p, h->stab.p, scap);
        // bucket and scatter must split the records the same way (same grid)
        const int grec = h->num_sms;
        launch_pdl(sel_bucket_kernel, grec, 1024, kSelBucketSmem, st, h->sctl.p, static_cast<const SelRec*>(h->srec.p),
                   static_cast<const uint32_t*>(h->sspl.p), static_cast<const uint32_t*>(h->stab.p), h->sbid.p, bcnt,
                   bw);
        launch_pdl(sel_scan_kernel, 1, 1024, 0, st, h->sctl.p, excess, static_cast<const unsigned long long*>(bcnt),
                   static_cast<const unsigned long long*>(bw), h->sboff.p, h->sbcur.p);
        launch_pdl(sel_scatter_kernel, grec, 1024, 0, st, static_cast<const SelCtl*>(h->sctl.p),
                   static_cast<const SelRec*>(h->srec.p), static_cast<const uint16_t*>(h->sbid.p),
                   static_cast<const int64_t*>(h->sboff.p), h->sbcur.p, h->srec2.p);
        launch_pdl(sel_sort_kernel, 3 * h->num_sms, kSelSortThreads, kSelCountSmem, st, h->sctl.p, excess, slot_tie,
                   static_cast<const int64_t*>(h->ids), static_cast<const uint32_t*>(h->sspl.p),
                   static_cast<const SelRec*>(h->srec2.p), static_cast<const int64_t*>(h->sboff.p),
                   static_cast<const unsigned long long*>(bcnt), h->sbig.p, h->vids.p, scap, oslot);
        launch_pdl(sel_big_kernel, h->num_sms, kSelSortThreads, kSelSortSmem, st, h->sctl.p, excess, slot_tie,
                   static_cast<const int64_t*>(h->ids), h->srec2.p, h->srec.p, static_cast<const int64_t*>(h->sboff.p),
                   static_cast<const unsigned long long*>(bcnt), static_cast<const int32_t*>(h->sbig.p), h->vids.p,
                   scap, oslot);
        h->launches += 7;
        CK(cudaGetLastError());
        record(h, 4, st);
        CK(cudaMemcpyAsync(h->sctl_h.p, h->sctl.p, sizeof(SelCtl), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        if (!h->sctl_h.p->retry) break;
        all = true;  // the sampled bound fell short of the excess: take every slot
    }
    const int64_t V = h->sctl_h.p->V;
    if (V > cap) fail(SINE_EINVAL, "output buffer too small for the victim list");
    CK(cudaMemcpyAsync(out, h->vids.p, V * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    std::vector<int64_t> slots;
    if (remove && V > 0) {
        slots.resize(V);
        if (oslot) CK(cudaMemcpyAsync(slots.data(), oslot, V * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    }
    CK(cudaStreamSynchronize(st));
    *nout = V;
    if (h->timing) CK(cudaEventElapsedTime(&h->t_evict, h->ev[3], h->ev[4]));
    if (remove && V > 0) {
        if (!oslot)
            for (int64_t i = 0; i < V; ++i) slots[i] = find_slot(h, out[i]);
        remove_slots(h, slots, oslot);
    }
}

bool certify_in_flight(const sine_index* h) {
    for (const auto& t : h->tickets)
        if (t.busy && t.certify) return true;
    return false;
}

// Called before a tombstone is written: certified tickets in flight that
// have no snapshot yet get a copy of the current bitmap (their submission
// state: nothing was removed since), enqueued ahead of the tombstone.
void snapshot_bitmap_for_tickets(sine_index* h) {
    std::shared_ptr<DevBitmap> snap;
    for (auto& t : h->tickets) {
        if (!t.busy || !t.certify || t.valid_snap) continue;
        if (!snap) {
            snap = std::make_shared<DevBitmap>();
            const int64_t words = (h->nslots + 31) / 32;
            CK(cudaMalloc(&snap->p, std::max<int64_t>(words, 1) * sizeof(uint32_t)));
            CK(cudaMemcpyAsync(snap->p, h->valid, words * sizeof(uint32_t), cudaMemcpyDeviceToDevice, h->stream));
        }
        t.valid_snap = snap;
    }
}

void maybe_compact(sine_index* h) {
    const int64_t dead = h->nslots - h->nlive;
    if (dead <= std::max<int64_t>(64, h->nlive / 4)) return;
    if (certify_in_flight(h)) {  // slots must not move under a pending re-run
        h->compact_pending = true;
        return;
    }
    h->compact_pending = false;
    compact(h);
}

// ExactCosineIndex.remove's bookkeeping (index.py:80-92): the last id moves
// into the removed id's position.
void order_remove(sine_index* h, int64_t slot);

void order_flush(sine_index* h) {
    for (const int64_t op : h->order_log) {
        if (op >= 0) {
            order_remove(h, op);
        } else {
            const int64_t s = ~op;
            if (static_cast<int64_t>(h->order_pos.size()) <= s) h->order_pos.resize(s + 1, -1);
            h->order_pos[s] = static_cast<int64_t>(h->order_slot.size());
            h->order_slot.push_back(s);
        }
    }
    h->order_log.clear();
}

void order_append(sine_index* h, int64_t slot) {
    if (h->order_log.empty()) {
        if (static_cast<int64_t>(h->order_pos.size()) <= slot) h->order_pos.resize(slot + 1, -1);
        h->order_pos[slot] = static_cast<int64_t>(h->order_slot.size());
        h->order_slot.push_back(slot);
    } else {
        h->order_log.push_back(~slot);
    }
}

void order_removed(sine_index* h, int64_t slot) {
    h->order_log.push_back(slot);
    if (static_cast<int64_t>(h->order_log.size()) > 2 * (h->nslots + 1024)) order_flush(h);
}

void order_remove(sine_index* h, int64_t slot) {
    const int64_t p = h->order_pos[slot];
    const int64_t last = h->order_slot.back();
    if (p != static_cast<int64_t>(h->order_slot.size()) - 1) {
        h->order_slot[p] = last;
        h->order_pos[last] = p;
    }
    h->order_slot.pop_back();
    h->order_pos[slot] = -1;
}

// slots removed in the given order (the caller's removal sequence)
// Tombstone `slots` (device copy `dslots` when the caller already has one).
void remove_slots(sine_index* h, const std::vector<int64_t>& slots, const int64_t* dslots = nullptr) {
    if (slots.empty()) return;
    DevBuf<int64_t> d;
    snapshot_bitmap_for_tickets(h);
    if (!dslots) {
        d.ensure(slots.size());
        CK(cudaMemcpyAsync(d.p, slots.data(), slots.size() * sizeof(int64_t), cudaMemcpyHostToDevice, h->stream));
        dslots = d.p;
    }
    set_bits_kernel<<<grid_for(slots.size(), 256, h->num_sms), 256, 0, h->stream>>>(h->valid, dslots, slots.size(), 0);
    ++h->launches;
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(h->stream));
    d.release();
    for (int64_t s : slots) {
        if (!h->ids_ascending) h->pos.erase(h->ids_h[s]);
        h->live_h[s] = 0;
        order_removed(h, s);
    }
    h->nlive -= static_cast<int64_t>(slots.size());
    maybe_compact(h);
}

// fp64 master rows of `n` slots -> host [n][dim]: one gather on the device
// and one copy back per 256 MB chunk (snapshots of 1M rows)
void gather_rows_host(sine_index* h, int64_t n, const int64_t* slots, double* out) {
    if (n <= 0) return;
    const int64_t chunk = std::max<int64_t>(1, (256ll << 20) / (h->dim * 8));
    DevBuf<int64_t> dslots;
    DevBuf<double> drows;
    dslots.ensure(std::min(n, chunk));
    drows.ensure(std::min(n, chunk) * h->dim);
    for (int64_t i0 = 0; i0 < n; i0 += chunk) {
        const int64_t m = std::min(chunk, n - i0);
        CK(cudaMemcpyAsync(dslots.p, slots + i0, m * 8, cudaMemcpyHostToDevice, h->stream));
        gather_rows64_kernel<<<grid_for(m * h->dim, 256, h->num_sms), 256, 0, h->stream>>>(h->rows64, dslots.p, m,
                                                                                          h->dim, drows.p);
        ++h->launches;
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(out + i0 * h->dim, drows.p, m * h->dim * 8, cudaMemcpyDeviceToHost, h->stream));
        CK(cudaStreamSynchronize(h->stream));
    }
    dslots.release();
    drows.release();
}

}  // namespace

// ====================================================================== C ABI

extern "C" {

const char* sine_last_error(void) { return g_err.c_str(); }

// not in the public header: other translation units (group.cu) report
// their failures through the same thread-local message
void sine_internal_set_error(const char* msg) { g_err = msg ? msg : ""; }
int sine_version(void) { return 1; }

int sine_device_count(int* n) {
    return guarded([&] { CK(cudaGetDeviceCount(n)); });
}

int sine_create(int device, int64_t dim, uint32_t flags, int64_t reserve_rows, sine_index_t** out) {
    return guarded([&] {
        if (!out) fail(SINE_EINVAL, "null output handle");
        if (dim < 1) fail(SINE_EINVAL, "dimension must be >= 1");
        if (!(flags & (SINE_STORE_F32 | SINE_STORE_BF16))) flags |= SINE_STORE_F32;
        CK(cudaSetDevice(device));
        auto* h = new sine_index();
        h->device = device;
        h->dim = dim;
        h->flags = flags;
        h->stride32 = round_up(dim, 32);
        h->stride16 = round_up(dim, 64);
        CK(cudaDeviceGetAttribute(&h->num_sms, cudaDevAttrMultiProcessorCount, device));
        CK(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
        for (auto& e : h->ev) CK(cudaEventCreate(&e));
        CK(cudaEventCreateWithFlags(&h->ws_ev, cudaEventDisableTiming));
        h->ws_stream = h->stream;
        if (reserve_rows > 0) grow(h, reserve_rows);
        *out = h;
    });
}

int sine_destroy(sine_index_t* h) {
    return guarded([&] {
        if (!h) return;
        cudaSetDevice(h->device);
        if (h->ws_stream != h->stream) cudaEventSynchronize(h->ws_ev);  // caller-stream queries drain first
        cudaStreamSynchronize(h->stream);
        free_master(h, h->rows64);
        for (void* p : {(void*)h->rows32, (void*)h->rows16, (void*)h->ids, (void*)h->valid,
                        (void*)h->lf, (void*)h->lc, (void*)h->ll, (void*)h->ls, (void*)h->created,
                        (void*)h->expiration, (void*)h->last_access, (void*)h->freq, (void*)h->size})
            if (p) cudaFree(p);
        // the DevBuf / HostBuf workspaces free themselves with the handle
        for (auto& t : h->tickets)
            if (t.done) cudaEventDestroy(t.done);
        for (auto& e : h->ev) cudaEventDestroy(e);
        cudaEventDestroy(h->ws_ev);
        cudaStreamDestroy(h->stream);
        delete h;
    });
}

int sine_reserve(sine_index_t* h, int64_t rows) {
    return guarded([&] {
        std::lock_guard<std::mutex> g(h->mu);
        CK(cudaSetDevice(h->device));
        ws_acquire(h, h->stream);
        grow(h, rows);
    });
}

int sine_insert(sine_index_t* h, int64_t n, const int64_t* ids, const double* rows, const sine_meta_cols_t* meta,
                uint32_t flags) {
    return guarded([&] {
        if (n <= 0) return;
        if (!ids || !rows) fail(SINE_EINVAL, "null ids/rows");
        std::lock_guard<std::mutex> g(h->mu);
        CK(cudaSetDevice(h->device));
        ws_acquire(h, h->stream);
        if (!(flags & SINE_NO_NORM_CHECK)) check_rows_host(h, n, rows);
        check_new_ids(h, n, ids);
        append(h, n, ids, rows, false, meta);
    });
}

int sine_insert_device(sine_index_t* h, int64_t n, const int64_t* ids, const double* rows_dev,
                       const sine_meta_cols_t* meta, uint32_t flags) {
    (void)flags;
    return guarded([&] {
        if (n <= 0) return;
        std::lock_guard<std::mutex> g(h->mu);
        CK(cudaSetDevice(h->device));
        ws_acquire(h, h->stream);
        check_new_ids(h, n, ids);
        // the rows may come from any stream (e.g. a torch kernel that just
        // wrote them): order the copy after all prior device work
        CK(cudaDeviceSynchronize());
        append(h, n, ids, rows_dev, true, meta);
    });
}

int sine_remove(sine_index_t* h, int64_t n, const int64_t* ids) {
    return guarded([&] {
        std::lock_guard<std::mutex> g(h->mu);
        CK(cudaSetDevice(h->device));
        ws_acquire(h, h->stream);
        std::vector<int64_t> slots;
        slots.reserve(n);
        bool asc = true;
        for (int64_t i = 1; asc && i < n; ++i) asc = ids[i] > ids[i - 1];
        std::unordered_set<int64_t> seen;
        for (int64_t i = 0; i < n; ++i) {
            const int64_t sl = find_slot(h, ids[i]);
            if (sl < 0 || (!asc && !seen.insert(ids[i]).second))
                fail(SINE_ENOTFOUND, "unknown id " + std::to_string(ids[i]));
            slots.push_back(sl);
        }
        remove_slots(h, slots);
    });
}

int sine_size(sine_index_t* h, int64_t* live, int64_t* slots) {
    return guarded([&] {
        std::lock_guard<std::mutex> g(h->mu);
        if (live) *live = h->nlive;
        if (slots) *slots = h->nslots;
    });
}

int sine_ids(sine_index_t* h, int64_t* out, int64_t cap, int64_t* n) {
    return guarded([&] {
        std::lock_guard<std::mutex> g(h->mu);
        order_flush(h);
        const int64_t m = static_cast<int64_t>(h->order_slot.size());
        for (int64_t j = 0; j < std::min(m, cap); ++j) out[j] = h->ids_h[h->order_slot[j]];
        *n = m;
    });
}

int sine_get_rows(sine_index_t* h, int64_t n, const int64_t* ids, double* out) {
    return guarded([&] {
        if (n <= 0) return;
        std::lock_guard<std::mutex> g(h->mu);
        CK(cudaSetDevice(h->device));
        ws_acquire(h, h->stream);
        std::vector<int64_t> slots(n);
        for (int64_t i = 0; i < n; ++i) {
            slots[i] = find_slot(h, ids[i]);
            if (slots[i] < 0) fail(SINE_ENOTFOUND, "unknown id " + std::to_string(ids[i]));
        }
        gather_rows_host(h, n, slots.data(), out);
    });
}

int sine_snapshot(sine_index_t* h, int64_t cap, int64_t* ids, double* rows, int64_t* n) {
    return guarded([&] {
        std::lock_guard<std::mutex> g(h->mu);
        CK(cudaSetDevice(h->device));
        ws_acquire(h, h->stream);
        order_flush(h);
        const int64_t m = static_cast<int64_t>(h->order_slot.size());
        *n = m;
        if (m > cap) fail(SINE_EINVAL, "snapshot buffers hold " + std::to_string(cap) + " rows, need " +
                                           std::to_string(m));
        for (int64_t j = 0; j < m; ++j) ids[j] = h->ids_h[h->order_slot[j]];
        gather_rows_host(h, m, h->order_slot.data(), rows);
    });
}

int sine_query(sine_index_t* h, int64_t B, const double* q, int k, double min_sim, uint32_t mode, int64_t* out_ids,
               double* out_sims, int32_t* out_counts) {
    return guarded([&] {
        if (B <= 0) return;
        if (k < 1) fail(SINE_EINVAL, "k must be >= 1");
        if (!(mode & SINE_NO_NORM_CHECK)) check_queries_host(h, B, q);
        std::lock_guard<std::mutex> g(h->mu);
        CK(cudaSetDevice(h->device));
        ws_acquire(h, h->stream);
        h->q64.ensure(B * h->dim);
        h->o_ids.ensure(B * k);
        h->o_sims.ensure(B * k);
        h->o_cnt.ensure(B);
        CK(cudaMemcpyAsync(h->q64.p, q, B * h->dim * sizeof(double), cudaMemcpyHostToDevice, h->stream));
        const bool certify = (mode & SINE_RERANK_F64) && (h->flags & SINE_STORE_F32) && h->nlive > 0;
        if (h->nlive > 0) {
            // results (and certificates) written by the merge kernel straight
            // into pinned, device-mapped staging: one host sync, no copies
            h->ids_zc.ensure(B * k);
            h->sims_zc.ensure(B * k);
            h->cnt_zc.ensure(B);
            if (certify) h->cert_h.ensure(B);
            int64_t* d_ids;
            double* d_sims;
            int32_t* d_cnt;
            uint8_t* d_cert = nullptr;
            CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&d_ids), h->ids_zc.p, 0));
            CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&d_sims), h->sims_zc.p, 0));
            CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&d_cnt), h->cnt_zc.p, 0));
            if (certify) CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&d_cert), h->cert_h.p, 0));
            {
                struct Reset {
                    sine_index* h;
                    ~Reset() { h->cert_out = nullptr; }
                } reset{h};
                h->cert_out = d_cert;
                query_device_impl(h, B, h->q64.p, k, min_sim, mode, d_ids, d_sims, d_cnt, h->stream);
            }
            CK(cudaStreamSynchronize(h->stream));
            h->uncertified = 0;
            if (certify)  // re-runs write the same mapped staging, synchronised
                h->uncertified = certify_and_fix(h, B, h->q64.p, k, min_sim, mode, d_ids, d_sims, d_cnt, h->stream,
                                                 h->cert_h.p);
            std::memcpy(out_ids, h->ids_zc.p, B * k * sizeof(int64_t));
            std::memcpy(out_sims, h->sims_zc.p, B * k * sizeof(double));
            std::memcpy(out_counts, h->cnt_zc.p, B * sizeof(int32_t));
            if (h->timing) scan_merge_times(h);
            return;
        }
        query_device_impl(h, B, h->q64.p, k, min_sim, mode, h->o_ids.p, h->o_sims.p, h->o_cnt.p, h->stream);
        // results and certificates come back together: one host sync in the
        // common (all certified) case
        if (certify) {
            h->cert_h.ensure(B);
            CK(cudaMemcpyAsync(h->cert_h.p, h->cert.p, B, cudaMemcpyDeviceToHost, h->stream));
        }
        CK(cudaMemcpyAsync(out_ids, h->o_ids.p, B * k * sizeof(int64_t), cudaMemcpyDeviceToHost, h->stream));
        CK(cudaMemcpyAsync(out_sims, h->o_sims.p, B * k * sizeof(double), cudaMemcpyDeviceToHost, h->stream));
        CK(cudaMemcpyAsync(out_counts, h->o_cnt.p, B * sizeof(int32_t), cudaMemcpyDeviceToHost, h->stream));
        CK(cudaStreamSynchronize(h->stream));
        h->uncertified = 0;
        if (certify) {
            h->uncertified = certify_and_fix(h, B, h->q64.p, k, min_sim, mode, h->o_ids.p, h->o_sims.p, h->o_cnt.p,
                                             h->stream, h->cert_h.p);
            if (h->uncertified) {
                CK(cudaMemcpyAsync(out_ids, h->o_ids.p, B * k * sizeof(int64_t), cudaMemcpyDeviceToHost, h->stream));
                CK(cudaMemcpyAsync(out_sims, h->o_sims.p, B * k * sizeof(double), cudaMemcpyDeviceToHost,
                                   h->stream));
                CK(cudaMemcpyAsync(out_counts, h->o_cnt.p, B * sizeof(int32_t), cudaMemcpyDeviceToHost, h->stream));
                CK(cudaStreamSynchronize(h->stream));
            }
        }
        if (h->timing) scan_merge_times(h);
    });
}

int sine_query_submit(sine_index_t* h, int64_t B, const double* q, int k, double min_sim, uint32_t mode,
                      int64_t* out_ids, double* out_sims, int32_t* out_counts, int64_t* ticket) {
    return guarded([&] {
        if (B <= 0) fail(SINE_EINVAL, "empty batch");
        if (k < 1) fail(SINE_EINVAL, "k must be >= 1");
        if (!(mode & SINE_NO_NORM_CHECK)) check_queries_host(h, B, q);
        std::lock_guard<std::mutex> g(h->mu);
        CK(cudaSetDevice(h->device));
        ws_acquire(h, h->stream);
        size_t slot = 0;
        while (slot < h->tickets.size() && h->tickets[slot].busy) ++slot;
        if (slot == h->tickets.size()) {
            if (slot >= 16) fail(SINE_EINVAL, "too many queries in flight (max 16)");
            h->tickets.emplace_back();
            CK(cudaEventCreateWithFlags(&h->tickets[slot].done, cudaEventDisableTiming));
        }
        auto& t = h->tickets[slot];
        h->q64.ensure(B * h->dim);
        h->o_ids.ensure(B * k);
        h->o_sims.ensure(B * k);
        h->o_cnt.ensure(B);
        CK(cudaMemcpyAsync(h->q64.p, q, B * h->dim * sizeof(double), cudaMemcpyHostToDevice, h->stream));
        t.certify = (mode & SINE_RERANK_F64) && (h->flags & SINE_STORE_F32) && h->nlive > 0;
        if (t.certify) t.cert.ensure(B);
        t.nslots = h->nslots;
        t.valid_snap.reset();
        t.zero_copy = h->nlive > 0;
        if (t.zero_copy) {
            // results land in this ticket's pinned staging (mapped into the
            // device address space); sine_query_wait copies them out
            t.sids.ensure(B * k);
            t.ssims.ensure(B * k);
            t.scnt.ensure(B);
            int64_t* d_ids;
            double* d_sims;
            int32_t* d_cnt;
            uint8_t* d_cert = nullptr;
            CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&d_ids), t.sids.p, 0));
            CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&d_sims), t.ssims.p, 0));
            CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&d_cnt), t.scnt.p, 0));
            if (t.certify) CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&d_cert), t.cert.p, 0));
            struct Reset {
                sine_index* h;
                ~Reset() { h->cert_out = nullptr; }
            } reset{h};
            h->cert_out = d_cert;
            query_device_impl(h, B, h->q64.p, k, min_sim, mode, d_ids, d_sims, d_cnt, h->stream);
        } else {
            query_device_impl(h, B, h->q64.p, k, min_sim, mode, h->o_ids.p, h->o_sims.p, h->o_cnt.p, h->stream);
            if (t.certify) CK(cudaMemcpyAsync(t.cert.p, h->cert.p, B, cudaMemcpyDeviceToHost, h->stream));
            CK(cudaMemcpyAsync(out_ids, h->o_ids.p, B * k * sizeof(int64_t), cudaMemcpyDeviceToHost, h->stream));
            CK(cudaMemcpyAsync(out_sims, h->o_sims.p, B * k * sizeof(double), cudaMemcpyDeviceToHost, h->stream));
            CK(cudaMemcpyAsync(out_counts, h->o_cnt.p, B * sizeof(int32_t), cudaMemcpyDeviceToHost, h->stream));
        }
        CK(cudaEventRecord(t.done, h->stream));
        t.busy = true;
        t.B = B, t.k = k, t.min_sim = min_sim, t.mode = mode;
        t.q = q, t.ids = out_ids, t.sims = out_sims, t.counts = out_counts;
        *ticket = static_cast<int64_t>(slot);
    });
}

int sine_query_wait(sine_index_t* h, int64_t ticket) {
    return guarded([&] {
        cudaEvent_t ev;
        {
            std::lock_guard<std::mutex> g(h->mu);
            if (ticket < 0 || ticket >= static_cast<int64_t>(h->tickets.size()) || !h->tickets[ticket].busy)
                fail(SINE_EINVAL, "unknown query ticket");
            ev = h->tickets[ticket].done;
        }
        CK(cudaEventSynchronize(ev));  // without the handle lock: other calls proceed
        std::lock_guard<std::mutex> g(h->mu);
        CK(cudaSetDevice(h->device));
        ws_acquire(h, h->stream);
        auto& t = h->tickets[ticket];
        t.busy = false;
        h->uncertified = 0;
        if (t.zero_copy) {
            std::memcpy(t.ids, t.sids.p, t.B * t.k * sizeof(int64_t));
            std::memcpy(t.sims, t.ssims.p, t.B * t.k * sizeof(double));
            std::memcpy(t.counts, t.scnt.p, t.B * sizeof(int32_t));
        }
        struct Retire {  // the ticket's snapshot goes; a deferred compaction may run
            sine_index* h;
            sine_index::Ticket& t;
            ~Retire() {
                t.valid_snap.reset();
                if (h->compact_pending) try {
                        maybe_compact(h);
                    } catch (...) {
                    }
            }
        } retire{h, t};
        if (!t.certify) return;
        // uncertified queries are re-run on the fp32 CUDA-core scan (2e-6
        // error bound) against the SUBMIT-time store -- the slots that
        // existed then and the bitmap of that moment -- in one batch, from
        // the caller's host copy of the queries (the device workspace may
        // already hold a later batch)
        std::vector<int64_t> redo;
        for (int64_t b = 0; b < t.B; ++b)
            if (!t.cert.p[b]) redo.push_back(b);
        if (redo.empty()) return;
        const int64_t R = static_cast<int64_t>(redo.size());
        std::vector<double> qh(R * h->dim);
        for (int64_t r = 0; r < R; ++r)
            std::memcpy(qh.data() + r * h->dim, t.q + redo[r] * h->dim, h->dim * sizeof(double));
        DevBuf<double> q1;
        DevBuf<int64_t> i1;
        DevBuf<double> s1;
        DevBuf<int32_t> c1;
        q1.ensure(R * h->dim), i1.ensure(R * t.k), s1.ensure(R * t.k), c1.ensure(R);
        CK(cudaMemcpyAsync(q1.p, qh.data(), R * h->dim * 8, cudaMemcpyHostToDevice, h->stream));
        {
            struct Snap {
                sine_index* h;
                ~Snap() { h->snap_nslots = -1, h->snap_valid = nullptr; }
            } snap{h};
            h->snap_nslots = t.nslots;
            h->snap_valid = t.valid_snap ? t.valid_snap->p : nullptr;
            query_device_impl(h, R, q1.p, t.k, t.min_sim, SINE_SCAN_F32 | SINE_RERANK_F64 | SINE_SCAN_CUDA_CORE, i1.p,
                              s1.p, c1.p, h->stream);
        }
        std::vector<int64_t> ih(R * t.k);
        std::vector<double> sh(R * t.k);
        std::vector<int32_t> ch(R);
        CK(cudaMemcpyAsync(ih.data(), i1.p, R * t.k * 8, cudaMemcpyDeviceToHost, h->stream));
        CK(cudaMemcpyAsync(sh.data(), s1.p, R * t.k * 8, cudaMemcpyDeviceToHost, h->stream));
        CK(cudaMemcpyAsync(ch.data(), c1.p, R * 4, cudaMemcpyDeviceToHost, h->stream));
        CK(cudaStreamSynchronize(h->stream));
        for (int64_t r = 0; r < R; ++r) {
            const int64_t b = redo[r];
            std::memcpy(t.ids + b * t.k, ih.data() + r * t.k, t.k * 8);
            std::memcpy(t.sims + b * t.k, sh.data() + r * t.k, t.k * 8);
            t.counts[b] = ch[r];
        }
        h->uncertified = R;
        q1.release(), i1.release(), s1.release(), c1.release();
    });
}

int sine_query_device(sine_index_t* h, int64_t B, const double* q_dev, int k, double min_sim, uint32_t mode,
                      int64_t* ids_dev, double* sims_dev, int32_t* counts_dev, void* stream) {
    return guarded([&] {
        std::lock_guard<std::mutex> g(h->mu);
        CK(cudaSetDevice(h->device));
        
        cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : h->stream;
        ws_acquire(h, st);
        query_device_impl(h, B, q_dev, k, min_sim, mode, ids_dev, sims_dev, counts_dev, st);
        if (mode & SINE_CERTIFY)
            h->uncertified = certify_and_fix(h, B, q_dev, k, min_sim, mode, ids_dev, sims_dev, counts_dev, st);
        ws_release(h, st);
    });
}

int sine_query_device_cert(sine_index_t* h, int64_t B, const double* q_dev, int k, double min_sim, uint32_t mode,
                           int64_t* ids_dev, double* sims_dev, int32_t* counts_dev, uint8_t* cert_dev,
                           void* stream) {
    return guarded([&] {
        std::lock_guard<std::mutex> g(h->mu);
        CK(cudaSetDevice(h->device));
        
        cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : h->stream;
        ws_acquire(h, st);
        struct Reset {
            sine_index* h;
            ~Reset() { h->cert_out = nullptr; }
        } reset{h};
        h->cert_out = cert_dev;
        if (h->nlive == 0 || !(mode & SINE_RERANK_F64))  // nothing to prove: every answer is exact
            CK(cudaMemsetAsync(cert_dev, 1, B, st));
        query_device_impl(h, B, q_dev, k, min_sim, mode & ~SINE_CERTIFY, ids_dev, sims_dev, counts_dev, st);
        ws_release(h, st);
    });
}

int sine_update_meta(sine_index_t* h, int64_t n, const int64_t* ids, const double* log_freq,
                     const int64_t* frequency, const double* last_access) {
    return guarded([&] {
        if (n <= 0) return;
        std::lock_guard<std::mutex> g(h->mu);
        if (!(h->flags & SINE_STORE_META)) fail(SINE_EINVAL, "index has no LCFU metadata");
        CK(cudaSetDevice(h->device));
        ws_acquire(h, h->stream);
        std::vector<int64_t> slots(n);
        for (int64_t i = 0; i < n; ++i) {
            slots[i] = find_slot(h, ids[i]);
            if (slots[i] < 0) fail(SINE_ENOTFOUND, "unknown id " + std::to_string(ids[i]));
        }
        if (n == 1) {
            const int64_t s = slots[0];
            CK(cudaMemcpyAsync(h->lf + s, log_freq, sizeof(double), cudaMemcpyHostToDevice, h->stream));
            CK(cudaMemcpyAsync(h->freq + s, frequency, sizeof(int64_t), cudaMemcpyHostToDevice, h->stream));
            CK(cudaMemcpyAsync(h->last_access + s, last_access, sizeof(double), cudaMemcpyHostToDevice, h->stream));
        } else {
            DevBuf<int64_t> ds, dfq;
            DevBuf<double> dlf, dla;
            ds.ensure(n), dfq.ensure(n), dlf.ensure(n), dla.ensure(n);
            CK(cudaMemcpyAsync(ds.p, slots.data(), n * 8, cudaMemcpyHostToDevice, h->stream));
            CK(cudaMemcpyAsync(dlf.p, log_freq, n * 8, cudaMemcpyHostToDevice, h->stream));
            CK(cudaMemcpyAsync(dfq.p, frequency, n * 8, cudaMemcpyHostToDevice, h->stream));
            CK(cudaMemcpyAsync(dla.p, last_access, n * 8, cudaMemcpyHostToDevice, h->stream));
            scatter_meta_kernel<<<grid_for(n, 256, h->num_sms), 256, 0, h->stream>>>(ds.p, n, dlf.p, dfq.p, dla.p,
                                                                                      h->lf, h->freq, h->last_access);
            ++h->launches;
            CK(cudaGetLastError());
            CK(cudaStreamSynchronize(h->stream));
        }
        CK(cudaStreamSynchronize(h->stream));
    });
}

int sine_expired(sine_index_t* h, double now, int remove, int64_t* out, int64_t cap, int64_t* n) {
    return guarded([&] {
        std::lock_guard<std::mutex> g(h->mu);
        if (!(h->flags & SINE_STORE_META)) fail(SINE_EINVAL, "index has no LCFU metadata");
        CK(cudaSetDevice(h->device));
        ws_acquire(h, h->stream);
        *n = 0;
        if (h->nlive == 0) return;
        const int nb = static_cast<int>((h->nslots + kExpChunk - 1) / kExpChunk);
        h->scratch_i32.ensure(nb);
        h->exp_off.ensure(nb + 1);
        h->cnt_h.ensure(2);
        expire_count_kernel<<<nb, 256, 0, h->stream>>>(h->expiration, h->valid, h->nslots, now, h->scratch_i32.p);
        expire_scan_kernel<<<1, 1024, 0, h->stream>>>(h->scratch_i32.p, nb, h->exp_off.p);
        h->launches += 2;
        CK(cudaGetLastError());
        int64_t total = 0;
        CK(cudaMemcpyAsync(&total, h->exp_off.p + nb, sizeof(int64_t), cudaMemcpyDeviceToHost, h->stream));
        CK(cudaStreamSynchronize(h->stream));
        *n = total;
        if (total == 0) return;
        if (total > cap) fail(SINE_EINVAL, "output buffer too small for expired ids");
        h->vids.ensure(total);
        h->vslots.ensure(total);
        expire_write_kernel<<<nb, 256, 0, h->stream>>>(h->expiration, h->valid, h->ids, h->nslots, now,
                                                       h->exp_off.p, h->vids.p, h->vslots.p);
        ++h->launches;
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(out, h->vids.p, total * 8, cudaMemcpyDeviceToHost, h->stream));
        int32_t* slots = nullptr;  // pinned staging: the host tables drop these slots
        h->cnt_h.ensure(total);    // sized by listing calls too: a later purge finds it ready
        if (remove) {
            slots = h->cnt_h.p;
            CK(cudaMemcpyAsync(slots, h->vslots.p, total * 4, cudaMemcpyDeviceToHost, h->stream));
        }
        CK(cudaStreamSynchronize(h->stream));
        if (!h->ids_ascending) std::sort(out, out + total);
        if (remove) {
            // tombstone on the device straight from the slot list
            snapshot_bitmap_for_tickets(h);
            set_bits32_kernel<<<grid_for(total, 256, h->num_sms), 256, 0, h->stream>>>(h->valid, h->vslots.p, total);
            ++h->launches;
            CK(cudaGetLastError());
            CK(cudaStreamSynchronize(h->stream));
            // the reference removes sorted(expired): with slots in id order the
            // slot list already is that order (no copy, no sort)
            std::vector<int32_t> by_id;
            const int32_t* order = slots;
            if (!h->ids_ascending) {
                by_id.assign(slots, slots + total);
                std::sort(by_id.begin(), by_id.end(),
                          [&](int32_t a, int32_t b) { return h->ids_h[a] < h->ids_h[b]; });
                order = by_id.data();
                for (int64_t i = 0; i < total; ++i) h->pos.erase(h->ids_h[order[i]]);
            }
            uint8_t* live = h->live_h.data();
            for (int64_t i = 0; i < total; ++i) live[order[i]] = 0;
            h->order_log.reserve(h->order_log.size() + total);
            for (int64_t i = 0; i < total; ++i) order_removed(h, order[i]);
            h->nlive -= total;
            maybe_compact(h);
        }
    });
}

int sine_select_victims(sine_index_t* h, int policy, double now, int64_t excess, int64_t* out, int64_t cap,
                        int64_t* n) {
    return guarded([&] {
        if (policy < 0 || policy > 2) fail(SINE_EINVAL, "unknown eviction policy");
        std::lock_guard<std::mutex> g(h->mu);
        CK(cudaSetDevice(h->device));
        ws_acquire(h, h->stream);
        select_victims_impl(h, policy, now, excess, out, cap, n);
    });
}

int sine_stream(sine_index_t* h, void** stream) {
    return guarded([&] { *stream = h->stream; });
}

int sine_evict(sine_index_t* h, int policy, double now, int64_t excess, int64_t* out, int64_t cap, int64_t* n) {
    return guarded([&] {
        if (policy < 0 || policy > 2) fail(SINE_EINVAL, "unknown eviction policy");
        std::lock_guard<std::mutex> g(h->mu);
        CK(cudaSetDevice(h->device));
        ws_acquire(h, h->stream);
        select_victims_impl(h, policy, now, excess, out, cap, n, true);
    });
}

int sine_set_select_cap(sine_index_t* h, int cap) {
    return guarded([&] {
        if (cap < 2 || cap > kSelCap) fail(SINE_EINVAL, "select cap must be in [2, 6144]");
        std::lock_guard<std::mutex> g(h->mu);
        h->sel_cap = cap;
    });
}

int sine_set_timing(sine_index_t* h, int on) {
    return guarded([&] { h->timing = on != 0; });
}

int sine_last_timing(sine_index_t* h, float* scan_ms, float* merge_ms, float* evict_ms) {
    return guarded([&] {
        if (scan_ms) *scan_ms = h->t_scan;
        if (merge_ms) *merge_ms = h->t_merge;
        if (evict_ms) *evict_ms = h->t_evict;
    });
}

int sine_timing_totals(sine_index_t* h, int kind, double* total_ms, int64_t* launches, int reset) {
    return guarded([&] {
        std::lock_guard<std::mutex> g(h->mu);
        double tot = 0.0;
        int64_t n = 0;
        for (size_t i = 0; i < h->tused; ++i) {
            auto& t = h->tpool[i];
            if (t.kind != kind) continue;
            CK(cudaEventSynchronize(t.b));
            float ms = 0.f;
            CK(cudaEventElapsedTime(&ms, t.a, t.b));
            tot += ms;
            ++n;
        }
        *total_ms = tot;
        *launches = n;
        if (reset) h->tused = 0;
    });
}

int sine_copy_certificates(sine_index_t* h, int64_t B, void* dst_dev, void* stream) {
    return guarded([&] {
        std::lock_guard<std::mutex> g(h->mu);
        if (!h->cert.p || static_cast<int64_t>(h->cert.n) < B) fail(SINE_EINVAL, "no certificates for that batch");
        cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : h->stream;
        CK(cudaMemcpyAsync(dst_dev, h->cert.p, B, cudaMemcpyDeviceToDevice, st));
    });
}

int sine_uncertified(sine_index_t* h, int64_t* n) {
    return guarded([&] { *n = h->uncertified; });
}

int sine_gemm_overflows(sine_index_t* h, int64_t* n) {
    return guarded([&] { *n = h->gemm_overflows; });
}

int sine_kernel_launches(sine_index_t* h, int64_t* n) {
    return guarded([&] { *n = h->launches; });
}

int sine_merge_shards(int device, int P, int64_t B, int k, const int64_t* ids_dev, const double* sims_dev,
                      int64_t rank_stride, int64_t* out_ids, double* out_sims, int32_t* out_counts, void* stream) {
    return guarded([&] {
        if (P < 1 || B < 0 || k < 1) fail(SINE_EINVAL, "bad shard merge shape");
        if (B == 0) return;
        const size_t smem = static_cast<size_t>(P) * k * 16;
        if (smem > 160 * 1024) fail(SINE_EINVAL, "P * k too large for the shard merge");
        CK(cudaSetDevice(device));
        smem_optin(reinterpret_cast<const void*>(shard_merge_kernel), 160 * 1024);
        shard_merge_kernel<<<static_cast<unsigned>(B), kShardMergeThreads, smem, static_cast<cudaStream_t>(stream)>>>(
            ids_dev, sims_dev, P, B, k, rank_stride ? rank_stride : B * k, out_ids, out_sims, out_counts);
        CK(cudaGetLastError());
    });
}

uint64_t sine_blake2b64(const uint8_t* msg, int64_t len, uint64_t key) { return blake2b64_keyed(msg, len, key); }

int sine_embed_hashed_bag(int device, uint64_t seed, int64_t dim, const uint8_t* tok_bytes, int64_t nbytes,
                          const int64_t* tok_off, int64_t ntok, const int64_t* q_off, int64_t B, double* out_rows) {
    return guarded([&] {
        if (dim < 1 || B < 0 || ntok < 0) fail(SINE_EINVAL, "bad embedding batch shape");
        if (B == 0) return;
        for (int64_t b = 0; b < B; ++b)
            if (q_off[b + 1] <= q_off[b]) fail(SINE_EINVAL, "cannot embed text with no tokens");
        if (q_off[0] != 0 || q_off[B] != ntok) fail(SINE_EINVAL, "query token ranges do not cover the tokens");
        CK(cudaSetDevice(device));
        std::vector<int32_t> tok_q(ntok);
        for (int64_t b = 0; b < B; ++b)
            for (int64_t t = q_off[b]; t < q_off[b + 1]; ++t) tok_q[t] = static_cast<int32_t>(b);
        DevBuf<uint8_t> dbytes;
        DevBuf<int64_t> doff;
        DevBuf<int32_t> dq;
        DevBuf<double> dcounts;
        dbytes.ensure(std::max<int64_t>(nbytes, 1));
        doff.ensure(ntok + 1);
        dq.ensure(std::max<int64_t>(ntok, 1));
        dcounts.ensure(B * dim);
        cudaStream_t st = nullptr;
        CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
        if (nbytes) CK(cudaMemcpyAsync(dbytes.p, tok_bytes, nbytes, cudaMemcpyHostToDevice, st));
        CK(cudaMemcpyAsync(doff.p, tok_off, (ntok + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, st));
        CK(cudaMemcpyAsync(dq.p, tok_q.data(), ntok * sizeof(int32_t), cudaMemcpyHostToDevice, st));
        CK(cudaMemsetAsync(dcounts.p, 0, B * dim * sizeof(double), st));
        embed_count_kernel<<<grid_for(ntok, 128, 148), 128, 0, st>>>(dbytes.p, doff.p, ntok, dq.p, seed, dim,
                                                                      dcounts.p);
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(out_rows, dcounts.p, B * dim * sizeof(double), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        CK(cudaStreamDestroy(st));
        // counts / (sum(c * c) ** 0.5): integer-valued sums are exact in any
        // order; the power is taken with the host libm like CPython's x ** 0.5
        for (int64_t b = 0; b < B; ++b) {
            double* r = out_rows + b * dim;
            double ss = 0.0;
            for (int64_t j = 0; j < dim; ++j) ss += r[j] * r[j];
            const double norm = std::pow(ss, 0.5);
            for (int64_t j = 0; j < dim; ++j) r[j] = r[j] / norm;
        }
    });
}

int64_t sine_hex_bound(int64_t n, int64_t d, int with_ids) {
    return n * ((with_ids ? hexio::kMaxId : 0) + d * (hexio::kMaxTok + 1) + 1);
}

int sine_hex_format(const int64_t* ids, const double* rows, int64_t n, int64_t d, char* out, int64_t cap,
                    int64_t* len) {
    return guarded([&] {
        if (n < 0 || d < 1) fail(SINE_EINVAL, "bad row block shape");
        if (cap < sine_hex_bound(n, d, ids != nullptr)) fail(SINE_EINVAL, "output buffer below sine_hex_bound");
        *len = n ? hexio::format_rows(ids, rows, n, d, out) : 0;
    });
}

int sine_hex_parse(const char* text, int64_t len, int64_t n, int64_t d, int64_t* ids, double* rows) {
    return guarded([&] {
        if (n < 0 || d < 1) fail(SINE_EINVAL, "bad row block shape");
        const std::string err = hexio::parse_rows(text, len, n, d, ids, rows);
        if (!err.empty()) fail(SINE_EINVAL, "snapshot " + err);
    });
}

int sine_host_alloc(size_t bytes, void** p) {
    return guarded([&] { CK(cudaMallocHost(p, bytes)); });
}

int sine_host_free(void* p) {
    return guarded([&] { CK(cudaFreeHost(p)); });
}

}  // extern "C"
