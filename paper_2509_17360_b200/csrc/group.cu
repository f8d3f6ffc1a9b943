// Single-process multi-GPU stage-1: one handle over P row shards (one
// sine_index per device entry; entries may repeat a device).
//
// The reference's engine is single-process and holds ONE index
// (pkg/src/semcache/engine.py:103-109); this group lets that engine use
// every GPU of a node through the same duck type (paper_2509_17360_b200/
// multidev.py).  A query runs on all shards at once -- one persistent worker
// thread per shard: H2D of the queries, the shard's exact top-k with its
// certificate re-run (sine_query_device + SINE_CERTIFY), and a peer copy
// of its [B][k] block into the root device's gather buffer (NVLink / NVSwitch
// peer DMA between GPUs, a device copy within one) -- then the root merges
// the P blocks with sine_merge_shards by (similarity desc, id asc): the
// same order a single ExactCosineIndex.query gives (index.py:42-46, :94-102).
//
// Built only on the public C ABI (include/sine_b200.h).

#include <cuda_runtime.h>

#include <condition_variable>
#include <deque>
#include <cstring>
#include <exception>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/sine_b200.h"

extern "C" void sine_internal_set_error(const char* msg);  // capi.cu: sine_last_error()

namespace {

struct GroupError {
    int code;
    std::string msg;
};

void ck(cudaError_t e) {
    if (e != cudaSuccess) throw GroupError{SINE_ECUDA, cudaGetErrorString(e)};
}
void ok(int st) {
    if (st != SINE_OK) throw GroupError{st, sine_last_error()};
}

template <typename T>
struct DBuf {
    T* p = nullptr;
    size_t n = 0;
    void ensure(size_t want) {
        if (want <= n) return;
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
        ck(cudaMalloc(&p, want * sizeof(T)));
        n = want;
    }
    ~DBuf() {
        if (p) cudaFree(p);
    }
};

}  // namespace

struct sine_group {
    struct Shard {
        sine_index_t* h = nullptr;
        int device = 0;
        cudaStream_t stream = nullptr;
        DBuf<double> q;
        DBuf<int64_t> ids;
        DBuf<double> sims;
        DBuf<int32_t> cnt;
        std::thread worker;
        int err = SINE_OK;
        std::string msg;
    };
    std::deque<Shard> shards;  // stable addresses (workers hold references)
    int root = 0;  // device of shard 0
    cudaStream_t root_stream = nullptr;
    DBuf<int64_t> g_ids;  // [P][B][k] on the root device
    DBuf<double> g_sims;
    DBuf<int64_t> o_ids;
    DBuf<double> o_sims;
    DBuf<int32_t> o_cnt;
    int64_t dim = 0;

    // job board: one query at a time (mu_query), workers woken per job
    std::mutex mu_query;
    std::mutex mu;
    std::condition_variable cv, cv_done;
    uint64_t gen = 0;
    int pending = 0;
    bool quit = false;
    struct Job {
        int64_t B;
        const double* q;
        int k;
        double min_sim;
        uint32_t mode;
    } job{};
};

namespace {

void run_shard(sine_group* g, int p) {
    auto& s = g->shards[p];
    const auto& j = g->job;
    ck(cudaSetDevice(s.device));
    s.q.ensure(static_cast<size_t>(j.B) * g->dim);
    s.ids.ensure(static_cast<size_t>(j.B) * j.k);
    s.sims.ensure(static_cast<size_t>(j.B) * j.k);
    s.cnt.ensure(static_cast<size_t>(j.B));
    ck(cudaMemcpyAsync(s.q.p, j.q, j.B * g->dim * sizeof(double), cudaMemcpyHostToDevice, s.stream));
    // an empty shard contributes padding (id -1) only
    ck(cudaMemsetAsync(s.ids.p, 0xff, static_cast<size_t>(j.B) * j.k * sizeof(int64_t), s.stream));
    ck(cudaMemsetAsync(s.sims.p, 0, static_cast<size_t>(j.B) * j.k * sizeof(double), s.stream));
    ok(sine_query_device(s.h, j.B, s.q.p, j.k, j.min_sim, j.mode | SINE_CERTIFY, s.ids.p, s.sims.p, s.cnt.p,
                         s.stream));
    const size_t blk = static_cast<size_t>(j.B) * j.k;
    ck(cudaMemcpyPeerAsync(g->g_ids.p + p * blk, g->root, s.ids.p, s.device, blk * sizeof(int64_t), s.stream));
    ck(cudaMemcpyPeerAsync(g->g_sims.p + p * blk, g->root, s.sims.p, s.device, blk * sizeof(double), s.stream));
    ck(cudaStreamSynchronize(s.stream));
}

void worker_loop(sine_group* g, int p) {
    uint64_t seen = 0;
    for (;;) {
        {
            std::unique_lock<std::mutex> lk(g->mu);
            g->cv.wait(lk, [&] { return g->quit || g->gen != seen; });
            if (g->quit) return;
            seen = g->gen;
        }
        auto& s = g->shards[p];
        s.err = SINE_OK;
        try {
            run_shard(g, p);
        } catch (const GroupError& e) {
            s.err = e.code;
            s.msg = e.msg;
        } catch (const std::exception& e) {
            s.err = SINE_ECUDA;
            s.msg = e.what();
        }
        std::lock_guard<std::mutex> lk(g->mu);
        if (--g->pending == 0) g->cv_done.notify_all();
    }
}

template <typename F>
int group_guarded(F&& f) {
    try {
        f();
        return SINE_OK;
    } catch (const GroupError& e) {
        sine_internal_set_error(e.msg.c_str());
        return e.code;
    } catch (const std::bad_alloc&) {
        sine_internal_set_error("out of host memory");
        return SINE_ENOMEM;
    } catch (const std::exception& e) {
        sine_internal_set_error(e.what());
        return SINE_ECUDA;
    }
}

}  // namespace

extern "C" {

int sine_group_create(sine_index_t* const* shards, const int* devices, int n, int64_t dim, sine_group_t** out) {
    return group_guarded([&] {
        if (!out || !shards || !devices || n < 1 || dim < 1) throw GroupError{SINE_EINVAL, "bad group shape"};
        auto* g = new sine_group();
        g->dim = dim;
        for (int p = 0; p < n; ++p) g->shards.emplace_back();
        g->root = devices[0];
        for (int p = 0; p < n; ++p) {
            auto& s = g->shards[p];
            s.h = shards[p];
            s.device = devices[p];
            ck(cudaSetDevice(s.device));
            ck(cudaStreamCreateWithFlags(&s.stream, cudaStreamNonBlocking));
        }
        // peer access between distinct devices (NVLink / NVSwitch); copies
        // stage through the host where the driver refuses it
        for (int p = 0; p < n; ++p)
            for (int r = 0; r < n; ++r) {
                const int a = devices[p], b = devices[r];
                if (a == b) continue;
                int can = 0;
                ck(cudaDeviceCanAccessPeer(&can, a, b));
                if (!can) continue;
                ck(cudaSetDevice(a));
                const cudaError_t e = cudaDeviceEnablePeerAccess(b, 0);
                if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) ck(e);
                cudaGetLastError();
            }
        ck(cudaSetDevice(g->root));
        ck(cudaStreamCreateWithFlags(&g->root_stream, cudaStreamNonBlocking));
        for (int p = 0; p < n; ++p) g->shards[p].worker = std::thread(worker_loop, g, p);
        *out = g;
    });
}

int sine_group_destroy(sine_group_t* g) {
    return group_guarded([&] {
        if (!g) return;
        std::unique_lock<std::mutex> one(g->mu_query);  // a running query finishes first
        {
            std::lock_guard<std::mutex> lk(g->mu);
            g->quit = true;
        }
        g->cv.notify_all();
        for (auto& s : g->shards)
            if (s.worker.joinable()) s.worker.join();
        for (auto& s : g->shards) {
            cudaSetDevice(s.device);
            cudaStreamDestroy(s.stream);
        }
        cudaSetDevice(g->root);
        cudaStreamDestroy(g->root_stream);
        one.unlock();  // before the mutex goes away with the group
        delete g;
    });
}

int sine_group_query(sine_group_t* g, int64_t B, const double* q, int k, double min_sim, uint32_t mode,
                     int64_t* out_ids, double* out_sims, int32_t* out_counts) {
    return group_guarded([&] {
        if (!g) throw GroupError{SINE_EINVAL, "null group"};
        if (k < 1) throw GroupError{SINE_EINVAL, "k must be >= 1"};
        if (B <= 0) return;
        std::lock_guard<std::mutex> one(g->mu_query);
        const int P = static_cast<int>(g->shards.size());
        const size_t blk = static_cast<size_t>(B) * k;
        ck(cudaSetDevice(g->root));
        g->g_ids.ensure(P * blk);
        g->g_sims.ensure(P * blk);
        g->o_ids.ensure(blk);
        g->o_sims.ensure(blk);
        g->o_cnt.ensure(static_cast<size_t>(B));
        {
            std::lock_guard<std::mutex> lk(g->mu);
            g->job = sine_group::Job{B, q, k, min_sim, mode};
            g->pending = P;
            ++g->gen;
        }
        g->cv.notify_all();
        {
            std::unique_lock<std::mutex> lk(g->mu);
            g->cv_done.wait(lk, [&] { return g->pending == 0; });
        }
        for (auto& s : g->shards)
            if (s.err != SINE_OK) throw GroupError{s.err, "shard on device " + std::to_string(s.device) + ": " + s.msg};
        ck(cudaSetDevice(g->root));
        ok(sine_merge_shards(g->root, P, B, k, g->g_ids.p, g->g_sims.p, static_cast<int64_t>(blk), g->o_ids.p,
                             g->o_sims.p, g->o_cnt.p, g->root_stream));
        ck(cudaMemcpyAsync(out_ids, g->o_ids.p, blk * sizeof(int64_t), cudaMemcpyDeviceToHost, g->root_stream));
        ck(cudaMemcpyAsync(out_sims, g->o_sims.p, blk * sizeof(double), cudaMemcpyDeviceToHost, g->root_stream));
        ck(cudaMemcpyAsync(out_counts, g->o_cnt.p, B * sizeof(int32_t), cudaMemcpyDeviceToHost, g->root_stream));
        ck(cudaStreamSynchronize(g->root_stream));
    });
}

}  // extern "C"
