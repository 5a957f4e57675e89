#include "runtime.h"

#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstdlib>

#include "kernels.h"

namespace h2f {

namespace {
Context* g_ctx = nullptr;
std::atomic<int64_t> g_launches{0};
constexpr size_t ALIGN = 256;
inline size_t align_up(size_t x) { return (x + ALIGN - 1) & ~(ALIGN - 1); }
}  // namespace

void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
int64_t kernel_launch_count() { return g_launches.load(); }
void add_launches(int64_t n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

// ---------------------------------------------------------------- Arena
void Arena::init(size_t bytes) {
    bytes &= ~(ALIGN - 1);
    void* p = nullptr;
    H2F_CUDA(cudaMalloc(&p, bytes));
    base_ = static_cast<char*>(p);
    cap_ = bytes;
    free_.clear();
    used_.clear();
    free_[0] = bytes;
}

void* Arena::alloc(size_t bytes) {
    bytes = align_up(bytes ? bytes : 1);
    for (auto it = free_.begin(); it != free_.end(); ++it) {
        if (it->second >= bytes) {
            const size_t off = it->first, sz = it->second;
            free_.erase(it);
            if (sz > bytes) free_[off + bytes] = sz - bytes;
            used_[off] = bytes;
            in_use_ += bytes;
            peak_ = std::max(peak_, in_use_);
            return base_ + off;
        }
    }
    throw Error(H2F_E_NOMEM, "device arena exhausted: need " + std::to_string(bytes) + " B, in use " +
                                 std::to_string(in_use_) + " of " + std::to_string(cap_));
}

void Arena::free(void* p) {
    if (!p) return;
    const size_t off = static_cast<char*>(p) - base_;
    auto u = used_.find(off);
    if (u == used_.end()) throw Error(H2F_E_INTERNAL, "arena free of unknown pointer");
    size_t sz = u->second;
    used_.erase(u);
    in_use_ -= sz;
    size_t start = off;
    auto next = free_.lower_bound(off);
    if (next != free_.begin()) {
        auto prev = std::prev(next);
        if (prev->first + prev->second == off) {
            start = prev->first;
            sz += prev->second;
            free_.erase(prev);
        }
    }
    next = free_.lower_bound(start + sz);
    if (next != free_.end() && next->first == start + sz) {
        sz += next->second;
        free_.erase(next);
    }
    free_[start] = sz;
}

// ---------------------------------------------------------------- Region
Region& Region::operator=(Region&& o) noexcept {
    if (this != &o) {
        release();
        chunk_ = o.chunk_;
        chunks_ = std::move(o.chunks_);
        cur_ = o.cur_;
        off_ = o.off_;
        used_ = o.used_;
        o.chunks_.clear();
        o.cur_ = o.off_ = o.used_ = 0;
    }
    return *this;
}

void* Region::alloc(size_t bytes) {
    bytes = align_up(bytes ? bytes : 1);
    while (cur_ < chunks_.size()) {
        auto& c = chunks_[cur_];
        if (off_ + bytes <= c.second) {
            void* p = c.first + off_;
            off_ += bytes;
            used_ += bytes;
            return p;
        }
        ++cur_;
        off_ = 0;
    }
    const size_t sz = std::max(chunk_, bytes);
    char* p = static_cast<char*>(ctx().arena.alloc(sz));
    chunks_.push_back({p, sz});
    cur_ = chunks_.size() - 1;
    off_ = bytes;
    used_ += bytes;
    return p;
}

void Region::release() {
    if (g_ctx)
        for (auto& c : chunks_) g_ctx->arena.free(c.first);
    chunks_.clear();
    cur_ = off_ = used_ = 0;
}

void Region::reset() {
    cur_ = 0;
    off_ = 0;
    used_ = 0;
}

// ---------------------------------------------------------------- Uploader
void* Uploader::put_bytes(const void* src, size_t bytes) {
    void* host = nullptr;
    void* d = reserve_bytes(bytes, &host);
    if (bytes >= (size_t(2) << 20)) {
        // large task arrays (a leaf-level Schur launch carries ~1e5 tasks):
        // the staging copy into pinned memory in parallel slices
        const int64_t nsl = int64_t(std::min<size_t>(16, bytes >> 19));
#pragma omp parallel for schedule(static)
        for (int64_t q = 0; q < nsl; ++q) {
            const size_t lo = bytes * size_t(q) / size_t(nsl), hi = bytes * size_t(q + 1) / size_t(nsl);
            std::memcpy(static_cast<char*>(host) + lo, static_cast<const char*>(src) + lo, hi - lo);
        }
    } else if (bytes) {
        std::memcpy(host, src, bytes);
    }
    return d;
}

void* Uploader::reserve_bytes(size_t bytes, void** host) {
    const size_t need = align_up(bytes ? bytes : 1);
    if (chunks_.empty() || used_ + need > chunks_[cur_].cap) {
        if (!chunks_.empty()) {
            flush(ctx().stream);  // what was put into this chunk must ship first
            ++cur_;
        }
        while (cur_ < chunks_.size() && chunks_[cur_].cap < need) ++cur_;
        if (cur_ >= chunks_.size()) {
            Chunk c;
            c.cap = std::max<size_t>(size_t(16) << 20, need * 2);
            H2F_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&c.host), c.cap, cudaHostAllocDefault));
            c.dev = static_cast<char*>(ctx().arena.alloc(c.cap));
            chunks_.push_back(c);
            cur_ = chunks_.size() - 1;
        }
        used_ = flushed_ = 0;
    }
    Chunk& c = chunks_[cur_];
    *host = c.host + used_;
    void* d = c.dev + used_;
    used_ += need;
    return d;
}

void Uploader::flush(cudaStream_t st) {
    if (cur_ >= chunks_.size() || used_ == flushed_) return;
    Chunk& c = chunks_[cur_];
    H2F_CUDA(cudaMemcpyAsync(c.dev + flushed_, c.host + flushed_, used_ - flushed_,
                             cudaMemcpyHostToDevice, st));
    flushed_ = used_;
}

void Uploader::reset() {
    cur_ = 0;
    used_ = flushed_ = 0;
}

Uploader::~Uploader() {
    for (auto& c : chunks_) cudaFreeHost(c.host);
}

// ---------------------------------------------------------------- Profiler
const char* kernel_name(int kid) {
    static const char* names[K_COUNT] = {
        "gemm_augment", "gemm_project", "gemm_schur", "gemm_fill_create", "gemm_top_update", "copy_tasks",
        "qr_r", "jacobi_svd", "complement", "lu_redundant", "trsm_eliminator", "norm_reduce", "top_panel_lu",
        "top_misc", "solve_fwd_clusters", "solve_fwd_scatter", "solve_bwd_clusters", "solve_top",
        "solve_misc", "matvec_gemv", "vector_ops", "qr_r_blocked", "jacobi_svd_coop", "complement_v"};
    return (kid >= 0 && kid < K_COUNT) ? names[kid] : "?";
}

cudaEvent_t Profiler::get_event() {
    if (!pool_.empty()) {
        cudaEvent_t e = pool_.back();
        pool_.pop_back();
        return e;
    }
    cudaEvent_t e;
    H2F_CUDA(cudaEventCreate(&e));
    return e;
}

int Profiler::begin(int kid, double flops, double bytes, double units) {
    if (!on || kid < 0) return -1;
    Rec r{kid, get_event(), get_event(), flops, bytes, units};
    H2F_CUDA(cudaEventRecord(r.a, ctx().stream));
    pending_.push_back(r);
    return int(pending_.size()) - 1;
}

void Profiler::end(int slot) {
    if (slot < 0 || slot >= int(pending_.size())) return;
    H2F_CUDA(cudaEventRecord(pending_[slot].b, ctx().stream));
}

void Profiler::collect() {
    if (pending_.empty()) return;
    H2F_CUDA(cudaStreamSynchronize(ctx().stream));
    // H2F_PROF_LOG=path: one line per launch "kernel flops bytes units ms" (development aid)
    static FILE* log = [] {
        const char* p = std::getenv("H2F_PROF_LOG");
        return p ? std::fopen(p, "a") : nullptr;
    }();
    for (auto& r : pending_) {
        float ms = 0.f;
        H2F_CUDA(cudaEventElapsedTime(&ms, r.a, r.b));
        if (log) std::fprintf(log, "%s %.6g %.6g %.6g %.6g\n", kernel_name(r.kid), r.flops, r.bytes, r.units, ms);
        Total& t = totals[r.kid];
        t.launches += 1;
        t.seconds += ms * 1e-3;
        t.flops += r.flops;
        t.bytes += r.bytes;
        pool_.push_back(r.a);
        pool_.push_back(r.b);
    }
    pending_.clear();
}

void Profiler::reset() {
    collect();
    for (auto& t : totals) t = Total{};
}

Profiler::~Profiler() {
    for (auto e : pool_) cudaEventDestroy(e);
}

ProfScope::ProfScope(int kid, double flops, double bytes, double units) {
    if (ctx_ready() && ctx().prof.on) slot = ctx().prof.begin(kid, flops, bytes, units);
}

ProfScope::~ProfScope() {
    if (slot >= 0) ctx().prof.end(slot);
}

// ---------------------------------------------------------------- Context
void* Context::pinned_buf(size_t bytes) {
    if (bytes > pinned_cap) {
        if (pinned) cudaFreeHost(pinned);
        pinned_cap = std::max(bytes, size_t(1) << 20);
        H2F_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&pinned), pinned_cap, cudaHostAllocDefault));
    }
    return pinned;
}

void Context::sync() {
    H2F_CUDA(cudaStreamSynchronize(stream));
    H2F_CUDA(cudaGetLastError());
    up.reset();
}

Context& ctx() {
    if (!g_ctx) throw Error(H2F_E_ARG, "h2f_init() has not been called");
    return *g_ctx;
}

bool ctx_ready() { return g_ctx != nullptr; }

void ctx_init(int device, double arena_gb) {
    if (g_ctx) {
        if (g_ctx->device != device) throw Error(H2F_E_ARG, "h2f already initialised on another device");
        return;
    }
    H2F_CUDA(cudaSetDevice(device));
    auto* c = new Context();
    c->device = device;
    H2F_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    size_t fr = 0, tot = 0;
    H2F_CUDA(cudaMemGetInfo(&fr, &tot));
    if (const char* env = std::getenv("H2F_ARENA_GB")) arena_gb = std::atof(env);
    size_t want;
    if (arena_gb > 0) want = size_t(arena_gb * double(size_t(1) << 30));
    else want = fr > (size_t(6) << 30) ? size_t(double(fr - (size_t(4) << 30)) * 0.92) : fr / 2;
    if (want > fr) want = size_t(double(fr) * 0.95);
    c->arena.init(want);
    g_ctx = c;
}

}  // namespace h2f
