// Host runtime: device context, the workspace arena (north-star subsystem 4),
// task uploads, error plumbing.
//
// The reference allocates every block dynamically (np.hstack / dict inserts;
// the paper's prefix-sum arena, is not implemented there).  Here
// one cudaMalloc at h2f_init() reserves a slab; everything a factorization
// needs is carved out of it by exclusive scans of block-dimension products
// (Region::alloc is a bump pointer), so no device allocation happens inside
// factorize()/solve().
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <map>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/h2f.h"

namespace h2f {

struct Error : std::runtime_error {
    int code;
    int cluster = -1, level = -1;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define H2F_CUDA(call)                                                                 \
    do {                                                                               \
        cudaError_t e_ = (call);                                                       \
        if (e_ != cudaSuccess)                                                         \
            throw ::h2f::Error(H2F_E_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
    } while (0)

#define H2F_ASSERT(cond, msg)                                                          \
    do {                                                                               \
        if (!(cond)) throw ::h2f::Error(H2F_E_INTERNAL, std::string("assertion: ") + (msg)); \
    } while (0)

// first-fit allocator over one device slab
class Arena {
  public:
    void init(size_t bytes);
    void* alloc(size_t bytes);
    void free(void* p);
    size_t capacity() const { return cap_; }
    size_t in_use() const { return in_use_; }
    size_t peak() const { return peak_; }
    char* base() const { return base_; }

  private:
    char* base_ = nullptr;
    size_t cap_ = 0, in_use_ = 0, peak_ = 0;
    std::map<size_t, size_t> free_;          // offset -> size
    std::unordered_map<size_t, size_t> used_;
};

// bump allocator over arena chunks; release() returns everything at once
class Region {
  public:
    explicit Region(size_t chunk = size_t(64) << 20) : chunk_(chunk) {}
    Region(const Region&) = delete;
    Region& operator=(const Region&) = delete;
    Region(Region&& o) noexcept { *this = std::move(o); }
    Region& operator=(Region&& o) noexcept;
    ~Region() { release(); }
    void* alloc(size_t bytes);
    template <class T> T* alloc_n(int64_t n) { return static_cast<T*>(alloc(sizeof(T) * (n > 0 ? n : 1))); }
    void release();
    void reset();  // keep chunks, rewind
    size_t used() const { return used_; }

  private:
    size_t chunk_;
    std::vector<std::pair<char*, size_t>> chunks_;
    size_t cur_ = 0, off_ = 0, used_ = 0;
};

// packs host task arrays into pinned memory and ships them with one async copy
class Uploader {
  public:
    template <class T> T* put(const std::vector<T>& v) {
        return static_cast<T*>(put_bytes(v.data(), v.size() * sizeof(T)));
    }
    void* put_bytes(const void* src, size_t bytes);
    // space for `bytes` that the caller fills through *host before the next
    // flush (avoids a staging copy for large task arrays)
    void* reserve_bytes(size_t bytes, void** host);
    template <class T> T* reserve(size_t n, T** host) {
        void* h = nullptr;
        T* d = static_cast<T*>(reserve_bytes(n * sizeof(T), &h));
        *host = static_cast<T*>(h);
        return d;
    }
    void flush(cudaStream_t st);
    void reset();  // only after the stream has drained
    ~Uploader();

  private:
    struct Chunk { char* host; char* dev; size_t cap; };
    std::vector<Chunk> chunks_;
    size_t cur_ = 0, used_ = 0, flushed_ = 0;
};

// ---- per-kernel profiler (CUDA events around launches; off by default) ------
enum KernelId : int {
    K_GEMM_AUG = 0, K_GEMM_PROJECT, K_GEMM_SCHUR, K_GEMM_CREATE, K_GEMM_TOP, K_COPY, K_QR, K_JACOBI,
    K_COMPLEMENT, K_LU, K_TRSM, K_REDUCE, K_TOP_PANEL, K_TOP_MISC, K_SOLVE_FWD, K_SOLVE_SCATTER,
    K_SOLVE_BWD, K_SOLVE_TOP, K_SOLVE_MISC, K_MATVEC, K_VECTOR, K_QR_BIG, K_JACOBI_BIG, K_COMPLEMENT_V,
    K_COUNT
};
const char* kernel_name(int kid);

class Profiler {
  public:
    bool on = false;
    int begin(int kid, double flops, double bytes, double units = 0);
    void end(int slot);
    void collect();  // syncs the stream, folds finished pairs into the totals
    void reset();
    struct Total { int64_t launches = 0; double seconds = 0, flops = 0, bytes = 0; };
    Total totals[K_COUNT];
    ~Profiler();

  private:
    struct Rec { int kid; cudaEvent_t a, b; double flops, bytes, units; };
    std::vector<Rec> pending_;
    std::vector<cudaEvent_t> pool_;
    cudaEvent_t get_event();
};

struct ProfScope {
    int slot = -1;
    ProfScope(int kid, double flops = 0, double bytes = 0, double units = 0);
    ~ProfScope();
};

struct Context {
    int device = 0;
    cudaStream_t stream = nullptr;
    Arena arena;
    Uploader up;
    // pinned staging for small device->host reads
    char* pinned = nullptr;
    size_t pinned_cap = 0;
    Profiler prof;
    void* pinned_buf(size_t bytes);
    void sync();  // stream sync + uploader reset
};

Context& ctx();
bool ctx_ready();
void ctx_init(int device, double arena_gb);

inline void* dalloc(size_t bytes) { return ctx().arena.alloc(bytes); }
inline void dfree(void* p) { ctx().arena.free(p); }

// round helpers
inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

}  // namespace h2f
