// DeviceObjective and its building blocks (see objective.cuh).
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <atomic>
#include <cmath>
#include <cstdlib>
#include <cstring>

#include <cstdint>
#include <map>
#include <mutex>
#include <string>

#include "objective.cuh"
#include "cg.cuh"
#include "fused.cuh"

namespace mfreg_b200 {

bool no_lazy_state();

namespace {
// bytes of freed device memory the pool keeps for reuse (MFREG_POOL_KEEP_GB; only blocks below
// kBigAllocBytes come from the pool). Default: all of it — the pool then never trims itself at a
// synchronisation; with an 8 GB threshold the trim after a C4 registration's teardown stalled
// the next registration's first allocations by 0.4-1 s (c4_reg.py REPS=3: 7.4 / 6.3 / 7.2 s ->
// 6.4 / 6.6 / 6.3 s). Memory goes back when an allocation fails (device_alloc trims and retries).
std::uint64_t pool_keep_bytes() {
    const char* e = std::getenv("MFREG_POOL_KEEP_GB");
    if (!e || !*e) return ~std::uint64_t(0);
    return static_cast<std::uint64_t>(std::max(0.0, std::atof(e)) * static_cast<double>(1ull << 30));
}
cudaMemPool_t default_pool() {
    int dev = 0;
    MFREG_CUDA(cudaGetDevice(&dev));
    cudaMemPool_t pool = nullptr;
    MFREG_CUDA(cudaDeviceGetDefaultMemPool(&pool, dev));
    static thread_local int configured = -1;
    if (configured != dev) {
        std::uint64_t keep = pool_keep_bytes();
        MFREG_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
        configured = dev;
    }
    return pool;
}
}  // namespace

namespace {
// Freed blocks of kBigAllocBytes and more are kept for reuse by an allocation of the same size
// (MFREG_BIG_CACHE_GB, default 64: a C4 registration's levels need ~30 GB; 0 = plain cudaFree): objectives are created per pyramid level
// and per call, and cudaFree of their tens of GB of state measured up to ~1 s per teardown at C4,
// growing with repeated registrations (scripts/c4_reg.py, MFREG_TRACE_TIME=1). A cached block is
// handed out again only after a device synchronisation at its release (cudaFree's own ordering),
// and the cache is emptied before cudaMalloc is retried on an out-of-memory error.
struct BigCache {
    std::mutex mu;
    std::multimap<std::size_t, std::pair<int, void*>> blocks;  // requested bytes -> (device, pointer)
    std::size_t bytes = 0;
};
BigCache& big_cache() {
    static BigCache* c = new BigCache;  // never destroyed: frees may come from static destructors
    return *c;
}
std::size_t big_cache_limit() {
    static const std::size_t lim = [] {
        const char* e = std::getenv("MFREG_BIG_CACHE_GB");
        const double gb = e ? std::atof(e) : 64.0;
        return static_cast<std::size_t>(std::max(0.0, gb) * static_cast<double>(1ull << 30));
    }();
    return lim;
}
void* big_take(std::size_t bytes) {
    int dev = 0;
    MFREG_CUDA(cudaGetDevice(&dev));
    BigCache& c = big_cache();
    std::lock_guard<std::mutex> lk(c.mu);
    auto range = c.blocks.equal_range(bytes);
    for (auto it = range.first; it != range.second; ++it)
        if (it->second.first == dev) {
            void* p = it->second.second;
            c.blocks.erase(it);
            c.bytes -= bytes;
            return p;
        }
    return nullptr;
}
bool big_put(void* p, std::size_t bytes) {
    if (bytes > big_cache_limit()) return false;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return false;
    BigCache& c = big_cache();
    std::lock_guard<std::mutex> lk(c.mu);
    if (c.bytes + bytes > big_cache_limit()) return false;
    if (cudaDeviceSynchronize() != cudaSuccess) return false;  // the block's last users are done
    c.blocks.emplace(bytes, std::make_pair(dev, p));
    c.bytes += bytes;
    return true;
}
void big_release_all() {
    int dev = 0;
    MFREG_CUDA(cudaGetDevice(&dev));
    BigCache& c = big_cache();
    std::lock_guard<std::mutex> lk(c.mu);
    for (auto it = c.blocks.begin(); it != c.blocks.end();) {
        if (it->second.first == dev) {
            cudaFree(it->second.second);
            c.bytes -= it->first;
            it = c.blocks.erase(it);
        } else {
            ++it;
        }
    }
}
}  // namespace

namespace {
struct PinnedPool {
    std::mutex mu;
    std::vector<void*> free;
};
PinnedPool& pinned_pool() {
    static PinnedPool* p = new PinnedPool;  // never destroyed (frees from static destructors)
    return *p;
}
}  // namespace

void* pinned_small_alloc(std::size_t bytes) {
    if (bytes > kPinnedSmall) throw std::invalid_argument("pinned_small_alloc: block too large");
    {
        PinnedPool& pp = pinned_pool();
        std::lock_guard<std::mutex> lk(pp.mu);
        if (!pp.free.empty()) {
            void* p = pp.free.back();
            pp.free.pop_back();
            return p;
        }
    }
    void* p = nullptr;
    MFREG_CUDA(cudaHostAlloc(&p, kPinnedSmall, cudaHostAllocMapped | cudaHostAllocPortable));
    return p;
}

void pinned_small_free(void* p) {
    if (!p) return;
    PinnedPool& pp = pinned_pool();
    std::lock_guard<std::mutex> lk(pp.mu);
    pp.free.push_back(p);
}

namespace {
std::atomic<long long> g_mem_cur{0}, g_mem_peak{0};  // library device allocations (live bytes, high-water mark)
void mem_note(long long delta) {
    const long long now = g_mem_cur.fetch_add(delta) + delta;
    long long peak = g_mem_peak.load();
    while (now > peak && !g_mem_peak.compare_exchange_weak(peak, now)) {
    }
}
}  // namespace

long long device_memory_peak(bool reset) {
    const long long p = g_mem_peak.load();
    if (reset) g_mem_peak.store(g_mem_cur.load());
    return p;
}

namespace {
// MFREG_TRACE_TIME=1: allocations slower than 20 ms on stderr
struct AllocTimer {
    const char* path = "pool";
    std::size_t bytes;
    std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
    explicit AllocTimer(std::size_t b) : bytes(b) {}
    ~AllocTimer() {
        static const bool tr = [] {
            const char* e = std::getenv("MFREG_TRACE_TIME");
            return e && *e && *e != '0';
        }();
        if (!tr) return;
        const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        if (ms > 20.0) std::fprintf(stderr, "  slow device_alloc(%zu bytes, %s): %.1f ms\n", bytes, path, ms);
    }
};
}  // namespace

void* device_alloc(std::size_t bytes) {
    mem_note(static_cast<long long>(bytes));
    AllocTimer at(bytes);
    void* p = nullptr;
    if (bytes >= kBigAllocBytes) {
        at.path = "big cache";
        if ((p = big_take(bytes))) return p;
        at.path = "cudaMalloc";
        cudaError_t e = cudaMalloc(&p, bytes);
        if (e == cudaErrorMemoryAllocation) {  // cached blocks may hold the memory: release, retry
            cudaGetLastError();
            MFREG_CUDA(cudaDeviceSynchronize());
            big_release_all();
            MFREG_CUDA(cudaMemPoolTrimTo(default_pool(), 0));
            e = cudaMalloc(&p, bytes);
        }
        if (e != cudaSuccess) {
            cudaGetLastError();
            throw CudaError(std::string("cudaMalloc(") + std::to_string(bytes) + " bytes): " + cudaGetErrorString(e));
        }
        return p;
    }
    cudaMemPool_t pool = default_pool();
    cudaError_t e = cudaMallocAsync(&p, bytes, 0);
    if (e == cudaErrorMemoryAllocation) {  // give the cached blocks back and retry once
        cudaGetLastError();
        MFREG_CUDA(cudaDeviceSynchronize());
        big_release_all();
        MFREG_CUDA(cudaMemPoolTrimTo(pool, 0));
        e = cudaMallocAsync(&p, bytes, 0);
    }
    if (e != cudaSuccess) {
        cudaGetLastError();
        throw CudaError(std::string("cudaMallocAsync(") + std::to_string(bytes) + " bytes): " + cudaGetErrorString(e));
    }
    return p;
}

void device_free(void* p, std::size_t bytes) {
    if (!p) return;
    mem_note(-static_cast<long long>(bytes));
    if (bytes >= kBigAllocBytes) {
        if (!big_put(p, bytes)) cudaFree(p);
    } else {
        cudaFreeAsync(p, 0);
    }
}

void check_launch(const char* what) {
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}

void validate_grid(const Grid& g, bool nodal) {  // grid.hpp:103-119
    for (int a = 0; a < 3; ++a) {
        if (g.m[a] < 1) throw std::invalid_argument("GridDesc: all m components must be >= 1");
        if (!(g.h[a] > 0.0)) throw std::invalid_argument("GridDesc: all h components must be > 0");
    }
    if (nodal)
        for (int a = 0; a < 3; ++a)
            if (g.m[a] < 2) throw std::invalid_argument("GridDesc: nodal grids need >= 2 points per axis");
}

Grid make_deform_grid(const Grid& image, const idx_t points[3]) {  // grid.hpp:131-146
    Grid g{};
    for (int a = 0; a < 3; ++a) {
        g.m[a] = points[a];
        if (points[a] < 2) throw std::invalid_argument("deformation grid needs >= 2 points per axis");
        if (points[a] - 1 > image.m[a]) throw std::invalid_argument("deformation grid finer than image grid");
        g.h[a] = (static_cast<double>(image.m[a]) * image.h[a]) / static_cast<double>(points[a] - 1);
    }
    return g;
}

Grid deformation_grid_for(const Grid& image, idx_t ratio) {  // multilevel.cpp:39-49
    if (ratio < 1) throw std::invalid_argument("deformation_grid_for: ratio must be >= 1");
    idx_t pts[3];
    for (int a = 0; a < 3; ++a) pts[a] = std::max<idx_t>(2, (image.m[a] + ratio - 1) / ratio + 1);
    return make_deform_grid(image, pts);
}

std::vector<int> plan_base_axis(idx_t mt, idx_t ms) {
    std::vector<int> hb(mt);
    for (idx_t k = 0; k < mt; ++k) {  // transfer.cpp:24-35, same expression as DevicePlanOwner
        const double c = (static_cast<double>(k) + 0.5) * static_cast<double>(ms - 1) / static_cast<double>(mt);
        hb[k] = static_cast<int>(std::clamp<idx_t>(static_cast<idx_t>(std::floor(c)), 0, ms - 2));
    }
    return hb;
}

std::vector<SlabInfo> slab_partition(const Grid& img, const Grid& dg, int nr, bool parity) {
    validate_grid(dg, true);
    validate_grid(img, false);
    if (nr < 1) throw std::invalid_argument("slab_partition: nranks must be >= 1");
    const int mz = static_cast<int>(img.m[2]), ms = static_cast<int>(dg.m[2]);
    const std::vector<int> b = plan_base_axis(mz, ms);
    // split planes: first image plane of a nodal cell, at or after the even split
    std::vector<int> zb(nr + 1, 0);
    zb[nr] = mz;
    for (int r = 1; r < nr; ++r) {
        int z = std::max(zb[r - 1] + 1, static_cast<int>((static_cast<long long>(r) * mz + nr / 2) / nr));
        while (z < mz && b[z] == b[z - 1]) ++z;
        if (z >= mz) throw std::invalid_argument("slab_partition: too many ranks for the z extent");
        zb[r] = z;
    }
    std::vector<SlabInfo> out(nr);
    for (int r = 0; r < nr; ++r) {
        SlabInfo& s = out[r];
        s.zlo = zb[r];
        s.zhi = zb[r + 1];
        s.own_lo = r == 0 ? 0 : b[s.zlo];
        s.own_hi = r == nr - 1 ? ms : b[s.zhi];
        s.bnd = r == nr - 1 ? 0 : std::max(0, b[s.zhi - 1] + 2 - s.own_hi);
        // operand planes read: the warp over [zlo-3, zhi+3) and the curvature stencil
        // (Lap Lap: +-2 nodal planes) of the owned planes
        int wlo = std::max(0, s.zlo - 3), whi = std::min(mz, s.zhi + 3);
        if (parity) {  // the warp over [first plane of nodal slab own_lo - 1, zhi) +- 2 planes
            int z = s.zlo;
            if (s.own_lo > 0)
                while (z > 0 && b[z - 1] >= s.own_lo - 1) --z;
            wlo = std::max(0, z - 2);
            whi = std::min(mz, s.zhi + 2);
        }
        s.need_lo = std::max(0, std::min(b[wlo], s.own_lo - 2));
        s.need_hi = std::min(ms, std::max(b[whi - 1] + 2, s.own_hi + 2));
    }
    for (int r = 0; r < nr; ++r) {
        const SlabInfo& s = out[r];
        if ((r > 0 && s.need_lo < out[r - 1].own_lo) || (r + 1 < nr && s.need_hi > out[r + 1].own_hi) ||
            (r + 1 < nr && s.own_hi + s.bnd > out[r + 1].own_hi) || s.own_hi <= s.own_lo)
            throw std::invalid_argument("slab_partition: slabs thinner than the halo (too many ranks)");
    }
    return out;
}

DevicePlanOwner::DevicePlanOwner(const Grid& nodal, const Grid& image) {
    validate_grid(nodal, true);
    validate_grid(image, false);
    view_.src = nodal;
    view_.tgt = image;
    for (int a = 0; a < 3; ++a) {
        const idx_t mt = image.m[a], ms = nodal.m[a];
        auto& hb = host_base[a];
        auto& hr = host_rem[a];
        hb = plan_base_axis(mt, ms);
        hr.resize(mt);
        for (idx_t k = 0; k < mt; ++k) {  // transfer.cpp:24-39, same expression
            const double c = (static_cast<double>(k) + 0.5) * static_cast<double>(ms - 1) / static_cast<double>(mt);
            hr[k] = c - static_cast<double>(hb[k]);
            if (hr[k] < 0.0 || hr[k] > 1.0) throw std::invalid_argument("transfer plan: coverage invariant violated");
        }
        std::vector<int> lo(ms - 1, 0), hi(ms - 1, 0);
        for (idx_t k = 0; k < mt; ++k) {
            const int c = hb[k];
            if (lo[c] == hi[c]) lo[c] = static_cast<int>(k);
            hi[c] = static_cast<int>(k) + 1;
        }
        base_[a].resize(mt);
        rem_[a].resize(mt);
        lo_[a].resize(ms - 1);
        hi_[a].resize(ms - 1);
        MFREG_CUDA(cudaMemcpy(base_[a].get(), hb.data(), mt * sizeof(int), cudaMemcpyHostToDevice));
        MFREG_CUDA(cudaMemcpy(rem_[a].get(), hr.data(), mt * sizeof(double), cudaMemcpyHostToDevice));
        MFREG_CUDA(cudaMemcpy(lo_[a].get(), lo.data(), (ms - 1) * sizeof(int), cudaMemcpyHostToDevice));
        MFREG_CUDA(cudaMemcpy(hi_[a].get(), hi.data(), (ms - 1) * sizeof(int), cudaMemcpyHostToDevice));
        view_.base[a] = base_[a].get();
        view_.rem[a] = rem_[a].get();
        view_.cell_lo[a] = lo_[a].get();
        view_.cell_hi[a] = hi_[a].get();
    }
}

Reducer::Reducer(Mode mode, idx_t max_n) : mode_(mode) {
    partials_.resize(static_cast<std::size_t>(std::max<idx_t>(16, std::max(chunk_count(max_n), tree_blocks(max_n)))));
}

void Reducer::sum(int kind, idx_t n, const double* a, const double* b, double* out_dev, double scale,
                  cudaStream_t s) {
    const idx_t need = mode_ == Mode::Parity ? chunk_count(n) : tree_blocks(n);
    if (static_cast<std::size_t>(need) > partials_.size()) partials_.resize(static_cast<std::size_t>(need));
    if (mode_ == Mode::Parity) launch_chunked_sum(kind, n, a, b, partials_.get(), out_dev, scale, s);
    else launch_tree_sum(kind, n, a, b, partials_.get(), out_dev, scale, s);
    check_launch("reduction");
}

void Reducer::sum3(int kind, idx_t n, const double* a, const double* b, double* out_dev, double scale,
                   cudaStream_t s) {
    if (mode_ != Mode::Parity) {
        for (int d = 0; d < 3; ++d) sum(kind, n, a + d * n, b ? b + d * n : nullptr, out_dev + d, scale, s);
        return;
    }
    const idx_t need = 3 * chunk_count(n);
    if (static_cast<std::size_t>(need) > partials_.size()) partials_.resize(static_cast<std::size_t>(need));
    launch_chunked_sum3(kind, n, a, b, partials_.get(), out_dev, scale, s);
    check_launch("reduction (3 segments)");
}

Scalars::Scalars(int n) : d_(static_cast<std::size_t>(n)) {
    h_ = static_cast<double*>(pinned_small_alloc(n * sizeof(double)));
    MFREG_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&hd_), h_, 0));
    MFREG_CUDA(cudaMemset(d_.get(), 0, n * sizeof(double)));
}
Scalars::~Scalars() { pinned_small_free(h_); }
void Scalars::fetch_async(int n, cudaStream_t s) {
    MFREG_CUDA(cudaMemcpyAsync(h_, d_.get(), n * sizeof(double), cudaMemcpyDeviceToHost, s));
}

const double* Scalars::fetch(int n, cudaStream_t s) {
    MFREG_CUDA(cudaMemcpyAsync(h_, d_.get(), n * sizeof(double), cudaMemcpyDeviceToHost, s));
    MFREG_CUDA(cudaStreamSynchronize(s));
    return h_;
}

// ------------------------------------------------------------------ DeviceNgf
DeviceNgf::DeviceNgf(const Grid& img, const double* R_dev, double tau, double rho, Mode mode, cudaStream_t s)
    : g_(img), tau_(tau), rho_(rho), mode_(mode), s_(s), R_(R_dev), red_(mode, img.count()) {
    if (!(rho > 0.0)) throw std::invalid_argument("NGF: rho must be > 0");  // ngf.cpp:168-170
    const std::size_t n = static_cast<std::size_t>(img.count());
    if (mode == Mode::Fast32) {  // single-precision state; R converted once per level
        R32.resize(n);
        Tw32.resize(n);
        dT32.resize(3 * n);
        frh32.resize(6 * n);
        launch_to_float(static_cast<idx_t>(n), R_dev, R32.get(), s);
    } else {
        Tw.resize(n);
        dT.resize(3 * n);
        if (mode == Mode::Parity) ensure_ws();
        else frh.resize(6 * n);
    }
    tab_ = make_hv_table(img);
}

void DeviceNgf::ensure_ws() {
    // per-voxel workspace of the unfused kernels (parity mode, and the kernel-level
    // NGF API in either mode); the fused fast-mode objective only keeps frh.
    const std::size_t n = static_cast<std::size_t>(g_.count());
    if (r.size() == n) return;
    r.resize(n);
    inv1.resize(n);
    inv2.resize(n);
    rh.resize(7 * n);
    sv.resize(n);
    if (mode_ != Mode::Parity) wbuf.resize(n);
}

void DeviceNgf::populate_points(const double* T_dev, const double* pts_dev) {
    ensure_ws();
    if (!(tau_ > 0.0) || !(rho_ > 0.0)) throw std::invalid_argument("NGF: tau and rho must be > 0");
    launch_sample(g_, T_dev, pts_dev, g_.count(), Tw.get(), dT.get(), s_);
    launch_ngf_ws(g_, R_, Tw.get(), tau_, rho_, r.get(), inv1.get(), inv2.get(), rh.get(), s_);
    check_launch("populate_ngf_workspace");
}

void DeviceNgf::populate_warp(const DevPlan& P, const double* y_dev, const double* T_dev, int wlo, int whi, int slo,
                              int shi) {
    ensure_ws();
    if (!(tau_ > 0.0) || !(rho_ > 0.0)) throw std::invalid_argument("NGF: tau and rho must be > 0");
    const int mz = static_cast<int>(g_.m[2]);
    launch_warp(P, y_dev, T_dev, Tw.get(), dT.get(), s_, std::max(0, wlo), whi < 0 ? -1 : std::min(whi, mz));
    launch_ngf_ws(g_, R_, Tw.get(), tau_, rho_, r.get(), inv1.get(), inv2.get(), rh.get(), s_, slo, shi);
    check_launch("warp + workspace");
}

void DeviceNgf::value_async(double* out_dev) {
    red_.sum(SUM_ONE_MINUS_SQ, g_.count(), r.get(), nullptr, out_dev, g_.cell_volume(), s_);
}

void DeviceNgf::gradient(double* out3n, int zlo, int zhi) {
    launch_ngf_gradient(g_, r.get(), rh.get(), dT.get(), out3n, s_, zlo, zhi);
    check_launch("ngf_gradient");
}

void DeviceNgf::hessian_vec_image(const double* svp, double* out3n, int zlo, int zhi) {
    if (mode_ == Mode::Parity) launch_hv_closed(g_, tab_, rh.get(), svp, dT.get(), out3n, s_, zlo, zhi);
    else launch_hv_factored(g_, rh.get(), svp, dT.get(), wbuf.get(), out3n, s_);
    check_launch("ngf_hessian_vec");
}

namespace {
__global__ void k_dot3(long long n, const double* __restrict__ dT, const double* __restrict__ p,
                       double* __restrict__ sv) {
    const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) sv[i] = dT[i] * p[i] + dT[n + i] * p[n + i] + dT[2 * n + i] * p[2 * n + i];
}
}  // namespace

void DeviceNgf::hessian_vec(const double* p3n, double* out3n) {
    const idx_t n = g_.count();
    note_launch(), k_dot3<<<static_cast<unsigned>((n + 255) / 256), 256, 0, s_>>>(n, dT.get(), p3n, sv.get());
    hessian_vec_image(sv.get(), out3n);
}

// ------------------------------------------------------------ DeviceObjective
DeviceObjective::DeviceObjective(const double* R_dev, const double* T_dev, const Grid& image, const Grid& deform,
                                 double tau, double rho, double alpha, Mode mode, cudaStream_t s, const SlabSpec& slab)
    : img_(image),
      dg_(deform),
      slab_(slab),
      alpha_(alpha),
      s_(s),
      T_(T_dev),
      plan_(deform, image),
      ngf_(image, R_dev, tau, rho, mode, s) {
    const std::size_t ny = static_cast<std::size_t>(dg_.count());
    xid_.resize(3 * ny);
    u_.resize(3 * ny);
    lapu_.resize(3 * ny);
    lapp_.resize(3 * ny);
    img3_.resize(3 * static_cast<std::size_t>(img_.count()));
    launch_identity(dg_, xid_.get(), s_);
    check_launch("identity");
    sliced_ = !slab.full(static_cast<int>(img_.m[2]), static_cast<int>(dg_.m[2]));
    if (sliced_) {
        if (mode == Mode::Fast32) throw std::invalid_argument("z slabs run in fast or parity mode");
        const auto parts = slab_partition(img_, dg_, 1);  // validates the grids
        (void)parts;
        const int mz = static_cast<int>(img_.m[2]), msz = static_cast<int>(dg_.m[2]);
        if (!(0 <= slab.zlo && slab.zlo < slab.zhi && slab.zhi <= mz && 0 <= slab.own_lo &&
              slab.own_lo < slab.own_hi && slab.own_hi <= msz))
            throw std::invalid_argument("slab: invalid z window");
        if (mode == Mode::Parity) {
            // the owned nodes' P^T reads the image planes of nodal slabs own_lo-1 .. own_hi-1, i.e.
            // [wlo, zhi); their per-voxel terms read the workspace one plane further, which reads
            // T_w one more; s = dT.(P p) is read two planes out by the 25-point Hv stencil
            const auto& bz = plan_.host_base[2];
            int wlo = 0;
            if (slab.own_lo > 0) {
                wlo = slab.zlo;
                while (wlo > 0 && bz[wlo - 1] >= slab.own_lo - 1) --wlo;
            }
            pw_.out_lo = wlo;
            pw_.out_hi = slab.zhi;
            pw_.ws_lo = std::max(0, wlo - 1);
            pw_.ws_hi = std::min(mz, slab.zhi + 1);
            pw_.warp_lo = pw_.s_lo = std::max(0, wlo - 2);
            pw_.warp_hi = pw_.s_hi = std::min(mz, slab.zhi + 2);
            pw_.n_lo = slab.own_lo;
            pw_.n_hi = slab.own_hi;
            pw_.l_lo = std::max(0, slab.own_lo - 1);
            pw_.l_hi = std::min(msz, slab.own_hi + 1);
        }
    }
    if (mode != Mode::Parity) {
        fused_ = std::make_unique<FusedPlan>(plan_, ngf_.state_R(), ngf_.state_Tw(), ngf_.state_dT(), ngf_.state_frh(),
                                             slab_, mode == Mode::Fast32);
        MFREG_CUDA(cudaStreamCreateWithFlags(&s2_, cudaStreamNonBlocking));
        MFREG_CUDA(cudaEventCreateWithFlags(&ev_fork_, cudaEventDisableTiming));
        MFREG_CUDA(cudaEventCreateWithFlags(&ev_join_, cudaEventDisableTiming));
        red2_ = std::make_unique<Reducer>(Mode::Fast, 3 * dg_.count());
        curv_.resize(3 * ny);
        sc2_.resize(4);
        // the lazy value-only state's y copy, allocated here rather than inside the first Armijo
        // trial: allocated there (stream-ordered pool, behind the CG's queued work) it measured
        // 0.3-0.8 s stalls on the first trial of each C4 level-0 solve after the first registration
        if (!sliced_ && !no_lazy_state()) ylazy_.resize(3 * ny);
    }
}

DeviceObjective::~DeviceObjective() {
    static const bool trace = [] {  // MFREG_TRACE_TIME=1 (as the solvers' per-iteration split)
        const char* e = std::getenv("MFREG_TRACE_TIME");
        return e && *e && *e != '0';
    }();
    if (trace) {  // (teardown cost breakdown; the members would go in this order anyway)
        auto t = std::chrono::steady_clock::now();
        auto lap = [&](const char* what) {
            const auto n = std::chrono::steady_clock::now();
            std::fprintf(stderr, "  teardown %s %.2f ms\n", what, std::chrono::duration<double, std::milli>(n - t).count());
            t = n;
        };
        fused_.reset();
        lap("fused");
        red2_.reset();
        lap("red2");
        graphs_.clear();
        lap("graphs");
        ngf_.release();
        lap("ngf");
    }
    if (ev_fork_) cudaEventDestroy(ev_fork_);
    if (ev_join_) cudaEventDestroy(ev_join_);
    if (s2_) cudaStreamDestroy(s2_);
    for (auto* v : {&pipe_.evh, &pipe_.eve, &pipe_.evf})
        for (cudaEvent_t e : *v) cudaEventDestroy(e);
    if (pipe_.ev0) cudaEventDestroy(pipe_.ev0);
    if (pipe_.evd) cudaEventDestroy(pipe_.evd);
    for (cudaStream_t q : {pipe_.h2d, pipe_.d2h, pipe_.fin})
        if (q) cudaStreamDestroy(q);
}

double DeviceObjective::min_spacing() const { return std::min({dg_.h[0], dg_.h[1], dg_.h[2]}); }

// fast-mode warp into the state arrays of the objective's precision
void DeviceObjective::warp_state(const double* y, cudaStream_t s, int zlo, int zhi, bool state) {
    if (ngf_.fp32())
        launch_warp_fast(plan_.view(), y, T_, ngf_.Tw32.get(), state ? ngf_.dT32.get() : nullptr, s, zlo, zhi);
    else
        launch_warp_fast(plan_.view(), y, T_, ngf_.Tw.get(), state ? ngf_.dT.get() : nullptr, s, zlo, zhi);
}

double* DeviceObjective::frh_out() {
    return fused_->hv3_recompute() ? nullptr : static_cast<double*>(ngf_.state_frh());
}

// a14: Hv uses the state of the last eval, value-only included. A lazy value-only
// eval skipped writing that state (dT, rho-hat); rebuild it at the recorded point.
void DeviceObjective::refresh_state() {
    if (!stale_) return;
    warp_state(ylazy_.get(), s_, 0, -1, true);
    if (!fused_->hv3_recompute())  // (the recomputing Hv pass: T_w and dT are the whole state)
        launch_eval_fused(plan_, *fused_, ngf_.R_, ngf_.Tw.get(), ngf_.dT.get(), ngf_.tau_, ngf_.rho_,
                          static_cast<double*>(ngf_.state_frh()), false, s_);
    check_launch("Objective: Hv state refresh");
    stale_ = false;
}

// fast mode: the launch sequence of eval (captured once per (y, grad) into a CUDA graph)
void DeviceObjective::enqueue_eval_fast(const double* y, double* grad, cudaStream_t s, bool state) {
    const idx_t ny = dg_.count();
    if (!state) MFREG_CUDA(cudaMemcpyAsync(ylazy_.get(), y, 3 * ny * sizeof(double), cudaMemcpyDeviceToDevice, s));
    const int mz = static_cast<int>(img_.m[2]);
    // (sliced: the slab's planes + 3 halo planes, the state of the 2 halo planes the Hv reads)
    const int wlo = sliced_ ? std::max(0, slab_.zlo - 3) : 0, whi = sliced_ ? std::min(mz, slab_.zhi + 3) : -1;
    // curvature value / gradient on the side stream (it needs only y), overlapping the
    // warp and the image pass
    MFREG_CUDA(cudaEventRecord(ev_fork_, s));
    MFREG_CUDA(cudaStreamWaitEvent(s2_, ev_fork_, 0));
    launch_sub(3 * ny, y, xid_.get(), u_.get(), s2_);
    launch_lap3(dg_, u_.get(), lapu_.get(), s2_, 0, -1, false);  // (fast: reciprocal multiplies)
    const idx_t pn = dg_.m[0] * dg_.m[1];
    if (sliced_)  // owned nodal planes only, per component
        for (int d = 0; d < 3; ++d)
            red2_->sum(SUM_SQ, (slab_.own_hi - slab_.own_lo) * pn, lapu_.get() + d * ny + slab_.own_lo * pn, nullptr,
                       sc2_.get() + d, 1.0, s2_);
    else
        red2_->sum(SUM_SQ, 3 * ny, lapu_.get(), nullptr, sc2_.get(), 1.0, s2_);
    // two-CTA eval kernel (whole domain): D comes from its last CTA and alpha S from the side
    // stream, both straight into the host scalars; the finalize is then a pure gather
    const bool scalars_direct = !sliced_ && fused_->ev2();
    if (scalars_direct) launch_curv_value(sc2_.get(), dg_.cell_volume(), alpha_, sc_.dev(1), sc_.host_dev() + 1, s2_);
    if (grad && alpha_ != 0.0)
        launch_bilap(dg_, lapu_.get(), alpha_ * (2.0 * dg_.cell_volume()), 0, 0.0, 0.0, nullptr, curv_.get(), s2_, 0,
                     -1, false);
    MFREG_CUDA(cudaEventRecord(ev_join_, s2_));
    warp_state(y, s, wlo, whi, state);
    launch_eval_fused(plan_, *fused_, ngf_.R_, ngf_.Tw.get(), ngf_.dT.get(), ngf_.tau_, ngf_.rho_,
                      state ? frh_out() : nullptr, grad != nullptr, s,
                      scalars_direct ? sc_.dev(0) : nullptr, scalars_direct ? sc_.host_dev() : nullptr);
    MFREG_CUDA(cudaStreamWaitEvent(s, ev_join_, 0));
    if (scalars_direct) {
        if (grad) {
            FinalizeSpec f;
            f.add = alpha_ != 0.0 ? curv_.get() : nullptr;
            f.out = grad;
            launch_nodal_finalize(plan_, *fused_, f, s);
        }
        check_launch("Objective::eval (fused)");
        return;
    }
    FinalizeSpec f;
    f.add = (grad && alpha_ != 0.0) ? curv_.get() : nullptr;
    f.S = sc2_.get();
    f.nS = sliced_ ? 3 : 1;
    f.alpha = alpha_;
    f.out = grad;
    f.value = true;
    f.sc = sc_.dev(0);
    f.sc_host = sc_.host_dev();  // D, alpha S straight to the host (eval_end reads them)
    launch_nodal_finalize(plan_, *fused_, f, s);
    check_launch("Objective::eval (fused)");
}

// fast mode: GN Hv (alpha 2 h^y Lap(Lap p) on the side stream, overlapping the image
// pass), optionally <dot_a, q> into sc
void DeviceObjective::enqueue_hv_fast(const double* p, double* q, const double* dot_a, double* sc, const int* skip,
                                      cudaStream_t s) {
    if (alpha_ != 0.0) {
        MFREG_CUDA(cudaEventRecord(ev_fork_, s));
        MFREG_CUDA(cudaStreamWaitEvent(s2_, ev_fork_, 0));
        launch_lap3(dg_, p, lapp_.get(), s2_, 0, -1, false);
        launch_bilap(dg_, lapp_.get(), alpha_ * (2.0 * dg_.cell_volume()), 0, 0.0, 0.0, nullptr, curv_.get(), s2_, 0, -1,
                     false);
        MFREG_CUDA(cudaEventRecord(ev_join_, s2_));
    }
    launch_hv_fused(plan_, *fused_, ngf_.frh.get(), ngf_.dT.get(), p, ngf_.tau_, ngf_.rho_, s, skip);
    if (alpha_ != 0.0) MFREG_CUDA(cudaStreamWaitEvent(s, ev_join_, 0));
    FinalizeSpec f;
    f.add = alpha_ != 0.0 ? curv_.get() : nullptr;
    f.out = q;
    f.dot_a = dot_a;
    f.sc = sc;
    f.skip = skip;
    f.hv_pass = true;
    launch_nodal_finalize(plan_, *fused_, f, s);
    check_launch("Objective::gn_hessian_vec (fused)");
}

double DeviceObjective::profile_kernel(int which, const double* p, int reps, std::size_t flush_bytes) {
    if (!fused_) throw std::logic_error("profile_kernel: fast mode only");
    refresh_state();
    DevArray<unsigned char> scratch(flush_bytes);
    cudaEvent_t e0, e1;
    MFREG_CUDA(cudaEventCreate(&e0));
    MFREG_CUDA(cudaEventCreate(&e1));
    double total = 0.0;
    for (int r = 0; r < reps; ++r) {
        if (flush_bytes) MFREG_CUDA(cudaMemsetAsync(scratch.get(), r & 0xff, flush_bytes, s_));
        MFREG_CUDA(cudaEventRecord(e0, s_));
        if (which == 0)
            launch_hv_fused(plan_, *fused_, ngf_.frh.get(), ngf_.dT.get(), p, ngf_.tau_, ngf_.rho_, s_);
        else if (which == 1)
            launch_eval_fused(plan_, *fused_, ngf_.R_, ngf_.Tw.get(), ngf_.dT.get(), ngf_.tau_, ngf_.rho_,
                              frh_out(), true, s_);
        else
            warp_state(p, s_, 0, -1);
        MFREG_CUDA(cudaEventRecord(e1, s_));
        MFREG_CUDA(cudaEventSynchronize(e1));
        float ms = 0.0f;
        MFREG_CUDA(cudaEventElapsedTime(&ms, e0, e1));
        total += ms;
    }
    check_launch("profile_kernel");
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    return total / std::max(1, reps);
}

// ---- host-buffer pipeline (eval_host / hv_host)
// Plan, once per objective: G <= 4 z groups of the two-CTA passes' z tile chunks; per group the
// image planes it covers, the nodal planes its warp / Hv pass reads (H2D chunk bounds: nodal
// planes up to base_z + 1 of the group's last plane read, the Hv tiles two steps past it) and the
// nodes complete after it (P^T of plane i touches base_z(i), base_z(i) + 1, so once the groups up
// to g ran, the nodes below base_z of the next group's first plane are final).
namespace {
// MFREG_PIPE_TRACE=1: timing events along the host pipeline, printed per call (stderr)
struct PipeTrace {
    bool on = false;
    std::vector<std::pair<std::string, cudaEvent_t>> ev;
    PipeTrace() {
        const char* e = std::getenv("MFREG_PIPE_TRACE");
        on = e && e[0] == '1';
    }
    void mark(const std::string& what, cudaStream_t s) {
        if (!on) return;
        cudaEvent_t e;
        cudaEventCreate(&e);
        cudaEventRecord(e, s);
        ev.emplace_back(what, e);
    }
    void dump(const char* call) {
        if (!on || ev.empty()) return;
        cudaDeviceSynchronize();
        std::fprintf(stderr, "%s:", call);
        for (auto& [w, e] : ev) {
            float ms = 0.0f;
            cudaEventElapsedTime(&ms, ev[0].second, e);
            std::fprintf(stderr, " %s %.3f", w.c_str(), ms);
        }
        std::fprintf(stderr, "\n");
        for (auto& [w, e] : ev) cudaEventDestroy(e);
        ev.clear();
    }
};
PipeTrace& ptrace() {
    static PipeTrace t;
    return t;
}
}  // namespace

bool DeviceObjective::pipe_ready() {
    if (pipe_.state) return pipe_.state == 1;
    pipe_.state = 2;
    const char* off = std::getenv("MFREG_NO_PIPE");
    if ((off && off[0] == '1') || !fused_ || sliced_ || !fused_->hv2() || !fused_->ev2() || fused_->hv3()) return false;
    const idx_t ny = dg_.count();
    const char* mb = std::getenv("MFREG_PIPE_MIN_MB");  // (tests force it on small grids)
    const long long min_bytes = (mb && *mb ? std::atoll(mb) : 16LL) << 20;
    if (3 * ny * static_cast<idx_t>(sizeof(double)) < min_bytes) return false;  // copies too small to hide
    // A plan of its own, on z chunks of <= 128 planes: the pipeline's granularity is the z tile
    // chunk, and the device-call plan's long chunks (2 x 450 planes at C4, 3% faster passes) would
    // leave it half of the operand to copy before the first group and half to copy back after the
    // last (e2e 33.4 -> 28.5 Gvoxel/s). Same kernels and state arrays; the results differ from the
    // device calls' in the last bits (per-tile sums over other plane ranges).
    pipe_.fp = std::make_unique<FusedPlan>(plan_, ngf_.state_R(), ngf_.state_Tw(), ngf_.state_dT(), ngf_.state_frh(),
                                           slab_, ngf_.fp32(), 128);
    if (!pipe_.fp->hv2() || !pipe_.fp->ev2() || pipe_.fp->hv3()) {
        pipe_.fp.reset();
        return false;
    }
    const TileMeta& t = pipe_.fp->meta();
    if (t.ntz < 2) {  // one z chunk: nothing to pipeline
        pipe_.fp.reset();
        return false;
    }
    const int G = t.ntz >= 4 ? 2 + std::min(3, t.ntz - 2) : t.ntz, mz = static_cast<int>(img_.m[2]), msz = static_cast<int>(dg_.m[2]);
    const auto& bz = plan_.host_base[2];
    Pipe& q = pipe_;
    q.G = G;
    q.cb.resize(G + 1);
    // one z tile chunk in the first group (the first H2D chunk is all the pipeline waits for) and
    // in the last (its finalize and D2H are what remains exposed), the rest in up to three groups
    // whose D2H each fits under the next group's pass; sizes 1, 2, 2, 2, 1 at C4 (8 chunks)
    if (t.ntz >= 4) {
        const int mid = G - 2;
        q.cb[0] = 0;
        for (int k = 0; k <= mid; ++k) q.cb[1 + k] = 1 + static_cast<int>((static_cast<long long>(k) * (t.ntz - 2)) / mid);
        q.cb[G] = t.ntz;
    } else
        for (int g = 0; g <= G; ++g) q.cb[g] = static_cast<int>((static_cast<long long>(g) * t.ntz) / G);
    q.za.resize(G);
    q.zb.resize(G);
    q.hb_warp.assign(G + 1, 0);
    q.hb_hv.assign(G + 1, 0);
    q.fb.assign(G + 1, 0);
    for (int g = 0; g < G; ++g) {
        q.za[g] = t.zlo + q.cb[g] * t.zc;
        q.zb[g] = std::min(t.zhi, t.zlo + q.cb[g + 1] * t.zc);
        const int lw = q.zb[g] - 1, lh = std::min(mz - 1, q.zb[g] + 1);
        q.hb_warp[g + 1] = std::max(q.hb_warp[g], std::min(msz, bz[lw] + 2));
        q.hb_hv[g + 1] = std::max(q.hb_hv[g], std::min(msz, bz[lh] + 2));
        q.fb[g + 1] = g + 1 < G ? std::max(q.fb[g], bz[t.zlo + q.cb[g + 1] * t.zc]) : msz;
    }
    q.hb_warp[G] = q.hb_hv[G] = msz;
    q.din.resize(3 * static_cast<std::size_t>(ny));
    q.dout.resize(3 * static_cast<std::size_t>(ny));
    for (cudaStream_t* st : {&q.h2d, &q.d2h}) MFREG_CUDA(cudaStreamCreateWithFlags(st, cudaStreamNonBlocking));
    // the per-group finalize at the highest priority: otherwise the block scheduler keeps handing
    // the SMs to the next group's image-pass CTAs and the gathers (and their D2H) slip to the end
    int lo_prio = 0, hi_prio = 0;
    MFREG_CUDA(cudaDeviceGetStreamPriorityRange(&lo_prio, &hi_prio));
    MFREG_CUDA(cudaStreamCreateWithPriority(&q.fin, cudaStreamNonBlocking, hi_prio));
    auto mk = [](std::vector<cudaEvent_t>& v, int n) {
        v.resize(n);
        for (auto& e : v) MFREG_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    };
    mk(q.evh, G);
    mk(q.eve, G);
    mk(q.evf, G);
    MFREG_CUDA(cudaEventCreateWithFlags(&q.ev0, cudaEventDisableTiming));
    MFREG_CUDA(cudaEventCreateWithFlags(&q.evd, cudaEventDisableTiming));
    pipe_.state = 1;
    return true;
}

void DeviceObjective::pipe_in(const double* host, const std::vector<int>& hb) {
    Pipe& q = pipe_;
    const idx_t ny = dg_.count(), pn = dg_.m[0] * dg_.m[1];
    MFREG_CUDA(cudaEventRecord(q.ev0, s_));  // pin_in_ is free once the work before this call ran
    MFREG_CUDA(cudaStreamWaitEvent(q.h2d, q.ev0, 0));
    ptrace().mark("t0", q.h2d);
    for (int g = 0; g < q.G; ++g) {
        if (hb[g + 1] > hb[g])
            for (int d = 0; d < 3; ++d) {
                const idx_t off = d * ny + hb[g] * pn;
                MFREG_CUDA(cudaMemcpyAsync(q.din.get() + off, host + off, (hb[g + 1] - hb[g]) * pn * sizeof(double),
                                           cudaMemcpyHostToDevice, q.h2d));
            }
        MFREG_CUDA(cudaEventRecord(q.evh[g], q.h2d));
        ptrace().mark("h2d" + std::to_string(g), q.h2d);
    }
}

// group g's pass was just enqueued on s_: its nodes are gathered on the finalize stream and copied
// out on the D2H stream while the next group runs
void DeviceObjective::pipe_out(int g, double* host, bool hv) {
    Pipe& q = pipe_;
    const idx_t ny = dg_.count(), pn = dg_.m[0] * dg_.m[1];
    MFREG_CUDA(cudaEventRecord(q.eve[g], s_));
    ptrace().mark("pass" + std::to_string(g), s_);
    MFREG_CUDA(cudaStreamWaitEvent(q.fin, q.eve[g], 0));
    if (q.fb[g + 1] > q.fb[g]) {
        FinalizeSpec f;
        f.add = alpha_ != 0.0 ? curv_.get() : nullptr;
        f.out = q.dout.get();
        f.hv_pass = hv;
        f.nlo = q.fb[g];
        f.nhi = q.fb[g + 1];
        launch_nodal_finalize(plan_, *q.fp, f, q.fin);
    }
    MFREG_CUDA(cudaEventRecord(q.evf[g], q.fin));
    ptrace().mark("fin" + std::to_string(g), q.fin);
    MFREG_CUDA(cudaStreamWaitEvent(q.d2h, q.evf[g], 0));
    if (q.fb[g + 1] > q.fb[g])
        for (int d = 0; d < 3; ++d) {
            const idx_t off = d * ny + q.fb[g] * pn;
            MFREG_CUDA(cudaMemcpyAsync(host + off, q.dout.get() + off, (q.fb[g + 1] - q.fb[g]) * pn * sizeof(double),
                                       cudaMemcpyDeviceToHost, q.d2h));
        }
    ptrace().mark("d2h" + std::to_string(g), q.d2h);
}

void DeviceObjective::pipe_sync() {
    MFREG_CUDA(cudaEventRecord(pipe_.evd, pipe_.d2h));
    MFREG_CUDA(cudaStreamWaitEvent(s_, pipe_.evd, 0));
    MFREG_CUDA(cudaStreamSynchronize(s_));
}

bool DeviceObjective::eval_host(const double* y_host, double* grad_host, double* j) {
    if (!y_host || !grad_host || !pipe_ready()) return false;
    if (!(ngf_.tau_ > 0.0) || !(ngf_.rho_ > 0.0)) throw std::invalid_argument("NGF: tau and rho must be > 0");
    Pipe& q = pipe_;
    const idx_t ny = dg_.count();
    const double* y = q.din.get();
    pipe_in(y_host, q.hb_warp);
    // curvature value / gradient once the whole operand is in, on the high-priority finalize
    // stream (ahead of the group finalizes that add it): at normal priority its kernels queue
    // behind the next image-pass group's CTAs and hold every finalize back to the last group
    const cudaStream_t cs = q.fin;
    MFREG_CUDA(cudaStreamWaitEvent(cs, q.evh[q.G - 1], 0));
    launch_sub(3 * ny, y, xid_.get(), u_.get(), cs);
    launch_lap3(dg_, u_.get(), lapu_.get(), cs, 0, -1, false);
    red2_->sum(SUM_SQ, 3 * ny, lapu_.get(), nullptr, sc2_.get(), 1.0, cs);
    launch_curv_value(sc2_.get(), dg_.cell_volume(), alpha_, sc_.dev(1), sc_.host_dev() + 1, cs);
    if (alpha_ != 0.0)
        launch_bilap(dg_, lapu_.get(), alpha_ * (2.0 * dg_.cell_volume()), 0, 0.0, 0.0, nullptr, curv_.get(), cs, 0,
                     -1, false);
    // warp per z group as its nodal planes arrive, then the eval pass per group
    for (int g = 0; g < q.G; ++g) {
        MFREG_CUDA(cudaStreamWaitEvent(s_, q.evh[g], 0));  // chunk g completes the group's nodal planes
        warp_state(y, s_, q.za[g], q.zb[g], true);
        ptrace().mark("warp" + std::to_string(g), s_);
    }
    struct NoPdl {
        NoPdl() { pdl_suspended() = true; }
        ~NoPdl() { pdl_suspended() = false; }
    } nopdl;
    for (int g = 0; g < q.G; ++g) {
        launch_eval_fused(plan_, *q.fp, ngf_.R_, ngf_.Tw.get(), ngf_.dT.get(), ngf_.tau_, ngf_.rho_, frh_out(), true,
                          s_, sc_.dev(0), sc_.host_dev(), q.cb[g], q.cb[g + 1]);
        pipe_out(g, grad_host, false);
    }
    check_launch("Objective::eval (host pipeline)");
    pipe_sync();
    ptrace().dump("eval_host");
    stale_ = false;
    const double v = eval_end();
    if (j) *j = v;
    return true;
}

bool DeviceObjective::hv_host(const double* p_host, double* q_host) {
    if (!p_host || !q_host || !pipe_ready()) return false;
    Pipe& q = pipe_;
    refresh_state();
    const double* p = q.din.get();
    pipe_in(p_host, q.hb_hv);
    if (alpha_ != 0.0) {  // (on the finalize stream, as in eval_host)
        MFREG_CUDA(cudaStreamWaitEvent(q.fin, q.evh[q.G - 1], 0));
        launch_lap3(dg_, p, lapp_.get(), q.fin, 0, -1, false);
        launch_bilap(dg_, lapp_.get(), alpha_ * (2.0 * dg_.cell_volume()), 0, 0.0, 0.0, nullptr, curv_.get(), q.fin, 0,
                     -1, false);
    }
    struct NoPdl {
        NoPdl() { pdl_suspended() = true; }
        ~NoPdl() { pdl_suspended() = false; }
    } nopdl;
    for (int g = 0; g < q.G; ++g) {
        MFREG_CUDA(cudaStreamWaitEvent(s_, q.evh[g], 0));  // chunk g completes group g's planes
        launch_hv_fused(plan_, *q.fp, ngf_.frh.get(), ngf_.dT.get(), p, ngf_.tau_, ngf_.rho_, s_, nullptr, q.cb[g],
                        q.cb[g + 1]);
        pipe_out(g, q_host, true);
    }
    check_launch("Objective::gn_hessian_vec (host pipeline)");
    pipe_sync();
    ptrace().dump("hv_host");
    return true;
}

// optimizer.cpp:64-92
double DeviceObjective::eval(const double* y, double* grad) {
    eval_begin(y, grad);
    MFREG_CUDA(cudaStreamSynchronize(s_));
    return eval_end();
}

void DeviceObjective::eval_begin(const double* y, double* grad) {
    const idx_t ny = dg_.count();
    if (fused_) {
        if (!(ngf_.tau_ > 0.0) || !(ngf_.rho_ > 0.0)) throw std::invalid_argument("NGF: tau and rho must be > 0");
        // value-only calls (Armijo trials) skip the Hv state; refresh_state() rebuilds it if an
        // Hv follows without a gradient evaluation in between
        const bool lazy = grad == nullptr && !sliced_ && !no_lazy_state();
        if (lazy && ylazy_.size() < static_cast<std::size_t>(3 * ny)) ylazy_.resize(static_cast<std::size_t>(3 * ny));
        graphs_.run({y, grad, nullptr, nullptr, nullptr, reinterpret_cast<const void*>(lazy ? 4 : 1)}, s_,
                    [&](cudaStream_t cs) { enqueue_eval_fast(y, grad, cs, !lazy); });
        stale_ = lazy;
        return;  // the finalize wrote D and alpha S to the mapped host scalars
    }
    if (sliced_) throw std::logic_error("parity z slab: eval through SlabProblem");
    ngf_.populate_warp(plan_.view(), y, T_);
    ngf_.value_async(sc_.dev(0));
    launch_sub(3 * ny, y, xid_.get(), u_.get(), s_);
    launch_lap3(dg_, u_.get(), lapu_.get(), s_);
    ngf_.reducer().sum3(SUM_SQ, ny, lapu_.get(), nullptr, sc_.dev(4), 1.0, s_);
    launch_curv_finalize(sc_.dev(4), dg_.cell_volume(), alpha_, sc_.dev(1), s_);
    if (grad) {
        ngf_.gradient(img3_.get());
        launch_transfer_T(plan_.view(), img3_.get(), grad, s_);
        if (alpha_ != 0.0) launch_bilap(dg_, lapu_.get(), 2.0 * dg_.cell_volume(), 1, alpha_, 0.0, nullptr, grad, s_);
    }
    check_launch("Objective::eval");
    sc_.fetch_async(2, s_);
}

void DeviceObjective::parity_eval_local(const double* y, double* grad) {
    if (fused_) throw std::logic_error("parity_eval_local: parity-mode objectives only");
    const idx_t ny = dg_.count();
    ngf_.populate_warp(plan_.view(), y, T_, pw_.warp_lo, pw_.warp_hi, pw_.ws_lo, pw_.ws_hi);
    launch_sub(3 * ny, y, xid_.get(), u_.get(), s_);
    launch_lap3(dg_, u_.get(), lapu_.get(), s_, pw_.l_lo, pw_.l_hi);
    if (grad) {
        ngf_.gradient(img3_.get(), pw_.out_lo, pw_.out_hi);
        launch_transfer_T(plan_.view(), img3_.get(), grad, s_, pw_.n_lo, pw_.n_hi);
        if (alpha_ != 0.0)
            launch_bilap(dg_, lapu_.get(), 2.0 * dg_.cell_volume(), 1, alpha_, 0.0, nullptr, grad, s_, pw_.n_lo, pw_.n_hi);
    }
    check_launch("Objective::eval (parity slab)");
}

double DeviceObjective::eval_end() {
    const double* h = sc_.host();
    last_distance_ = h[0];
    last_regularizer_ = h[1];
    return last_distance_ + last_regularizer_;
}

// optimizer.cpp:94-104
void DeviceObjective::gn_hessian_vec(const double* p, double* q) {
    if (fused_) {
        refresh_state();
        graphs_.run({p, q, nullptr, nullptr, nullptr, reinterpret_cast<const void*>(2)}, s_,
                    [&](cudaStream_t cs) { enqueue_hv_fast(p, q, nullptr, nullptr, nullptr, cs); });
        return;
    }
    launch_Pp_s(plan_.view(), p, ngf_.dT.get(), ngf_.sv.get(), s_, pw_.s_lo, pw_.s_hi);
    ngf_.hessian_vec_image(ngf_.sv.get(), img3_.get(), pw_.out_lo, pw_.out_hi);
    launch_transfer_T(plan_.view(), img3_.get(), q, s_, pw_.n_lo, pw_.n_hi);
    if (alpha_ != 0.0) {
        launch_lap3(dg_, p, lapp_.get(), s_, pw_.l_lo, pw_.l_hi);
        launch_bilap(dg_, lapp_.get(), 2.0 * dg_.cell_volume(), 1, alpha_, 0.0, nullptr, q, s_, pw_.n_lo, pw_.n_hi);
    }
    check_launch("Objective::gn_hessian_vec");
}

// optimizer.cpp:106-111
void DeviceObjective::seed_hessian_vec(const double* p, double gamma, double* q) {
    launch_lap3(dg_, p, lapp_.get(), s_, pw_.l_lo, pw_.l_hi);
    launch_bilap(dg_, lapp_.get(), 2.0 * dg_.cell_volume(), 2, 0.0, gamma, p, q, s_, pw_.n_lo, pw_.n_hi);
    check_launch("Objective::seed_hessian_vec");
}

double DeviceObjective::dot(const double* a, const double* b) {
    if (sliced_) {  // owned nodal planes, per component, added in component order
        const idx_t ny = dg_.count(), pn = dg_.m[0] * dg_.m[1], off = slab_.own_lo * pn;
        for (int d = 0; d < 3; ++d)
            ngf_.reducer().sum(SUM_DOT, (slab_.own_hi - slab_.own_lo) * pn, a + d * ny + off, b + d * ny + off,
                               sc_.dev(12 + d), 1.0, s_);
        const double* h = sc_.fetch(15, s_);
        return (h[12] + h[13]) + h[14];
    }
    ngf_.reducer().sum(SUM_DOT, dof(), a, b, sc_.dev(8), 1.0, s_);
    return sc_.fetch(9, s_)[8];
}

void DeviceObjective::dot_async(const double* a, const double* b, double* out_dev) {
    ngf_.reducer().sum(SUM_DOT, dof(), a, b, out_dev, 1.0, s_);
}

void DeviceObjective::apply_dot(int op, double gamma, const double* p, double* q, double* pq_dev, const int* skip) {
    if (!fused_ || op != 0) {
        DeviceProblem::apply_dot(op, gamma, p, q, pq_dev, skip);
        return;
    }
    // fused GN Hv with <p, q> folded into the nodal finalize
    refresh_state();
    graphs_.run({p, q, pq_dev, skip, nullptr, reinterpret_cast<const void*>(3)}, s_,
                [&](cudaStream_t cs) { enqueue_hv_fast(p, q, p, pq_dev, skip, cs); });
}

// MFREG_NO_LAZY_STATE=1: value-only evaluations write the Hv state eagerly (A/B switch)
bool no_lazy_state() {
    static const bool off = [] {
        const char* e = std::getenv("MFREG_NO_LAZY_STATE");
        return e && e[0] == '1';
    }();
    return off;
}

// ------------------------------------------------------------------ GraphCache
GraphCache::GraphCache(std::size_t cap) : cap_(cap) {
    const char* off = std::getenv("MFREG_NO_GRAPHS");
    enabled_ = !(off && off[0] == '1');
}

GraphCache::~GraphCache() { clear(); }

void GraphCache::clear() {
    for (auto& e : entries_)
        if (e.exec) cudaGraphExecDestroy(e.exec);
    entries_.clear();
    if (cs_) cudaStreamDestroy(cs_);
    cs_ = nullptr;
}

GraphCache::Entry* GraphCache::find(const Key& k) {
    for (auto& e : entries_)
        if (e.key == k) {
            e.last_use = ++clock_;
            return &e;
        }
    return nullptr;
}

bool GraphCache::promote(const Key& k) {
    for (auto& e : seen_)
        if (e.first == k) return ++e.second >= kPromote;
    if (seen_.size() >= 4 * cap_) seen_.erase(seen_.begin());
    seen_.emplace_back(k, 1);
    return kPromote <= 1;
}

void GraphCache::begin() {
    if (!cs_) MFREG_CUDA(cudaStreamCreateWithFlags(&cs_, cudaStreamNonBlocking));
    l0_ = launch_counter();
    MFREG_CUDA(cudaStreamBeginCapture(cs_, cudaStreamCaptureModeRelaxed));
}

void GraphCache::abort() {
    cudaGraph_t g = nullptr;
    cudaStreamEndCapture(cs_, &g);
    if (g) cudaGraphDestroy(g);
    cudaGetLastError();
}

GraphCache::Entry* GraphCache::end(const Key& k) {
    cudaGraph_t g = nullptr;
    MFREG_CUDA(cudaStreamEndCapture(cs_, &g));
    cudaGraphExec_t ex = nullptr;
    const cudaError_t err = cudaGraphInstantiate(&ex, g, 0);
    cudaGraphDestroy(g);
    MFREG_CUDA(err);
    const long long n = launch_counter() - l0_;
    note_launches(-n);  // counted again on every replay
    if (entries_.size() >= cap_) {  // evict the least recently used
        auto it = std::min_element(entries_.begin(), entries_.end(),
                                   [](const Entry& a, const Entry& b) { return a.last_use < b.last_use; });
        cudaGraphExecDestroy(it->exec);
        entries_.erase(it);
    }
    entries_.push_back(Entry{k, ex, n, ++clock_});
    return &entries_.back();
}

void GraphCache::launch(Entry* e, cudaStream_t s) {
    MFREG_CUDA(cudaGraphLaunch(e->exec, s));
    note_launches(e->launches);
}

DeviceCg& DeviceProblem::cg_workspace() {
    if (!cg_) cg_ = std::make_shared<DeviceCg>(dof());
    return *cg_;
}

double DeviceObjective::inf_norm(const double* a, double scale) {
    launch_inf_norm(dof(), a, scale, sc_.dev(10), s_);
    check_launch("inf_norm");
    return sc_.fetch(11, s_)[10];
}

}  // namespace mfreg_b200
