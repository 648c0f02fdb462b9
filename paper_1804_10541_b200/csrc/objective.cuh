// Host-side C++ runtime for the device-resident hot path: device buffers, the
// transfer plan, the NGF state, DeviceObjective (reference Objective,
// optimizer.hpp:53-106), the device-resident solvers (optimizer.cpp:113-407) and
// the multilevel driver (multilevel.cpp:117-145).
#pragma once

#include <cuda_runtime.h>

#include <array>
#include <cmath>
#include <cstdint>
#include <deque>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "kernels.cuh"

namespace mfreg_b200 {

struct CudaError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

#define MFREG_CUDA(call)                                                                                  \
    do {                                                                                                  \
        cudaError_t e_ = (call);                                                                          \
        if (e_ != cudaSuccess)                                                                            \
            throw ::mfreg_b200::CudaError(std::string(#call) + ": " + cudaGetErrorString(e_));          \
    } while (0)

void check_launch(const char* what);

// Parity: bitwise = reference; Fast: fused kernels, fp64; Fast32: fused kernels with the
// image-grid state (T_w, dT, rho-hat) and the fused arithmetic in fp32 (north star's optional
// fp32 mode, tolerance 1e-4); nodal vectors, reductions and solvers stay fp64.
enum class Mode : int { Parity = 0, Fast = 1, Fast32 = 2 };

// Device allocations come from the device's default stream-ordered pool (allocated and
// freed on the legacy stream, which all library work is ordered with) with up to
// MFREG_POOL_KEEP_GB kept cached: objectives are created per pyramid level and per call, and
// cudaMalloc/cudaFree of their state cost tens of milliseconds with a wide spread.
// (blocks of kBigAllocBytes and more use cudaMalloc and an exact-size cache of freed blocks:
// growing the pool by tens of GB on first use measured 0.6-4 s against 0.05 s for cudaMalloc, and
// pool allocations of 90-180 MB measured 0.1-0.5 s stalls when a registration's level objectives
// were rebuilt — the 256 MB threshold of earlier let the per-level nodal and partial arrays
// through the pool)
constexpr std::size_t kBigAllocBytes = std::size_t(32) << 20;
void* device_alloc(std::size_t bytes);
// high-water mark of the library's live device allocations since load (or the last reset)
long long device_memory_peak(bool reset);
void device_free(void* p, std::size_t bytes);
// small mapped pinned host blocks (<= kPinnedSmall bytes), recycled across objectives:
// cudaFreeHost synchronises the device and measured tens to hundreds of ms per teardown
constexpr std::size_t kPinnedSmall = 4096;
void* pinned_small_alloc(std::size_t bytes);
void pinned_small_free(void* p);

// RAII device array of doubles (or raw bytes).
template <typename T>
class DevArray {
public:
    DevArray() = default;
    explicit DevArray(std::size_t n) { resize(n); }
    ~DevArray() { release(); }
    DevArray(const DevArray&) = delete;
    DevArray& operator=(const DevArray&) = delete;
    DevArray(DevArray&& o) noexcept : p_(o.p_), n_(o.n_) {
        o.p_ = nullptr;
        o.n_ = 0;
    }
    DevArray& operator=(DevArray&& o) noexcept {
        if (this != &o) {
            release();
            p_ = o.p_;
            n_ = o.n_;
            o.p_ = nullptr;
            o.n_ = 0;
        }
        return *this;
    }
    void resize(std::size_t n) {
        if (n == n_) return;
        release();
        if (n) p_ = static_cast<T*>(device_alloc(n * sizeof(T)));
        n_ = n;
    }
    void release() {
        if (p_) device_free(p_, n_ * sizeof(T));
        p_ = nullptr;
        n_ = 0;
    }
    T* get() { return p_; }
    const T* get() const { return p_; }
    std::size_t size() const { return n_; }

private:
    T* p_ = nullptr;
    std::size_t n_ = 0;
};
using DVec = DevArray<double>;

// Validation mirroring grid.hpp:103-146 (messages identical to the reference).
void validate_grid(const Grid& g, bool nodal);
Grid make_deform_grid(const Grid& image, const idx_t points[3]);
Grid deformation_grid_for(const Grid& image, idx_t ratio);

// transfer.cpp:11-47 computed on the host bit-identically, uploaded once per level.
class DevicePlanOwner {
public:
    DevicePlanOwner(const Grid& nodal, const Grid& image);
    const DevPlan& view() const { return view_; }
    std::vector<int> host_base[3];
    std::vector<double> host_rem[3];

private:
    DevArray<int> base_[3], lo_[3], hi_[3];
    DVec rem_[3];
    DevPlan view_{};
};

// transfer.cpp:24-35 on one axis: image index -> nodal cell (host, no device state)
std::vector<int> plan_base_axis(idx_t image_m, idx_t nodal_m);

// z-slab decomposition: rank r outputs the image planes
// [zlo, zhi) (D and the P^T contributions of those planes) and owns the nodal
// planes [own_lo, own_hi) (curvature term, dot products). Splits fall on nodal
// cell boundaries, so neighbouring ranks share exactly the P^T planes
// [own_hi, own_hi + bnd) (summed on the upper rank). Before an operator call the
// nodal operand must be valid on [need_lo, need_hi) (halo from the neighbours).
struct SlabSpec {
    int zlo = 0, zhi = -1, own_lo = 0, own_hi = -1;
    bool full(int mz, int msz) const { return zhi < 0 || (zlo == 0 && zhi == mz && own_lo == 0 && own_hi == msz); }
};
struct SlabInfo {
    int zlo, zhi, own_lo, own_hi, need_lo, need_hi, bnd;
};
// parity: the operand halo of the parity-mode slabs (their owned nodes' P^T reads the image
// planes of the nodal slab below the first owned plane, recomputed from the operand)
std::vector<SlabInfo> slab_partition(const Grid& image, const Grid& deform, int nranks, bool parity = false);

// CUDA graphs for fixed launch sequences, keyed by the pointers they bake in
// (replayed on the caller's stream; LRU-bounded). MFREG_NO_GRAPHS=1 disables.
class GraphCache {
public:
    // set while this thread captures an enclosing graph (DeviceCg windows): nested calls enqueue
    // their work inline instead of launching their own graphs
    static bool& capturing() {
        static thread_local bool flag = false;
        return flag;
    }
    using Key = std::array<const void*, 6>;
    explicit GraphCache(std::size_t cap = 8);
    ~GraphCache();
    void clear();  // destroy every cached graph
    GraphCache(const GraphCache&) = delete;
    GraphCache& operator=(const GraphCache&) = delete;
    bool enabled() const { return enabled_; }
    template <class F>
    void run(const Key& k, cudaStream_t s, F&& enqueue) {
        if (!enabled_ || capturing()) {
            enqueue(s);  // graphs off, or an enclosing graph (CG window) is being captured
            return;
        }
        Entry* e = find(k);
        if (!e && !promote(k)) {  // keys seen fewer than kPromote times run eagerly
            enqueue(s);
            return;
        }
        if (!e) {
            begin();
            try {
                enqueue(cs_);
            } catch (...) {
                abort();
                throw;
            }
            e = end(k);
        }
        launch(e, s);
    }

private:
    struct Entry {
        Key key;
        cudaGraphExec_t exec;
        long long launches;
        unsigned long long last_use;
    };
    Entry* find(const Key& k);
    bool promote(const Key& k);  // counts a miss; true once the key is worth a graph
    static constexpr int kPromote = 3;
    std::vector<std::pair<Key, int>> seen_;
    void begin();
    void abort();
    Entry* end(const Key& k);
    void launch(Entry* e, cudaStream_t s);
    std::vector<Entry> entries_;
    std::size_t cap_;
    bool enabled_ = true;
    cudaStream_t cs_ = nullptr;
    long long l0_ = 0;
    unsigned long long clock_ = 0;
};

// Reduction helpers: exact 4096-chunk order (parity) or fixed-order tree (fast).
class Reducer {
public:
    Reducer(Mode mode, idx_t max_n);
    // device result into out_dev (scaled)
    void sum(int kind, idx_t n, const double* a, const double* b, double* out_dev, double scale, cudaStream_t s);
    // three segments a + d n (d = 0..2) into out_dev[0..2], each exactly as sum(); one launch pair
    void sum3(int kind, idx_t n, const double* a, const double* b, double* out_dev, double scale, cudaStream_t s);
    Mode mode() const { return mode_; }

private:
    Mode mode_;
    DVec partials_;
};

// Scalar staging: a few device doubles mirrored into pinned host memory.
class Scalars {
public:
    explicit Scalars(int n = 32);
    ~Scalars();
    double* dev(int i) { return d_.get() + i; }
    // copies [0, n) to host and synchronises the stream
    const double* fetch(int n, cudaStream_t s);
    // enqueues the copy of [0, n) only; host() is valid after the stream is synchronised
    void fetch_async(int n, cudaStream_t s);
    const double* host() const { return h_; }
    // device view of the (mapped, pinned) host buffer: a kernel that writes a scalar here
    // makes it readable by the host after the stream synchronises, with no copy
    double* host_dev() { return hd_; }

private:
    DVec d_;
    double* h_ = nullptr;
    double* hd_ = nullptr;
};

// Abstract problem the device-resident solvers drive (reference Problem,
// optimizer.hpp:36-48), with the vector-space operations the solvers need so a
// sharded implementation can reduce across GPUs.
class DeviceProblem {
public:
    virtual ~DeviceProblem() = default;
    virtual idx_t dof() const = 0;  // local length of y
    virtual double eval(const double* y, double* grad) = 0;
    virtual void gn_hessian_vec(const double* p, double* q) = 0;
    virtual void seed_hessian_vec(const double* p, double gamma, double* q) = 0;
    virtual double min_spacing() const = 0;
    virtual double alpha() const = 0;
    virtual double last_distance() const = 0;
    virtual double last_regularizer() const = 0;
    virtual double dot(const double* a, const double* b) = 0;  // vec_dot (optimizer.cpp:12-19)
    virtual double inf_norm(const double* a, double scale) = 0;  // max |scale * a_i|
    virtual cudaStream_t stream() const = 0;
    double norm(const double* a) { return std::sqrt(dot(a, a)); }
    // asynchronous vec_dot with a device result (exact chunk order in parity mode)
    virtual void dot_async(const double* a, const double* b, double* out_dev) = 0;
    // fixed-order tree reductions allowed (fast mode)
    virtual bool fast_reductions() const = 0;
    // q = A p and <p, q> into pq_dev (A = GN operator, op 0, or seed operator, op 1);
    // `skip` (device flag, nullable): work may be skipped when *skip != 0
    virtual void apply_dot(int op, double gamma, const double* p, double* q, double* pq_dev, const int* skip) {
        (void)skip;
        if (op == 1) seed_hessian_vec(p, gamma, q);
        else gn_hessian_vec(p, q);
        dot_async(p, q, pq_dev);
    }
    // the CG loop may be captured into CUDA graphs (everything apply_dot / dot_async enqueue
    // is device work on stream(), no host synchronisation or allocation)
    virtual bool cg_graphable() const { return false; }
    // route the problem's work to `s` (the CG graph capture stream) until redirected back
    virtual void redirect_stream(cudaStream_t s) { (void)s; }
    // make the operator's cached state current (called before a CG loop is captured)
    virtual void prepare_operator() {}
    // device-resident CG workspace (created on first use)
    class DeviceCg& cg_workspace();

private:
    std::shared_ptr<class DeviceCg> cg_;
};

// NGF state on the image grid: reference image (+ its owner), sampled template
// state and the per-iterate workspace (ngf.hpp:21-37).
class DeviceNgf {
public:
    DeviceNgf(const Grid& img, const double* R_dev, double tau, double rho, Mode mode, cudaStream_t s);
    // populate from explicit sample points (ngf.cpp:185-214), both device pointers
    void ensure_ws();
    void populate_points(const double* T_dev, const double* pts_dev);
    // populate from the nodal deformation (transfer_apply + populate fused)
    // (windows: image planes [lo, hi) of the warp / workspace / outputs, default the whole grid;
    // parity-mode z slabs compute only what their owned nodes read)
    void populate_warp(const DevPlan& P, const double* y_dev, const double* T_dev, int wlo = 0, int whi = -1,
                       int slo = 0, int shi = -1);
    void value_async(double* out_dev);                 // D (ngf.cpp:225-231)
    void gradient(double* out3n, int zlo = 0, int zhi = -1);  // dD/dP (ngf.cpp:66-103)
    void hessian_vec_image(const double* sv, double* out3n, int zlo = 0, int zhi = -1);  // from s = dT.(P p)
    void hessian_vec(const double* p3n, double* out3n);        // image-grid p (ngf.cpp:253-258)
    const Grid& grid() const { return g_; }
    Mode mode() const { return mode_; }
    cudaStream_t stream() const { return s_; }
    Reducer& reducer() { return red_; }

    Grid g_;
    double tau_, rho_;
    Mode mode_;
    cudaStream_t s_;
    const double* R_;  // borrowed
    DVec Tw, dT, r, inv1, inv2, rh, sv, wbuf;
    DVec frh;  // fast mode: rho-hat [6][n] (-x,+x,-y,+y,-z,+z), the Hv state
    DevArray<float> R32, Tw32, dT32, frh32;  // Fast32 state
    void release() {  // free the image-grid state now (the destructor would)
        for (DVec* v : {&Tw, &dT, &r, &inv1, &inv2, &rh, &sv, &wbuf, &frh}) v->release();
        for (DevArray<float>* v : {&R32, &Tw32, &dT32, &frh32}) v->release();
    }
    bool fp32() const { return mode_ == Mode::Fast32; }
    const void* state_R() const { return fp32() ? static_cast<const void*>(R32.get()) : R_; }
    void* state_Tw() { return fp32() ? static_cast<void*>(Tw32.get()) : Tw.get(); }
    void* state_dT() { return fp32() ? static_cast<void*>(dT32.get()) : dT.get(); }
    void* state_frh() { return fp32() ? static_cast<void*>(frh32.get()) : frh.get(); }
    HvTable tab_;
    Reducer red_;
};

class DeviceObjective : public DeviceProblem {
public:
    // R_dev/T_dev: device arrays over `image` that must outlive the objective
    // (the reference Objective also stores references, optimizer.hpp:87-88).
    // `slab`: this rank's z window (fast mode only); default: the whole domain
    DeviceObjective(const double* R_dev, const double* T_dev, const Grid& image, const Grid& deform, double tau,
                    double rho, double alpha, Mode mode, cudaStream_t s, const SlabSpec& slab = SlabSpec{});
    ~DeviceObjective() override;
    idx_t dof() const override { return 3 * dg_.count(); }
    double eval(const double* y, double* grad) override;
    // eval split for host-buffer callers: enqueue everything (incl. the scalar copy-out),
    // let the caller enqueue its own copies, synchronise once, then read J
    void eval_begin(const double* y, double* grad);
    double eval_end();
    // host-buffer calls with the copies pipelined against the passes: the H2D of
    // the operand in nodal z chunks ahead of the warp / Hv pass launched in z groups, each group's
    // nodes finalized and copied out while the next group runs. Returns false (nothing done) when
    // the pipeline does not apply (parity mode, z slabs, legacy kernels, small grids,
    // MFREG_NO_PIPE=1); the caller then stages the buffers whole.
    bool eval_host(const double* y_host, double* grad_host, double* j);
    bool hv_host(const double* p_host, double* q_host);
    void gn_hessian_vec(const double* p, double* q) override;
    void seed_hessian_vec(const double* p, double gamma, double* q) override;
    double min_spacing() const override;
    double alpha() const override { return alpha_; }
    double last_distance() const override { return last_distance_; }
    double last_regularizer() const override { return last_regularizer_; }
    double dot(const double* a, const double* b) override;
    double inf_norm(const double* a, double scale) override;
    cudaStream_t stream() const override { return s_; }
    void dot_async(const double* a, const double* b, double* out_dev) override;
    bool fast_reductions() const override { return fused_ != nullptr; }
    bool cg_graphable() const override { return fused_ != nullptr && !sliced_ && graphs_.enabled(); }
    void redirect_stream(cudaStream_t s) override { s_ = s; }
    void prepare_operator() override { refresh_state(); }
    void apply_dot(int op, double gamma, const double* p, double* q, double* pq_dev, const int* skip) override;
    const double* identity_dev() const { return xid_.get(); }
    // parity-mode z slabs (slab.cu): the windowed eval without its value reductions; the slab
    // problem assembles D and S across ranks (DistSum) from r and Lap u
    void parity_eval_local(const double* y, double* grad);
    const double* parity_r() const { return ngf_.r.get(); }
    const double* lap_u() const { return lapu_.get(); }
    const Grid& image_grid() const { return img_; }
    const Grid& deform_grid() const { return dg_; }
    DeviceNgf& ngf() { return ngf_; }
    const DevicePlanOwner& plan() const { return plan_; }
    bool sliced() const { return sliced_; }
    // bench support: average device time (CUDA events on the launching stream) of one
    // image-pass kernel of the fast path: 0 = GN Hv pass (operand p), 1 = eval pass
    // (gradient), 2 = warp; `flush_bytes` > 0 writes a scratch buffer that large before
    // every timed launch (L2 flush, outside the timed interval). Needs a prior eval.
    double profile_kernel(int which, const double* p, int reps, std::size_t flush_bytes);

private:
    // state=false: value-only evaluation that leaves the Hv state (dT, rho-hat) unwritten and
    // records y in ylazy_; refresh_state() rebuilds that state before the next Hv needs it
    void enqueue_eval_fast(const double* y, double* grad, cudaStream_t s, bool state = true);
    void warp_state(const double* y, cudaStream_t s, int zlo, int zhi, bool state = true);
    void refresh_state();
    // where the eval pass stores rho-hat: nowhere when the Hv pass recomputes it (hv3)
    double* frh_out();
    void enqueue_hv_fast(const double* p, double* q, const double* dot_a, double* sc, const int* skip, cudaStream_t s);
    bool pipe_ready();
    void pipe_in(const double* host, const std::vector<int>& hb);  // H2D by nodal z chunks -> pin_in_
    void pipe_out(int g, double* host, bool hv);                   // finalize group g's nodes -> D2H
    void pipe_sync();
    struct Pipe {
        int state = 0;                        // 0 unset, 1 on, 2 off
        int G = 0;                            // z groups
        std::vector<int> cb;                  // [G + 1] z tile chunk bounds of the groups
        std::vector<int> za, zb;              // image planes of group g
        std::vector<int> hb_warp, hb_hv;      // [G + 1] nodal z bounds of the H2D chunks (eval / Hv)
        std::vector<int> fb;                  // [G + 1] nodal z bounds of the per-group finalize
        cudaStream_t h2d = nullptr, d2h = nullptr, fin = nullptr;
        std::vector<cudaEvent_t> evh, eve, evf;
        cudaEvent_t ev0 = nullptr, evd = nullptr;
        DVec din, dout;
        std::unique_ptr<class FusedPlan> fp;  // the same passes on z chunks of <= 128 planes
    } pipe_;
    Grid img_, dg_;
    SlabSpec slab_;
    bool sliced_ = false;
    // parity-mode slab windows: warp, workspace, image outputs, s (image planes); P^T / curvature
    // outputs and Lap (nodal planes). Whole grid by default.
    struct PWin {
        int warp_lo = 0, warp_hi = -1, ws_lo = 0, ws_hi = -1, out_lo = 0, out_hi = -1, s_lo = 0, s_hi = -1;
        int n_lo = 0, n_hi = -1, l_lo = 0, l_hi = -1;
    } pw_;
    bool stale_ = false;  // Hv state belongs to ylazy_, not yet rebuilt (lazy value-only eval)
    DVec ylazy_;
    double alpha_;
    cudaStream_t s_;
    const double* T_;
    DevicePlanOwner plan_;
    DeviceNgf ngf_;
    DVec xid_, u_, lapu_, lapp_, img3_;
    std::unique_ptr<class FusedPlan> fused_;  // fast mode: fused single-pass kernels
    cudaStream_t s2_ = nullptr;                // fast mode: side stream (nodal curvature terms)
    cudaEvent_t ev_fork_ = nullptr, ev_join_ = nullptr;
    std::unique_ptr<Reducer> red2_;
    DVec curv_, sc2_;
    Scalars sc_;
    GraphCache graphs_;
    double last_distance_ = 0.0, last_regularizer_ = 0.0;
};

// ---- solvers (optimizer.hpp:108-166), vectors on the device
struct CgConfig {
    int max_iters = 50;
    double rel_tol = 1e-2;
};
struct CgResult {
    int iters = 0;
    double relres = 0.0;
    bool breakdown = false;
};
struct ArmijoConfig {
    double c1 = 1e-4;
    double beta = 0.5;
    int max_backtracks = 10;
};
struct OptimizerConfig {
    int max_iters = 20;
    ArmijoConfig armijo{};
    CgConfig cg{50, 1e-2};
    CgConfig h0_cg{20, 1e-2};
    int lbfgs_history = 5;
    double gamma = -1.0;
    double tol_rel_j = 1e-4;
    double tol_grad = 1e-4;
    double tol_step = 1e-3;
};
struct IterationRecord {
    int iter = 0;
    int cg_iters = 0;
    double j = 0.0, distance = 0.0, regularizer = 0.0, grad_norm = 0.0, step = 0.0;
};
struct MinimizeResult {
    std::vector<IterationRecord> trace;
    bool line_search_failed = false;
};

// op: 0 = Gauss-Newton operator, 1 = L-BFGS seed (Hess S + gamma I)
CgResult cg_solve(DeviceProblem& P, int op, double gamma, const double* b, double* x, const CgConfig& cfg);
MinimizeResult gauss_newton_minimize(DeviceProblem& P, const double* y0, double* y, const OptimizerConfig& cfg);
MinimizeResult lbfgs_minimize(DeviceProblem& P, const double* y0, double* y, const OptimizerConfig& cfg);

enum class Method : int { Lbfgs = 0, GaussNewton = 1 };
struct MultilevelConfig {
    int levels = 3;
    idx_t deform_ratio = 4;
    double tau = 10.0, rho = 10.0;
    double alpha = 1.0;
    Method method = Method::Lbfgs;
    Mode mode = Mode::Parity;
    OptimizerConfig opt{};
    bool keep_level_y = false;  // LevelResult::y (multilevel.hpp:47-51 result.y) for every level
};
struct LevelResult {
    Grid image_grid, deform_grid;
    MinimizeResult result;
    DVec y;  // the level's final deformation (when MultilevelConfig::keep_level_y)
};
struct MultilevelResult {
    DVec y;
    Grid deform_grid;
    std::vector<LevelResult> levels;  // coarsest first
};
MultilevelResult register_multilevel(const double* R_dev, const double* T_dev, const Grid& image,
                                     const MultilevelConfig& cfg, cudaStream_t s);

}  // namespace mfreg_b200
