// The rest of the reference's public API over the C ABI (include/mfreg_cuda.h, "drop-in
// API" section): per-point volume / curvature / nodal-interpolation helpers, the NGF
// precompute, the offset table, the deterministic vector reductions, and a host-defined
// Problem (reference optimizer.hpp:36-48) driven by the device-resident solvers.
//
// Every computation runs on the GPU in the reference's operation order (the library is
// built with --fmad=false), so the parity-mode results are bitwise those of the reference.
#include <algorithm>
#include <cmath>
#include <map>
#include <vector>

#include "capi_util.cuh"
#include "cg.cuh"

using namespace mfreg_b200;
using namespace mfreg_b200::capi;

namespace {

__device__ __forceinline__ long long clamp_ll(long long v, long long hi) { return v < 0 ? 0 : (v > hi ? hi : v); }

// volume.cpp:96-109 — backward x,y,z then forward x,y,z, clamped neighbours, IEEE quotient by h
__device__ __forceinline__ void dgrad6_at(const double* __restrict__ v, const Grid& g, long long i, double r[6]) {
    const long long m0 = g.m[0], m1 = g.m[1], m2 = g.m[2];
    const long long x = i % m0, y = (i / m0) % m1, z = i / (m0 * m1);
    const double vi = v[i];
    const long long nb[6] = {g.lin(clamp_ll(x - 1, m0 - 1), y, z), g.lin(x, clamp_ll(y - 1, m1 - 1), z),
                             g.lin(x, y, clamp_ll(z - 1, m2 - 1)), g.lin(clamp_ll(x + 1, m0 - 1), y, z),
                             g.lin(x, clamp_ll(y + 1, m1 - 1), z), g.lin(x, y, clamp_ll(z + 1, m2 - 1))};
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        r[a] = __ddiv_rn(vi - v[nb[a]], g.h[a]);
        r[a + 3] = __ddiv_rn(v[nb[a + 3]] - vi, g.h[a]);
    }
}

// volume.cpp:115-121
__device__ __forceinline__ double eps_norm_dev(const double g[6], double eps) {
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < 6; ++k) s += g[k] * g[k];
    return sqrt(0.5 * s + eps * eps);
}

// discrete_gradient at idx[k] (all voxels when idx is null) -> out[6k..6k+5]; with
// `norm_eps` >= 0 also eps_norm of it -> norm[k] (make_ngf_precomp, ngf.cpp:167-183)
__global__ void k_dgrad(Grid g, const double* __restrict__ v, const long long* __restrict__ idx, long long n,
                        double* __restrict__ out6, double norm_eps, double* __restrict__ norm) {
    const long long k = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (k >= n) return;
    double r[6];
    dgrad6_at(v, g, idx ? idx[k] : k, r);
    if (out6)
        for (int c = 0; c < 6; ++c) out6[6 * k + c] = r[c];
    if (norm) norm[k] = eps_norm_dev(r, norm_eps);
}

__global__ void k_eps_norm(const double* __restrict__ g6, long long n, double eps, double* __restrict__ out) {
    const long long k = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (k >= n) return;
    double r[6];
    for (int c = 0; c < 6; ++c) r[c] = g6[6 * k + c];
    out[k] = eps_norm_dev(r, eps);
}

// curvature.cpp:9-21 at node idx[k]
__global__ void k_lap_at(Grid g, const double* __restrict__ u, const long long* __restrict__ idx, long long n,
                         double* __restrict__ out) {
    const long long k = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (k >= n) return;
    const long long i = idx[k], m0 = g.m[0], m1 = g.m[1], m2 = g.m[2];
    const long long c[3] = {i % m0, (i / m0) % m1, i / (m0 * m1)};
    const long long st[3] = {1, m0, m0 * m1};
    const long long mm[3] = {m0, m1, m2};
    const double ui = u[i];
    double s = 0.0;
    for (int a = 0; a < 3; ++a) {
        const long long lo = c[a] > 0 ? i - st[a] : i, hi = c[a] < mm[a] - 1 ? i + st[a] : i;
        const double h = g.h[a];
        s += (u[lo] - 2.0 * ui + u[hi]) / (h * h);
    }
    out[k] = s;
}

// multilevel.cpp:51-76 at the points p[3k..3k+2]
__global__ void k_nodal_interp(Grid g, const double* __restrict__ comp, const double* __restrict__ pts, long long n,
                               double* __restrict__ out) {
    const long long k = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (k >= n) return;
    long long b[3];
    double w[3];
    for (int a = 0; a < 3; ++a) {
        const long long ma = g.m[a];
        double s = pts[3 * k + a] / g.h[a];
        const double hi = static_cast<double>(ma - 1);
        s = s < 0.0 ? 0.0 : (hi < s ? hi : s);
        long long base = static_cast<long long>(floor(s));
        base = base < 0 ? 0 : (base > ma - 2 ? ma - 2 : base);
        b[a] = base;
        w[a] = s - static_cast<double>(base);
    }
    double v = 0.0;
    for (int c = 0; c < 2; ++c)
        for (int bb = 0; bb < 2; ++bb)
            for (int aa = 0; aa < 2; ++aa) {
                const double weight = (aa ? w[0] : 1.0 - w[0]) * (bb ? w[1] : 1.0 - w[1]) * (c ? w[2] : 1.0 - w[2]);
                v += weight * comp[g.lin(b[0] + aa, b[1] + bb, b[2] + c)];
            }
    out[k] = v;
}

inline unsigned blocks_for(long long n) { return static_cast<unsigned>(std::max<long long>(1, (n + 255) / 256)); }

// host index list -> device
struct Idx {
    Idx(const int64_t* idx, long long n) {
        if (!idx || n <= 0) return;
        buf.resize(static_cast<std::size_t>(n));
        MFREG_CUDA(cudaMemcpyAsync(buf.get(), idx, n * sizeof(long long), cudaMemcpyHostToDevice, kStream));
    }
    DevArray<long long> buf;
    const long long* ptr() const { return buf.size() ? buf.get() : nullptr; }
};

// ---- a host-defined Problem (optimizer.hpp:36-48) for the device-resident solvers. The
// solver vectors live in HBM; each operator call stages its operand to pinned host memory,
// runs the host callback and stages the result back. Reductions are the reference's exact
// 4096-chunk sums (vec_dot, optimizer.cpp:12-19), so traces are bitwise the reference's.
class CallbackProblem : public DeviceProblem {
public:
    CallbackProblem(const mfreg_cu_problem_ops& ops, idx_t n)
        : ops_(ops), n_(n), red_(Mode::Parity, n), sc_(16) {
        if (!ops.eval || !ops.gn_hessian_vec || !ops.seed_hessian_vec || !ops.min_spacing)
            throw std::invalid_argument("problem: eval, gn_hessian_vec, seed_hessian_vec and min_spacing are required");
        MFREG_CUDA(cudaMallocHost(&h_in_, std::max<idx_t>(1, n) * sizeof(double)));
        MFREG_CUDA(cudaMallocHost(&h_out_, std::max<idx_t>(1, n) * sizeof(double)));
    }
    ~CallbackProblem() override {
        cudaFreeHost(h_in_);
        cudaFreeHost(h_out_);
    }
    idx_t dof() const override { return n_; }
    double eval(const double* y, double* grad) override {
        down(y);
        double j = 0.0;
        call(ops_.eval(ops_.ctx, h_in_, grad ? h_out_ : nullptr, &j), "eval");
        if (grad) up(grad);
        return j;
    }
    void gn_hessian_vec(const double* p, double* q) override {
        down(p);
        call(ops_.gn_hessian_vec(ops_.ctx, h_in_, h_out_), "gn_hessian_vec");
        up(q);
    }
    void seed_hessian_vec(const double* p, double gamma, double* q) override {
        down(p);
        call(ops_.seed_hessian_vec(ops_.ctx, h_in_, gamma, h_out_), "seed_hessian_vec");
        up(q);
    }
    double min_spacing() const override { return ops_.min_spacing(ops_.ctx); }
    double alpha() const override { return ops_.alpha ? ops_.alpha(ops_.ctx) : 0.0; }
    double last_distance() const override { return ops_.last_distance ? ops_.last_distance(ops_.ctx) : 0.0; }
    double last_regularizer() const override {
        return ops_.last_regularizer ? ops_.last_regularizer(ops_.ctx) : 0.0;
    }
    double dot(const double* a, const double* b) override {
        red_.sum(SUM_DOT, n_, a, b, sc_.dev(0), 1.0, kStream);
        return sc_.fetch(1, kStream)[0];
    }
    double inf_norm(const double* a, double scale) override {
        launch_inf_norm(n_, a, scale, sc_.dev(2), kStream);
        check_launch("inf_norm");
        return sc_.fetch(3, kStream)[2];
    }
    cudaStream_t stream() const override { return kStream; }
    void dot_async(const double* a, const double* b, double* out_dev) override {
        red_.sum(SUM_DOT, n_, a, b, out_dev, 1.0, kStream);
    }
    bool fast_reductions() const override { return false; }

private:
    void down(const double* d) {
        MFREG_CUDA(cudaMemcpyAsync(h_in_, d, n_ * sizeof(double), cudaMemcpyDeviceToHost, kStream));
        MFREG_CUDA(cudaStreamSynchronize(kStream));
    }
    void up(double* d) {
        MFREG_CUDA(cudaMemcpyAsync(d, h_out_, n_ * sizeof(double), cudaMemcpyHostToDevice, kStream));
        MFREG_CUDA(cudaStreamSynchronize(kStream));
    }
    static void call(int rc, const char* what) {
        if (rc != 0) throw std::runtime_error(std::string("problem callback failed: ") + what);
    }
    mfreg_cu_problem_ops ops_;
    idx_t n_;
    Reducer red_;
    Scalars sc_;
    double* h_in_ = nullptr;
    double* h_out_ = nullptr;
};

void get_trace(const MinimizeResult& res, mfreg_cu_iter_record* trace, int cap, int* ntrace, int* lsf) {
    const int n = copy_trace(res.trace, trace, cap);
    if (ntrace) *ntrace = n;
    if (lsf) *lsf = res.line_search_failed ? 1 : 0;
}

}  // namespace

extern "C" {

// ---- vec_dot / vec_norm / vec_inf_norm (optimizer.cpp:12-29)
int mfreg_cu_vec_dot(const double* a, const double* b, int64_t n, int where, double* out) {
    return guard([&] {
        if (n < 0) throw std::invalid_argument("vec_dot: length mismatch");
        In ai(a, n, where, kStream), bi(b, n, where, kStream);
        Reducer red(Mode::Parity, n);
        Scalars sc(2);
        red.sum(SUM_DOT, n, ai.ptr, bi.ptr, sc.dev(0), 1.0, kStream);
        *out = sc.fetch(1, kStream)[0];
    });
}
int mfreg_cu_vec_inf_norm(const double* a, int64_t n, int where, double* out) {
    return guard([&] {
        In ai(a, n, where, kStream);
        Scalars sc(2);
        launch_inf_norm(n, ai.ptr, 1.0, sc.dev(0), kStream);
        check_launch("vec_inf_norm");
        *out = sc.fetch(1, kStream)[0];
    });
}

// ---- make_transfer_plan (transfer.cpp:11-47): per-axis base / rem, image axes concatenated
int mfreg_cu_transfer_plan(const mfreg_cu_grid* nodal, const mfreg_cu_grid* image, int64_t* base, double* rem) {
    return guard([&] {
        DevicePlanOwner plan(to_grid(nodal), to_grid(image));
        std::size_t o = 0;
        for (int a = 0; a < 3; ++a)
            for (std::size_t k = 0; k < plan.host_base[a].size(); ++k, ++o) {
                if (base) base[o] = plan.host_base[a][k];
                if (rem) rem[o] = plan.host_rem[a][k];
            }
    });
}

// ---- volume.hpp helpers
int mfreg_cu_discrete_gradient(const mfreg_cu_grid* image, const double* v, const int64_t* idx, int64_t n,
                               double* out6, int where) {
    return guard([&] {
        const Grid g = to_grid(image);
        validate_grid(g, false);
        const long long cnt = idx ? n : g.count();
        if (idx)
            for (long long k = 0; k < n; ++k)
                if (idx[k] < 0 || idx[k] >= g.count()) throw std::invalid_argument("discrete_gradient: index out of range");
        In vi(v, g.count(), where, kStream);
        Idx ix(idx, n);
        Out o(out6, 6 * cnt, where);
        if (cnt > 0) k_dgrad<<<blocks_for(cnt), 256, 0, kStream>>>(g, vi.ptr, ix.ptr(), cnt, o.ptr, -1.0, nullptr);
        note_launch();
        check_launch("discrete_gradient");
        o.finish(kStream);
    });
}
int mfreg_cu_eps_norm(const double* g6, int64_t n, double eps, double* out, int where) {
    return guard([&] {
        In gi(g6, 6 * n, where, kStream);
        Out o(out, n, where);
        if (n > 0) k_eps_norm<<<blocks_for(n), 256, 0, kStream>>>(gi.ptr, n, eps, o.ptr);
        note_launch();
        check_launch("eps_norm");
        o.finish(kStream);
    });
}

// ---- curvature.hpp: laplacian(u_comp, g, i) at a list of nodes
int mfreg_cu_laplacian_at(const mfreg_cu_grid* nodal, const double* u_comp, const int64_t* idx, int64_t n, double* out,
                          int where) {
    return guard([&] {
        const Grid g = to_grid(nodal);
        for (long long k = 0; k < n; ++k)
            if (idx[k] < 0 || idx[k] >= g.count()) throw std::invalid_argument("laplacian: index out of range");
        In ui(u_comp, g.count(), where, kStream);
        Idx ix(idx, n);
        Out o(out, n, where);
        if (n > 0) k_lap_at<<<blocks_for(n), 256, 0, kStream>>>(g, ui.ptr, ix.ptr(), n, o.ptr);
        note_launch();
        check_launch("laplacian");
        o.finish(kStream);
    });
}

// ---- multilevel.hpp: nodal_interpolate(comp, g, p) at a list of points (x, y, z interleaved)
int mfreg_cu_nodal_interpolate(const mfreg_cu_grid* nodal, const double* comp, const double* pts, int64_t n,
                               double* out, int where) {
    return guard([&] {
        const Grid g = to_grid(nodal);
        In ci(comp, g.count(), where, kStream), pi(pts, 3 * n, where, kStream);
        Out o(out, n, where);
        if (n > 0) k_nodal_interp<<<blocks_for(n), 256, 0, kStream>>>(g, ci.ptr, pi.ptr, n, o.ptr);
        note_launch();
        check_launch("nodal_interpolate");
        o.finish(kStream);
    });
}

// ---- ngf.hpp: make_ngf_precomp (ref_grads AoS [m][6], ref_norms [m])
int mfreg_cu_ngf_precomp(const double* ref, const mfreg_cu_grid* image, double rho, double* ref_grads,
                         double* ref_norms, int where) {
    return guard([&] {
        if (!(rho > 0.0)) throw std::invalid_argument("NGF: rho must be > 0");
        const Grid g = to_grid(image);
        validate_grid(g, false);
        const long long n = g.count();
        In ri(ref, n, where, kStream);
        Out og(ref_grads, 6 * n, where), on(ref_norms, n, where);
        k_dgrad<<<blocks_for(n), 256, 0, kStream>>>(g, ri.ptr, nullptr, n, og.ptr, rho, on.ptr);
        note_launch();
        check_launch("make_ngf_precomp");
        og.finish(kStream);
        on.finish(kStream);
    });
}
// the workspace's template gradients tpl_grads (AoS [m][6]) of the last populate
int mfreg_cu_ngf_tpl_grads(mfreg_cu_ngf* h, double* tpl_grads, int where) {
    return guard([&] {
        if (!h || !h->ngf) throw std::invalid_argument("null NGF context");
        const Grid g = h->g;
        const long long n = g.count();
        Out o(tpl_grads, 6 * n, where);
        k_dgrad<<<blocks_for(n), 256, 0, kStream>>>(g, h->ngf->Tw.get(), nullptr, n, o.ptr, -1.0, nullptr);
        note_launch();
        check_launch("tpl_grads");
        o.finish(kStream);
    });
}

// ---- ngf.hpp: make_offset_table (ngf.cpp:267-300), grouped by linear kappa as the reference
int mfreg_cu_offset_table(const mfreg_cu_grid* image, int* nentries, int64_t* kappa, int* npairs, int* pairs) {
    return guard([&] {
        const Grid g = to_grid(image);
        auto mu = [&](int d) -> long long {
            switch (d) {
            case NEGZ: return -g.m[0] * g.m[1];
            case NEGY: return -g.m[0];
            case NEGX: return -1;
            case CENTER: return 0;
            case POSX: return 1;
            case POSY: return g.m[0];
            default: return g.m[0] * g.m[1];
            }
        };
        std::map<long long, std::vector<std::pair<int, int>>> groups;
        for (int da = 0; da < 7; ++da)
            for (int db = 0; db < 7; ++db) groups[mu(db) - mu(da)].emplace_back(da, db);
        if (groups.size() == 25) {  // closed-form cross-check (ngf.cpp:282-297)
            const long long m1 = g.m[0], m12 = g.m[0] * g.m[1];
            std::vector<long long> e = {-2 * m12, -m12 - m1, -m12 - 1, -m12, -m12 + 1, -m12 + m1, -2 * m1, -m1 - 1,
                                        -m1,      -m1 + 1,   -2,       -1,   0,        1,         2,       m1 - 1,
                                        m1,       m1 + 1,    2 * m1,   m12 - m1, m12 - 1, m12,    m12 + 1, m12 + m1,
                                        2 * m12};
            std::sort(e.begin(), e.end());
            std::size_t i = 0;
            for (const auto& kv : groups)
                if (kv.first != e[i++]) throw std::logic_error("offset table mismatch against closed-form list");
        }
        int ne = 0, np = 0;
        for (const auto& kv : groups) {
            if (kappa) kappa[ne] = kv.first;
            if (npairs) npairs[ne] = static_cast<int>(kv.second.size());
            for (const auto& pr : kv.second) {
                if (pairs) {
                    pairs[2 * np] = pr.first;
                    pairs[2 * np + 1] = pr.second;
                }
                ++np;
            }
            ++ne;
        }
        *nentries = ne;
    });
}

// ---- optimizer.hpp: armijo_search (optimizer.cpp:156-175) on a host phi
int mfreg_cu_armijo_search(double (*phi)(void* ctx, double eta, int* err), void* ctx, double f0, double gdotd,
                           double c1, double beta, int max_backtracks, double eta0, double* eta, int* accepted,
                           int* descent, double* f_new) {
    return guard([&] {
        *eta = 0.0;
        *accepted = 0;
        *descent = 1;
        *f_new = 0.0;
        if (!(gdotd < 0.0)) {
            *descent = 0;
            return;
        }
        double e = eta0;
        for (int k = 0; k <= max_backtracks; ++k) {
            int err = 0;
            const double f = phi(ctx, e, &err);
            if (err) throw std::runtime_error("problem callback failed: phi");
            if (std::isfinite(f) && f <= f0 + c1 * e * gdotd) {
                *eta = e;
                *accepted = 1;
                *f_new = f;
                return;
            }
            e *= beta;
        }
    });
}

// ---- a host Problem driven by the device-resident solvers
int mfreg_cu_problem_minimize(const mfreg_cu_problem_ops* ops, int64_t n, int method, const double* y0,
                              const mfreg_cu_opt_config* cfg, double* y_out, mfreg_cu_iter_record* trace, int cap,
                              int* ntrace, int* line_search_failed, int where) {
    return guard([&] {
        if (!ops) throw std::invalid_argument("null problem");
        if (method != MFREG_CU_LBFGS && method != MFREG_CU_GAUSS_NEWTON) throw std::invalid_argument("unknown method");
        CallbackProblem P(*ops, n);
        In yi(y0, n, where, kStream);
        Out yo(y_out, n, where);
        const OptimizerConfig c = to_cfg(cfg);
        const MinimizeResult res = method == MFREG_CU_LBFGS ? lbfgs_minimize(P, yi.ptr, yo.ptr, c)
                                                            : gauss_newton_minimize(P, yi.ptr, yo.ptr, c);
        yo.finish(kStream);
        MFREG_CUDA(cudaStreamSynchronize(kStream));
        get_trace(res, trace, cap, ntrace, line_search_failed);
    });
}

// cg_solve(apply, b, cfg) (optimizer.cpp:113-154): `apply` is ops->gn_hessian_vec (op 0) or
// ops->seed_hessian_vec with gamma (op 1)
int mfreg_cu_problem_cg_solve(const mfreg_cu_problem_ops* ops, int64_t n, int op, double gamma, const double* b,
                              int max_iters, double rel_tol, double* x, int* iters, double* relres, int* breakdown,
                              int where) {
    return guard([&] {
        if (!ops) throw std::invalid_argument("null problem");
        CallbackProblem P(*ops, n);
        In bi(b, n, where, kStream);
        Out xo(x, n, where);
        const CgResult r = cg_solve(P, op, gamma, bi.ptr, xo.ptr, CgConfig{max_iters, rel_tol});
        xo.finish(kStream);
        MFREG_CUDA(cudaStreamSynchronize(kStream));
        *iters = r.iters;
        *relres = r.relres;
        *breakdown = r.breakdown ? 1 : 0;
    });
}

}  // extern "C"
