// TEST INFRASTRUCTURE ONLY — never linked into or called by the product.
//
// extern "C" wrapper around the UNMODIFIED reference library (mfreg, compiled
// from /root/reference/proj/src by oracle/Makefile into oracle/_ref/). Only
// tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
// reference leg may load the resulting libmfreg_ref.so. Every entry point
// forwards to the reference symbol named in its comment; nothing here
// re-implements reference arithmetic.
#include <cstdint>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <string>
#include <vector>

#include "mfreg/curvature.hpp"
#include "mfreg/io.hpp"
#include "mfreg/multilevel.hpp"
#include "mfreg/ngf.hpp"
#include "mfreg/optimizer.hpp"
#include "mfreg/oracle.hpp"
#include "mfreg/parallel.hpp"
#include "mfreg/synthetic.hpp"
#include "mfreg/transfer.hpp"
#include "mfreg/volume.hpp"

using namespace mfreg;

namespace {

thread_local std::string g_err;

// 0 ok, 1 invalid_argument, 2 logic_error, 3 other
template <typename Fn>
int guard(Fn&& fn) {
    try {
        fn();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::logic_error& e) {
        g_err = e.what();
        return 2;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 3;
    }
}

std::array<index_t, 3> M(const std::int64_t* m) { return {m[0], m[1], m[2]}; }
std::array<double, 3> H(const double* h) { return {h[0], h[1], h[2]}; }

Volume make_vol(const double* data, const std::int64_t* m, const double* h) {
    Volume v;
    v.grid = make_image_grid(M(m), H(h));
    v.data.assign(data, data + v.grid.count());
    return v;
}

GridDesc nodal(const std::int64_t* m, const double* h) {
    GridDesc g{M(m), H(h), GridKind::Nodal};
    return g;
}

struct NgfCtx {
    Volume ref;
    NgfParams params;
    NgfPrecomp pre;
    NgfWorkspace ws;
    Volume tpl;
};

struct ObjCtx {
    Volume ref;
    Volume tpl;
    GridDesc dg;
    Objective* obj = nullptr;
    ~ObjCtx() { delete obj; }
};

} // namespace

extern "C" {

// Mirrors mfreg::OptimizerConfig (optimizer.hpp:145-155) field by field.
struct mref_opt_config {
    int max_iters;
    double c1;
    double beta;
    int max_backtracks;
    int cg_max_iters;
    double cg_rel_tol;
    int h0_max_iters;
    double h0_rel_tol;
    int lbfgs_history;
    double gamma;
    double tol_rel_j;
    double tol_grad;
    double tol_step;
};

// Mirrors mfreg::IterationRecord (optimizer.hpp:22-30).
struct mref_iter_record {
    int iter;
    int cg_iters;
    double j;
    double distance;
    double regularizer;
    double grad_norm;
    double step;
};

const char* mref_last_error() { return g_err.c_str(); }

void mref_set_threads(int n) { set_thread_count(n); }
int mref_thread_count() { return thread_count(); }

// synthetic.cpp:15-63
int mref_make_phantom(const std::int64_t* m, const double* h, double* out) {
    return guard([&] {
        const Volume v = synthetic::make_phantom(M(m), H(h));
        std::memcpy(out, v.data.data(), v.data.size() * sizeof(double));
    });
}

// synthetic.cpp:65-90
int mref_make_random_volume(const std::int64_t* m, const double* h, std::uint64_t seed, int passes,
                            double* out) {
    return guard([&] {
        const Volume v = synthetic::make_random_volume(M(m), H(h), seed, passes);
        std::memcpy(out, v.data.data(), v.data.size() * sizeof(double));
    });
}

// synthetic.cpp:110-143 — terms of make_sinusoid_warp (amp[3][3], freq[3][3], phase[3][3])
int mref_sinusoid_terms(const double* extent, double max_amp, std::uint64_t seed, double* amp,
                        int* freq, double* phase) {
    return guard([&] {
        const auto w = synthetic::make_sinusoid_warp({extent[0], extent[1], extent[2]}, max_amp, seed);
        for (int t = 0; t < 3; ++t) {
            for (int d = 0; d < 3; ++d) {
                amp[t * 3 + d] = w.terms[t].amp[d];
                freq[t * 3 + d] = w.terms[t].freq[d];
                phase[t * 3 + d] = w.terms[t].phase[d];
            }
        }
    });
}

// synthetic.cpp:145-159 with make_sinusoid_warp(extent(vol), max_amp, seed)
int mref_warp_sinusoid(const double* vol, const std::int64_t* m, const double* h, double max_amp,
                       std::uint64_t seed, double* out) {
    return guard([&] {
        const Volume v = make_vol(vol, m, h);
        const auto w = synthetic::make_sinusoid_warp(
            {v.grid.extent(0), v.grid.extent(1), v.grid.extent(2)}, max_amp, seed);
        const Volume o = synthetic::warp_with(v, w);
        std::memcpy(out, o.data.data(), o.data.size() * sizeof(double));
    });
}

// synthetic.cpp:161-175 — ground-truth phi at the nodal points of (my, image extent)
int mref_warp_field(const std::int64_t* m, const double* h, double max_amp, std::uint64_t seed,
                    const std::int64_t* my, double* out) {
    return guard([&] {
        const GridDesc img = make_image_grid(M(m), H(h));
        const auto w = synthetic::make_sinusoid_warp({img.extent(0), img.extent(1), img.extent(2)},
                                                     max_amp, seed);
        const GridDesc dg = make_deform_grid(img, M(my));
        const auto y = synthetic::warp_field(w, dg);
        std::memcpy(out, y.data(), y.size() * sizeof(double));
    });
}

// grid.hpp:131-146
int mref_make_deform_grid(const std::int64_t* m, const double* h, const std::int64_t* my,
                          double* hy) {
    return guard([&] {
        const GridDesc g = make_deform_grid(make_image_grid(M(m), H(h)), M(my));
        for (int a = 0; a < 3; ++a) hy[a] = g.h[a];
    });
}

// multilevel.cpp:39-49
int mref_deformation_grid_for(const std::int64_t* m, const double* h, std::int64_t ratio,
                              std::int64_t* my, double* hy) {
    return guard([&] {
        const GridDesc g = deformation_grid_for(make_image_grid(M(m), H(h)), ratio);
        for (int a = 0; a < 3; ++a) {
            my[a] = g.m[a];
            hy[a] = g.h[a];
        }
    });
}

// transfer.cpp:11-47
int mref_transfer_plan(const std::int64_t* ms, const double* hs, const std::int64_t* mt,
                       const double* ht, std::int64_t* base, double* rem) {
    return guard([&] {
        const auto plan = make_transfer_plan(nodal(ms, hs), make_image_grid(M(mt), H(ht)));
        std::size_t o = 0;
        for (int a = 0; a < 3; ++a) {
            for (std::size_t k = 0; k < plan.base[a].size(); ++k, ++o) {
                base[o] = plan.base[a][k];
                rem[o] = plan.rem[a][k];
            }
        }
    });
}

// transfer.cpp:49-86
int mref_transfer_apply(const std::int64_t* ms, const double* hs, const std::int64_t* mt,
                        const double* ht, const double* y, double* out) {
    return guard([&] {
        const auto plan = make_transfer_plan(nodal(ms, hs), make_image_grid(M(mt), H(ht)));
        const std::size_t ns = plan.source.count(), nt = plan.target.count();
        transfer_apply(plan, {y, 3 * ns}, {out, 3 * nt});
    });
}

// transfer.cpp:131-150
int mref_transfer_apply_transpose(const std::int64_t* ms, const double* hs, const std::int64_t* mt,
                                  const double* ht, const double* w, double* out) {
    return guard([&] {
        const auto plan = make_transfer_plan(nodal(ms, hs), make_image_grid(M(mt), H(ht)));
        const std::size_t ns = plan.source.count(), nt = plan.target.count();
        transfer_apply_transpose(plan, {w, 3 * nt}, {out, 3 * ns});
    });
}

// volume.cpp:29-74
int mref_interpolate(const double* t, const std::int64_t* m, const double* h, const double* p,
                     double* value, double* grad) {
    return guard([&] {
        const Volume v = make_vol(t, m, h);
        const auto r = interpolate(v, {p[0], p[1], p[2]});
        *value = r.value;
        for (int a = 0; a < 3; ++a) grad[a] = r.grad[a];
    });
}

// volume.cpp:76-94
int mref_sample_deformed(const double* t, const std::int64_t* m, const double* h,
                         const double* points, std::int64_t n, double* values, double* partials) {
    return guard([&] {
        const Volume v = make_vol(t, m, h);
        SampledTemplate s;
        sample_deformed(v, {points, static_cast<std::size_t>(3 * n)}, s);
        std::memcpy(values, s.values.data(), n * sizeof(double));
        for (int a = 0; a < 3; ++a) std::memcpy(partials + a * n, s.partials[a].data(), n * sizeof(double));
    });
}

// volume.cpp:123-160
int mref_downsample(const double* v, const std::int64_t* m, const double* h, double* out,
                    std::int64_t* mo, double* ho) {
    return guard([&] {
        const Volume c = downsample(make_vol(v, m, h));
        std::memcpy(out, c.data.data(), c.data.size() * sizeof(double));
        for (int a = 0; a < 3; ++a) {
            mo[a] = c.grid.m[a];
            ho[a] = c.grid.h[a];
        }
    });
}

// ---- NGF kernel API (ngf.hpp:26-85) through an opaque context ----
void* mref_ngf_create(const double* ref, const std::int64_t* m, const double* h, double tau,
                      double rho) {
    auto* c = new NgfCtx;
    int rc = guard([&] {
        c->ref = make_vol(ref, m, h);
        c->params = {tau, rho};
        c->pre = make_ngf_precomp(c->ref, rho);
    });
    if (rc) {
        delete c;
        return nullptr;
    }
    return c;
}

void mref_ngf_destroy(void* p) { delete static_cast<NgfCtx*>(p); }

// ngf.cpp:185-214
int mref_ngf_populate(void* p, const double* tpl, const double* points) {
    auto* c = static_cast<NgfCtx*>(p);
    return guard([&] {
        c->tpl = make_vol(tpl, c->ref.grid.m.data(), c->ref.grid.h.data());
        const std::size_t n = c->ref.grid.count();
        populate_ngf_workspace(c->ws, c->tpl, {points, 3 * n}, c->pre, c->params, c->ref.grid);
    });
}

int mref_ngf_workspace(void* p, double* values, double* partials, double* tpl_grads,
                       double* residual, double* inv1, double* inv2, double* ref_grads,
                       double* ref_norms) {
    auto* c = static_cast<NgfCtx*>(p);
    return guard([&] {
        const std::size_t n = c->ref.grid.count();
        for (std::size_t i = 0; i < n; ++i) {
            if (values) values[i] = c->ws.sampled.values[i];
            if (partials)
                for (int a = 0; a < 3; ++a) partials[a * n + i] = c->ws.sampled.partials[a][i];
            if (tpl_grads)
                for (int k = 0; k < 6; ++k) tpl_grads[k * n + i] = c->ws.tpl_grads[i][k];
            if (ref_grads)
                for (int k = 0; k < 6; ++k) ref_grads[k * n + i] = c->pre.ref_grads[i][k];
            if (ref_norms) ref_norms[i] = c->pre.ref_norms[i];
            if (residual) residual[i] = c->ws.residual[i];
            if (inv1) inv1[i] = c->ws.inv1[i];
            if (inv2) inv2[i] = c->ws.inv2[i];
        }
    });
}

// ngf.cpp:225-231
int mref_ngf_value(void* p, double* out) {
    auto* c = static_cast<NgfCtx*>(p);
    return guard([&] { *out = ngf_value(c->ws, c->ref.grid); });
}

// ngf.cpp:233-236
int mref_ngf_gradient(void* p, double* out) {
    auto* c = static_cast<NgfCtx*>(p);
    return guard([&] {
        ngf_gradient(c->ws, c->pre, c->ref.grid, {out, 3 * static_cast<std::size_t>(c->ref.grid.count())});
    });
}

// ngf.cpp:253-258
int mref_ngf_hessian_vec(void* p, const double* v, double* out) {
    auto* c = static_cast<NgfCtx*>(p);
    return guard([&] {
        const std::size_t n3 = 3 * static_cast<std::size_t>(c->ref.grid.count());
        ngf_hessian_vec({v, n3}, c->ws, c->pre, c->ref.grid, {out, n3});
    });
}

// ngf.cpp:220-223
int mref_ngf_rho(void* p, std::int64_t i, int k, double* out) {
    auto* c = static_cast<NgfCtx*>(p);
    return guard([&] { *out = ngf_rho(i, static_cast<Dir>(k), c->ws, c->pre, c->ref.grid); });
}

// oracle.cpp:223-293 — independent sparse-matrix chain (the paper's MBC baseline)
int mref_oracle_image(void* p, const std::int64_t* my, const double* v, double* grad_out,
                      double* hvp_out) {
    auto* c = static_cast<NgfCtx*>(p);
    return guard([&] {
        const GridDesc dg = make_deform_grid(c->ref.grid, M(my));
        const auto plan = make_transfer_plan(dg, c->ref.grid);
        oracle::Derivatives der(c->ref, c->ws.sampled, c->params, c->ref.grid, plan, dg);
        const auto g = der.distance_gradient_image();
        std::memcpy(grad_out, g.data(), g.size() * sizeof(double));
        const std::size_t n3 = 3 * static_cast<std::size_t>(c->ref.grid.count());
        const auto hv = der.distance_hvp_image({v, n3});
        std::memcpy(hvp_out, hv.data(), hv.size() * sizeof(double));
    });
}

// ---- curvature (curvature.hpp:13-31), nodal grid (m, h) ----
int mref_laplacian_apply(const double* u, const std::int64_t* m, const double* h, double* out) {
    return guard([&] {
        const GridDesc g = nodal(m, h);
        const std::size_t n = g.count();
        laplacian_apply({u, n}, g, {out, n});
    });
}

int mref_curvature_value(const double* u, const std::int64_t* m, const double* h, double* out) {
    return guard([&] {
        const GridDesc g = nodal(m, h);
        *out = curvature_value({u, 3 * static_cast<std::size_t>(g.count())}, g);
    });
}

int mref_curvature_gradient(const double* u, const std::int64_t* m, const double* h, double* out) {
    return guard([&] {
        const GridDesc g = nodal(m, h);
        const auto r = curvature_gradient({u, 3 * static_cast<std::size_t>(g.count())}, g);
        std::memcpy(out, r.data(), r.size() * sizeof(double));
    });
}

int mref_curvature_hessian_vec(const double* u, const std::int64_t* m, const double* h,
                               double* out) {
    return guard([&] {
        const GridDesc g = nodal(m, h);
        const auto r = curvature_hessian_vec({u, 3 * static_cast<std::size_t>(g.count())}, g);
        std::memcpy(out, r.data(), r.size() * sizeof(double));
    });
}

// ---- Objective (optimizer.hpp:53-106) ----
void* mref_objective_create(const double* ref, const double* tpl, const std::int64_t* m,
                            const double* h, const std::int64_t* my, double tau, double rho,
                            double alpha) {
    auto* c = new ObjCtx;
    int rc = guard([&] {
        c->ref = make_vol(ref, m, h);
        c->tpl = make_vol(tpl, m, h);
        c->dg = make_deform_grid(c->ref.grid, M(my));
        c->obj = new Objective(c->ref, c->tpl, c->dg, {tau, rho}, alpha);
    });
    if (rc) {
        delete c;
        return nullptr;
    }
    return c;
}

void mref_objective_destroy(void* p) { delete static_cast<ObjCtx*>(p); }

std::int64_t mref_objective_dof(void* p) { return static_cast<ObjCtx*>(p)->obj->dof(); }

int mref_objective_identity(void* p, double* out) {
    auto* c = static_cast<ObjCtx*>(p);
    return guard([&] {
        const auto x = c->obj->identity();
        std::memcpy(out, x.data(), x.size() * sizeof(double));
    });
}

// optimizer.cpp:64-92
int mref_objective_eval(void* p, const double* y, double* grad, double* j, double* dist,
                        double* reg) {
    auto* c = static_cast<ObjCtx*>(p);
    return guard([&] {
        const std::size_t n = c->obj->dof();
        *j = c->obj->eval({y, n}, grad ? std::span<double>(grad, n) : std::span<double>());
        *dist = c->obj->last_distance();
        *reg = c->obj->last_regularizer();
    });
}

// optimizer.cpp:94-104
int mref_objective_gn_hessian_vec(void* p, const double* v, double* q) {
    auto* c = static_cast<ObjCtx*>(p);
    return guard([&] {
        const std::size_t n = c->obj->dof();
        c->obj->gn_hessian_vec({v, n}, {q, n});
    });
}

// optimizer.cpp:106-111
int mref_objective_seed_hessian_vec(void* p, const double* v, double gamma, double* q) {
    auto* c = static_cast<ObjCtx*>(p);
    return guard([&] {
        const std::size_t n = c->obj->dof();
        c->obj->seed_hessian_vec({v, n}, gamma, {q, n});
    });
}

static OptimizerConfig to_cfg(const mref_opt_config* k) {
    OptimizerConfig c;
    c.max_iters = k->max_iters;
    c.armijo = {k->c1, k->beta, k->max_backtracks};
    c.cg = {k->cg_max_iters, k->cg_rel_tol};
    c.h0_cg = {k->h0_max_iters, k->h0_rel_tol};
    c.lbfgs_history = k->lbfgs_history;
    c.gamma = k->gamma;
    c.tol_rel_j = k->tol_rel_j;
    c.tol_grad = k->tol_grad;
    c.tol_step = k->tol_step;
    return c;
}

static int copy_trace(const IterationTrace& t, mref_iter_record* out, int cap) {
    int n = 0;
    for (const auto& r : t) {
        if (n < cap) {
            out[n] = {r.iter, r.cg_iters, r.j, r.distance, r.regularizer, r.grad_norm, r.step};
        }
        ++n;
    }
    return n;
}

// optimizer.cpp:113-154 on the Gauss-Newton operator (seed=0) or H0 (seed=1, gamma)
int mref_cg_solve(void* p, int seed, double gamma, const double* b, int max_iters, double rel_tol,
                  double* x, int* iters, double* relres, int* breakdown) {
    auto* c = static_cast<ObjCtx*>(p);
    return guard([&] {
        const std::size_t n = c->obj->dof();
        LinearOperator op;
        if (seed) {
            op = [&](std::span<const double> v, std::span<double> o) { c->obj->seed_hessian_vec(v, gamma, o); };
        } else {
            op = [&](std::span<const double> v, std::span<double> o) { c->obj->gn_hessian_vec(v, o); };
        }
        const auto r = cg_solve(op, {b, n}, {max_iters, rel_tol});
        std::memcpy(x, r.x.data(), n * sizeof(double));
        *iters = r.iters;
        *relres = r.relres;
        *breakdown = r.breakdown ? 1 : 0;
    });
}

// optimizer.cpp:272-407; method 0 = L-BFGS, 1 = Gauss-Newton
int mref_minimize(void* p, int method, const double* y0, const mref_opt_config* cfg, double* y_out,
                  mref_iter_record* trace, int cap, int* ntrace, int* ls_failed) {
    auto* c = static_cast<ObjCtx*>(p);
    return guard([&] {
        const std::size_t n = c->obj->dof();
        const auto oc = to_cfg(cfg);
        const MinimizeResult r = method == 1 ? gauss_newton_minimize(*c->obj, {y0, n}, oc)
                                             : lbfgs_minimize(*c->obj, {y0, n}, oc);
        std::memcpy(y_out, r.y.data(), n * sizeof(double));
        *ntrace = copy_trace(r.trace, trace, cap);
        *ls_failed = r.line_search_failed ? 1 : 0;
    });
}

// multilevel.cpp:78-115
int mref_prolong(const double* yc, const std::int64_t* mc, const double* hc, const std::int64_t* mf,
                 const double* hf, double* out) {
    return guard([&] {
        const GridDesc c = nodal(mc, hc), f = nodal(mf, hf);
        const auto y = prolong({yc, 3 * static_cast<std::size_t>(c.count())}, c, f);
        std::memcpy(out, y.data(), y.size() * sizeof(double));
    });
}

// multilevel.cpp:117-145. Outputs: finest y (caller sizes it from the finest
// deformation grid), per-level traces packed back to back (coarsest first),
// level_iters[levels], ls_failed[levels].
int mref_register_multilevel(const double* ref, const double* tpl, const std::int64_t* m,
                             const double* h, int levels, std::int64_t ratio, double tau,
                             double rho, double alpha, int method, const mref_opt_config* cfg,
                             double* y_out, mref_iter_record* trace, int cap, int* level_iters,
                             int* ls_failed) {
    return guard([&] {
        const Volume r = make_vol(ref, m, h);
        const Volume t = make_vol(tpl, m, h);
        MultilevelConfig mc;
        mc.levels = levels;
        mc.deform_ratio = ratio;
        mc.ngf = {tau, rho};
        mc.alpha = alpha;
        mc.method = method == 1 ? Method::GaussNewton : Method::Lbfgs;
        mc.opt = to_cfg(cfg);
        const auto res = register_multilevel(r, t, mc);
        std::memcpy(y_out, res.y.data(), res.y.size() * sizeof(double));
        int off = 0;
        for (std::size_t l = 0; l < res.levels.size(); ++l) {
            const int k = copy_trace(res.levels[l].result.trace, trace + off, cap - off);
            level_iters[l] = k;
            ls_failed[l] = res.levels[l].result.line_search_failed ? 1 : 0;
            off += k;
        }
    });
}

// ---- io.hpp
// io::read_volume (io.cpp:111-164); data may be NULL (dims / spacing only)
int mref_io_read_volume(const char* path, std::int64_t* m, double* h, double* data) {
    return guard([&] {
        const Volume v = io::read_volume(path);
        for (int a = 0; a < 3; ++a) {
            m[a] = v.grid.m[a];
            h[a] = v.grid.h[a];
        }
        if (data) std::memcpy(data, v.data.data(), v.data.size() * sizeof(double));
    });
}

// io::write_volume (io.cpp:166-188)
int mref_io_write_volume(const char* path, const std::int64_t* m, const double* h, const double* data) {
    return guard([&] { io::write_volume(path, make_vol(data, m, h)); });
}

// io::write_deformation (io.cpp:200-229)
int mref_io_write_deformation(const char* path, const double* y, std::int64_t n, const std::int64_t* m,
                              const double* h) {
    return guard([&] { io::write_deformation(path, {y, static_cast<std::size_t>(n)}, nodal(m, h)); });
}

// io::read_deformation_grid (io.cpp:231-253)
int mref_io_read_deformation_grid(const char* path, std::int64_t* m, double* h) {
    return guard([&] {
        const GridDesc g = io::read_deformation_grid(path);
        for (int a = 0; a < 3; ++a) {
            m[a] = g.m[a];
            h[a] = g.h[a];
        }
    });
}

// io::read_deformation (io.cpp:255-274)
int mref_io_read_deformation(const char* path, const std::int64_t* m, const double* h, double* y) {
    return guard([&] {
        const auto v = io::read_deformation(path, nodal(m, h));
        std::memcpy(y, v.data(), v.size() * sizeof(double));
    });
}

// io::read_landmarks (io.cpp:276-303)
int mref_io_read_landmarks(const char* path, const double* spacing, double* out, std::int64_t cap,
                           std::int64_t* count) {
    return guard([&] {
        const auto v = io::read_landmarks(path, {spacing[0], spacing[1], spacing[2]});
        *count = static_cast<std::int64_t>(v.size());
        for (std::size_t i = 0; out && i < v.size() && static_cast<std::int64_t>(i) < cap; ++i)
            for (int a = 0; a < 3; ++a) out[3 * i + a] = v[i][a];
    });
}

// io::landmark_error (io.cpp:305-348)
int mref_io_landmark_error(const double* fixed, std::int64_t nf, const double* moving, std::int64_t nm,
                           const double* y, std::int64_t ny, const std::int64_t* m, const double* h, double* mean,
                           double* stddev, std::int64_t* count) {
    return guard([&] {
        std::vector<std::array<double, 3>> f(static_cast<std::size_t>(nf)), mv(static_cast<std::size_t>(nm));
        for (std::int64_t i = 0; i < nf; ++i) f[i] = {fixed[3 * i], fixed[3 * i + 1], fixed[3 * i + 2]};
        for (std::int64_t i = 0; i < nm; ++i) mv[i] = {moving[3 * i], moving[3 * i + 1], moving[3 * i + 2]};
        const auto st = io::landmark_error(f, mv, {y, static_cast<std::size_t>(ny)}, nodal(m, h));
        *mean = st.mean;
        *stddev = st.stddev;
        *count = static_cast<std::int64_t>(st.count);
    });
}

} // extern "C"
