// extern "C" boundary (include/mfreg_cuda.h). Maps the reference's exceptions to
// status codes and stages host buffers when `where == MFREG_CU_HOST`.
#include <atomic>
#include <cstring>
#include <memory>
#include <random>
#include <string>

#include "../../include/mfreg_cuda.h"
#include "capi_util.cuh"
#include "io.cuh"
#include "objective.cuh"

using namespace mfreg_b200;
using namespace mfreg_b200::capi;

std::string& mfreg_b200::capi::last_error() {
    static thread_local std::string e;
    return e;
}

namespace {

// synthetic.cpp:110-143, computed with the same libstdc++ engine/distributions
WarpTerms sinusoid_terms(const double extent[3], double max_amp, std::uint64_t seed) {
    WarpTerms w{};
    for (int a = 0; a < 3; ++a) w.extent[a] = extent[a];
    std::mt19937_64 rng(seed);
    std::uniform_real_distribution<double> amp_dist(-1.0, 1.0);
    std::uniform_int_distribution<int> freq_dist(1, 2);
    std::uniform_real_distribution<double> phase_dist(-0.5, 0.5);
    for (int t = 0; t < 3; ++t)
        for (int d = 0; d < 3; ++d) {
            w.amp[t][d] = amp_dist(rng);
            w.freq[t][d] = freq_dist(rng);
            w.phase[t][d] = phase_dist(rng);
        }
    double bound = 0.0;
    for (int d = 0; d < 3; ++d) {
        double s = 0.0;
        for (int t = 0; t < 3; ++t) s += std::abs(w.amp[t][d]);
        bound = std::max(bound, s);
    }
    const double scale = bound > 0.0 ? max_amp / (bound * std::sqrt(3.0)) : 0.0;
    for (int t = 0; t < 3; ++t)
        for (int d = 0; d < 3; ++d) w.amp[t][d] *= scale;
    return w;
}

}  // namespace

extern "C" {

const char* mfreg_cu_last_error(void) { return last_error().c_str(); }
int mfreg_cu_version(void) { return 1; }
int mfreg_cu_device_count(int* n) { return guard([&] { MFREG_CUDA(cudaGetDeviceCount(n)); }); }
int mfreg_cu_set_device(int device) { return guard([&] { MFREG_CUDA(cudaSetDevice(device)); }); }
int mfreg_cu_synchronize(void) { return guard([&] { MFREG_CUDA(cudaDeviceSynchronize()); }); }
int mfreg_cu_device_memory_peak(int reset, int64_t* bytes) {
    return guard([&] { *bytes = device_memory_peak(reset != 0); });
}

int mfreg_cu_make_deform_grid(const mfreg_cu_grid* image, const int64_t points[3], mfreg_cu_grid* out) {
    return guard([&] {
        const idx_t p[3] = {points[0], points[1], points[2]};
        from_grid(make_deform_grid(to_grid(image), p), out);
    });
}

int mfreg_cu_deformation_grid_for(const mfreg_cu_grid* image, int64_t ratio, mfreg_cu_grid* out) {
    return guard([&] { from_grid(deformation_grid_for(to_grid(image), ratio), out); });
}

int mfreg_cu_transfer_apply(const mfreg_cu_grid* nodal, const mfreg_cu_grid* image, const double* y, double* out,
                            int where) {
    return guard([&] {
        DevicePlanOwner plan(to_grid(nodal), to_grid(image));
        const auto& P = plan.view();
        In yi(y, 3 * P.src.count(), where, kStream);
        Out o(out, 3 * P.tgt.count(), where);
        launch_transfer_apply(P, yi.ptr, o.ptr, kStream);
        check_launch("transfer_apply");
        o.finish(kStream);
    });
}

int mfreg_cu_transfer_apply_transpose(const mfreg_cu_grid* nodal, const mfreg_cu_grid* image, const double* w,
                                      double* out, int where) {
    return guard([&] {
        DevicePlanOwner plan(to_grid(nodal), to_grid(image));
        const auto& P = plan.view();
        In wi(w, 3 * P.tgt.count(), where, kStream);
        Out o(out, 3 * P.src.count(), where);
        launch_transfer_T(P, wi.ptr, o.ptr, kStream);
        check_launch("transfer_apply_transpose");
        o.finish(kStream);
    });
}

int mfreg_cu_sample_deformed(const mfreg_cu_grid* image, const double* tpl, const double* points, int64_t n,
                             double* values, double* partials, int where) {
    return guard([&] {
        const Grid g = to_grid(image);
        validate_grid(g, false);
        if (n < 0) throw std::invalid_argument("sample_deformed: points length must be a multiple of 3");
        In t(tpl, g.count(), where, kStream);
        In p(points, 3 * n, where, kStream);
        Out v(values, n, where), d(partials, 3 * n, where);
        if (n > 0) launch_sample(g, t.ptr, p.ptr, n, v.ptr, d.ptr, kStream);
        check_launch("sample_deformed");
        v.finish(kStream);
        d.finish(kStream);
    });
}

int mfreg_cu_downsample(const mfreg_cu_grid* image, const double* v, double* out, mfreg_cu_grid* out_grid,
                        int where) {
    return guard([&] {
        const Grid g = to_grid(image);
        for (int a = 0; a < 3; ++a)
            if (g.m[a] < 2) throw std::invalid_argument("downsample: all axes must have m >= 2");
        Grid c{};
        for (int a = 0; a < 3; ++a) {
            c.m[a] = (g.m[a] + 1) / 2;
            c.h[a] = 2.0 * g.h[a];
        }
        if (out_grid) from_grid(c, out_grid);
        if (!out) return;
        In vi(v, g.count(), where, kStream);
        Out o(out, c.count(), where);
        launch_downsample(g, c, vi.ptr, o.ptr, kStream);
        check_launch("downsample");
        o.finish(kStream);
    });
}

int mfreg_cu_laplacian_apply(const mfreg_cu_grid* nodal, const double* u_comp, double* out, int where) {
    return guard([&] {
        // one component: run the 3-component kernel on a zero-padded triple
        const Grid g = to_grid(nodal);
        const std::size_t n = g.count();
        DVec u3(3 * n), o3(3 * n);
        MFREG_CUDA(cudaMemsetAsync(u3.get(), 0, 3 * n * sizeof(double), kStream));
        MFREG_CUDA(cudaMemcpyAsync(u3.get(), u_comp, n * sizeof(double),
                                   where == MFREG_CU_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice, kStream));
        launch_lap3(g, u3.get(), o3.get(), kStream);
        check_launch("laplacian_apply");
        MFREG_CUDA(cudaMemcpyAsync(out, o3.get(), n * sizeof(double),
                                   where == MFREG_CU_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice, kStream));
        MFREG_CUDA(cudaStreamSynchronize(kStream));
    });
}

int mfreg_cu_curvature_value(const mfreg_cu_grid* nodal, const double* u, double* out, int mode, int where) {
    return guard([&] {
        const Grid g = to_grid(nodal);
        const idx_t n = g.count();
        In ui(u, 3 * n, where, kStream);
        DVec l(3 * n), sc(8);
        Reducer red(to_mode(mode), n);
        launch_lap3(g, ui.ptr, l.get(), kStream);
        for (int d = 0; d < 3; ++d) red.sum(SUM_SQ, n, l.get() + d * n, nullptr, sc.get() + d, 1.0, kStream);
        launch_curv_finalize(sc.get(), g.cell_volume(), 1.0, sc.get() + 4, kStream);
        check_launch("curvature_value");
        MFREG_CUDA(cudaMemcpyAsync(out, sc.get() + 4, sizeof(double), cudaMemcpyDeviceToHost, kStream));
        MFREG_CUDA(cudaStreamSynchronize(kStream));
    });
}

static int curvature_bilap(const mfreg_cu_grid* nodal, const double* u, double* out, int where) {
    return guard([&] {
        const Grid g = to_grid(nodal);
        const idx_t n = g.count();
        In ui(u, 3 * n, where, kStream);
        Out o(out, 3 * n, where);
        DVec l(3 * n);
        launch_lap3(g, ui.ptr, l.get(), kStream);
        launch_bilap(g, l.get(), 2.0 * g.cell_volume(), 0, 0.0, 0.0, nullptr, o.ptr, kStream);
        check_launch("curvature_gradient");
        o.finish(kStream);
    });
}
int mfreg_cu_curvature_gradient(const mfreg_cu_grid* nodal, const double* u, double* out, int where) {
    return curvature_bilap(nodal, u, out, where);
}
int mfreg_cu_curvature_hessian_vec(const mfreg_cu_grid* nodal, const double* p, double* out, int where) {
    return curvature_bilap(nodal, p, out, where);
}

// ---- NGF
int mfreg_cu_ngf_create(const double* ref, const mfreg_cu_grid* image, double tau, double rho, int mode, int where,
                        mfreg_cu_ngf** out) {
    return guard([&] {
        if (mode == MFREG_CU_FAST32)  // DeviceNgf's unfused kernels need the fp64 state
            throw std::invalid_argument("NGF kernel API: FAST32 is an Objective mode (the kernel-level NGF API is fp64)");
        auto h = std::make_unique<mfreg_cu_ngf>();
        h->g = to_grid(image);
        validate_grid(h->g, false);
        const std::size_t n = h->g.count();
        h->R.resize(n);
        check_where(where);
        MFREG_CUDA(cudaMemcpy(h->R.get(), ref, n * sizeof(double),
                              where == MFREG_CU_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice));
        h->ngf = std::make_unique<DeviceNgf>(h->g, h->R.get(), tau, rho, to_mode(mode), kStream);
        *out = h.release();
    });
}
int mfreg_cu_ngf_destroy(mfreg_cu_ngf* ngf) {
    return guard([&] { delete ngf; });
}
int mfreg_cu_ngf_populate(mfreg_cu_ngf* h, const double* tpl, const double* points, int where) {
    return guard([&] {
        const idx_t n = h->g.count();
        In t(tpl, n, where, kStream), p(points, 3 * n, where, kStream);
        h->ngf->populate_points(t.ptr, p.ptr);
        MFREG_CUDA(cudaStreamSynchronize(kStream));
    });
}
int mfreg_cu_ngf_value(mfreg_cu_ngf* h, double* out) {
    return guard([&] {
        DVec d(1);
        h->ngf->value_async(d.get());
        MFREG_CUDA(cudaMemcpyAsync(out, d.get(), sizeof(double), cudaMemcpyDeviceToHost, kStream));
        MFREG_CUDA(cudaStreamSynchronize(kStream));
    });
}
int mfreg_cu_ngf_gradient(mfreg_cu_ngf* h, double* out, int where) {
    return guard([&] {
        Out o(out, 3 * h->g.count(), where);
        h->ngf->gradient(o.ptr);
        o.finish(kStream);
    });
}
int mfreg_cu_ngf_hessian_vec(mfreg_cu_ngf* h, const double* p, double* out, int where) {
    return guard([&] {
        const idx_t n = h->g.count();
        In pi(p, 3 * n, where, kStream);
        Out o(out, 3 * n, where);
        h->ngf->hessian_vec(pi.ptr, o.ptr);
        o.finish(kStream);
    });
}
int mfreg_cu_ngf_workspace(mfreg_cu_ngf* h, double* values, double* partials, double* residual, double* inv1,
                           double* inv2, double* rho_hat, int where) {
    return guard([&] {
        check_where(where);
        const std::size_t n = h->g.count();
        const auto kind = where == MFREG_CU_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice;
        auto cp = [&](double* dst, const DVec& src, std::size_t k) {
            if (dst) MFREG_CUDA(cudaMemcpyAsync(dst, src.get(), k * n * sizeof(double), kind, kStream));
        };
        cp(values, h->ngf->Tw, 1);
        cp(partials, h->ngf->dT, 3);
        cp(residual, h->ngf->r, 1);
        cp(inv1, h->ngf->inv1, 1);
        cp(inv2, h->ngf->inv2, 1);
        cp(rho_hat, h->ngf->rh, 7);
        MFREG_CUDA(cudaStreamSynchronize(kStream));
    });
}

// ---- Objective
int mfreg_cu_objective_create(const double* ref, const double* tpl, const mfreg_cu_grid* image,
                              const mfreg_cu_grid* deform, double tau, double rho, double alpha, int mode, int where,
                              mfreg_cu_objective** out) {
    return guard([&] {
        check_where(where);
        auto h = std::make_unique<mfreg_cu_objective>();
        h->img = to_grid(image);
        h->dg = to_grid(deform);
        validate_grid(h->img, false);
        const std::size_t n = h->img.count();
        h->R.resize(n);
        h->T.resize(n);
        const auto kind = where == MFREG_CU_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice;
        MFREG_CUDA(cudaMemcpy(h->R.get(), ref, n * sizeof(double), kind));
        MFREG_CUDA(cudaMemcpy(h->T.get(), tpl, n * sizeof(double), kind));
        h->obj = std::make_unique<DeviceObjective>(h->R.get(), h->T.get(), h->img, h->dg, tau, rho, alpha,
                                                   to_mode(mode), kStream);
        MFREG_CUDA(cudaStreamSynchronize(kStream));
        *out = h.release();
    });
}
int mfreg_cu_objective_create_slab(const double* ref, const double* tpl, const mfreg_cu_grid* image,
                                   const mfreg_cu_grid* deform, double tau, double rho, double alpha,
                                   const int32_t slab[4], int where, mfreg_cu_objective** out) {
    return guard([&] {
        check_where(where);
        if (!slab) throw std::invalid_argument("slab: null window");
        auto h = std::make_unique<mfreg_cu_objective>();
        h->img = to_grid(image);
        h->dg = to_grid(deform);
        validate_grid(h->img, false);
        const std::size_t n = h->img.count();
        h->R.resize(n);
        h->T.resize(n);
        const auto kind = where == MFREG_CU_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice;
        MFREG_CUDA(cudaMemcpy(h->R.get(), ref, n * sizeof(double), kind));
        MFREG_CUDA(cudaMemcpy(h->T.get(), tpl, n * sizeof(double), kind));
        SlabSpec sp;
        sp.zlo = slab[0];
        sp.zhi = slab[1];
        sp.own_lo = slab[2];
        sp.own_hi = slab[3];
        h->obj = std::make_unique<DeviceObjective>(h->R.get(), h->T.get(), h->img, h->dg, tau, rho, alpha, Mode::Fast,
                                                   kStream, sp);
        MFREG_CUDA(cudaStreamSynchronize(kStream));
        *out = h.release();
    });
}
int mfreg_cu_slab_partition(const mfreg_cu_grid* image, const mfreg_cu_grid* deform, int nranks, int32_t* table) {
    return mfreg_cu_slab_partition_mode(image, deform, nranks, MFREG_CU_FAST, table);
}
int mfreg_cu_slab_partition_mode(const mfreg_cu_grid* image, const mfreg_cu_grid* deform, int nranks, int mode,
                                 int32_t* table) {
    return guard([&] {
        const auto parts = slab_partition(to_grid(image), to_grid(deform), nranks, to_mode(mode) == Mode::Parity);
        for (int r = 0; r < nranks; ++r) {
            const SlabInfo& s = parts[r];
            const int32_t v[7] = {s.zlo, s.zhi, s.own_lo, s.own_hi, s.need_lo, s.need_hi, s.bnd};
            std::memcpy(table + 7 * r, v, sizeof(v));
        }
    });
}
int mfreg_cu_objective_dot(mfreg_cu_objective* obj, const double* a, const double* b, int where, double* out) {
    return guard([&] {
        const idx_t nd = obj->obj->dof();
        In ai(a, nd, where, kStream);
        In bi(b, nd, where, kStream);
        *out = obj->obj->dot(ai.ptr, bi.ptr);
    });
}
int mfreg_cu_objective_destroy(mfreg_cu_objective* obj) {
    return guard([&] { delete obj; });
}
int mfreg_cu_objective_dof(mfreg_cu_objective* obj, int64_t* dof) {
    return guard([&] { *dof = obj->obj->dof(); });
}
int mfreg_cu_objective_min_spacing(mfreg_cu_objective* obj, double* out) {
    return guard([&] { *out = obj->obj->min_spacing(); });
}
int mfreg_cu_objective_identity(mfreg_cu_objective* obj, double* out, int where) {
    return guard([&] {
        check_where(where);
        MFREG_CUDA(cudaMemcpyAsync(out, obj->obj->identity_dev(), obj->obj->dof() * sizeof(double),
                                   where == MFREG_CU_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice,
                                   kStream));
        MFREG_CUDA(cudaStreamSynchronize(kStream));
    });
}
int mfreg_cu_objective_eval(mfreg_cu_objective* obj, const double* y, double* grad, int where, double* j) {
    return guard([&] {
        const idx_t nd = obj->obj->dof();
        if (!y) throw std::invalid_argument("Objective::eval: y length mismatch");
        check_where(where);
        if (where == MFREG_CU_HOST && grad && obj->obj->eval_host(y, grad, j)) return;  // copies pipelined
        In yi(y, nd, where, kStream, &obj->stage[0]);
        Out g(grad, nd, where, &obj->stage[1]);
        // one synchronisation: the gradient copy-out rides behind the scalar copy-out
        obj->obj->eval_begin(yi.ptr, g.ptr);
        if (where == MFREG_CU_HOST && grad)
            MFREG_CUDA(cudaMemcpyAsync(grad, g.ptr, nd * sizeof(double), cudaMemcpyDeviceToHost, kStream));
        MFREG_CUDA(cudaStreamSynchronize(kStream));
        const double v = obj->obj->eval_end();
        if (j) *j = v;
    });
}
int mfreg_cu_objective_last(mfreg_cu_objective* obj, double* distance, double* regularizer) {
    return guard([&] {
        if (distance) *distance = obj->obj->last_distance();
        if (regularizer) *regularizer = obj->obj->last_regularizer();
    });
}
int mfreg_cu_objective_gn_hessian_vec(mfreg_cu_objective* obj, const double* p, double* q, int where) {
    return guard([&] {
        const idx_t nd = obj->obj->dof();
        check_where(where);
        if (where == MFREG_CU_HOST && p && q && obj->obj->hv_host(p, q)) return;  // copies pipelined
        In pi(p, nd, where, kStream, &obj->stage[2]);
        Out o(q, nd, where, &obj->stage[3]);
        obj->obj->gn_hessian_vec(pi.ptr, o.ptr);
        o.finish(kStream);
    });
}
int mfreg_cu_objective_profile_kernel(mfreg_cu_objective* obj, int which, const double* operand, int reps,
                                      long long flush_bytes, double* ms) {
    return guard([&] {
        const idx_t nd = obj->obj->dof();
        const double* dev = operand;
        DVec tmp;
        if (cudaPointerAttributes at{}; cudaPointerGetAttributes(&at, operand) != cudaSuccess ||
                                         at.type != cudaMemoryTypeDevice) {
            cudaGetLastError();
            tmp.resize(nd);
            MFREG_CUDA(cudaMemcpy(tmp.get(), operand, nd * sizeof(double), cudaMemcpyHostToDevice));
            dev = tmp.get();
        }
        *ms = obj->obj->profile_kernel(which, dev, reps, static_cast<std::size_t>(std::max(0LL, flush_bytes)));
    });
}
int mfreg_cu_objective_seed_hessian_vec(mfreg_cu_objective* obj, const double* p, double gamma, double* q,
                                        int where) {
    return guard([&] {
        const idx_t nd = obj->obj->dof();
        In pi(p, nd, where, kStream, &obj->stage[2]);
        Out o(q, nd, where);
        obj->obj->seed_hessian_vec(pi.ptr, gamma, o.ptr);
        o.finish(kStream);
    });
}

int mfreg_cu_cg_solve(mfreg_cu_objective* obj, int op, double gamma, const double* b, int max_iters, double rel_tol,
                      double* x, int* iters, double* relres, int* breakdown, int where) {
    return guard([&] {
        if (obj->obj->sliced()) throw std::logic_error("slab objectives are driven by the distributed solver (slab.py)");
        const idx_t nd = obj->obj->dof();
        In bi(b, nd, where, kStream);
        Out xo(x, nd, where);
        const CgResult r = cg_solve(*obj->obj, op, gamma, bi.ptr, xo.ptr, {max_iters, rel_tol});
        xo.finish(kStream);
        if (iters) *iters = r.iters;
        if (relres) *relres = r.relres;
        if (breakdown) *breakdown = r.breakdown ? 1 : 0;
    });
}

int mfreg_cu_minimize(mfreg_cu_objective* obj, int method, const double* y0, const mfreg_cu_opt_config* cfg,
                      double* y_out, mfreg_cu_iter_record* trace, int cap, int* ntrace, int* line_search_failed,
                      int where) {
    return guard([&] {
        if (obj->obj->sliced()) throw std::logic_error("slab objectives are driven by the distributed solver (slab.py)");
        const idx_t nd = obj->obj->dof();
        In yi(y0, nd, where, kStream);
        Out yo(y_out, nd, where);
        const OptimizerConfig c = to_cfg(cfg);
        const MinimizeResult r = method == MFREG_CU_GAUSS_NEWTON ? gauss_newton_minimize(*obj->obj, yi.ptr, yo.ptr, c)
                                                                 : lbfgs_minimize(*obj->obj, yi.ptr, yo.ptr, c);
        yo.finish(kStream);
        MFREG_CUDA(cudaStreamSynchronize(kStream));
        const int n = copy_trace(r.trace, trace, cap);
        if (ntrace) *ntrace = n;
        if (line_search_failed) *line_search_failed = r.line_search_failed ? 1 : 0;
    });
}

int mfreg_cu_prolong(const mfreg_cu_grid* coarse, const mfreg_cu_grid* fine, const double* y_coarse, double* y_fine,
                     int where) {
    return guard([&] {
        const Grid c = to_grid(coarse), f = to_grid(fine);
        validate_grid(c, true);
        validate_grid(f, true);
        for (int a = 0; a < 3; ++a) {  // multilevel.cpp:83-91
            const double tol = std::max(c.h[a], f.h[a]);
            const double ec = static_cast<double>(c.m[a] - 1) * c.h[a], ef = static_cast<double>(f.m[a] - 1) * f.h[a];
            if (std::abs(ec - ef) > tol) throw std::invalid_argument("prolong: grid extents differ");
        }
        In yi(y_coarse, 3 * c.count(), where, kStream);
        Out yo(y_fine, 3 * f.count(), where);
        launch_prolong(c, f, yi.ptr, yo.ptr, kStream);
        check_launch("prolong");
        yo.finish(kStream);
    });
}

static int register_multilevel_impl(const double* ref, const double* tpl, const mfreg_cu_grid* image,
                                    const mfreg_cu_ml_config* cfg, double* y_out, mfreg_cu_grid* deform_out,
                                    mfreg_cu_iter_record* trace, int cap, int* level_iters, int* line_search_failed,
                                    mfreg_cu_grid* level_image, mfreg_cu_grid* level_deform, double* level_y,
                                    int64_t level_y_cap, int where) {
    return guard([&] {
        const Grid g = to_grid(image);
        validate_grid(g, false);
        const idx_t n = g.count();
        In r(ref, n, where, kStream), t(tpl, n, where, kStream);
        MultilevelConfig mc;
        mc.levels = cfg->levels;
        mc.deform_ratio = cfg->deform_ratio;
        mc.tau = cfg->tau;
        mc.rho = cfg->rho;
        mc.alpha = cfg->alpha;
        mc.method = cfg->method == MFREG_CU_GAUSS_NEWTON ? Method::GaussNewton : Method::Lbfgs;
        mc.mode = to_mode(cfg->mode);
        mc.opt = to_cfg(&cfg->opt);
        mc.keep_level_y = level_y != nullptr;
        MultilevelResult res = register_multilevel(r.ptr, t.ptr, g, mc, kStream);
        if (deform_out) from_grid(res.deform_grid, deform_out);
        check_where(where);
        const cudaMemcpyKind kind = where == MFREG_CU_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice;
        if (y_out) MFREG_CUDA(cudaMemcpyAsync(y_out, res.y.get(), res.y.size() * sizeof(double), kind, kStream));
        int64_t yoff = 0;
        for (std::size_t l = 0; l < res.levels.size(); ++l) {
            if (level_image) from_grid(res.levels[l].image_grid, level_image + l);
            if (level_deform) from_grid(res.levels[l].deform_grid, level_deform + l);
            if (level_y) {
                const auto& yl = res.levels[l].y;
                if (yoff + static_cast<int64_t>(yl.size()) > level_y_cap)
                    throw std::invalid_argument("register_multilevel: level_y buffer too small");
                MFREG_CUDA(cudaMemcpyAsync(level_y + yoff, yl.get(), yl.size() * sizeof(double), kind, kStream));
                yoff += static_cast<int64_t>(yl.size());
            }
        }
        MFREG_CUDA(cudaStreamSynchronize(kStream));
        int off = 0;
        for (std::size_t l = 0; l < res.levels.size(); ++l) {
            const int k = copy_trace(res.levels[l].result.trace, trace ? trace + std::min(off, cap) : nullptr,
                                     std::max(0, cap - off));
            if (level_iters) level_iters[l] = k;
            if (line_search_failed) line_search_failed[l] = res.levels[l].result.line_search_failed ? 1 : 0;
            off += k;
        }
    });
}

int mfreg_cu_register_multilevel(const double* ref, const double* tpl, const mfreg_cu_grid* image,
                                 const mfreg_cu_ml_config* cfg, double* y_out, mfreg_cu_grid* deform_out,
                                 mfreg_cu_iter_record* trace, int cap, int* level_iters, int* line_search_failed,
                                 int where) {
    return register_multilevel_impl(ref, tpl, image, cfg, y_out, deform_out, trace, cap, level_iters,
                                    line_search_failed, nullptr, nullptr, nullptr, 0, where);
}

int mfreg_cu_register_multilevel_ex(const double* ref, const double* tpl, const mfreg_cu_grid* image,
                                    const mfreg_cu_ml_config* cfg, double* y_out, mfreg_cu_grid* deform_out,
                                    mfreg_cu_iter_record* trace, int cap, int* level_iters, int* line_search_failed,
                                    mfreg_cu_grid* level_image_grids, mfreg_cu_grid* level_deform_grids,
                                    double* level_y, int64_t level_y_cap, int where) {
    return register_multilevel_impl(ref, tpl, image, cfg, y_out, deform_out, trace, cap, level_iters,
                                    line_search_failed, level_image_grids, level_deform_grids, level_y, level_y_cap,
                                    where);
}

int mfreg_cu_make_phantom(const mfreg_cu_grid* image, double* out, int where) {
    return guard([&] {
        const Grid g = to_grid(image);
        validate_grid(g, false);
        Out o(out, g.count(), where);
        launch_phantom(g, o.ptr, kStream);
        check_launch("make_phantom");
        o.finish(kStream);
    });
}

int mfreg_cu_warp_sinusoid(const mfreg_cu_grid* image, const double* vol, double max_amp, uint64_t seed, double* out,
                           int where) {
    return guard([&] {
        const Grid g = to_grid(image);
        validate_grid(g, false);
        const double ext[3] = {static_cast<double>(g.m[0]) * g.h[0], static_cast<double>(g.m[1]) * g.h[1],
                               static_cast<double>(g.m[2]) * g.h[2]};
        const WarpTerms w = sinusoid_terms(ext, max_amp, seed);
        In v(vol, g.count(), where, kStream);
        Out o(out, g.count(), where);
        launch_warp_with(g, w, v.ptr, o.ptr, kStream);
        check_launch("warp_with");
        o.finish(kStream);
    });
}

int mfreg_cu_scale(int64_t n, double a, double* x, int where) {
    return guard([&] {
        if (where != MFREG_CU_DEVICE) throw std::invalid_argument("mfreg_cu_scale expects device memory");
        launch_scale_inplace(n, a, x, kStream);
        check_launch("scale");
    });
}

int64_t mfreg_cu_launch_count(void) { return mfreg_b200::launch_counter(); }

// ---- volume / deformation / landmark files (io.cuh)
int mfreg_cu_read_volume(const char* path, mfreg_cu_grid* grid, double* data, int where) {
    return guard([&] {
        check_where(where);
        const io::VolumeHeader h = io::read_volume_header(path);
        if (grid) from_grid(h.grid, grid);
        if (!data) return;
        if (where == MFREG_CU_DEVICE) {
            io::read_volume(path, data, kStream);
        } else {
            DVec d(h.grid.count());
            io::read_volume(path, d.get(), kStream);
            MFREG_CUDA(cudaMemcpy(data, d.get(), h.grid.count() * sizeof(double), cudaMemcpyDeviceToHost));
        }
    });
}

int mfreg_cu_write_volume(const char* path, const mfreg_cu_grid* grid, const double* data, int where) {
    return guard([&] {
        check_where(where);
        const Grid g = to_grid(grid);
        validate_grid(g, false);
        if (where == MFREG_CU_DEVICE) {
            std::vector<double> h(g.count());
            MFREG_CUDA(cudaMemcpy(h.data(), data, h.size() * sizeof(double), cudaMemcpyDeviceToHost));
            io::write_volume(path, g, h.data());
        } else {
            io::write_volume(path, g, data);
        }
    });
}

int mfreg_cu_write_deformation(const char* path, const double* y, int64_t n, const mfreg_cu_grid* nodal, int where) {
    return guard([&] {
        check_where(where);
        const Grid g = to_grid(nodal);
        if (where == MFREG_CU_DEVICE && n == 3 * g.count()) {
            std::vector<double> h(static_cast<std::size_t>(n));
            MFREG_CUDA(cudaMemcpy(h.data(), y, h.size() * sizeof(double), cudaMemcpyDeviceToHost));
            io::write_deformation(path, h.data(), h.size(), g);
        } else {
            io::write_deformation(path, y, static_cast<std::size_t>(std::max<int64_t>(0, n)), g);
        }
    });
}

int mfreg_cu_read_deformation_grid(const char* path, mfreg_cu_grid* nodal) {
    return guard([&] { from_grid(io::read_deformation_grid(path), nodal); });
}

int mfreg_cu_read_deformation(const char* path, const mfreg_cu_grid* nodal, double* y, int where) {
    return guard([&] {
        check_where(where);
        const std::vector<double> v = io::read_deformation(path, to_grid(nodal));
        if (where == MFREG_CU_DEVICE)
            MFREG_CUDA(cudaMemcpy(y, v.data(), v.size() * sizeof(double), cudaMemcpyHostToDevice));
        else
            std::memcpy(y, v.data(), v.size() * sizeof(double));
    });
}

int mfreg_cu_read_landmarks(const char* path, const double spacing[3], double* out, int64_t cap, int64_t* count) {
    return guard([&] {
        const auto v = io::read_landmarks(path, {spacing[0], spacing[1], spacing[2]});
        *count = static_cast<int64_t>(v.size());
        for (std::size_t i = 0; out && i < v.size() && static_cast<int64_t>(i) < cap; ++i)
            for (int a = 0; a < 3; ++a) out[3 * i + a] = v[i][a];
    });
}

int mfreg_cu_landmark_error(const double* fixed, int64_t n_fixed, const double* moving, int64_t n_moving,
                            const double* y, int64_t ny, const mfreg_cu_grid* nodal, int where, double* mean,
                            double* stddev, int64_t* count) {
    return guard([&] {
        if (n_fixed != n_moving) throw std::invalid_argument("landmark_error: list sizes differ");
        Grid g = to_grid(nodal);
        if (ny != 3 * g.count()) throw std::invalid_argument("landmark_error: field length mismatch");
        In yi(y, static_cast<std::size_t>(ny), where, kStream);
        const io::LandmarkStats st =
            io::landmark_error(fixed, moving, static_cast<std::size_t>(n_fixed), yi.ptr, g, kStream);
        *mean = st.mean;
        *stddev = st.stddev;
        *count = static_cast<int64_t>(st.count);
    });
}

int mfreg_cu_warp_volume(const double* vol, const mfreg_cu_grid* image, const double* y, const mfreg_cu_grid* nodal,
                         double* out, int where) {
    return guard([&] {
        Grid gi = to_grid(image), gn = to_grid(nodal);
        validate_grid(gi, false);
        validate_grid(gn, true);
        In vi(vol, gi.count(), where, kStream);
        In yi(y, 3 * gn.count(), where, kStream);
        Out o(out, gi.count(), where);
        io::warp_volume(vi.ptr, gi, yi.ptr, gn, o.ptr, kStream);
        o.finish(kStream);
    });
}

}  // extern "C"
