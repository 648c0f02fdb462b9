// Reference-style client of the mfreg public API (optimizer.hpp, ngf.hpp, volume.hpp,
// transfer.hpp, curvature.hpp, multilevel.hpp, grid.hpp). The same source compiles
//   * against the reference headers + the unmodified reference library (-DMFREG_REFERENCE;
//     tests/golden/gen_api_client.py, in the build container), and
//   * against include/mfreg_b200.hpp + libmfreg_cuda.so (namespace mfreg = mfreg_b200).
// It prints every result as exact bit patterns / byte hashes, so the two outputs are compared
// line by line (tests/test_cpp_drop_in.py). Inputs are closed-form (no generator library).
#include <cinttypes>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#ifdef MFREG_REFERENCE
#include "mfreg/multilevel.hpp"
#else
#include "mfreg_b200.hpp"
namespace mfreg = mfreg_b200;
#endif

namespace {

std::uint64_t bits(double v) {
    std::uint64_t u;
    std::memcpy(&u, &v, 8);
    return u;
}
std::uint64_t hash(std::span<const double> a) {  // FNV-1a over the bit patterns
    std::uint64_t h = 1469598103934665603ull;
    for (double v : a) {
        const std::uint64_t u = bits(v);
        for (int k = 0; k < 8; ++k) {
            h ^= (u >> (8 * k)) & 0xffu;
            h *= 1099511628211ull;
        }
    }
    return h;
}
void pd(const char* key, double v) { std::printf("%s %016" PRIx64 "\n", key, bits(v)); }
void pv(const char* key, std::span<const double> a) { std::printf("%s n=%zu %016" PRIx64 "\n", key, a.size(), hash(a)); }
void pi(const char* key, long long v) { std::printf("%s %lld\n", key, v); }

// f(y) = 1/2 sum d_i y_i^2 (the shape of tests/test_optimizer.cpp's Quadratic)
class Quadratic : public mfreg::Problem {
public:
    explicit Quadratic(std::vector<double> diag) : diag_(std::move(diag)) {}
    double eval(std::span<const double> y, std::span<double> grad) override {
        double f = 0.0;
        for (std::size_t i = 0; i < y.size(); ++i) {
            f += 0.5 * diag_[i] * y[i] * y[i];
            if (!grad.empty()) grad[i] = diag_[i] * y[i];
        }
        return f;
    }
    void gn_hessian_vec(std::span<const double> p, std::span<double> q) override {
        for (std::size_t i = 0; i < p.size(); ++i) q[i] = diag_[i] * p[i];
    }
    void seed_hessian_vec(std::span<const double> p, double gamma, std::span<double> q) override {
        for (std::size_t i = 0; i < p.size(); ++i) q[i] = (1.0 + gamma) * p[i];
    }
    double min_spacing() const override { return 1.0; }

private:
    std::vector<double> diag_;
};

mfreg::Volume field(std::array<mfreg::index_t, 3> m, std::array<double, 3> h, double a, double b) {
    mfreg::Volume v = mfreg::make_volume(m, h);
    for (mfreg::index_t i = 0; i < v.grid.count(); ++i) {
        const auto p = v.grid.point_coords(i);
        v.data[static_cast<std::size_t>(i)] =
            1000.0 * (std::sin(a * p[0] + 0.3) * std::cos(b * p[1] - 0.2) + 0.5 * std::sin(0.37 * p[2] + a * b));
    }
    return v;
}

void trace(const char* key, const mfreg::MinimizeResult& r) {
    for (const auto& t : r.trace)
        std::printf("%s it %d cg %d j %016" PRIx64 " d %016" PRIx64 " s %016" PRIx64 " g %016" PRIx64 " step %016" PRIx64
                    "\n",
                    key, t.iter, t.cg_iters, bits(t.j), bits(t.distance), bits(t.regularizer), bits(t.grad_norm),
                    bits(t.step));
    pv((std::string(key) + " y").c_str(), r.y);
    pi((std::string(key) + " lsf").c_str(), r.line_search_failed ? 1 : 0);
}

}  // namespace

int main() {
    // ---- vec_dot / vec_norm / vec_inf_norm (chunks of 4096 crossed)
    std::vector<double> a(10007), b(10007);
    for (std::size_t i = 0; i < a.size(); ++i) {
        a[i] = std::sin(0.01 * static_cast<double>(i)) * 3.7;
        b[i] = std::cos(0.013 * static_cast<double>(i)) - 0.25;
    }
    pd("vec_dot", mfreg::vec_dot(a, b));
    pd("vec_norm", mfreg::vec_norm(a));
    pd("vec_inf_norm", mfreg::vec_inf_norm(b));
    try {
        (void)mfreg::vec_dot(a, std::span<const double>(b).first(5));
    } catch (const std::invalid_argument& e) {
        std::printf("vec_dot throws %s\n", e.what());
    }

    // ---- a user Problem through the generic solvers
    {
        std::vector<double> d(300), y0(300);
        for (std::size_t i = 0; i < d.size(); ++i) {
            d[i] = 1.0 + 0.5 * static_cast<double>(i % 17);
            y0[i] = std::cos(0.3 * static_cast<double>(i)) * 2.0;
        }
        Quadratic q(d);
        mfreg::OptimizerConfig cfg;
        cfg.max_iters = 6;
        trace("quad_gn", mfreg::gauss_newton_minimize(q, y0, cfg));
        trace("quad_lbfgs", mfreg::lbfgs_minimize(q, y0, cfg));
    }
    // ---- cg_solve with a LinearOperator, armijo_search with a phi
    {
        const std::size_t n = 5000;
        mfreg::LinearOperator op = [&](std::span<const double> p, std::span<double> out) {
            for (std::size_t i = 0; i < n; ++i) {
                double v = 2.5 * p[i];
                if (i > 0) v -= p[i - 1];
                if (i + 1 < n) v -= p[i + 1];
                out[i] = v;
            }
        };
        std::vector<double> rhs(n);
        for (std::size_t i = 0; i < n; ++i) rhs[i] = std::sin(0.001 * static_cast<double>(i * i % 997));
        const auto r = mfreg::cg_solve(op, rhs, mfreg::CgConfig{40, 1e-6});
        pi("cg iters", r.iters);
        pd("cg relres", r.relres);
        pv("cg x", r.x);
        const auto phi = [](double eta) { return (eta - 0.3) * (eta - 0.3) + 1.0; };
        const auto ar = mfreg::armijo_search(phi, 1.09, -0.6, mfreg::ArmijoConfig{}, 1.0);
        pd("armijo eta", ar.eta);
        pi("armijo accepted", ar.accepted);
        pd("armijo f_new", ar.f_new);
        const auto ar2 = mfreg::armijo_search(phi, 1.09, 0.5, mfreg::ArmijoConfig{});
        pi("armijo descent", ar2.descent);
    }

    // ---- grids
    const auto img = mfreg::make_image_grid({18, 14, 12}, {0.97, 0.97, 2.5});
    const auto dg = mfreg::deformation_grid_for(img, 4);
    std::printf("deform %lld %lld %lld %016" PRIx64 " %016" PRIx64 " %016" PRIx64 "\n", (long long)dg.m[0],
                (long long)dg.m[1], (long long)dg.m[2], bits(dg.h[0]), bits(dg.h[1]), bits(dg.h[2]));
    pi("neighbor", img.neighbor(img.linear(0, 5, 11), mfreg::Dir::PosZ) + 7 * img.neighbor(37, mfreg::Dir::NegX));
    try {
        (void)mfreg::make_deform_grid(img, {40, 4, 4});
    } catch (const std::invalid_argument& e) {
        std::printf("make_deform_grid throws %s\n", e.what());
    }

    // ---- volume.hpp
    const mfreg::Volume R = field(img.m, img.h, 0.41, 0.23), T = field(img.m, img.h, 0.38, 0.27);
    {
        const auto ir = mfreg::interpolate(T, {3.3, 6.79, 12.5});
        pd("interp v", ir.value);
        pd("interp gx", ir.grad[0]);
        pd("interp gz", ir.grad[2]);
        const auto ir2 = mfreg::interpolate(T, {-3.0, 2.0, 2.0});  // Dirichlet zero
        pd("interp out", ir2.value);
        const auto g6 = mfreg::discrete_gradient(R, 17 + 18 * 13);
        pv("dgrad", g6);
        pd("eps_norm", mfreg::eps_norm(g6, 10.0));
        const auto ds = mfreg::downsample(R);
        pi("downsample m", ds.grid.m[0] * 10000 + ds.grid.m[1] * 100 + ds.grid.m[2]);
        pv("downsample", ds.data);
    }
    // ---- transfer.hpp
    const auto plan = mfreg::make_transfer_plan(dg, img);
    {
        std::vector<double> bb;
        for (int ax = 0; ax < 3; ++ax)
            for (std::size_t k = 0; k < plan.base[ax].size(); ++k) bb.push_back(static_cast<double>(plan.base[ax][k]) + plan.rem[ax][k]);
        pv("plan", bb);
        long long sp = 0;
        for (std::size_t s = 0; s < plan.slab_planes.size(); ++s)
            for (auto k : plan.slab_planes[s]) sp = sp * 31 + static_cast<long long>(s * 100 + static_cast<std::size_t>(k));
        pi("slab_planes", sp);
    }
    std::vector<double> y(3 * static_cast<std::size_t>(dg.count()));
    for (mfreg::index_t i = 0; i < dg.count(); ++i) {
        const auto p = dg.point_coords(i);
        for (int d = 0; d < 3; ++d)
            y[static_cast<std::size_t>(d * dg.count() + i)] = p[d] + 0.4 * std::sin(1.7 * static_cast<double>(i) + d);
    }
    std::vector<double> yhat(3 * static_cast<std::size_t>(img.count())), back(y.size());
    mfreg::transfer_apply(plan, y, yhat);
    pv("P y", yhat);
    mfreg::transfer_apply_transpose(plan, yhat, back);
    pv("PT w", back);
    // ---- curvature.hpp
    {
        std::vector<double> u(y.size()), lap(static_cast<std::size_t>(dg.count()));
        for (std::size_t i = 0; i < u.size(); ++i) u[i] = std::cos(0.7 * static_cast<double>(i));
        pd("laplacian", mfreg::laplacian(std::span<const double>(u).first(lap.size()), dg, 5));
        mfreg::laplacian_apply(std::span<const double>(u).first(lap.size()), dg, lap);
        pv("laplacian_apply", lap);
        pd("curv value", mfreg::curvature_value(u, dg));
        pv("curv grad", mfreg::curvature_gradient(u, dg));
        std::vector<double> scratch(lap.size()), out(u.size());
        mfreg::curvature_hessian_vec(u, dg, scratch, out);
        pv("curv hv", out);
        try {
            mfreg::curvature_hessian_vec(u, dg, std::span<double>(scratch).first(3), out);
        } catch (const std::invalid_argument& e) {
            std::printf("curvature throws %s\n", e.what());
        }
    }
    // ---- ngf.hpp
    {
        const mfreg::NgfParams prm{};
        const auto pre = mfreg::make_ngf_precomp(R, prm.rho);
        std::vector<double> rg;
        for (const auto& g : pre.ref_grads) rg.insert(rg.end(), g.begin(), g.end());
        pv("precomp grads", rg);
        pv("precomp norms", pre.ref_norms);
        mfreg::NgfWorkspace ws;
        mfreg::populate_ngf_workspace(ws, T, yhat, pre, prm, img);
        pv("ws values", ws.sampled.values);
        pv("ws partials z", ws.sampled.partials[2]);
        std::vector<double> tg;
        for (const auto& g : ws.tpl_grads) tg.insert(tg.end(), g.begin(), g.end());
        pv("ws tpl_grads", tg);
        pv("ws residual", ws.residual);
        pv("ws inv2", ws.inv2);
        pd("ngf_residual", mfreg::ngf_residual(100, ws));
        pd("ngf_rho", mfreg::ngf_rho(100, mfreg::Dir::PosY, ws, pre, img) + mfreg::ngf_rho(7, mfreg::Dir::Center, ws, pre, img));
        pd("ngf_value", mfreg::ngf_value(ws, img));
        std::vector<double> gout(yhat.size()), hv(yhat.size()), p(yhat.size());
        mfreg::ngf_gradient(ws, pre, img, gout);
        pv("ngf_gradient", gout);
        for (std::size_t i = 0; i < p.size(); ++i) p[i] = std::sin(0.11 * static_cast<double>(i));
        mfreg::ngf_hessian_vec(p, ws, pre, img, hv);
        pv("ngf_hessian_vec", hv);
        const auto tab = mfreg::make_offset_table(img);
        long long ts = 0;
        for (const auto& e : tab.entries) {
            ts = ts * 7 + e.kappa;
            for (const auto& pr : e.pairs) ts = ts * 3 + static_cast<int>(pr.first) * 7 + static_cast<int>(pr.second);
        }
        pi("offset table", static_cast<long long>(tab.entries.size()) * 1000 + static_cast<long long>(tab.pair_count()));
        pi("offset hash", ts);
    }
    // ---- Objective (Problem) and the solvers on it
    {
        mfreg::Objective obj(R, T, dg, mfreg::NgfParams{}, 1.0);
        std::vector<double> grad(y.size()), q(y.size()), p(y.size());
        const double j = obj.eval(y, grad);
        pd("obj J", j);
        pd("obj D", obj.last_distance());
        pd("obj S", obj.last_regularizer());
        pv("obj grad", grad);
        for (std::size_t i = 0; i < p.size(); ++i) p[i] = std::cos(0.05 * static_cast<double>(i));
        obj.gn_hessian_vec(p, q);
        pv("obj gnhv", q);
        obj.seed_hessian_vec(p, 0.25, q);
        pv("obj seedhv", q);
        pv("obj workspace residual", obj.workspace().residual);
        pd("obj min_spacing", obj.min_spacing());
        pi("obj plan", static_cast<long long>(obj.plan().base[2].size()));
        try {
            obj.gn_hessian_vec(std::span<const double>(p).first(10), q);
        } catch (const std::invalid_argument& e) {
            std::printf("gn_hessian_vec throws %s\n", e.what());
        }
        mfreg::OptimizerConfig cfg;
        cfg.max_iters = 3;
        trace("obj_gn", mfreg::gauss_newton_minimize(obj, obj.identity(), cfg));
        trace("obj_lbfgs", mfreg::lbfgs_minimize(obj, obj.identity(), cfg));
    }
    // ---- multilevel.hpp
    {
        const auto pyr = mfreg::build_pyramid(R, T, 2);
        pv("pyramid", pyr[1].tpl.data);
        const auto cg = mfreg::deformation_grid_for(pyr[1].reference.grid, 4);
        std::vector<double> yc(3 * static_cast<std::size_t>(cg.count()));
        for (mfreg::index_t i = 0; i < cg.count(); ++i) {
            const auto pc = cg.point_coords(i);
            for (int d = 0; d < 3; ++d) yc[static_cast<std::size_t>(d * cg.count() + i)] = pc[d] + 0.2 * std::cos(static_cast<double>(i) + d);
        }
        pd("nodal_interpolate", mfreg::nodal_interpolate(std::span<const double>(yc).first(static_cast<std::size_t>(cg.count())), cg, {3.1, 2.2, 9.9}));
        pv("prolong", mfreg::prolong(yc, cg, dg));
        try {
            (void)mfreg::build_pyramid(R, T, 9);
        } catch (const std::invalid_argument& e) {
            std::printf("build_pyramid throws %s\n", e.what());
        }
        mfreg::MultilevelConfig mc;
        mc.levels = 2;
        mc.method = mfreg::Method::GaussNewton;
        mc.opt.max_iters = 3;
        const auto res = mfreg::register_multilevel(R, T, mc);
        pv("ml y", res.y);
        for (const auto& lv : res.levels) {
            std::printf("ml level image %lld %lld %lld deform %lld %lld %lld\n", (long long)lv.image_grid.m[0],
                        (long long)lv.image_grid.m[1], (long long)lv.image_grid.m[2], (long long)lv.deform_grid.m[0],
                        (long long)lv.deform_grid.m[1], (long long)lv.deform_grid.m[2]);
            trace("ml", lv.result);
        }
    }
    return 0;
}
