// mfreg_b200.hpp — header-only C++ drop-in for the reference mfreg API
// (/root/reference/proj/include/mfreg/*.hpp) over the C ABI in mfreg_cuda.h.
//
// Same type names, member functions, argument meaning, defaults and exception
// types as the reference; a caller switches with
//     namespace mfreg = mfreg_b200;
// Host std::span / std::vector arguments are staged through the C ABI; the
// derivative evaluations, solver loops and multilevel driver run on the GPU.
// The extra trailing ExecMode argument selects `Parity` (bitwise identical to the
// reference, default) or `Fast` (fused kernels, max-rel <= 1e-9 per operator).
#ifndef MFREG_B200_HPP
#define MFREG_B200_HPP

#include <array>
#include <filesystem>
#include <cstdint>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "mfreg_cuda.h"

namespace mfreg_b200 {

using index_t = std::int64_t;

enum class GridKind { CellCentered, Nodal };  // grid.hpp:14
enum class ExecMode : int { Parity = MFREG_CU_PARITY, Fast = MFREG_CU_FAST };

namespace detail {
inline void check(int rc) {
    if (rc == MFREG_CU_OK) return;
    const std::string msg = mfreg_cu_last_error();
    if (rc == MFREG_CU_EINVAL) throw std::invalid_argument(msg);
    if (rc == MFREG_CU_ELOGIC) throw std::logic_error(msg);
    throw std::runtime_error(msg);
}
}  // namespace detail

// grid.hpp:50-120
struct GridDesc {
    std::array<index_t, 3> m{1, 1, 1};
    std::array<double, 3> h{1.0, 1.0, 1.0};
    GridKind kind = GridKind::CellCentered;

    index_t count() const { return m[0] * m[1] * m[2]; }
    double cell_volume() const { return h[0] * h[1] * h[2]; }
    double extent(int axis) const {
        return kind == GridKind::CellCentered ? static_cast<double>(m[axis]) * h[axis]
                                              : static_cast<double>(m[axis] - 1) * h[axis];
    }
    index_t linear(index_t i, index_t j, index_t k) const { return i + j * m[0] + k * m[0] * m[1]; }
    mfreg_cu_grid c() const { return mfreg_cu_grid{{m[0], m[1], m[2]}, {h[0], h[1], h[2]}}; }
};

inline GridDesc from_c(const mfreg_cu_grid& g, GridKind kind) {
    return GridDesc{{g.m[0], g.m[1], g.m[2]}, {g.h[0], g.h[1], g.h[2]}, kind};
}

inline GridDesc make_image_grid(std::array<index_t, 3> m, std::array<double, 3> h) {  // grid.hpp:122-127
    for (int a = 0; a < 3; ++a) {
        if (m[a] < 1) throw std::invalid_argument("GridDesc: all m components must be >= 1");
        if (!(h[a] > 0.0)) throw std::invalid_argument("GridDesc: all h components must be > 0");
    }
    return GridDesc{m, h, GridKind::CellCentered};
}

inline GridDesc make_deform_grid(const GridDesc& image, std::array<index_t, 3> points) {  // grid.hpp:131-146
    const mfreg_cu_grid img = image.c();
    mfreg_cu_grid out{};
    const int64_t p[3] = {points[0], points[1], points[2]};
    detail::check(mfreg_cu_make_deform_grid(&img, p, &out));
    return from_c(out, GridKind::Nodal);
}

inline GridDesc deformation_grid_for(const GridDesc& image, index_t ratio) {  // multilevel.cpp:39-49
    const mfreg_cu_grid img = image.c();
    mfreg_cu_grid out{};
    detail::check(mfreg_cu_deformation_grid_for(&img, ratio, &out));
    return from_c(out, GridKind::Nodal);
}

// volume.hpp:13-16
struct Volume {
    GridDesc grid;
    std::vector<double> data;
};

struct NgfParams {  // ngf.hpp:14-17
    double tau = 10.0;
    double rho = 10.0;
};

// ---- kernel-level API (transfer.hpp, curvature.hpp) -----------------------
inline void transfer_apply(const GridDesc& nodal, const GridDesc& image, std::span<const double> y,
                           std::span<double> out) {
    if (y.size() != static_cast<std::size_t>(3 * nodal.count()) ||
        out.size() != static_cast<std::size_t>(3 * image.count()))
        throw std::invalid_argument("transfer_apply: length mismatch");
    const mfreg_cu_grid s = nodal.c(), t = image.c();
    detail::check(mfreg_cu_transfer_apply(&s, &t, y.data(), out.data(), MFREG_CU_HOST));
}

inline void transfer_apply_transpose(const GridDesc& nodal, const GridDesc& image, std::span<const double> w,
                                     std::span<double> out) {
    if (w.size() != static_cast<std::size_t>(3 * image.count()) ||
        out.size() != static_cast<std::size_t>(3 * nodal.count()))
        throw std::invalid_argument("transfer_apply_transpose: length mismatch");
    const mfreg_cu_grid s = nodal.c(), t = image.c();
    detail::check(mfreg_cu_transfer_apply_transpose(&s, &t, w.data(), out.data(), MFREG_CU_HOST));
}

inline double curvature_value(std::span<const double> u, const GridDesc& g) {  // curvature.hpp:20
    if (u.size() != static_cast<std::size_t>(3 * g.count()))
        throw std::invalid_argument("curvature_value: length must be 3*m^y");
    const mfreg_cu_grid c = g.c();
    double v = 0.0;
    detail::check(mfreg_cu_curvature_value(&c, u.data(), &v, MFREG_CU_PARITY, MFREG_CU_HOST));
    return v;
}

inline std::vector<double> curvature_gradient(std::span<const double> u, const GridDesc& g) {  // curvature.hpp:30
    std::vector<double> out(u.size());
    const mfreg_cu_grid c = g.c();
    detail::check(mfreg_cu_curvature_gradient(&c, u.data(), out.data(), MFREG_CU_HOST));
    return out;
}

inline std::vector<double> curvature_hessian_vec(std::span<const double> p, const GridDesc& g) {
    std::vector<double> out(p.size());
    const mfreg_cu_grid c = g.c();
    detail::check(mfreg_cu_curvature_hessian_vec(&c, p.data(), out.data(), MFREG_CU_HOST));
    return out;
}

// ---- Objective (optimizer.hpp:53-106) ---------------------------------------
class Objective {
public:
    Objective(const Volume& reference, const Volume& tpl, const GridDesc& deform_grid, const NgfParams& params,
              double alpha, ExecMode mode = ExecMode::Parity)
        : image_grid_(reference.grid), deform_grid_(deform_grid), params_(params), alpha_(alpha) {
        deform_grid_.kind = GridKind::Nodal;
        const mfreg_cu_grid img = image_grid_.c(), dg = deform_grid_.c();
        detail::check(mfreg_cu_objective_create(reference.data.data(), tpl.data.data(), &img, &dg, params.tau,
                                                params.rho, alpha, static_cast<int>(mode), MFREG_CU_HOST, &h_));
    }
    ~Objective() {
        if (h_) mfreg_cu_objective_destroy(h_);
    }
    Objective(const Objective&) = delete;
    Objective& operator=(const Objective&) = delete;

    index_t dof() const { return 3 * deform_grid_.count(); }
    const GridDesc& image_grid() const { return image_grid_; }
    const GridDesc& deform_grid() const { return deform_grid_; }
    const NgfParams& params() const { return params_; }
    double alpha() const { return alpha_; }
    double min_spacing() const {
        double v = 0.0;
        detail::check(mfreg_cu_objective_min_spacing(h_, &v));
        return v;
    }
    std::vector<double> identity() const {
        std::vector<double> x(static_cast<std::size_t>(dof()));
        detail::check(mfreg_cu_objective_identity(h_, x.data(), MFREG_CU_HOST));
        return x;
    }
    // Evaluates J at y; fills grad if non-empty (optimizer.cpp:64-92).
    double eval(std::span<const double> y, std::span<double> grad) {
        if (y.size() != static_cast<std::size_t>(dof())) throw std::invalid_argument("Objective::eval: y length mismatch");
        if (!grad.empty() && grad.size() != y.size())
            throw std::invalid_argument("Objective::eval: grad length mismatch");
        double j = 0.0;
        detail::check(mfreg_cu_objective_eval(h_, y.data(), grad.empty() ? nullptr : grad.data(), MFREG_CU_HOST, &j));
        return j;
    }
    double last_distance() const {
        double d = 0.0, r = 0.0;
        detail::check(mfreg_cu_objective_last(h_, &d, &r));
        return d;
    }
    double last_regularizer() const {
        double d = 0.0, r = 0.0;
        detail::check(mfreg_cu_objective_last(h_, &d, &r));
        return r;
    }
    void gn_hessian_vec(std::span<const double> p, std::span<double> q) {
        detail::check(mfreg_cu_objective_gn_hessian_vec(h_, p.data(), q.data(), MFREG_CU_HOST));
    }
    void seed_hessian_vec(std::span<const double> p, double gamma, std::span<double> q) {
        detail::check(mfreg_cu_objective_seed_hessian_vec(h_, p.data(), gamma, q.data(), MFREG_CU_HOST));
    }
    mfreg_cu_objective* handle() const { return h_; }

private:
    GridDesc image_grid_, deform_grid_;
    NgfParams params_;
    double alpha_;
    mfreg_cu_objective* h_ = nullptr;
};

// ---- solvers (optimizer.hpp:108-166) ----------------------------------------
struct CgConfig {
    int max_iters = 50;
    double rel_tol = 1e-2;
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
    mfreg_cu_opt_config c() const {
        return mfreg_cu_opt_config{max_iters,   armijo.c1,    armijo.beta,   armijo.max_backtracks, cg.max_iters,
                                   cg.rel_tol,  h0_cg.max_iters, h0_cg.rel_tol, lbfgs_history,        gamma,
                                   tol_rel_j,   tol_grad,     tol_step};
    }
};
struct IterationRecord {
    int iter = 0;
    double j = 0.0, distance = 0.0, regularizer = 0.0, grad_norm = 0.0, step = 0.0;
    int cg_iters = 0;
};
using IterationTrace = std::vector<IterationRecord>;
struct MinimizeResult {
    std::vector<double> y;
    IterationTrace trace;
    bool line_search_failed = false;
};

namespace detail {
inline IterationTrace to_trace(const std::vector<mfreg_cu_iter_record>& r, int n) {
    IterationTrace t;
    for (int k = 0; k < n && k < static_cast<int>(r.size()); ++k)
        t.push_back({r[k].iter, r[k].j, r[k].distance, r[k].regularizer, r[k].grad_norm, r[k].step, r[k].cg_iters});
    return t;
}
inline MinimizeResult minimize(Objective& obj, std::span<const double> y0, const OptimizerConfig& cfg, int method) {
    MinimizeResult res;
    res.y.resize(static_cast<std::size_t>(obj.dof()));
    std::vector<mfreg_cu_iter_record> tr(static_cast<std::size_t>(cfg.max_iters + 8));
    int nt = 0, lsf = 0;
    const mfreg_cu_opt_config oc = cfg.c();
    check(mfreg_cu_minimize(obj.handle(), method, y0.data(), &oc, res.y.data(), tr.data(), static_cast<int>(tr.size()),
                            &nt, &lsf, MFREG_CU_HOST));
    res.trace = to_trace(tr, nt);
    res.line_search_failed = lsf != 0;
    return res;
}
}  // namespace detail

inline MinimizeResult lbfgs_minimize(Objective& obj, std::span<const double> y0, const OptimizerConfig& cfg) {
    return detail::minimize(obj, y0, cfg, MFREG_CU_LBFGS);
}
inline MinimizeResult gauss_newton_minimize(Objective& obj, std::span<const double> y0, const OptimizerConfig& cfg) {
    return detail::minimize(obj, y0, cfg, MFREG_CU_GAUSS_NEWTON);
}

// ---- multilevel (multilevel.hpp:36-64) ---------------------------------------
enum class Method { Lbfgs, GaussNewton };
struct MultilevelConfig {
    int levels = 3;
    index_t deform_ratio = 4;
    NgfParams ngf{};
    double alpha = 1.0;
    Method method = Method::Lbfgs;
    OptimizerConfig opt{};
    ExecMode mode = ExecMode::Parity;
};
struct LevelResult {
    GridDesc deform_grid;
    MinimizeResult result;
};
struct MultilevelResult {
    std::vector<double> y;
    GridDesc deform_grid;
    std::vector<LevelResult> levels;  // coarsest first (traces only)
};

inline MultilevelResult register_multilevel(const Volume& reference, const Volume& tpl, const MultilevelConfig& cfg) {
    const GridDesc dg = deformation_grid_for(reference.grid, cfg.deform_ratio);
    MultilevelResult out;
    out.y.resize(static_cast<std::size_t>(3 * dg.count()));
    const mfreg_cu_grid img = reference.grid.c();
    const mfreg_cu_ml_config mc{cfg.levels,
                                cfg.deform_ratio,
                                cfg.ngf.tau,
                                cfg.ngf.rho,
                                cfg.alpha,
                                cfg.method == Method::GaussNewton ? MFREG_CU_GAUSS_NEWTON : MFREG_CU_LBFGS,
                                static_cast<int>(cfg.mode),
                                cfg.opt.c()};
    const int cap = cfg.levels * (cfg.opt.max_iters + 2) + 8;
    std::vector<mfreg_cu_iter_record> tr(static_cast<std::size_t>(cap));
    std::vector<int> li(static_cast<std::size_t>(cfg.levels)), lsf(static_cast<std::size_t>(cfg.levels));
    mfreg_cu_grid og{};
    detail::check(mfreg_cu_register_multilevel(reference.data.data(), tpl.data.data(), &img, &mc, out.y.data(), &og,
                                               tr.data(), cap, li.data(), lsf.data(), MFREG_CU_HOST));
    out.deform_grid = from_c(og, GridKind::Nodal);
    int off = 0;
    for (int l = 0; l < cfg.levels; ++l) {
        LevelResult lr;
        std::vector<mfreg_cu_iter_record> seg(tr.begin() + off, tr.begin() + off + li[static_cast<std::size_t>(l)]);
        lr.result.trace = detail::to_trace(seg, li[static_cast<std::size_t>(l)]);
        lr.result.line_search_failed = lsf[static_cast<std::size_t>(l)] != 0;
        out.levels.push_back(std::move(lr));
        off += li[static_cast<std::size_t>(l)];
    }
    return out;
}

// ---- io.hpp (volume / deformation / landmark files; io.cpp:111-348)
namespace io {

inline Volume read_volume(const std::filesystem::path& path) {  // io.cpp:111-164
    mfreg_cu_grid g{};
    detail::check(mfreg_cu_read_volume(path.c_str(), &g, nullptr, MFREG_CU_HOST));
    Volume v{from_c(g, GridKind::CellCentered), {}};
    v.data.resize(static_cast<std::size_t>(v.grid.count()));
    detail::check(mfreg_cu_read_volume(path.c_str(), &g, v.data.data(), MFREG_CU_HOST));
    return v;
}
inline void write_volume(const std::filesystem::path& path, const Volume& v) {  // io.cpp:166-188
    const mfreg_cu_grid g = v.grid.c();
    detail::check(mfreg_cu_write_volume(path.c_str(), &g, v.data.data(), MFREG_CU_HOST));
}
inline void write_deformation(const std::filesystem::path& path, std::span<const double> y,
                              const GridDesc& grid) {  // io.cpp:200-229
    const mfreg_cu_grid g = grid.c();
    detail::check(mfreg_cu_write_deformation(path.c_str(), y.data(), static_cast<int64_t>(y.size()), &g, MFREG_CU_HOST));
}
inline GridDesc read_deformation_grid(const std::filesystem::path& path) {  // io.cpp:231-253
    mfreg_cu_grid g{};
    detail::check(mfreg_cu_read_deformation_grid(path.c_str(), &g));
    return from_c(g, GridKind::Nodal);
}
inline std::vector<double> read_deformation(const std::filesystem::path& path, const GridDesc& grid) {
    const mfreg_cu_grid g = grid.c();  // io.cpp:255-274
    std::vector<double> y(static_cast<std::size_t>(3 * grid.count()));
    detail::check(mfreg_cu_read_deformation(path.c_str(), &g, y.data(), MFREG_CU_HOST));
    return y;
}
inline std::vector<std::array<double, 3>> read_landmarks(const std::filesystem::path& path,
                                                         const std::array<double, 3>& spacing) {  // io.cpp:276-303
    int64_t n = 0;
    detail::check(mfreg_cu_read_landmarks(path.c_str(), spacing.data(), nullptr, 0, &n));
    std::vector<std::array<double, 3>> out(static_cast<std::size_t>(n));
    detail::check(mfreg_cu_read_landmarks(path.c_str(), spacing.data(), out.empty() ? nullptr : out[0].data(), n, &n));
    return out;
}
struct LandmarkStats {
    double mean = 0.0;
    double stddev = 0.0;
    std::size_t count = 0;
};
inline LandmarkStats landmark_error(const std::vector<std::array<double, 3>>& fixed,
                                    const std::vector<std::array<double, 3>>& moving, std::span<const double> y,
                                    const GridDesc& grid) {  // io.cpp:305-348
    const mfreg_cu_grid g = grid.c();
    LandmarkStats st;
    int64_t cnt = 0;
    detail::check(mfreg_cu_landmark_error(fixed.empty() ? nullptr : fixed[0].data(), static_cast<int64_t>(fixed.size()),
                                          moving.empty() ? nullptr : moving[0].data(),
                                          static_cast<int64_t>(moving.size()), y.data(), static_cast<int64_t>(y.size()),
                                          &g, MFREG_CU_HOST, &st.mean, &st.stddev, &cnt));
    st.count = static_cast<std::size_t>(cnt);
    return st;
}

}  // namespace io

}  // namespace mfreg_b200

#endif  // MFREG_B200_HPP
