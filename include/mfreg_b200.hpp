// mfreg_b200.hpp — header-only C++ drop-in for the reference mfreg API
// (/root/reference/proj/include/mfreg/*.hpp) over the C ABI in mfreg_cuda.h.
//
// Same type names, member functions, argument meaning, defaults and exception
// types as the reference; a caller switches with
//     namespace mfreg = mfreg_b200;
// Every computation runs on the GPU through libmfreg_cuda.so: host std::span /
// std::vector arguments are staged through the C ABI, and the derivative
// evaluations, the solver loops and the multilevel driver are device-resident. Only
// descriptor arithmetic (GridDesc index math, the grouping of a transfer plan's
// slab_planes) is inline here, as it is inline in the reference's grid.hpp.
// Objective takes an extra trailing ExecMode argument: `Parity` (bitwise identical to
// the reference, the default) or `Fast` (fused kernels, max-rel <= 1e-9 per operator).
//
// Differences a caller can observe: Objective copies `reference` and
// `tpl` to the GPU at construction (the reference keeps references and re-reads them);
// the NGF kernel functions act on the device copy of the workspace made by
// populate_ngf_workspace (editing NgfWorkspace's host vectors afterwards changes nothing);
// populate_ngf_workspace requires params.rho to equal the rho the precomp was made with;
// the *_counted variants do not update the reference's operation counters (counters.hpp,
// out of scope).
#ifndef MFREG_B200_HPP
#define MFREG_B200_HPP

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdint>
#include <exception>
#include <filesystem>
#include <functional>
#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "mfreg_cuda.h"

namespace mfreg_b200 {

using index_t = std::int64_t;

// ---- grid.hpp ---------------------------------------------------------------
enum class GridKind { CellCentered, Nodal };
enum class Dir : int { NegZ = 0, NegY, NegX, Center, PosX, PosY, PosZ };
inline constexpr std::array<Dir, 7> kAllDirs = {Dir::NegZ, Dir::NegY, Dir::NegX, Dir::Center,
                                                Dir::PosX, Dir::PosY, Dir::PosZ};
inline constexpr int dir_axis(Dir d) {
    return (d == Dir::NegX || d == Dir::PosX) ? 0 : (d == Dir::NegY || d == Dir::PosY) ? 1 : (d == Dir::Center ? -1 : 2);
}
inline constexpr int dir_sign(Dir d) {
    return static_cast<int>(d) < static_cast<int>(Dir::Center) ? -1 : (d == Dir::Center ? 0 : 1);
}
inline constexpr Dir dir_opposite(Dir d) { return static_cast<Dir>(6 - static_cast<int>(d)); }

enum class ExecMode : int { Parity = MFREG_CU_PARITY, Fast = MFREG_CU_FAST };

namespace detail {
inline void check(int rc) {
    if (rc == MFREG_CU_OK) return;
    const std::string msg = mfreg_cu_last_error();
    if (rc == MFREG_CU_EINVAL) throw std::invalid_argument(msg);
    if (rc == MFREG_CU_ELOGIC) throw std::logic_error(msg);
    throw std::runtime_error(msg);
}
inline std::size_t sz(index_t n) { return static_cast<std::size_t>(n); }
}  // namespace detail

// grid.hpp:50-120
struct GridDesc {
    std::array<index_t, 3> m{1, 1, 1};
    std::array<double, 3> h{1.0, 1.0, 1.0};
    GridKind kind = GridKind::CellCentered;

    index_t count() const { return m[0] * m[1] * m[2]; }
    double cell_volume() const { return h[0] * h[1] * h[2]; }
    double extent(int axis) const {
        return kind == GridKind::CellCentered ? static_cast<double>(m[detail::sz(axis)]) * h[detail::sz(axis)]
                                              : static_cast<double>(m[detail::sz(axis)] - 1) * h[detail::sz(axis)];
    }
    index_t linear(index_t i, index_t j, index_t k) const { return i + j * m[0] + k * m[0] * m[1]; }
    std::array<index_t, 3> decompose(index_t idx) const {
        return {idx % m[0], (idx / m[0]) % m[1], idx / (m[0] * m[1])};
    }
    index_t neighbor(index_t idx, Dir d) const {  // Neumann-clamped axis neighbour
        if (d == Dir::Center) return idx;
        auto c = decompose(idx);
        const auto a = detail::sz(dir_axis(d));
        c[a] = std::clamp<index_t>(c[a] + dir_sign(d), 0, m[a] - 1);
        return linear(c[0], c[1], c[2]);
    }
    std::array<double, 3> point_coords(index_t idx) const {
        const auto c = decompose(idx);
        std::array<double, 3> p{};
        for (std::size_t a = 0; a < 3; ++a) {
            const double base = static_cast<double>(c[a]);
            p[a] = kind == GridKind::CellCentered ? (base + 0.5) * h[a] : base * h[a];
        }
        return p;
    }
    void validate() const {
        for (std::size_t a = 0; a < 3; ++a) {
            if (m[a] < 1) throw std::invalid_argument("GridDesc: all m components must be >= 1");
            if (!(h[a] > 0.0)) throw std::invalid_argument("GridDesc: all h components must be > 0");
        }
        if (kind == GridKind::Nodal)
            for (std::size_t a = 0; a < 3; ++a)
                if (m[a] < 2) throw std::invalid_argument("GridDesc: nodal grids need >= 2 points per axis");
    }
    mfreg_cu_grid c() const { return mfreg_cu_grid{{m[0], m[1], m[2]}, {h[0], h[1], h[2]}}; }
};

inline GridDesc from_c(const mfreg_cu_grid& g, GridKind kind) {
    return GridDesc{{g.m[0], g.m[1], g.m[2]}, {g.h[0], g.h[1], g.h[2]}, kind};
}

inline GridDesc make_image_grid(std::array<index_t, 3> m, std::array<double, 3> h) {  // grid.hpp:122-127
    GridDesc g{m, h, GridKind::CellCentered};
    g.validate();
    return g;
}

inline GridDesc make_deform_grid(const GridDesc& image, std::array<index_t, 3> points) {  // grid.hpp:131-146
    const mfreg_cu_grid img = image.c();
    mfreg_cu_grid out{};
    const int64_t p[3] = {points[0], points[1], points[2]};
    detail::check(mfreg_cu_make_deform_grid(&img, p, &out));
    return from_c(out, GridKind::Nodal);
}

// ---- volume.hpp ---------------------------------------------------------------
struct Volume {  // volume.hpp:13-16
    GridDesc grid;
    std::vector<double> data;
};

inline Volume make_volume(std::array<index_t, 3> m, std::array<double, 3> h, double fill = 0.0) {
    Volume v{make_image_grid(m, h), {}};
    v.data.assign(detail::sz(v.grid.count()), fill);
    return v;
}

struct InterpResult {
    double value = 0.0;
    std::array<double, 3> grad{0.0, 0.0, 0.0};
};

// T(P(y)) samples plus the diagonal entries of dT/dP (volume.hpp:33-45)
struct SampledTemplate {
    std::vector<double> values;
    std::array<std::vector<double>, 3> partials;
    void resize(index_t n) {
        values.assign(detail::sz(n), 0.0);
        for (auto& p : partials) p.assign(detail::sz(n), 0.0);
    }
};

// points: component-major (all x, all y, all z), length 3n (volume.cpp:76-94)
inline void sample_deformed(const Volume& t, std::span<const double> points, SampledTemplate& out) {
    if (points.size() % 3 != 0) throw std::invalid_argument("sample_deformed: points length must be a multiple of 3");
    const index_t n = static_cast<index_t>(points.size() / 3);
    out.resize(n);
    std::vector<double> parts(detail::sz(3 * n));
    const mfreg_cu_grid g = t.grid.c();
    detail::check(mfreg_cu_sample_deformed(&g, t.data.data(), points.data(), n, out.values.data(), parts.data(),
                                           MFREG_CU_HOST));
    for (std::size_t d = 0; d < 3; ++d)
        std::copy(parts.begin() + static_cast<std::ptrdiff_t>(d * detail::sz(n)),
                  parts.begin() + static_cast<std::ptrdiff_t>((d + 1) * detail::sz(n)), out.partials[d].begin());
}

// volume.cpp:29-74: trilinear with Dirichlet zeros, analytic gradient, ties to the lower cell
inline InterpResult interpolate(const Volume& t, const std::array<double, 3>& p) {
    SampledTemplate s;
    sample_deformed(t, p, s);  // one point: (x, y, z) is its component-major layout
    return InterpResult{s.values[0], {s.partials[0][0], s.partials[1][0], s.partials[2][0]}};
}

// volume.cpp:96-109 (backward x,y,z then forward x,y,z, clamped neighbours)
inline std::array<double, 6> discrete_gradient(std::span<const double> data, const GridDesc& g, index_t i) {
    std::array<double, 6> r{};
    const mfreg_cu_grid c = g.c();
    const int64_t idx = i;
    detail::check(mfreg_cu_discrete_gradient(&c, data.data(), &idx, 1, r.data(), MFREG_CU_HOST));
    return r;
}
inline std::array<double, 6> discrete_gradient(const Volume& v, index_t i) { return discrete_gradient(v.data, v.grid, i); }

inline double eps_norm(const std::array<double, 6>& g, double eps) {  // volume.cpp:115-121
    double out = 0.0;
    detail::check(mfreg_cu_eps_norm(g.data(), 1, eps, &out, MFREG_CU_HOST));
    return out;
}

inline Volume downsample(const Volume& v) {  // volume.cpp:123-160
    const mfreg_cu_grid g = v.grid.c();
    mfreg_cu_grid og{};
    detail::check(mfreg_cu_downsample(&g, nullptr, nullptr, &og, MFREG_CU_HOST));
    Volume out{from_c(og, GridKind::CellCentered), std::vector<double>(detail::sz(og.m[0] * og.m[1] * og.m[2]))};
    detail::check(mfreg_cu_downsample(&g, v.data.data(), out.data.data(), nullptr, MFREG_CU_HOST));
    return out;
}

// ---- transfer.hpp -----------------------------------------------------------
struct TransferPlan {  // transfer.hpp:14-20
    GridDesc source;  // nodal
    GridDesc target;  // cell-centred
    std::array<std::vector<index_t>, 3> base;
    std::array<std::vector<double>, 3> rem;
    std::vector<std::vector<index_t>> slab_planes;  // image z-planes per deformation z-slab
};

inline TransferPlan make_transfer_plan(const GridDesc& source, const GridDesc& target) {  // transfer.cpp:11-47
    if (source.kind != GridKind::Nodal || target.kind != GridKind::CellCentered)
        throw std::invalid_argument("transfer plan needs nodal source and cell-centered target");
    source.validate();
    target.validate();
    TransferPlan plan{source, target, {}, {}, {}};
    const index_t tot = target.m[0] + target.m[1] + target.m[2];
    std::vector<int64_t> b(detail::sz(tot));
    std::vector<double> r(detail::sz(tot));
    const mfreg_cu_grid s = source.c(), t = target.c();
    detail::check(mfreg_cu_transfer_plan(&s, &t, b.data(), r.data()));
    std::size_t o = 0;
    for (std::size_t a = 0; a < 3; ++a) {
        plan.base[a].assign(b.begin() + static_cast<std::ptrdiff_t>(o),
                            b.begin() + static_cast<std::ptrdiff_t>(o + detail::sz(target.m[a])));
        plan.rem[a].assign(r.begin() + static_cast<std::ptrdiff_t>(o),
                           r.begin() + static_cast<std::ptrdiff_t>(o + detail::sz(target.m[a])));
        o += detail::sz(target.m[a]);
    }
    plan.slab_planes.assign(detail::sz(source.m[2] - 1), {});
    for (index_t k = 0; k < target.m[2]; ++k) plan.slab_planes[detail::sz(plan.base[2][detail::sz(k)])].push_back(k);
    return plan;
}

inline void transfer_apply(const GridDesc& nodal, const GridDesc& image, std::span<const double> y,
                           std::span<double> out) {
    if (y.size() != detail::sz(3 * nodal.count()) || out.size() != detail::sz(3 * image.count()))
        throw std::invalid_argument("transfer_apply: length mismatch");
    const mfreg_cu_grid s = nodal.c(), t = image.c();
    detail::check(mfreg_cu_transfer_apply(&s, &t, y.data(), out.data(), MFREG_CU_HOST));
}
inline void transfer_apply(const TransferPlan& plan, std::span<const double> y, std::span<double> out) {
    transfer_apply(plan.source, plan.target, y, out);  // transfer.cpp:49-86
}

inline void transfer_apply_transpose(const GridDesc& nodal, const GridDesc& image, std::span<const double> w,
                                     std::span<double> out) {
    if (w.size() != detail::sz(3 * image.count()) || out.size() != detail::sz(3 * nodal.count()))
        throw std::invalid_argument("transfer_apply_transpose: length mismatch");
    const mfreg_cu_grid s = nodal.c(), t = image.c();
    detail::check(mfreg_cu_transfer_apply_transpose(&s, &t, w.data(), out.data(), MFREG_CU_HOST));
}
inline void transfer_apply_transpose(const TransferPlan& plan, std::span<const double> w, std::span<double> out) {
    transfer_apply_transpose(plan.source, plan.target, w, out);  // transfer.cpp:131-150
}

// ---- curvature.hpp ----------------------------------------------------------
inline double laplacian(std::span<const double> u_comp, const GridDesc& g, index_t i) {  // curvature.cpp:9-21
    if (u_comp.size() != detail::sz(g.count())) throw std::invalid_argument("laplacian_apply: length mismatch");
    const mfreg_cu_grid c = g.c();
    const int64_t idx = i;
    double v = 0.0;
    detail::check(mfreg_cu_laplacian_at(&c, u_comp.data(), &idx, 1, &v, MFREG_CU_HOST));
    return v;
}

inline void laplacian_apply(std::span<const double> u_comp, const GridDesc& g, std::span<double> out) {
    if (u_comp.size() != detail::sz(g.count()) || out.size() != u_comp.size())
        throw std::invalid_argument("laplacian_apply: length mismatch");
    const mfreg_cu_grid c = g.c();
    detail::check(mfreg_cu_laplacian_apply(&c, u_comp.data(), out.data(), MFREG_CU_HOST));
}

inline double curvature_value(std::span<const double> u, const GridDesc& g) {  // curvature.cpp:35-49
    if (u.size() != detail::sz(3 * g.count())) throw std::invalid_argument("curvature_value: length must be 3*m^y");
    const mfreg_cu_grid c = g.c();
    double v = 0.0;
    detail::check(mfreg_cu_curvature_value(&c, u.data(), &v, MFREG_CU_PARITY, MFREG_CU_HOST));
    return v;
}

namespace detail {
inline void bilap_check(std::span<const double> v, const GridDesc& g, std::span<double> scratch, std::span<double> out) {
    if (v.size() != sz(3 * g.count()) || out.size() != v.size() || scratch.size() < sz(g.count()))
        throw std::invalid_argument("curvature: buffer length mismatch");
}
}  // namespace detail

// curvature.cpp:76-84 (the device scratch replaces the caller's; `scratch` is only checked)
inline void curvature_gradient(std::span<const double> u, const GridDesc& g, std::span<double> scratch,
                               std::span<double> out) {
    detail::bilap_check(u, g, scratch, out);
    const mfreg_cu_grid c = g.c();
    detail::check(mfreg_cu_curvature_gradient(&c, u.data(), out.data(), MFREG_CU_HOST));
}
inline void curvature_hessian_vec(std::span<const double> p, const GridDesc& g, std::span<double> scratch,
                                  std::span<double> out) {
    detail::bilap_check(p, g, scratch, out);
    const mfreg_cu_grid c = g.c();
    detail::check(mfreg_cu_curvature_hessian_vec(&c, p.data(), out.data(), MFREG_CU_HOST));
}
inline std::vector<double> curvature_gradient(std::span<const double> u, const GridDesc& g) {
    std::vector<double> scratch(detail::sz(g.count())), out(u.size());
    curvature_gradient(u, g, scratch, out);
    return out;
}
inline std::vector<double> curvature_hessian_vec(std::span<const double> p, const GridDesc& g) {
    std::vector<double> scratch(detail::sz(g.count())), out(p.size());
    curvature_hessian_vec(p, g, scratch, out);
    return out;
}

// ---- ngf.hpp ------------------------------------------------------------------
struct NgfParams {  // ngf.hpp:14-17
    double tau = 10.0;
    double rho = 10.0;
};

// ngf.hpp:21-24 (+ the reference volume the device context is built from)
struct NgfPrecomp {
    std::vector<std::array<double, 6>> ref_grads;
    std::vector<double> ref_norms;
    std::shared_ptr<const Volume> reference_;
    double rho_ = 0.0;
};

inline NgfPrecomp make_ngf_precomp(const Volume& reference, double rho) {  // ngf.cpp:167-183
    NgfPrecomp pre;
    const index_t n = reference.grid.count();
    pre.ref_grads.resize(detail::sz(n));
    pre.ref_norms.resize(detail::sz(n));
    const mfreg_cu_grid g = reference.grid.c();
    detail::check(mfreg_cu_ngf_precomp(reference.data.data(), &g, rho, pre.ref_grads.data()->data(),
                                       pre.ref_norms.data(), MFREG_CU_HOST));
    pre.reference_ = std::make_shared<const Volume>(reference);
    pre.rho_ = rho;
    return pre;
}

namespace detail {
struct NgfHandle {
    mfreg_cu_ngf* h = nullptr;
    GridDesc g;
    double tau = 0.0, rho = 0.0;
    const Volume* ref = nullptr;
    ~NgfHandle() {
        if (h) mfreg_cu_ngf_destroy(h);
    }
};
}  // namespace detail

// ngf.hpp:29-37; the device copy of the workspace (ctx_) is what the NGF kernels read
struct NgfWorkspace {
    SampledTemplate sampled;
    std::vector<std::array<double, 6>> tpl_grads;
    std::vector<double> residual;
    std::vector<double> inv1;
    std::vector<double> inv2;
    std::shared_ptr<detail::NgfHandle> ctx_;
    std::vector<double> rho_hat_;  // [7][m], kAllDirs order (ngf_rho)
};

inline void populate_ngf_workspace(NgfWorkspace& ws, const Volume& tpl, std::span<const double> points,
                                   const NgfPrecomp& pre, const NgfParams& params, const GridDesc& g) {
    if (!(params.tau > 0.0) || !(params.rho > 0.0)) throw std::invalid_argument("NGF: tau and rho must be > 0");
    if (!pre.reference_) throw std::invalid_argument("NGF: precomp was not made by make_ngf_precomp");
    if (pre.rho_ != params.rho) throw std::invalid_argument("NGF: precomp rho differs from params.rho");
    const index_t n = g.count();
    if (points.size() != detail::sz(3 * n)) throw std::invalid_argument("sample_deformed: points length mismatch");
    auto& c = ws.ctx_;
    if (!c || c->ref != pre.reference_.get() || c->tau != params.tau || c->rho != params.rho || c->g.m != g.m ||
        c->g.h != g.h) {
        c = std::make_shared<detail::NgfHandle>();
        const mfreg_cu_grid gc = g.c();
        detail::check(mfreg_cu_ngf_create(pre.reference_->data.data(), &gc, params.tau, params.rho, MFREG_CU_PARITY,
                                          MFREG_CU_HOST, &c->h));
        c->g = g;
        c->tau = params.tau;
        c->rho = params.rho;
        c->ref = pre.reference_.get();
    }
    detail::check(mfreg_cu_ngf_populate(c->h, tpl.data.data(), points.data(), MFREG_CU_HOST));
    ws.sampled.resize(n);
    std::vector<double> parts(detail::sz(3 * n));
    ws.residual.resize(detail::sz(n));
    ws.inv1.resize(detail::sz(n));
    ws.inv2.resize(detail::sz(n));
    ws.rho_hat_.resize(detail::sz(7 * n));
    ws.tpl_grads.resize(detail::sz(n));
    detail::check(mfreg_cu_ngf_workspace(c->h, ws.sampled.values.data(), parts.data(), ws.residual.data(),
                                         ws.inv1.data(), ws.inv2.data(), ws.rho_hat_.data(), MFREG_CU_HOST));
    detail::check(mfreg_cu_ngf_tpl_grads(c->h, ws.tpl_grads.data()->data(), MFREG_CU_HOST));
    for (std::size_t d = 0; d < 3; ++d)
        std::copy(parts.begin() + static_cast<std::ptrdiff_t>(d * detail::sz(n)),
                  parts.begin() + static_cast<std::ptrdiff_t>((d + 1) * detail::sz(n)), ws.sampled.partials[d].begin());
}

namespace detail {
inline mfreg_cu_ngf* ngf_of(const NgfWorkspace& ws) {
    if (!ws.ctx_) throw std::invalid_argument("NGF: workspace not populated");
    return ws.ctx_->h;
}
}  // namespace detail

inline double ngf_residual(index_t i, const NgfWorkspace& ws) { return ws.residual[detail::sz(i)]; }

inline double ngf_rho(index_t i, Dir k, const NgfWorkspace& ws, const NgfPrecomp&, const GridDesc& g) {
    (void)detail::ngf_of(ws);
    return ws.rho_hat_[detail::sz(static_cast<index_t>(k) * g.count() + i)];
}

inline double ngf_value(const NgfWorkspace& ws, const GridDesc&) {  // ngf.cpp:225-231
    double v = 0.0;
    detail::check(mfreg_cu_ngf_value(detail::ngf_of(ws), &v));
    return v;
}

inline void ngf_gradient(const NgfWorkspace& ws, const NgfPrecomp&, const GridDesc& g, std::span<double> out) {
    if (out.size() != detail::sz(3 * g.count())) throw std::invalid_argument("ngf_gradient: output length must be 3*m");
    detail::check(mfreg_cu_ngf_gradient(detail::ngf_of(ws), out.data(), MFREG_CU_HOST));
}
inline void ngf_gradient_counted(const NgfWorkspace& ws, const NgfPrecomp& pre, const GridDesc& g, std::span<double> out) {
    ngf_gradient(ws, pre, g, out);
}

inline void ngf_hessian_vec(std::span<const double> p, const NgfWorkspace& ws, const NgfPrecomp&, const GridDesc& g,
                            std::span<double> out) {
    if (p.size() != detail::sz(3 * g.count()) || out.size() != p.size())
        throw std::invalid_argument("ngf_hessian_vec: vector length must be 3*m");
    detail::check(mfreg_cu_ngf_hessian_vec(detail::ngf_of(ws), p.data(), out.data(), MFREG_CU_HOST));
}
inline void ngf_hessian_vec_counted(std::span<const double> p, const NgfWorkspace& ws, const NgfPrecomp& pre,
                                    const GridDesc& g, std::span<double> out) {
    ngf_hessian_vec(p, ws, pre, g, out);
}

struct OffsetTable {  // ngf.hpp:67-85
    struct Entry {
        index_t kappa;
        std::vector<std::pair<Dir, Dir>> pairs;
    };
    std::vector<Entry> entries;
    std::size_t pair_count() const {
        std::size_t n = 0;
        for (const auto& e : entries) n += e.pairs.size();
        return n;
    }
};

inline OffsetTable make_offset_table(const GridDesc& g) {  // ngf.cpp:267-300
    int ne = 0;
    int64_t kappa[49];
    int npairs[49], pairs[98];
    const mfreg_cu_grid c = g.c();
    detail::check(mfreg_cu_offset_table(&c, &ne, kappa, npairs, pairs));
    OffsetTable t;
    int q = 0;
    for (int e = 0; e < ne; ++e) {
        OffsetTable::Entry en{kappa[e], {}};
        for (int k = 0; k < npairs[e]; ++k, ++q) en.pairs.emplace_back(static_cast<Dir>(pairs[2 * q]), static_cast<Dir>(pairs[2 * q + 1]));
        t.entries.push_back(std::move(en));
    }
    return t;
}

// ---- optimizer.hpp ----------------------------------------------------------
inline double vec_dot(std::span<const double> a, std::span<const double> b) {  // optimizer.cpp:12-19
    if (a.size() != b.size()) throw std::invalid_argument("vec_dot: length mismatch");
    double v = 0.0;
    detail::check(mfreg_cu_vec_dot(a.data(), b.data(), static_cast<int64_t>(a.size()), MFREG_CU_HOST, &v));
    return v;
}
inline double vec_norm(std::span<const double> a) { return std::sqrt(vec_dot(a, a)); }
inline double vec_inf_norm(std::span<const double> a) {
    double v = 0.0;
    detail::check(mfreg_cu_vec_inf_norm(a.data(), static_cast<int64_t>(a.size()), MFREG_CU_HOST, &v));
    return v;
}

struct IterationRecord {  // optimizer.hpp:22-30
    int iter = 0;
    double j = 0.0;
    double distance = 0.0;
    double regularizer = 0.0;
    double grad_norm = 0.0;
    double step = 0.0;
    int cg_iters = 0;
};
using IterationTrace = std::vector<IterationRecord>;

// optimizer.hpp:36-48
class Problem {
public:
    virtual ~Problem() = default;
    virtual double eval(std::span<const double> y, std::span<double> grad) = 0;
    virtual void gn_hessian_vec(std::span<const double> p, std::span<double> q) = 0;
    virtual void seed_hessian_vec(std::span<const double> p, double gamma, std::span<double> q) = 0;
    virtual double min_spacing() const = 0;
    virtual double alpha() const { return 0.0; }
    virtual double last_distance() const { return 0.0; }
    virtual double last_regularizer() const { return 0.0; }
};

// optimizer.hpp:53-106: J(y) = D_NGF(P y) + alpha S(y), evaluated on the GPU
class Objective : public Problem {
public:
    Objective(const Volume& reference, const Volume& tpl, const GridDesc& deform_grid, const NgfParams& params,
              double alpha, ExecMode mode = ExecMode::Parity)
        : ref_(reference), tpl_(tpl), image_grid_(reference.grid), deform_grid_(deform_grid), params_(params),
          alpha_(alpha) {
        deform_grid_.kind = GridKind::Nodal;
        if (tpl.grid.m != reference.grid.m) throw std::invalid_argument("Objective: image sizes differ");
        const mfreg_cu_grid img = image_grid_.c(), dg = deform_grid_.c();
        detail::check(mfreg_cu_objective_create(reference.data.data(), tpl.data.data(), &img, &dg, params.tau,
                                                params.rho, alpha, static_cast<int>(mode), MFREG_CU_HOST, &h_));
    }
    ~Objective() override {
        if (h_) mfreg_cu_objective_destroy(h_);
    }
    Objective(const Objective&) = delete;
    Objective& operator=(const Objective&) = delete;

    index_t dof() const { return 3 * deform_grid_.count(); }
    const GridDesc& image_grid() const { return image_grid_; }
    const GridDesc& deform_grid() const { return deform_grid_; }
    const NgfParams& params() const { return params_; }
    double alpha() const override { return alpha_; }
    double min_spacing() const override {
        double v = 0.0;
        detail::check(mfreg_cu_objective_min_spacing(h_, &v));
        return v;
    }
    const TransferPlan& plan() const {
        if (!plan_) plan_ = std::make_unique<TransferPlan>(make_transfer_plan(deform_grid_, image_grid_));
        return *plan_;
    }
    const NgfPrecomp& precomp() const {
        if (!pre_) pre_ = std::make_unique<NgfPrecomp>(make_ngf_precomp(ref_, params_.rho));
        return *pre_;
    }
    // the NGF workspace at the last evaluated iterate, rebuilt on the GPU from it (parity order)
    const NgfWorkspace& workspace() const {
        if (ylast_.empty()) throw std::logic_error("Objective::workspace: no evaluation yet");
        if (!ws_fresh_) {
            std::vector<double> yhat(detail::sz(3 * image_grid_.count()));
            transfer_apply(plan(), ylast_, yhat);
            populate_ngf_workspace(ws_, tpl_, yhat, precomp(), params_, image_grid_);
            ws_fresh_ = true;
        }
        return ws_;
    }
    std::vector<double> identity() const {
        std::vector<double> x(detail::sz(dof()));
        detail::check(mfreg_cu_objective_identity(h_, x.data(), MFREG_CU_HOST));
        return x;
    }
    // Evaluates J at y; fills grad if non-empty (optimizer.cpp:64-92).
    double eval(std::span<const double> y, std::span<double> grad) override {
        if (y.size() != detail::sz(dof())) throw std::invalid_argument("Objective::eval: y length mismatch");
        if (!grad.empty() && grad.size() != y.size()) throw std::invalid_argument("Objective::eval: grad length mismatch");
        double j = 0.0;
        detail::check(mfreg_cu_objective_eval(h_, y.data(), grad.empty() ? nullptr : grad.data(), MFREG_CU_HOST, &j));
        ylast_.assign(y.begin(), y.end());
        ws_fresh_ = false;
        return j;
    }
    double last_distance() const override {
        double d = 0.0, r = 0.0;
        detail::check(mfreg_cu_objective_last(h_, &d, &r));
        return d;
    }
    double last_regularizer() const override {
        double d = 0.0, r = 0.0;
        detail::check(mfreg_cu_objective_last(h_, &d, &r));
        return r;
    }
    // P^T H^ P p + alpha Hess(S) p at the last evaluated iterate (optimizer.cpp:94-104)
    void gn_hessian_vec(std::span<const double> p, std::span<double> q) override {
        if (p.size() != detail::sz(dof())) throw std::invalid_argument("transfer_apply: length mismatch");
        if (q.size() != detail::sz(dof())) throw std::invalid_argument("transfer_apply_transpose: length mismatch");
        detail::check(mfreg_cu_objective_gn_hessian_vec(h_, p.data(), q.data(), MFREG_CU_HOST));
    }
    // (Hess(S) + gamma I) p (optimizer.cpp:106-111)
    void seed_hessian_vec(std::span<const double> p, double gamma, std::span<double> q) override {
        if (p.size() != detail::sz(dof()) || q.size() != p.size())
            throw std::invalid_argument("curvature: buffer length mismatch");
        detail::check(mfreg_cu_objective_seed_hessian_vec(h_, p.data(), gamma, q.data(), MFREG_CU_HOST));
    }
    mfreg_cu_objective* handle() const { return h_; }

private:
    const Volume& ref_;
    const Volume& tpl_;
    GridDesc image_grid_, deform_grid_;
    NgfParams params_;
    double alpha_;
    mfreg_cu_objective* h_ = nullptr;
    std::vector<double> ylast_;
    mutable bool ws_fresh_ = false;
    mutable std::unique_ptr<TransferPlan> plan_;
    mutable std::unique_ptr<NgfPrecomp> pre_;
    mutable NgfWorkspace ws_;
};

struct CgConfig {
    int max_iters = 50;
    double rel_tol = 1e-2;
};
struct CgResult {
    std::vector<double> x;
    int iters = 0;
    double relres = 0.0;
    bool breakdown = false;
};
using LinearOperator = std::function<void(std::span<const double>, std::span<double>)>;

struct ArmijoConfig {
    double c1 = 1e-4;
    double beta = 0.5;
    int max_backtracks = 10;
};
struct ArmijoResult {
    double eta = 0.0;
    bool accepted = false;
    bool descent = true;
    double f_new = 0.0;
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
        return mfreg_cu_opt_config{max_iters,  armijo.c1,       armijo.beta,   armijo.max_backtracks, cg.max_iters,
                                   cg.rel_tol, h0_cg.max_iters, h0_cg.rel_tol, lbfgs_history,        gamma,
                                   tol_rel_j,  tol_grad,        tol_step};
    }
};
struct MinimizeResult {
    std::vector<double> y;
    IterationTrace trace;
    bool line_search_failed = false;
};

namespace detail {
inline IterationTrace to_trace(const mfreg_cu_iter_record* r, int n) {
    IterationTrace t;
    for (int k = 0; k < n; ++k)
        t.push_back({r[k].iter, r[k].j, r[k].distance, r[k].regularizer, r[k].grad_norm, r[k].step, r[k].cg_iters});
    return t;
}

// a host Problem behind the C callbacks; exceptions are carried across the C ABI and rethrown
struct ProblemCtx {
    Problem* p = nullptr;
    const LinearOperator* op = nullptr;
    std::size_t n = 0;
    std::exception_ptr err;
};
template <class F>
inline int guarded(void* c, F&& f) {
    auto* x = static_cast<ProblemCtx*>(c);
    try {
        f(*x);
        return 0;
    } catch (...) {
        x->err = std::current_exception();
        return 1;
    }
}
inline int cb_eval(void* c, const double* y, double* g, double* j) {
    return guarded(c, [&](ProblemCtx& x) {
        *j = x.p->eval({y, x.n}, g ? std::span<double>(g, x.n) : std::span<double>());
    });
}
inline int cb_gn(void* c, const double* p, double* q) {
    return guarded(c, [&](ProblemCtx& x) {
        if (x.op) (*x.op)({p, x.n}, {q, x.n});
        else x.p->gn_hessian_vec({p, x.n}, {q, x.n});
    });
}
inline int cb_seed(void* c, const double* p, double gamma, double* q) {
    return guarded(c, [&](ProblemCtx& x) { x.p->seed_hessian_vec({p, x.n}, gamma, {q, x.n}); });
}
template <double (Problem::*M)() const>
inline double cb_scalar(void* c) {
    auto* x = static_cast<ProblemCtx*>(c);
    try {
        return (x->p->*M)();
    } catch (...) {
        x->err = std::current_exception();
        return std::nan("");
    }
}
inline int cb_unused(void*, const double*, double*, double*) { return 1; }
inline int cb_unused_seed(void*, const double*, double, double*) { return 1; }
inline double cb_one(void*) { return 1.0; }
inline mfreg_cu_problem_ops ops_for(ProblemCtx& c) {
    if (c.op) return mfreg_cu_problem_ops{&c, cb_unused, cb_gn, cb_unused_seed, cb_one, nullptr, nullptr, nullptr};
    return mfreg_cu_problem_ops{&c,
                                cb_eval,
                                cb_gn,
                                cb_seed,
                                cb_scalar<&Problem::min_spacing>,
                                cb_scalar<&Problem::alpha>,
                                cb_scalar<&Problem::last_distance>,
                                cb_scalar<&Problem::last_regularizer>};
}
inline void finish(int rc, ProblemCtx& c) {
    if (c.err) std::rethrow_exception(c.err);
    check(rc);
}

inline MinimizeResult minimize(Problem& prob, std::span<const double> y0, const OptimizerConfig& cfg, int method) {
    MinimizeResult res;
    std::vector<mfreg_cu_iter_record> tr(sz(std::max(cfg.max_iters, 0) + 8));
    int nt = 0, lsf = 0;
    const mfreg_cu_opt_config oc = cfg.c();
    if (auto* obj = dynamic_cast<Objective*>(&prob)) {  // the registration objective: all on the GPU
        if (y0.size() != sz(obj->dof())) throw std::invalid_argument("Objective::eval: y length mismatch");
        res.y.resize(sz(obj->dof()));
        check(mfreg_cu_minimize(obj->handle(), method, y0.data(), &oc, res.y.data(), tr.data(), static_cast<int>(tr.size()),
                                &nt, &lsf, MFREG_CU_HOST));
    } else {  // any other Problem: device-resident solver loop, host operator callbacks
        ProblemCtx c{&prob, nullptr, y0.size(), nullptr};
        const mfreg_cu_problem_ops ops = ops_for(c);
        res.y.resize(y0.size());
        finish(mfreg_cu_problem_minimize(&ops, static_cast<int64_t>(y0.size()), method, y0.data(), &oc, res.y.data(),
                                         tr.data(), static_cast<int>(tr.size()), &nt, &lsf, MFREG_CU_HOST),
               c);
    }
    res.trace = to_trace(tr.data(), std::min(nt, static_cast<int>(tr.size())));
    res.line_search_failed = lsf != 0;
    return res;
}
}  // namespace detail

// optimizer.cpp:113-154: plain CG for a symmetric PSD operator, x0 = 0
inline CgResult cg_solve(const LinearOperator& apply, std::span<const double> b, const CgConfig& cfg) {
    detail::ProblemCtx c{nullptr, &apply, b.size(), nullptr};
    const mfreg_cu_problem_ops ops = detail::ops_for(c);
    CgResult r;
    r.x.resize(b.size());
    int it = 0, br = 0;
    double rr = 0.0;
    detail::finish(mfreg_cu_problem_cg_solve(&ops, static_cast<int64_t>(b.size()), 0, 0.0, b.data(), cfg.max_iters,
                                             cfg.rel_tol, r.x.data(), &it, &rr, &br, MFREG_CU_HOST),
                   c);
    r.iters = it;
    r.relres = rr;
    r.breakdown = br != 0;
    return r;
}

// optimizer.cpp:156-175
inline ArmijoResult armijo_search(const std::function<double(double)>& phi, double f0, double gdotd,
                                  const ArmijoConfig& cfg, double eta0 = 1.0) {
    struct Ctx {
        const std::function<double(double)>* phi;
        std::exception_ptr err;
    } c{&phi, nullptr};
    auto tramp = [](void* p, double eta, int* err) -> double {
        auto* x = static_cast<Ctx*>(p);
        try {
            return (*x->phi)(eta);
        } catch (...) {
            x->err = std::current_exception();
            *err = 1;
            return 0.0;
        }
    };
    ArmijoResult r;
    int acc = 0, desc = 1;
    const int rc = mfreg_cu_armijo_search(tramp, &c, f0, gdotd, cfg.c1, cfg.beta, cfg.max_backtracks, eta0, &r.eta, &acc,
                                          &desc, &r.f_new);
    if (c.err) std::rethrow_exception(c.err);
    detail::check(rc);
    r.accepted = acc != 0;
    r.descent = desc != 0;
    return r;
}

inline MinimizeResult lbfgs_minimize(Problem& obj, std::span<const double> y0, const OptimizerConfig& cfg) {
    return detail::minimize(obj, y0, cfg, MFREG_CU_LBFGS);
}
inline MinimizeResult gauss_newton_minimize(Problem& obj, std::span<const double> y0, const OptimizerConfig& cfg) {
    return detail::minimize(obj, y0, cfg, MFREG_CU_GAUSS_NEWTON);
}

// ---- multilevel.hpp -----------------------------------------------------------
struct LevelImages {
    Volume reference;
    Volume tpl;
};

// multilevel.cpp:9-37 (block-mean halving on the GPU)
inline std::vector<LevelImages> build_pyramid(const Volume& reference, const Volume& tpl, int levels) {
    if (levels < 1) throw std::invalid_argument("build_pyramid: levels must be >= 1");
    for (std::size_t a = 0; a < 3; ++a) {
        if (reference.grid.m[a] != tpl.grid.m[a]) throw std::invalid_argument("build_pyramid: image sizes differ");
        index_t m = reference.grid.m[a];
        for (int l = 1; l < levels; ++l) {
            if (m < 2) throw std::invalid_argument("build_pyramid: too many levels for this size");
            m = (m + 1) / 2;
        }
        if (m < 2) throw std::invalid_argument("build_pyramid: too many levels for this size");
    }
    std::vector<LevelImages> out;
    out.push_back({reference, tpl});
    for (int l = 1; l < levels; ++l) out.push_back({downsample(out.back().reference), downsample(out.back().tpl)});
    return out;
}

inline GridDesc deformation_grid_for(const GridDesc& image, index_t ratio) {  // multilevel.cpp:39-49
    const mfreg_cu_grid img = image.c();
    mfreg_cu_grid out{};
    detail::check(mfreg_cu_deformation_grid_for(&img, ratio, &out));
    return from_c(out, GridKind::Nodal);
}

inline double nodal_interpolate(std::span<const double> comp, const GridDesc& g, const std::array<double, 3>& p) {
    if (comp.size() != detail::sz(g.count())) throw std::invalid_argument("nodal_interpolate: length mismatch");
    const mfreg_cu_grid c = g.c();
    double v = 0.0;
    detail::check(mfreg_cu_nodal_interpolate(&c, comp.data(), p.data(), 1, &v, MFREG_CU_HOST));
    return v;
}

inline std::vector<double> prolong(std::span<const double> y_coarse, const GridDesc& coarse, const GridDesc& fine) {
    if (y_coarse.size() != detail::sz(3 * coarse.count())) throw std::invalid_argument("prolong: field length mismatch");
    std::vector<double> out(detail::sz(3 * fine.count()));
    const mfreg_cu_grid c = coarse.c(), f = fine.c();
    detail::check(mfreg_cu_prolong(&c, &f, y_coarse.data(), out.data(), MFREG_CU_HOST));
    return out;
}

enum class Method { Lbfgs, GaussNewton };
struct MultilevelConfig {  // multilevel.hpp:38-45 (+ execution mode)
    int levels = 3;
    index_t deform_ratio = 4;
    NgfParams ngf{};
    double alpha = 1.0;
    Method method = Method::Lbfgs;
    OptimizerConfig opt{};
    ExecMode mode = ExecMode::Parity;
};
struct LevelResult {  // multilevel.hpp:47-51
    GridDesc image_grid;
    GridDesc deform_grid;
    MinimizeResult result;
};
struct MultilevelResult {
    std::vector<double> y;
    GridDesc deform_grid;
    std::vector<LevelResult> levels;  // coarsest first
};

// multilevel.cpp:117-145: pyramid, per-level solve and prolongation all on the GPU
inline MultilevelResult register_multilevel(const Volume& reference, const Volume& tpl, const MultilevelConfig& cfg) {
    if (reference.grid.m != tpl.grid.m) throw std::invalid_argument("build_pyramid: image sizes differ");
    if (cfg.levels < 1) throw std::invalid_argument("build_pyramid: levels must be >= 1");
    const GridDesc dg = deformation_grid_for(reference.grid, cfg.deform_ratio);
    MultilevelResult out;
    out.y.resize(detail::sz(3 * dg.count()));
    const mfreg_cu_grid img = reference.grid.c();
    const mfreg_cu_ml_config mc{cfg.levels,
                                cfg.deform_ratio,
                                cfg.ngf.tau,
                                cfg.ngf.rho,
                                cfg.alpha,
                                cfg.method == Method::GaussNewton ? MFREG_CU_GAUSS_NEWTON : MFREG_CU_LBFGS,
                                static_cast<int>(cfg.mode),
                                cfg.opt.c()};
    const std::size_t L = detail::sz(cfg.levels);
    const int cap = cfg.levels * (std::max(cfg.opt.max_iters, 0) + 2) + 8;
    std::vector<mfreg_cu_iter_record> tr(detail::sz(cap));
    std::vector<int> li(L), lsf(L);
    std::vector<mfreg_cu_grid> gi(L), gd(L);
    // every level's deformation: coarse levels are 1/8 the size of the next, so <= 8/7 of the finest
    index_t ycap = 0;
    {
        GridDesc g = reference.grid;
        for (std::size_t l = 0; l < L; ++l) {
            ycap += 3 * deformation_grid_for(g, cfg.deform_ratio).count();
            for (std::size_t a = 0; a < 3; ++a) {
                g.m[a] = (g.m[a] + 1) / 2;
                g.h[a] *= 2.0;
            }
            if (std::min({g.m[0], g.m[1], g.m[2]}) < 1) break;
        }
    }
    std::vector<double> ly(detail::sz(ycap));
    mfreg_cu_grid og{};
    detail::check(mfreg_cu_register_multilevel_ex(reference.data.data(), tpl.data.data(), &img, &mc, out.y.data(), &og,
                                                  tr.data(), cap, li.data(), lsf.data(), gi.data(), gd.data(),
                                                  ly.data(), ycap, MFREG_CU_HOST));
    out.deform_grid = from_c(og, GridKind::Nodal);
    int off = 0;
    std::size_t yoff = 0;
    for (std::size_t l = 0; l < L; ++l) {
        LevelResult lr;
        lr.image_grid = from_c(gi[l], GridKind::CellCentered);
        lr.deform_grid = from_c(gd[l], GridKind::Nodal);
        lr.result.trace = detail::to_trace(tr.data() + std::min(off, cap), std::min(li[l], cap - std::min(off, cap)));
        lr.result.line_search_failed = lsf[l] != 0;
        const std::size_t ny = detail::sz(3 * lr.deform_grid.count());
        lr.result.y.assign(ly.begin() + static_cast<std::ptrdiff_t>(yoff), ly.begin() + static_cast<std::ptrdiff_t>(yoff + ny));
        yoff += ny;
        out.levels.push_back(std::move(lr));
        off += li[l];
    }
    return out;
}

// ---- io.hpp (volume / deformation / landmark files; io.cpp:111-348)
namespace io {

inline Volume read_volume(const std::filesystem::path& path) {  // io.cpp:111-164
    mfreg_cu_grid g{};
    detail::check(mfreg_cu_read_volume(path.c_str(), &g, nullptr, MFREG_CU_HOST));
    Volume v{from_c(g, GridKind::CellCentered), {}};
    v.data.resize(detail::sz(v.grid.count()));
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
    std::vector<double> y(detail::sz(3 * grid.count()));
    detail::check(mfreg_cu_read_deformation(path.c_str(), &g, y.data(), MFREG_CU_HOST));
    return y;
}
inline std::vector<std::array<double, 3>> read_landmarks(const std::filesystem::path& path,
                                                         const std::array<double, 3>& spacing) {  // io.cpp:276-303
    int64_t n = 0;
    detail::check(mfreg_cu_read_landmarks(path.c_str(), spacing.data(), nullptr, 0, &n));
    std::vector<std::array<double, 3>> out(detail::sz(n));
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
