// Device-resident solvers (reference optimizer.cpp:113-407) and the multilevel
// driver (multilevel.cpp:9-145). All vectors stay in HBM; only the scalars the
// reference's control flow branches on cross to the host.
#include <algorithm>
#include <cmath>
#include <deque>

#include <chrono>
#include <cstdio>
#include <cstdlib>

#include "cg.cuh"
#include "objective.cuh"

namespace mfreg_b200 {

namespace {

double effective_gamma(const OptimizerConfig& cfg, double alpha) {  // optimizer.cpp:179-181
    return cfg.gamma >= 0.0 ? cfg.gamma : 1e-3 * std::max(1.0, alpha);
}

bool should_stop(const OptimizerConfig& cfg, double g0, double min_hy, double j_prev, double j_cur, double gnorm,
                 double step_inf) {  // optimizer.cpp:188-200
    if (gnorm <= cfg.tol_grad * g0) return true;
    if (std::abs(j_prev - j_cur) <= cfg.tol_rel_j * std::max(1.0, std::abs(j_prev))) return true;
    if (step_inf <= cfg.tol_step * min_hy) return true;
    return false;
}

// MFREG_TRACE_TIME=1: per-iteration host wall split of the Gauss-Newton loop on stderr
bool trace_time() {
    static const bool on = [] {
        const char* e = std::getenv("MFREG_TRACE_TIME");
        return e && *e && *e != '0';
    }();
    return on;
}

// optimizer.cpp:156-175 with phi(eta) = J(y + eta d), value-only evaluation
bool armijo_search(DeviceProblem& P, const double* y, const double* dir, double* y_trial, double f0, double gdotd,
                   const ArmijoConfig& cfg, double eta0, double& eta_out) {
    if (!(gdotd < 0.0)) return false;
    double eta = eta0;
    for (int k = 0; k <= cfg.max_backtracks; ++k) {
        launch_axpy_to(P.dof(), y, eta, dir, y_trial, P.stream());
        const double f = P.eval(y_trial, nullptr);
        if (std::isfinite(f) && f <= f0 + cfg.c1 * eta * gdotd) {
            eta_out = eta;
            return true;
        }
        eta *= cfg.beta;
    }
    return false;
}

}  // namespace

// optimizer.cpp:113-154 — plain CG, x0 = 0, device-resident scalars (cg.cu)
CgResult cg_solve(DeviceProblem& P, int op, double gamma, const double* b, double* x, const CgConfig& cfg) {
    return P.cg_workspace().solve(P, op, gamma, b, x, cfg);
}

// optimizer.cpp:202-268 + 392-407
MinimizeResult gauss_newton_minimize(DeviceProblem& P, const double* y0, double* y, const OptimizerConfig& cfg) {
    const idx_t n = P.dof();
    cudaStream_t s = P.stream();
    MinimizeResult out;
    MFREG_CUDA(cudaMemcpyAsync(y, y0, n * sizeof(double), cudaMemcpyDeviceToDevice, s));
    if (cfg.max_iters <= 0) return out;
    DVec grad(n), dir(n), y_trial(n), b(n);
    double j = P.eval(y, grad.get());
    const double g0 = P.norm(grad.get());
    const double min_hy = P.min_spacing();
    for (int it = 0; it < cfg.max_iters; ++it) {
        IterationRecord rec;
        rec.iter = it;
        rec.j = j;
        rec.distance = P.last_distance();
        rec.regularizer = P.last_regularizer();
        rec.grad_norm = P.norm(grad.get());
        if (rec.grad_norm <= cfg.tol_grad * g0) {
            out.trace.push_back(rec);
            break;
        }
        const auto t_cg = std::chrono::steady_clock::now();
        launch_neg(n, grad.get(), b.get(), s);
        const CgResult sol = cg_solve(P, 0, 0.0, b.get(), dir.get(), cfg.cg);
        const auto t_ls = std::chrono::steady_clock::now();
        rec.cg_iters = sol.iters;
        const double gdotd = P.dot(grad.get(), dir.get());
        const double dinf = P.inf_norm(dir.get(), 1.0);
        const double eta0 = dinf > 0.0 ? std::min(1.0, P.min_spacing() / dinf) : 1.0;
        double eta = 0.0;
        if (!armijo_search(P, y, dir.get(), y_trial.get(), j, gdotd, cfg.armijo, eta0, eta)) {
            out.line_search_failed = true;
            out.trace.push_back(rec);
            break;
        }
        rec.step = eta;
        const double j_prev = j;
        launch_axpy_to(n, y, eta, dir.get(), y, s);
        const double step_inf = P.inf_norm(dir.get(), eta);
        const auto t_ev = std::chrono::steady_clock::now();
        j = P.eval(y, grad.get());
        out.trace.push_back(rec);
        if (trace_time()) {
            const auto t_end = std::chrono::steady_clock::now();
            auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
            std::fprintf(stderr, "gn it %d: cg %d iters %.2f ms, line search eta %.3g %.2f ms, eval %.2f ms\n", it,
                         sol.iters, ms(t_cg, t_ls), eta, ms(t_ls, t_ev), ms(t_ev, t_end));
        }
        if (should_stop(cfg, g0, min_hy, j_prev, j, P.norm(grad.get()), step_inf)) break;
    }
    return out;
}

// optimizer.cpp:272-390
MinimizeResult lbfgs_minimize(DeviceProblem& P, const double* y0, double* y, const OptimizerConfig& cfg) {
    const idx_t n = P.dof();
    cudaStream_t s = P.stream();
    const double gamma = effective_gamma(cfg, P.alpha());
    const int hist = std::max(1, cfg.lbfgs_history);
    MinimizeResult out;
    MFREG_CUDA(cudaMemcpyAsync(y, y0, n * sizeof(double), cudaMemcpyDeviceToDevice, s));
    if (cfg.max_iters <= 0) return out;

    // history slots: hist + 1 (one is filled before the oldest is popped)
    std::vector<DVec> S, Yv;
    for (int k = 0; k < hist + 1; ++k) {
        S.emplace_back(static_cast<std::size_t>(n));
        Yv.emplace_back(static_cast<std::size_t>(n));
    }
    struct Pair {
        int slot;
        double rho;
    };
    std::deque<Pair> history;
    auto free_slot = [&]() {
        for (int k = 0; k < hist + 1; ++k) {
            bool used = false;
            for (const auto& p : history) used |= (p.slot == k);
            if (!used) return k;
        }
        return 0;
    };

    DVec grad(n), grad_new(n), dir(n), y_trial(n), q(n), r(n);
    std::vector<double> alphas;
    double j = P.eval(y, grad.get());
    const double g0 = P.norm(grad.get());
    const double min_hy = P.min_spacing();

    for (int it = 0; it < cfg.max_iters; ++it) {
        IterationRecord rec;
        rec.iter = it;
        rec.j = j;
        rec.distance = P.last_distance();
        rec.regularizer = P.last_regularizer();
        rec.grad_norm = P.norm(grad.get());
        if (rec.grad_norm <= cfg.tol_grad * g0) {
            out.trace.push_back(rec);
            break;
        }
        // two-loop recursion, optimizer.cpp:285-312
        MFREG_CUDA(cudaMemcpyAsync(q.get(), grad.get(), n * sizeof(double), cudaMemcpyDeviceToDevice, s));
        alphas.assign(history.size(), 0.0);
        for (std::size_t k = history.size(); k-- > 0;) {
            const auto& hp = history[k];
            alphas[k] = hp.rho * P.dot(S[hp.slot].get(), q.get());
            launch_axpy_to(n, q.get(), -alphas[k], Yv[hp.slot].get(), q.get(), s);
        }
        const CgResult h0 = cg_solve(P, 1, gamma, q.get(), r.get(), cfg.h0_cg);
        for (std::size_t k = 0; k < history.size(); ++k) {
            const auto& hp = history[k];
            const double beta = hp.rho * P.dot(Yv[hp.slot].get(), r.get());
            launch_axpy_to(n, r.get(), alphas[k] - beta, S[hp.slot].get(), r.get(), s);
        }
        launch_neg(n, r.get(), dir.get(), s);
        rec.cg_iters = h0.iters;
        const double gdotd = P.dot(grad.get(), dir.get());
        const double dinf = P.inf_norm(dir.get(), 1.0);
        const double eta0 = dinf > 0.0 ? std::min(1.0, P.min_spacing() / dinf) : 1.0;
        double eta = 0.0;
        if (!armijo_search(P, y, dir.get(), y_trial.get(), j, gdotd, cfg.armijo, eta0, eta)) {
            out.line_search_failed = true;
            out.trace.push_back(rec);
            break;
        }
        rec.step = eta;
        const double j_prev = j;
        const int slot = free_slot();
        double* sv = S[slot].get();
        double* yv = Yv[slot].get();
        launch_scale_to(n, eta, dir.get(), sv, s);  // s = eta*dir
        launch_axpy_to(n, y, 1.0, sv, y, s);        // y += s (1.0*s is exact)
        const double step_inf = P.inf_norm(sv, 1.0);
        j = P.eval(y, grad_new.get());
        launch_sub(n, grad_new.get(), grad.get(), yv, s);
        const double sy = P.dot(sv, yv);
        if (sy > 1e-10 * P.norm(sv) * P.norm(yv)) {
            history.push_back({slot, 1.0 / sy});
            while (static_cast<int>(history.size()) > hist) history.pop_front();
        }
        std::swap(grad, grad_new);
        out.trace.push_back(rec);
        if (should_stop(cfg, g0, min_hy, j_prev, j, P.norm(grad.get()), step_inf)) break;
    }
    return out;
}

// multilevel.cpp:9-37 (pyramid), :117-145 (driver), :78-115 (prolong)
MultilevelResult register_multilevel(const double* R_dev, const double* T_dev, const Grid& image,
                                     const MultilevelConfig& cfg, cudaStream_t s) {
    if (cfg.levels < 1) throw std::invalid_argument("build_pyramid: levels must be >= 1");
    validate_grid(image, false);
    for (int a = 0; a < 3; ++a) {
        idx_t m = image.m[a];
        for (int l = 1; l < cfg.levels; ++l) {
            if (m < 2) throw std::invalid_argument("build_pyramid: too many levels for this size");
            m = (m + 1) / 2;
        }
        if (m < 2) throw std::invalid_argument("build_pyramid: too many levels for this size");
    }
    std::vector<Grid> G(cfg.levels);
    std::vector<DVec> R(cfg.levels), T(cfg.levels);
    G[0] = image;
    for (int l = 1; l < cfg.levels; ++l) {
        for (int a = 0; a < 3; ++a) {
            G[l].m[a] = (G[l - 1].m[a] + 1) / 2;
            G[l].h[a] = 2.0 * G[l - 1].h[a];
        }
        R[l].resize(static_cast<std::size_t>(G[l].count()));
        T[l].resize(static_cast<std::size_t>(G[l].count()));
        const double* rp = l == 1 ? R_dev : R[l - 1].get();
        const double* tp = l == 1 ? T_dev : T[l - 1].get();
        launch_downsample(G[l - 1], G[l], rp, R[l].get(), s);
        launch_downsample(G[l - 1], G[l], tp, T[l].get(), s);
    }
    check_launch("build_pyramid");
    const auto t_start = std::chrono::steady_clock::now();
    if (trace_time()) {
        MFREG_CUDA(cudaStreamSynchronize(s));
        std::fprintf(stderr, "pyramid built\n");
    }

    MultilevelResult out;
    DVec y, y0;
    Grid prev{};
    bool have_prev = false;
    auto ms_since = [](std::chrono::steady_clock::time_point t) {
        return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t).count();
    };
    auto t_prev_end = t_start;  // the previous level's objective is destroyed between its total and here
    for (int l = cfg.levels - 1; l >= 0; --l) {
        if (trace_time() && l != cfg.levels - 1)
            std::fprintf(stderr, "level %d: objective teardown %.2f ms\n", l + 1, ms_since(t_prev_end));
        const auto t_level = std::chrono::steady_clock::now();
        const Grid dg = deformation_grid_for(G[l], cfg.deform_ratio);
        const double* rp = l == 0 ? R_dev : R[l].get();
        const double* tp = l == 0 ? T_dev : T[l].get();
        DeviceObjective obj(rp, tp, G[l], dg, cfg.tau, cfg.rho, cfg.alpha, cfg.mode, s);
        if (trace_time()) {
            MFREG_CUDA(cudaStreamSynchronize(s));
            std::fprintf(stderr, "level %d: objective %.2f ms\n", l, ms_since(t_level));
        }
        y0.resize(static_cast<std::size_t>(obj.dof()));
        if (have_prev) launch_prolong(prev, dg, y.get(), y0.get(), s);
        else MFREG_CUDA(cudaMemcpyAsync(y0.get(), obj.identity_dev(), obj.dof() * sizeof(double),
                                        cudaMemcpyDeviceToDevice, s));
        check_launch("prolong");
        DVec yl(static_cast<std::size_t>(obj.dof()));
        MinimizeResult res = cfg.method == Method::Lbfgs ? lbfgs_minimize(obj, y0.get(), yl.get(), cfg.opt)
                                                         : gauss_newton_minimize(obj, y0.get(), yl.get(), cfg.opt);
        MFREG_CUDA(cudaStreamSynchronize(s));
        if (trace_time()) std::fprintf(stderr, "level %d: total %.2f ms\n", l, ms_since(t_level));
        t_prev_end = std::chrono::steady_clock::now();
        LevelResult lr{G[l], dg, std::move(res), DVec()};
        if (cfg.keep_level_y) {
            lr.y.resize(static_cast<std::size_t>(obj.dof()));
            MFREG_CUDA(cudaMemcpyAsync(lr.y.get(), yl.get(), obj.dof() * sizeof(double), cudaMemcpyDeviceToDevice, s));
        }
        y = std::move(yl);
        out.levels.push_back(std::move(lr));
        prev = dg;
        have_prev = true;
    }
    if (trace_time()) std::fprintf(stderr, "level 0: objective teardown %.2f ms\n", ms_since(t_prev_end));
    out.y = std::move(y);
    out.deform_grid = prev;
    return out;
}

}  // namespace mfreg_b200
