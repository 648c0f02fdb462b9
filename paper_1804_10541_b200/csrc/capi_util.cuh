// Helpers of the extern "C" boundary (capi.cu, capi_api.cu): exception -> status mapping,
// grid / config conversion and host <-> device staging of `where == MFREG_CU_HOST` buffers.
#pragma once

#include <string>
#include <vector>

#include "../../include/mfreg_cuda.h"
#include "objective.cuh"

namespace mfreg_b200 {
namespace capi {

// last error message of this thread (mfreg_cu_last_error)
std::string& last_error();

template <typename Fn>
int guard(Fn&& fn) {
    try {
        fn();
        return MFREG_CU_OK;
    } catch (const std::invalid_argument& e) {
        last_error() = e.what();
        return MFREG_CU_EINVAL;
    } catch (const CudaError& e) {
        last_error() = e.what();
        return MFREG_CU_ECUDA;
    } catch (const std::logic_error& e) {
        last_error() = e.what();
        return MFREG_CU_ELOGIC;
    } catch (const std::exception& e) {
        last_error() = e.what();
        return MFREG_CU_EOTHER;
    }
}

inline Grid to_grid(const mfreg_cu_grid* g) {
    if (!g) throw std::invalid_argument("null grid");
    Grid r{};
    for (int a = 0; a < 3; ++a) {
        r.m[a] = g->m[a];
        r.h[a] = g->h[a];
    }
    return r;
}
inline void from_grid(const Grid& g, mfreg_cu_grid* o) {
    for (int a = 0; a < 3; ++a) {
        o->m[a] = g.m[a];
        o->h[a] = g.h[a];
    }
}

inline void check_where(int where) {
    if (where != MFREG_CU_HOST && where != MFREG_CU_DEVICE) throw std::invalid_argument("where must be HOST or DEVICE");
}

// Read-only input: device view of a host or device array of n doubles.
// `cache`: a per-handle staging buffer reused across calls (no cudaMalloc/cudaFree
// on the per-iteration path); null = a temporary.
struct In {
    In(const double* p, std::size_t n, int where, cudaStream_t s, DVec* cache = nullptr) {
        check_where(where);
        if (where == MFREG_CU_DEVICE || !p) {
            ptr = p;
        } else {
            DVec& b = cache ? *cache : buf;
            if (b.size() < n) b.resize(n);
            MFREG_CUDA(cudaMemcpyAsync(b.get(), p, n * sizeof(double), cudaMemcpyHostToDevice, s));
            ptr = b.get();
        }
    }
    DVec buf;
    const double* ptr = nullptr;
};

// Output: device buffer written by kernels, copied back on finish() for host.
struct Out {
    Out(double* p, std::size_t n, int where, DVec* cache = nullptr) : host(p), n(n), where(where) {
        check_where(where);
        if (where == MFREG_CU_DEVICE || !p) {
            ptr = p;
        } else {
            DVec& b = cache ? *cache : buf;
            if (b.size() < n) b.resize(n);
            ptr = b.get();
        }
    }
    void finish(cudaStream_t s) {
        if (where == MFREG_CU_HOST && host) {
            MFREG_CUDA(cudaMemcpyAsync(host, ptr, n * sizeof(double), cudaMemcpyDeviceToHost, s));
            MFREG_CUDA(cudaStreamSynchronize(s));
        }
    }
    double* host;
    std::size_t n;
    int where;
    DVec buf;
    double* ptr = nullptr;
};

inline Mode to_mode(int mode) {
    if (mode != MFREG_CU_PARITY && mode != MFREG_CU_FAST && mode != MFREG_CU_FAST32)
        throw std::invalid_argument("mode must be PARITY, FAST or FAST32");
    return static_cast<Mode>(mode);
}

inline OptimizerConfig to_cfg(const mfreg_cu_opt_config* k) {
    OptimizerConfig c;
    if (!k) return c;
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

inline int copy_trace(const std::vector<IterationRecord>& t, mfreg_cu_iter_record* out, int cap) {
    int n = 0;
    for (const auto& r : t) {
        if (out && n < cap) out[n] = {r.iter, r.cg_iters, r.j, r.distance, r.regularizer, r.grad_norm, r.step};
        ++n;
    }
    return n;
}

constexpr cudaStream_t kStream = 0;  // legacy default stream: ordered with torch's default stream

}  // namespace capi
}  // namespace mfreg_b200

// opaque handles of the C ABI
struct mfreg_cu_ngf {
    mfreg_b200::Grid g;
    mfreg_b200::DVec R;
    std::unique_ptr<mfreg_b200::DeviceNgf> ngf;
};

struct mfreg_cu_objective {
    mfreg_b200::Grid img, dg;
    mfreg_b200::DVec R, T;
    std::unique_ptr<mfreg_b200::DeviceObjective> obj;
    mfreg_b200::DVec stage[4];  // host-call staging (y / p in, grad / q out), reused
};

