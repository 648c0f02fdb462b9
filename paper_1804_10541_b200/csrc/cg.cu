// Device-resident conjugate gradients (reference cg_solve, optimizer.cpp:113-154).
//
// The CG scalars live in device memory (CgState). Single-thread kernels apply the
// reference's scalar logic in the same IEEE operations and order (breakdown on a
// non-finite or non-positive <p,Ap>, relres = sqrt(rr_new)/||b||, stop at
// relres <= tol, beta = rr_new/rr); vector kernels become no-ops once `done` is
// set, so the host only polls `done` every few iterations instead of reading
// two scalars per iteration.
#include <cmath>

#include "cg.cuh"

namespace mfreg_b200 {

namespace {

__global__ void k_cg_init(CgState* st, const double* dotbb) {
    // bnorm = vec_norm(b); rr = vec_dot(r, r) with r = b (the same reduction)
    st->rr = *dotbb;
    st->bnorm = sqrt(*dotbb);
    st->iters = 0;
    st->relres = 0.0;
    st->breakdown = 0;
    st->done = st->bnorm == 0.0 ? 1 : 0;
}

__global__ void k_cg_alpha(CgState* st) {
    if (st->done) return;
    const double pap = st->pap;
    if (!isfinite(pap) || pap <= 0.0) {  // optimizer.cpp:127-131
        st->breakdown = !isfinite(pap) ? 1 : 0;
        st->done = 1;
        return;
    }
    st->alpha = st->rr / pap;
}

__global__ void k_cg_update_xr(long long n, const double* __restrict__ p, const double* __restrict__ ap,
                               double* __restrict__ x, double* __restrict__ r, const CgState* st) {
    if (st->done) return;
    const double alpha = st->alpha;
    const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) {
        x[i] += alpha * p[i];
        r[i] -= alpha * ap[i];
    }
}

__device__ __forceinline__ void cg_beta_logic(CgState* st, double rr_new, double tol) {
    st->iters += 1;  // optimizer.cpp:137-150
    st->relres = sqrt(rr_new) / st->bnorm;
    if (!isfinite(rr_new)) {
        st->breakdown = 1;
        st->done = 1;
        return;
    }
    if (st->relres <= tol) {
        st->done = 1;
        return;
    }
    st->beta = rr_new / st->rr;
    st->rr = rr_new;
}

__global__ void k_cg_beta(CgState* st, const double* rr_new, double tol) {
    if (st->done) return;
    cg_beta_logic(st, *rr_new, tol);
}

__global__ void k_cg_update_p(long long n, const double* __restrict__ r, double* __restrict__ p, const CgState* st) {
    if (st->done) return;
    const double beta = st->beta;
    const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) p[i] = r[i] + beta * p[i];
}

// fast mode: x += alpha p, r -= alpha Ap and <r, r> in one pass (fixed-order tree,
// last block applies the beta logic)
constexpr int UPD_THREADS = 256;
constexpr int kTicketGroups = 32;
__global__ void __launch_bounds__(UPD_THREADS) k_cg_update_fused(long long n, const double* __restrict__ p,
                                                                 const double* __restrict__ ap, double* __restrict__ x,
                                                                 double* __restrict__ r, CgState* st, double* red,
                                                                 unsigned int* counter, double tol) {
    __shared__ double sh[32];
    __shared__ bool last;
    if (st->done) return;  // uniform: every block sees the same flag (set only by a previous launch)
    // k_cg_alpha folded in: every block applies the same test to the same <p, Ap>
    const double pap = st->pap;
    if (!isfinite(pap) || pap <= 0.0) {  // optimizer.cpp:127-131
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            st->breakdown = !isfinite(pap) ? 1 : 0;
            st->done = 1;
        }
        return;
    }
    const double alpha = st->rr / pap;
    if (blockIdx.x == 0 && threadIdx.x == 0) st->alpha = alpha;
    double acc = 0.0;
    for (long long i = static_cast<long long>(blockIdx.x) * UPD_THREADS + threadIdx.x; i < n;
         i += static_cast<long long>(gridDim.x) * UPD_THREADS) {
        x[i] += alpha * p[i];
        const double ri = r[i] - alpha * ap[i];
        r[i] = ri;
        acc = fma(ri, ri, acc);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x < 32) {
        double v = threadIdx.x < (UPD_THREADS >> 5) ? sh[threadIdx.x] : 0.0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
        if (threadIdx.x == 0) {
            red[blockIdx.x] = v;
            __threadfence();
            // two-level completion ticket (group counters, then the top one): avoids ~10^3
            // same-address atomics per launch
            const unsigned g = blockIdx.x % kTicketGroups, ng = min(gridDim.x, static_cast<unsigned>(kTicketGroups));
            const unsigned gsize = (gridDim.x - g + kTicketGroups - 1) / kTicketGroups;
            bool lst = false;
            if (atomicAdd(counter + 1 + g, 1u) == gsize - 1) {
                counter[1 + g] = 0u;
                __threadfence();
                lst = atomicAdd(counter, 1u) == ng - 1;
            }
            last = lst;
        }
    }
    __syncthreads();
    if (!last || threadIdx.x >= 32) return;
    __threadfence();
    double v = 0.0;
    for (unsigned b = threadIdx.x; b < gridDim.x; b += 32) v += red[b];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if (threadIdx.x == 0) {
        *counter = 0u;
        cg_beta_logic(st, v, tol);
    }
}

// small systems (coarse pyramid levels): the whole CG update in one block — alpha test,
// x += alpha p, r -= alpha Ap, <r, r> (fixed-order block tree), the beta logic and
// p = r + beta p — one launch instead of three
constexpr int SMALL_THREADS = 1024;
constexpr long long kSmallN = 4 * 1024;
__global__ void __launch_bounds__(SMALL_THREADS) k_cg_step_small(long long n, double* __restrict__ p,
                                                                 const double* __restrict__ ap, double* __restrict__ x,
                                                                 double* __restrict__ r, CgState* st, double tol) {
    __shared__ double sh[32];
    __shared__ int go;
    if (st->done) return;
    const double pap = st->pap;
    if (!isfinite(pap) || pap <= 0.0) {
        if (threadIdx.x == 0) {
            st->breakdown = !isfinite(pap) ? 1 : 0;
            st->done = 1;
        }
        return;
    }
    const double alpha = st->rr / pap;
    double acc = 0.0;
    for (long long i = threadIdx.x; i < n; i += SMALL_THREADS) {
        x[i] += alpha * p[i];
        const double ri = r[i] - alpha * ap[i];
        r[i] = ri;
        acc = fma(ri, ri, acc);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x < 32) {
        double v = sh[threadIdx.x];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
        if (threadIdx.x == 0) {
            st->alpha = alpha;
            cg_beta_logic(st, v, tol);
            go = st->done ? 0 : 1;
        }
    }
    __syncthreads();
    if (!go) return;
    const double beta = st->beta;
    for (long long i = threadIdx.x; i < n; i += SMALL_THREADS) p[i] = r[i] + beta * p[i];
}

inline unsigned blocks_for(long long n, int t = 256) { return static_cast<unsigned>((n + t - 1) / t); }

}  // namespace

DeviceCg::DeviceCg(idx_t n) : n_(n), r_(n), p_(n), ap_(n), st_(1), red_(1024), counter_(1 + kTicketGroups) {
    static_assert(sizeof(CgState) <= kPinnedSmall, "CG state block");
    host_ = static_cast<CgState*>(pinned_small_alloc(sizeof(CgState)));
    MFREG_CUDA(cudaMemset(counter_.get(), 0, (1 + kTicketGroups) * sizeof(unsigned int)));
}

DeviceCg::~DeviceCg() {
    for (auto& g : graphs_)
        if (g.exec) cudaGraphExecDestroy(g.exec);
    if (cs_) cudaStreamDestroy(cs_);
    pinned_small_free(host_);
}

void DeviceCg::window(DeviceProblem& P, int op, double gamma, double* x, const CgConfig& cfg, int w,
                      bool fused_update) {
    const idx_t n = n_;
    cudaStream_t s = P.stream();
    CgState* st = st_.get();
    double* scal = reinterpret_cast<double*>(&st->scratch);
    const unsigned ub = static_cast<unsigned>(std::min<long long>(blocks_for(n, UPD_THREADS), 1024));
    for (int j = 0; j < w; ++j) {
        P.apply_dot(op, gamma, p_.get(), ap_.get(), &st->pap, &st->done);
        if (fused_update && n <= kSmallN) {
            note_launch(), k_cg_step_small<<<1, SMALL_THREADS, 0, s>>>(n, p_.get(), ap_.get(), x, r_.get(), st,
                                                                       cfg.rel_tol);
            continue;
        }
        if (fused_update) {
            note_launch(), k_cg_update_fused<<<ub, UPD_THREADS, 0, s>>>(n, p_.get(), ap_.get(), x, r_.get(), st,
                                                                        red_.get(), counter_.get(), cfg.rel_tol);
        } else {
            note_launch(), k_cg_alpha<<<1, 1, 0, s>>>(st);
            note_launch(), k_cg_update_xr<<<blocks_for(n), 256, 0, s>>>(n, p_.get(), ap_.get(), x, r_.get(), st);
            P.dot_async(r_.get(), r_.get(), scal);
            note_launch(), k_cg_beta<<<1, 1, 0, s>>>(st, scal, cfg.rel_tol);
        }
        note_launch(), k_cg_update_p<<<blocks_for(n), 256, 0, s>>>(n, r_.get(), p_.get(), st);
    }
    MFREG_CUDA(cudaMemcpyAsync(host_, st, sizeof(CgState), cudaMemcpyDeviceToHost, s));
}

CgResult DeviceCg::solve(DeviceProblem& P, int op, double gamma, const double* b, double* x, const CgConfig& cfg,
                         int poll) {
    const idx_t n = n_;
    cudaStream_t s = P.stream();
    CgState* st = st_.get();
    P.prepare_operator();  // outside any capture: the window graphs replay the operator as is
    MFREG_CUDA(cudaMemsetAsync(x, 0, n * sizeof(double), s));
    MFREG_CUDA(cudaMemcpyAsync(r_.get(), b, n * sizeof(double), cudaMemcpyDeviceToDevice, s));
    MFREG_CUDA(cudaMemcpyAsync(p_.get(), b, n * sizeof(double), cudaMemcpyDeviceToDevice, s));
    MFREG_CUDA(cudaMemsetAsync(ap_.get(), 0, n * sizeof(double), s));
    double* scal = reinterpret_cast<double*>(&st->scratch);
    P.dot_async(b, b, scal);
    note_launch(), k_cg_init<<<1, 1, 0, s>>>(st, scal);
    const bool fused_update = P.fast_reductions();
    // Windows of `poll` iterations between host checks of `done`. When the problem allows it
    // each window replays one CUDA graph (captured on first use per operator / x / window
    // length): the small per-iteration kernels then cost no host launch time, which is what
    // bounds CG on the coarse pyramid levels.
    const bool graphs = P.cg_graphable();
    if (cfg.max_iters <= 0) MFREG_CUDA(cudaMemcpyAsync(host_, st, sizeof(CgState), cudaMemcpyDeviceToHost, s));
    for (int it = 0; it < cfg.max_iters;) {
        const int w = std::min(poll, cfg.max_iters - it);
        if (it > 0) {
            MFREG_CUDA(cudaStreamSynchronize(s));
            if (host_->done) break;
        }
        if (!graphs) {
            window(P, op, gamma, x, cfg, w, fused_update);
        } else {
            GraphEntry* e = nullptr;
            for (auto& g : graphs_)
                if (g.P == &P && g.op == op && g.w == w && g.gamma == gamma && g.tol == cfg.rel_tol && g.x == x &&
                    g.fused == fused_update)
                    e = &g;
            if (!e) {
                if (!cs_) MFREG_CUDA(cudaStreamCreateWithFlags(&cs_, cudaStreamNonBlocking));
                const long long l0 = launch_counter();
                MFREG_CUDA(cudaStreamBeginCapture(cs_, cudaStreamCaptureModeRelaxed));
                P.redirect_stream(cs_);
                GraphCache::capturing() = true;
                try {
                    window(P, op, gamma, x, cfg, w, fused_update);
                } catch (...) {
                    GraphCache::capturing() = false;
                    P.redirect_stream(s);
                    cudaGraph_t g = nullptr;
                    cudaStreamEndCapture(cs_, &g);
                    if (g) cudaGraphDestroy(g);
                    cudaGetLastError();
                    throw;
                }
                GraphCache::capturing() = false;
                P.redirect_stream(s);
                cudaGraph_t g = nullptr;
                MFREG_CUDA(cudaStreamEndCapture(cs_, &g));
                cudaGraphExec_t ex = nullptr;
                const cudaError_t err = cudaGraphInstantiate(&ex, g, 0);
                cudaGraphDestroy(g);
                MFREG_CUDA(err);
                const long long nl = launch_counter() - l0;
                note_launches(-nl);  // counted on every replay instead
                if (graphs_.size() >= 8) {
                    cudaGraphExecDestroy(graphs_.front().exec);
                    graphs_.erase(graphs_.begin());
                }
                graphs_.push_back(GraphEntry{&P, op, w, gamma, cfg.rel_tol, x, fused_update, ex, nl});
                e = &graphs_.back();
            }
            MFREG_CUDA(cudaGraphLaunch(e->exec, s));
            note_launches(e->launches);
        }
        it += w;
    }
    check_launch("cg_solve (device)");
    MFREG_CUDA(cudaStreamSynchronize(s));
    CgResult res;
    res.iters = host_->iters;
    res.relres = host_->relres;
    res.breakdown = host_->breakdown != 0;
    return res;
}

}  // namespace mfreg_b200
