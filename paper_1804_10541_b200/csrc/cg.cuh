// Device-resident CG (see cg.cu).
#pragma once

#include <vector>

#include "objective.cuh"

namespace mfreg_b200 {

struct CgState {
    double rr, pap, alpha, beta, relres, bnorm;
    double scratch;  // device result of the exact/fast dot products
    int iters, done, breakdown, pad;
};

class DeviceCg {
public:
    explicit DeviceCg(idx_t n);
    ~DeviceCg();
    DeviceCg(const DeviceCg&) = delete;
    DeviceCg& operator=(const DeviceCg&) = delete;
    // cg_solve(op, b) -> x, x0 = 0; `poll`: iterations between host checks of `done`
    CgResult solve(DeviceProblem& P, int op, double gamma, const double* b, double* x, const CgConfig& cfg,
                   int poll = 8);

private:
    // `w` CG iterations (device-side early exit once done), then the state copy to host_
    void window(DeviceProblem& P, int op, double gamma, double* x, const CgConfig& cfg, int w, bool fused_update);
    struct GraphEntry {
        const void* P;
        int op, w;
        double gamma, tol;
        double* x;
        bool fused;
        cudaGraphExec_t exec;
        long long launches;
    };
    std::vector<GraphEntry> graphs_;
    cudaStream_t cs_ = nullptr;  // capture stream (the problem's own stream may be the legacy one)
    idx_t n_;
    DVec r_, p_, ap_;
    DevArray<CgState> st_;
    DVec red_;
    DevArray<unsigned int> counter_;
    CgState* host_ = nullptr;
};

}  // namespace mfreg_b200
