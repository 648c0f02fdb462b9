// Device-resident CG (see cg.cu).
#pragma once

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
    idx_t n_;
    DVec r_, p_, ap_;
    DevArray<CgState> st_;
    DVec red_;
    DevArray<unsigned int> counter_;
    CgState* host_ = nullptr;
};

}  // namespace mfreg_b200
