// Shared device-side definitions for the B200 NGF + curvature hot path.
//
// Layout: every image or nodal scalar field is a dense fp64
// array, x fastest (reference grid.hpp:63); 3-vectors are component-major
// (all x, then all y, then all z; reference ngf.cpp:75-77, transfer.cpp:70).
//
// The whole library is compiled with --fmad=false: every `a*b + c` below is a
// separately rounded multiply and add, exactly as the reference's baseline
// x86-64 build evaluates it. Kernels that are allowed to
// contract (the `fast` mode NGF Hv) call fma() explicitly.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace mfreg_b200 {

using idx_t = long long;

// Grid descriptor passed by value (reference GridDesc, grid.hpp:50-120).
struct Grid {
    idx_t m[3];
    double h[3];
    double ih[3];  // RN(1 / h), for the correctly rounded division div_rn (kernels.cu)
    __host__ __device__ idx_t count() const { return m[0] * m[1] * m[2]; }
    __host__ __device__ double cell_volume() const { return h[0] * h[1] * h[2]; }
    __host__ __device__ idx_t lin(idx_t i, idx_t j, idx_t k) const { return i + j * m[0] + k * m[0] * m[1]; }
    __host__ void set_inv() {
        for (int a = 0; a < 3; ++a) ih[a] = 1.0 / h[a];
    }
};

// Directions {-z,-y,-x,0,+x,+y,+z} (grid.hpp:16-18).
enum Dir : int { NEGZ = 0, NEGY = 1, NEGX = 2, CENTER = 3, POSX = 4, POSY = 5, POSZ = 6 };

__host__ __device__ inline int dir_axis(int d) {
    return (d == NEGX || d == POSX) ? 0 : (d == NEGY || d == POSY) ? 1 : (d == CENTER ? -1 : 2);
}
__host__ __device__ inline int dir_sign(int d) { return d < CENTER ? -1 : (d == CENTER ? 0 : 1); }
__host__ __device__ inline int dir_opp(int d) { return 6 - d; }
__host__ __device__ inline int dir_dx(int d) { return d == NEGX ? -1 : (d == POSX ? 1 : 0); }
__host__ __device__ inline int dir_dy(int d) { return d == NEGY ? -1 : (d == POSY ? 1 : 0); }
__host__ __device__ inline int dir_dz(int d) { return d == NEGZ ? -1 : (d == POSZ ? 1 : 0); }

// Device-resident grid-transfer plan (reference TransferPlan, transfer.hpp:14-20):
// per image axis index k the nodal cell base[k] and fraction rem[k], computed on
// the host bit-identically to transfer.cpp:24-35; plus, for the deterministic
// gather form of P^T, per nodal cell c the image index range [lo[c], hi[c]).
struct DevPlan {
    Grid src;  // nodal
    Grid tgt;  // cell-centred
    const int* base[3];
    const double* rem[3];
    const int* cell_lo[3];
    const int* cell_hi[3];
};

constexpr int kChunk = 4096;  // reference kReductionChunk (parallel.hpp:20)

}  // namespace mfreg_b200
