// sm_100a kernels for the NGF + curvature matrix-free derivative path.
// Compiled with --fmad=false (see common.cuh): every expression below keeps the
// reference's operation order and rounding so `parity` results are bitwise
// identical to the CPU reference.
#include <cstdlib>
#include <algorithm>
#include <atomic>
#include <cmath>
#include <map>
#include <vector>

#include "kernels.cuh"

namespace mfreg_b200 {

namespace {

constexpr int BX = 64, BY = 4;

inline dim3 grid3(const Grid& g) {
    return dim3(static_cast<unsigned>((g.m[0] + BX - 1) / BX), static_cast<unsigned>((g.m[1] + BY - 1) / BY),
                static_cast<unsigned>(g.m[2]));
}
inline dim3 block3() { return dim3(BX, BY, 1); }

inline unsigned blocks1(idx_t n, int t = 256) { return static_cast<unsigned>(std::max<idx_t>(1, (n + t - 1) / t)); }

__device__ __forceinline__ bool coords(const Grid& g, idx_t& x, idx_t& y, idx_t& z, int zoff = 0) {
    x = static_cast<idx_t>(blockIdx.x) * BX + threadIdx.x;
    y = static_cast<idx_t>(blockIdx.y) * BY + threadIdx.y;
    z = static_cast<idx_t>(blockIdx.z) + zoff;  // z window [zoff, zoff + gridDim.z) (parity z slabs)
    return x < g.m[0] && y < g.m[1];
}

__device__ __forceinline__ idx_t clampi(idx_t v, idx_t hi) { return v < 0 ? 0 : (v > hi ? hi : v); }

// volume.cpp:19-25
__device__ __forceinline__ double sample_or_zero(const double* __restrict__ t, const Grid& g, idx_t i, idx_t j,
                                                 idx_t k) {
    if (i < 0 || j < 0 || k < 0 || i >= g.m[0] || j >= g.m[1] || k >= g.m[2]) return 0.0;
    return __ldg(&t[g.lin(i, j, k)]);
}

// Correctly rounded p / h from the correctly rounded reciprocal ih = RN(1/h)
// (Markstein's correction: q0 = RN(p ih), r = p - q0 h exactly by FMA,
// q = RN(q0 + r ih)); identical to IEEE division, ~4x cheaper than __ddiv_rn.
// A zero quotient keeps the sign of p, as IEEE division does.
__device__ __forceinline__ double div_rn(double p, double h, double ih) {
    const double q0 = __dmul_rn(p, ih);
    const double r = __fma_rn(-q0, h, p);
    const double q = __fma_rn(r, ih, q0);
    return q == 0.0 ? q0 : q;
}

// volume.cpp:29-74 — trilinear sample with Dirichlet zeros; ties go to the lower
// cell (ceil(s)-1); IEEE division p/h (a reciprocal multiply flips ties).
__device__ __forceinline__ void interpolate(const double* __restrict__ t, const Grid& g, double px, double py,
                                            double pz, double& value, double& gx, double& gy, double& gz) {
    const double p[3] = {px, py, pz};
    idx_t base[3];
    double f[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        const double s = div_rn(p[a], g.h[a], g.ih[a]) - 0.5;
        const double c = ceil(s);
        base[a] = static_cast<idx_t>(c) - 1;
        f[a] = s - static_cast<double>(base[a]);
    }
    double v[2][2][2];
#pragma unroll
    for (int gg = 0; gg < 2; ++gg)
#pragma unroll
        for (int b = 0; b < 2; ++b)
#pragma unroll
            for (int a = 0; a < 2; ++a) v[gg][b][a] = sample_or_zero(t, g, base[0] + a, base[1] + b, base[2] + gg);
    const double fx = f[0], fy = f[1], fz = f[2];
    double cx[2][2], dx[2][2];
#pragma unroll
    for (int gg = 0; gg < 2; ++gg)
#pragma unroll
        for (int b = 0; b < 2; ++b) {
            cx[gg][b] = v[gg][b][0] * (1.0 - fx) + v[gg][b][1] * fx;
            dx[gg][b] = v[gg][b][1] - v[gg][b][0];
        }
    double cy[2], dyv[2], dxv[2];
#pragma unroll
    for (int gg = 0; gg < 2; ++gg) {
        cy[gg] = cx[gg][0] * (1.0 - fy) + cx[gg][1] * fy;
        dyv[gg] = cx[gg][1] - cx[gg][0];
        dxv[gg] = dx[gg][0] * (1.0 - fy) + dx[gg][1] * fy;
    }
    value = cy[0] * (1.0 - fz) + cy[1] * fz;
    const double ggx = dxv[0] * (1.0 - fz) + dxv[1] * fz;
    const double ggy = dyv[0] * (1.0 - fz) + dyv[1] * fz;
    const double ggz = cy[1] - cy[0];
    gx = div_rn(ggx, g.h[0], g.ih[0]);
    gy = div_rn(ggy, g.h[1], g.ih[1]);
    gz = div_rn(ggz, g.h[2], g.ih[2]);
}

// transfer.cpp:56-83 — acc += ((wx*wy)*wz)*y over corners in (g,b,a) order from 0.0
__device__ __forceinline__ void transfer_point(const DevPlan& P, const double* __restrict__ y, idx_t x, idx_t yy,
                                               idx_t z, double out[3]) {
    const idx_t bx = P.base[0][x], by = P.base[1][yy], bz = P.base[2][z];
    const double rx = P.rem[0][x], ry = P.rem[1][yy], rz = P.rem[2][z];
    const double wx[2] = {1.0 - rx, rx}, wy[2] = {1.0 - ry, ry}, wz[2] = {1.0 - rz, rz};
    const idx_t ns = P.src.count();
    const idx_t sm0 = P.src.m[0], sm01 = P.src.m[0] * P.src.m[1];
#pragma unroll
    for (int d = 0; d < 3; ++d) {
        const double* yd = y + d * ns;
        double acc = 0.0;
#pragma unroll
        for (int g = 0; g < 2; ++g)
#pragma unroll
            for (int b = 0; b < 2; ++b)
#pragma unroll
                for (int a = 0; a < 2; ++a) {
                    const idx_t src = (bx + a) + (by + b) * sm0 + (bz + g) * sm01;
                    acc += wx[a] * wy[b] * wz[g] * __ldg(&yd[src]);
                }
        out[d] = acc;
    }
}

__global__ void k_transfer_apply(DevPlan P, const double* __restrict__ y, double* __restrict__ out) {
    idx_t x, yy, z;
    if (!coords(P.tgt, x, yy, z)) return;
    double v[3];
    transfer_point(P, y, x, yy, z, v);
    const idx_t n = P.tgt.count(), i = P.tgt.lin(x, yy, z);
    out[i] = v[0];
    out[n + i] = v[1];
    out[2 * n + i] = v[2];
}

__global__ void k_warp(DevPlan P, const double* __restrict__ y, const double* __restrict__ T, double* __restrict__ Tw,
                       double* __restrict__ dT, int zoff) {
    idx_t x, yy, z;
    if (!coords(P.tgt, x, yy, z)) return;
    z += zoff;  // image-plane window (z slabs)
    double v[3];
    transfer_point(P, y, x, yy, z, v);
    double val, gx, gy, gz;
    interpolate(T, P.tgt, v[0], v[1], v[2], val, gx, gy, gz);
    const idx_t n = P.tgt.count(), i = P.tgt.lin(x, yy, z);
    Tw[i] = val;
    dT[i] = gx;
    dT[n + i] = gy;
    dT[2 * n + i] = gz;
}

// fast mode warp: the same P y (transfer.cpp:56-83 operation order, corner weights
// shared by the three components) and the same cell choice as the reference
// (IEEE p/h via div_rn, ties to the lower cell: at the identity every sample sits
// on a tie, and the one-sided gradient there depends on that choice), then the
// trilinear value / gradient with fused arithmetic (continuous in the cell
// fraction, so contraction only moves the last bits).
// (OutT = float: the FAST32 state; the cell choice and P y stay exact fp64)
// 6 resident blocks (48 warps) per SM: the kernel is global-load latency bound (two levels
// of dependent gathers, nodal y then the template), so occupancy beats registers — measured
// 40 regs / 6 blocks: -18% at 128^3, -25% at 512x512x256 against 48 regs / 5 blocks; 7 blocks
// spill (slower)
#ifndef MFREG_WARP_MINB
#define MFREG_WARP_MINB 6
#endif
// trilinear T at the sample point pt (the reference's cell choice) and its analytic
// gradient, stored at image index (x, yy, z); shared by the two fast warp kernels
// EXACT_S = false: the sample coordinate p/h - 0.5 as one FMA with the reciprocal (callers
// guarantee the point is not within 1e-9 of a cell face, so the cell is the reference's)
template <typename OutT, bool EXACT_S = true>
__device__ __forceinline__ void warp_sample_store(const DevPlan& P, const double* __restrict__ T, const double pt[3],
                                                  int x, int yy, int z, int mx, int my, int mz,
                                                  OutT* __restrict__ Tw, OutT* __restrict__ dT) {
    const int m3[3] = {mx, my, mz};
    int i0[3];
    double f[3];
    bool ok0[3], ok1[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        const double sa = EXACT_S ? div_rn(pt[a], P.tgt.h[a], P.tgt.ih[a]) - 0.5 : fma(pt[a], P.tgt.ih[a], -0.5);
        const double c = fmin(fmax(ceil(sa), -4.0), static_cast<double>(m3[a]) + 4.0);  // far outside: all zero
        const int b0 = static_cast<int>(c) - 1;
        f[a] = sa - static_cast<double>(static_cast<long long>(ceil(sa)) - 1);
        ok0[a] = b0 >= 0 && b0 < m3[a];
        ok1[a] = b0 + 1 >= 0 && b0 + 1 < m3[a];
        i0[a] = b0;
    }
    const int plane = mx * my;
    double t[2][2][2];
    const double* tr[2][2];
    tr[0][0] = T + (i0[0] + i0[1] * mx + i0[2] * plane);
    tr[0][1] = tr[0][0] + mx;
    tr[1][0] = tr[0][0] + plane;
    tr[1][1] = tr[1][0] + mx;
#pragma unroll
    for (int g = 0; g < 2; ++g)
#pragma unroll
        for (int b = 0; b < 2; ++b)
#pragma unroll
            for (int a = 0; a < 2; ++a) {
                const bool ok = (a ? ok1[0] : ok0[0]) && (b ? ok1[1] : ok0[1]) && (g ? ok1[2] : ok0[2]);
                t[g][b][a] = ok ? __ldg(tr[g][b] + a) : 0.0;
            }
    const double fx = f[0], fy = f[1], fz = f[2];
    double cx[2][2], dx[2][2];
#pragma unroll
    for (int g = 0; g < 2; ++g)
#pragma unroll
        for (int b = 0; b < 2; ++b) {
            dx[g][b] = t[g][b][1] - t[g][b][0];
            cx[g][b] = fma(fx, dx[g][b], t[g][b][0]);
        }
    double cy[2], dyv[2], dxv[2];
#pragma unroll
    for (int g = 0; g < 2; ++g) {
        dyv[g] = cx[g][1] - cx[g][0];
        cy[g] = fma(fy, dyv[g], cx[g][0]);
        dxv[g] = fma(fy, dx[g][1] - dx[g][0], dx[g][0]);
    }
    const double gzv = cy[1] - cy[0];
    const long long i = x + static_cast<long long>(yy) * mx + static_cast<long long>(z) * plane,
                    n = static_cast<long long>(plane) * mz;
    Tw[i] = static_cast<OutT>(fma(fz, gzv, cy[0]));
    if (dT == nullptr) return;  // value-only evaluation: the Hv state is refreshed lazily
    dT[i] = static_cast<OutT>(fma(fz, dxv[1] - dxv[0], dxv[0]) * P.tgt.ih[0]);
    dT[n + i] = static_cast<OutT>(fma(fz, dyv[1] - dyv[0], dyv[0]) * P.tgt.ih[1]);
    dT[2 * n + i] = static_cast<OutT>(gzv * P.tgt.ih[2]);
}

// Fast-P-y sample (k_warp_z, points not within 1e-9 of a cell face): the caller has the sample
// coordinate sa = p/h - 0.5 (FMA with the reciprocal), c = ceil(sa) and f = sa - (c - 1) (exactly
// the fraction warp_sample_store forms through an integer round trip). Interior cells (every tap
// inside the volume: all but a boundary shell) take 8 unpredicated loads from one base index;
// boundary cells the per-tap zero fill. Same arithmetic as warp_sample_store, bitwise.
template <typename OutT>
__device__ __forceinline__ void warp_sample_store_c(const DevPlan& P, const double* __restrict__ T, const double c[3],
                                                    const double f[3], int mx, int my, int mz, long long i, long long n,
                                                    OutT* __restrict__ Tw, OutT* __restrict__ dT) {
    const int m3[3] = {mx, my, mz};
    int b[3];
    bool inner = true;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        // (saturating conversion, then the clamp of warp_sample_store: far outside is all zero)
        b[a] = min(max(__double2int_rz(c[a]), -4), m3[a] + 4) - 1;
        inner = inner && static_cast<unsigned>(b[a]) < static_cast<unsigned>(m3[a] - 1);
    }
    const int plane = mx * my;
    double t[2][2][2];
    if (inner) {
        const double* t0 = T + (b[0] + b[1] * mx + b[2] * plane);
        const double* t1 = t0 + plane;
        t[0][0][0] = __ldg(t0);
        t[0][0][1] = __ldg(t0 + 1);
        t[0][1][0] = __ldg(t0 + mx);
        t[0][1][1] = __ldg(t0 + mx + 1);
        t[1][0][0] = __ldg(t1);
        t[1][0][1] = __ldg(t1 + 1);
        t[1][1][0] = __ldg(t1 + mx);
        t[1][1][1] = __ldg(t1 + mx + 1);
    } else {
#pragma unroll
        for (int g = 0; g < 2; ++g)
#pragma unroll
            for (int bb = 0; bb < 2; ++bb)
#pragma unroll
                for (int a = 0; a < 2; ++a) {
                    const int ix = b[0] + a, iy = b[1] + bb, iz = b[2] + g;
                    const bool ok = ix >= 0 && ix < mx && iy >= 0 && iy < my && iz >= 0 && iz < mz;
                    t[g][bb][a] = ok ? __ldg(T + (ix + iy * mx + static_cast<long long>(iz) * plane)) : 0.0;
                }
    }
    const double fx = f[0], fy = f[1], fz = f[2];
    double cx[2][2], dx[2][2];
#pragma unroll
    for (int g = 0; g < 2; ++g)
#pragma unroll
        for (int bb = 0; bb < 2; ++bb) {
            dx[g][bb] = t[g][bb][1] - t[g][bb][0];
            cx[g][bb] = fma(fx, dx[g][bb], t[g][bb][0]);
        }
    double cy[2], dyv[2], dxv[2];
#pragma unroll
    for (int g = 0; g < 2; ++g) {
        dyv[g] = cx[g][1] - cx[g][0];
        cy[g] = fma(fy, dyv[g], cx[g][0]);
        dxv[g] = fma(fy, dx[g][1] - dx[g][0], dx[g][0]);
    }
    const double gzv = cy[1] - cy[0];
    Tw[i] = static_cast<OutT>(fma(fz, gzv, cy[0]));
    if (dT == nullptr) return;
    dT[i] = static_cast<OutT>(fma(fz, dxv[1] - dxv[0], dxv[0]) * P.tgt.ih[0]);
    dT[n + i] = static_cast<OutT>(fma(fz, dyv[1] - dyv[0], dyv[0]) * P.tgt.ih[1]);
    dT[2 * n + i] = static_cast<OutT>(gzv * P.tgt.ih[2]);
}

__global__ void k_sample(Grid g, const double* __restrict__ T, const double* __restrict__ pts, idx_t n,
                         double* __restrict__ vals, double* __restrict__ dT) {
    const idx_t i = static_cast<idx_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double val, gx, gy, gz;
    interpolate(T, g, pts[i], pts[n + i], pts[2 * n + i], val, gx, gy, gz);
    vals[i] = val;
    dT[i] = gx;
    dT[n + i] = gy;
    dT[2 * n + i] = gz;
}

// transfer.cpp:92-150 as a per-node gather in the reference's exact accumulation
// order: odd deformation z-slab first, then even; inside a slab image planes,
// rows, columns ascending; each term ((wx*wy)*wz)*v. Deterministic, no atomics.
__global__ void k_transfer_T(DevPlan P, const double* __restrict__ w, double* __restrict__ out, int zoff) {
    idx_t nx, ny, nz;
    if (!coords(P.src, nx, ny, nz, zoff)) return;
    const idx_t nt = P.tgt.count(), ns = P.src.count();
    const idx_t tm0 = P.tgt.m[0], tm01 = P.tgt.m[0] * P.tgt.m[1];
    const idx_t ncx = P.src.m[0] - 1, ncy = P.src.m[1] - 1, ncz = P.src.m[2] - 1;
    double a0 = 0.0, a1 = 0.0, a2 = 0.0;
    // slab order: the odd one of {nz-1, nz} first (phase 0), then the even one
    idx_t slabs[2];
    int ns_ = 0;
    const idx_t s_lo = nz - 1, s_hi = nz;
    if (s_lo >= 0 && (s_lo & 1)) slabs[ns_++] = s_lo;
    if (s_hi < ncz && (s_hi & 1)) slabs[ns_++] = s_hi;
    if (s_lo >= 0 && !(s_lo & 1)) slabs[ns_++] = s_lo;
    if (s_hi < ncz && !(s_hi & 1)) slabs[ns_++] = s_hi;
    for (int si = 0; si < ns_; ++si) {
        const idx_t sl = slabs[si];
        const bool gz1 = (sl == nz - 1);
        for (idx_t kz = P.cell_lo[2][sl]; kz < P.cell_hi[2][sl]; ++kz) {
            const double rz = P.rem[2][kz];
            const double wz = gz1 ? rz : 1.0 - rz;
            for (int cyi = 0; cyi < 2; ++cyi) {
                const idx_t cy = ny - 1 + cyi;  // cell ny-1 (b=1) precedes cell ny (b=0)
                if (cy < 0 || cy >= ncy) continue;
                const bool b1 = (cyi == 0);
                for (idx_t ky = P.cell_lo[1][cy]; ky < P.cell_hi[1][cy]; ++ky) {
                    const double ry = P.rem[1][ky];
                    const double wy = b1 ? ry : 1.0 - ry;
                    for (int cxi = 0; cxi < 2; ++cxi) {
                        const idx_t cx = nx - 1 + cxi;
                        if (cx < 0 || cx >= ncx) continue;
                        const bool ax1 = (cxi == 0);
                        for (idx_t kx = P.cell_lo[0][cx]; kx < P.cell_hi[0][cx]; ++kx) {
                            const double rx = P.rem[0][kx];
                            const double wx = ax1 ? rx : 1.0 - rx;
                            const double wgt = wx * wy * wz;
                            const idx_t ti = kx + ky * tm0 + kz * tm01;
                            a0 += wgt * __ldg(&w[ti]);
                            a1 += wgt * __ldg(&w[nt + ti]);
                            a2 += wgt * __ldg(&w[2 * nt + ti]);
                        }
                    }
                }
            }
        }
    }
    const idx_t o = P.src.lin(nx, ny, nz);
    out[o] = a0;
    out[ns + o] = a1;
    out[2 * ns + o] = a2;
}

// volume.cpp:115-121
__device__ __forceinline__ double eps_norm6(const double g[6], double eps) {
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < 6; ++k) s += g[k] * g[k];
    return sqrt(0.5 * s + eps * eps);
}

// volume.cpp:96-109 — backward x,y,z then forward x,y,z with clamped neighbours
__device__ __forceinline__ void dgrad6(const double* __restrict__ v, const Grid& g, idx_t x, idx_t y, idx_t z,
                                       double r[6]) {
    const idx_t i = g.lin(x, y, z);
    const double vi = __ldg(&v[i]);
    const idx_t nb[6] = {g.lin(clampi(x - 1, g.m[0] - 1), y, z), g.lin(x, clampi(y - 1, g.m[1] - 1), z),
                         g.lin(x, y, clampi(z - 1, g.m[2] - 1)), g.lin(clampi(x + 1, g.m[0] - 1), y, z),
                         g.lin(x, clampi(y + 1, g.m[1] - 1), z), g.lin(x, y, clampi(z + 1, g.m[2] - 1))};
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        r[a] = div_rn(vi - __ldg(&v[nb[a]]), g.h[a], g.ih[a]);
        r[a + 3] = div_rn(__ldg(&v[nb[a + 3]]) - vi, g.h[a], g.ih[a]);
    }
}

// ngf.cpp:185-214 (workspace) fused with ngf.cpp:39-64 (rho-hat for all 7
// directions, stored direction-major rh[k*n+i]); rho-hat(0) summed over kAllDirs.
__global__ void k_ngf_ws(Grid g, const double* __restrict__ R, const double* __restrict__ Tw, double tau, double rho,
                         double* __restrict__ r, double* __restrict__ inv1o, double* __restrict__ inv2o,
                         double* __restrict__ rh, int zoff) {
    idx_t x, y, z;
    if (!coords(g, x, y, z, zoff)) return;
    const idx_t n = g.count(), i = g.lin(x, y, z);
    double gt[6], gr[6];
    dgrad6(Tw, g, x, y, z, gt);
    dgrad6(R, g, x, y, z, gr);
    const double tn = eps_norm6(gt, tau);
    const double rn = eps_norm6(gr, rho);
    double num = tau * rho;
#pragma unroll
    for (int c = 0; c < 6; ++c) num += 0.5 * gt[c] * gr[c];
    const double in1 = __ddiv_rn(1.0, tn * rn);
    const double in2 = __ddiv_rn(num, tn * tn * tn * rn);
    r[i] = num * in1;
    if (inv1o) inv1o[i] = in1;
    if (inv2o) inv2o[i] = in2;
    double hh[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) hh[a] = __ddiv_rn(1.0, 2.0 * g.h[a] * g.h[a]);
    double center = 0.0;
#pragma unroll
    for (int k = 0; k < 7; ++k) {
        if (k == CENTER) continue;
        const int a = dir_axis(k), sgn = dir_sign(k);
        const int comp = sgn > 0 ? a + 3 : a;
        const double h = g.h[a];
        const double dR = static_cast<double>(sgn) * h * gr[comp];
        const double dTv = static_cast<double>(sgn) * h * gt[comp];
        const double v = hh[a] * (dR * in1 - dTv * in2);
        rh[k * n + i] = v;
        center -= v;
    }
    rh[CENTER * n + i] = center;
}

// ngf.cpp:66-103 (Alg. 4.1): acc = sum_k r_{i+k} rho-hat_{i+k}(-k), kAllDirs order;
// out_d = (-2 h_bar * acc) * dT_d. 3-D neighbours: wrapped linear neighbours of the
// reference contribute exact zeros (clamped rho-hat), so skipping them is bitwise neutral.
__global__ void k_ngf_gradient(Grid g, double scale, const double* __restrict__ r, const double* __restrict__ rh,
                               const double* __restrict__ dT, double* __restrict__ out, int zoff) {
    idx_t x, y, z;
    if (!coords(g, x, y, z, zoff)) return;
    const idx_t n = g.count(), i = g.lin(x, y, z);
    double acc = 0.0;
#pragma unroll
    for (int k = 0; k < 7; ++k) {
        const idx_t jx = x + dir_dx(k), jy = y + dir_dy(k), jz = z + dir_dz(k);
        if (jx < 0 || jy < 0 || jz < 0 || jx >= g.m[0] || jy >= g.m[1] || jz >= g.m[2]) continue;
        const idx_t j = g.lin(jx, jy, jz);
        acc += __ldg(&r[j]) * __ldg(&rh[dir_opp(k) * n + j]);
    }
    const double s = scale * acc;
    out[i] = s * dT[i];
    out[n + i] = s * dT[n + i];
    out[2 * n + i] = s * dT[2 * n + i];
}

__global__ void k_Pp_s(DevPlan P, const double* __restrict__ p, const double* __restrict__ dT,
                       double* __restrict__ sv, int zoff) {
    idx_t x, yy, z;
    if (!coords(P.tgt, x, yy, z, zoff)) return;
    double v[3];
    transfer_point(P, p, x, yy, z, v);
    const idx_t n = P.tgt.count(), i = P.tgt.lin(x, yy, z);
    sv[i] = dT[i] * v[0] + dT[n + i] * v[1] + dT[2 * n + i] * v[2];
}

// ngf.cpp:105-163 (Alg. 4.2) bit-identical: entries by ascending kappa, pairs in
// (da, db) insertion order, drdr accumulated from 0.0, c = drdr * s, q += c * dT_i.
__global__ void k_hv_closed(Grid g, HvTable tab, double scale, const double* __restrict__ rh,
                            const double* __restrict__ sv, const double* __restrict__ dT, double* __restrict__ out,
                            int zoff) {
    idx_t x, y, z;
    if (!coords(g, x, y, z, zoff)) return;
    const idx_t n = g.count(), i = g.lin(x, y, z);
    double qx = 0.0, qy = 0.0, qz = 0.0;
    const double d0 = dT[i], d1 = dT[n + i], d2 = dT[2 * n + i];
    for (int e = 0; e < tab.ngroups; ++e) {
        const idx_t tx = x + tab.dx[e], ty = y + tab.dy[e], tz = z + tab.dz[e];
        if (tx < 0 || ty < 0 || tz < 0 || tx >= g.m[0] || ty >= g.m[1] || tz >= g.m[2]) continue;
        double drdr = 0.0;
        for (int q = 0; q < tab.npairs[e]; ++q) {
            const int da = tab.pa[e][q], db = tab.pb[e][q];
            const idx_t ux = x + dir_dx(db), uy = y + dir_dy(db), uz = z + dir_dz(db);
            if (ux < 0 || uy < 0 || uz < 0 || ux >= g.m[0] || uy >= g.m[1] || uz >= g.m[2]) continue;
            const idx_t t = g.lin(ux, uy, uz);
            drdr += __ldg(&rh[dir_opp(da) * n + t]) * __ldg(&rh[dir_opp(db) * n + t]);
        }
        const double c = drdr * __ldg(&sv[g.lin(tx, ty, tz)]);
        qx += c * d0;
        qy += c * d1;
        qz += c * d2;
    }
    out[i] = scale * qx;
    out[n + i] = scale * qy;
    out[2 * n + i] = scale * qz;
}

// The offset table of every grid with m_x, m_y >= 5 (kappa order = lexicographic (dz, dy, dx)
// order of the 25 3-D offsets), built at compile time so the closed-form Hv below runs with
// immediate offsets and fully unrolled group / pair loops; make_hv_table() output is compared
// with it on the host and the generic kernel serves every other grid.
struct CanonHvTable {
    int ngroups;
    int dx[25], dy[25], dz[25], npairs[25], pa[25][7], pb[25][7];
};
constexpr int cdx(int d) { return d == NEGX ? -1 : (d == POSX ? 1 : 0); }
constexpr int cdy(int d) { return d == NEGY ? -1 : (d == POSY ? 1 : 0); }
constexpr int cdz(int d) { return d == NEGZ ? -1 : (d == POSZ ? 1 : 0); }
constexpr CanonHvTable make_canon_hv_table() {
    CanonHvTable t{};
    long long kap[25] = {};
    int ng = 0;
    for (int da = 0; da < 7; ++da)
        for (int db = 0; db < 7; ++db) {
            const int dx = cdx(db) - cdx(da), dy = cdy(db) - cdy(da), dz = cdz(db) - cdz(da);
            int e = 0;
            while (e < ng && !(t.dx[e] == dx && t.dy[e] == dy && t.dz[e] == dz)) ++e;
            if (e == ng) {
                t.dx[e] = dx;
                t.dy[e] = dy;
                t.dz[e] = dz;
                kap[e] = dx + 1000LL * dy + 1000000LL * dz;
                ++ng;
            }
            t.pa[e][t.npairs[e]] = da;
            t.pb[e][t.npairs[e]] = db;
            ++t.npairs[e];
        }
    t.ngroups = ng;
    for (int i = 1; i < ng; ++i)  // stable insertion sort by kappa (std::stable_sort in make_hv_table)
        for (int j = i; j > 0 && kap[j] < kap[j - 1]; --j) {
            const long long tk = kap[j]; kap[j] = kap[j - 1]; kap[j - 1] = tk;
            int v = t.dx[j]; t.dx[j] = t.dx[j - 1]; t.dx[j - 1] = v;
            v = t.dy[j]; t.dy[j] = t.dy[j - 1]; t.dy[j - 1] = v;
            v = t.dz[j]; t.dz[j] = t.dz[j - 1]; t.dz[j - 1] = v;
            v = t.npairs[j]; t.npairs[j] = t.npairs[j - 1]; t.npairs[j - 1] = v;
            for (int q = 0; q < 7; ++q) {
                v = t.pa[j][q]; t.pa[j][q] = t.pa[j - 1][q]; t.pa[j - 1][q] = v;
                v = t.pb[j][q]; t.pb[j][q] = t.pb[j - 1][q]; t.pb[j - 1][q] = v;
            }
        }
    return t;
}
constexpr CanonHvTable kCanonHv = make_canon_hv_table();

bool is_canon_hv_table(const HvTable& t) {
    if (t.ngroups != kCanonHv.ngroups) return false;
    for (int e = 0; e < t.ngroups; ++e) {
        if (t.dx[e] != kCanonHv.dx[e] || t.dy[e] != kCanonHv.dy[e] || t.dz[e] != kCanonHv.dz[e] ||
            t.npairs[e] != kCanonHv.npairs[e])
            return false;
        for (int q = 0; q < t.npairs[e]; ++q)
            if (t.pa[e][q] != kCanonHv.pa[e][q] || t.pb[e][q] != kCanonHv.pb[e][q]) return false;
    }
    return true;
}

// k_hv_closed with the compile-time table: same groups, pairs, bounds tests and operation
// order per voxel (bitwise the generic kernel); the group and pair loops are unrolled by
// template recursion so every table entry is an immediate
struct CanonCtx {
    long long i, n, pl;
    int x, y, z, mx, my, mz;
    bool ok[7];
    long long off[7];
    const double* __restrict__ rh;
    const double* __restrict__ sv;
};

template <int E, int Q>
__device__ __forceinline__ void canon_pairs(const CanonCtx& c, double& drdr) {
    if constexpr (Q < kCanonHv.npairs[E]) {
        constexpr int da = kCanonHv.pa[E][Q], db = kCanonHv.pb[E][Q];
        if (c.ok[db]) {
            const long long t = c.i + c.off[db];
            drdr += __ldg(&c.rh[(6 - da) * c.n + t]) * __ldg(&c.rh[(6 - db) * c.n + t]);
        }
        canon_pairs<E, Q + 1>(c, drdr);
    }
}

template <int E>
__device__ __forceinline__ void canon_group(const CanonCtx& c, double d0, double d1, double d2, double& qx, double& qy,
                                            double& qz) {
    if constexpr (E < kCanonHv.ngroups) {
        constexpr int DX = kCanonHv.dx[E], DY = kCanonHv.dy[E], DZ = kCanonHv.dz[E];
        const int tx = c.x + DX, ty = c.y + DY, tz = c.z + DZ;
        if (!(tx < 0 || ty < 0 || tz < 0 || tx >= c.mx || ty >= c.my || tz >= c.mz)) {
            double drdr = 0.0;
            canon_pairs<E, 0>(c, drdr);
            const double cc = drdr * __ldg(&c.sv[c.i + DX + static_cast<long long>(DY) * c.mx + DZ * c.pl]);
            qx += cc * d0;
            qy += cc * d1;
            qz += cc * d2;
        }
        canon_group<E + 1>(c, d0, d1, d2, qx, qy, qz);
    }
}

__global__ void __launch_bounds__(BX * BY) k_hv_closed_canon(Grid g, double scale, const double* __restrict__ rh,
                                                             const double* __restrict__ sv,
                                                             const double* __restrict__ dT, double* __restrict__ out,
                                                             int zoff) {
    CanonCtx c;
    c.x = static_cast<int>(blockIdx.x) * BX + threadIdx.x;
    c.y = static_cast<int>(blockIdx.y) * BY + threadIdx.y;
    c.z = static_cast<int>(blockIdx.z) + zoff;
    c.mx = static_cast<int>(g.m[0]);
    c.my = static_cast<int>(g.m[1]);
    c.mz = static_cast<int>(g.m[2]);
    if (c.x >= c.mx || c.y >= c.my) return;
    c.pl = static_cast<long long>(c.mx) * c.my;
    c.n = c.pl * c.mz;
    c.i = c.x + static_cast<long long>(c.y) * c.mx + c.z * c.pl;
    c.rh = rh;
    c.sv = sv;
#pragma unroll
    for (int d = 0; d < 7; ++d) {
        const int ux = c.x + cdx(d), uy = c.y + cdy(d), uz = c.z + cdz(d);
        c.ok[d] = ux >= 0 && uy >= 0 && uz >= 0 && ux < c.mx && uy < c.my && uz < c.mz;
        c.off[d] = cdx(d) + static_cast<long long>(cdy(d)) * c.mx + cdz(d) * c.pl;
    }
    const long long i = c.i, n = c.n;
    double qx = 0.0, qy = 0.0, qz = 0.0;
    const double d0 = dT[i], d1 = dT[n + i], d2 = dT[2 * n + i];
    canon_group<0>(c, d0, d1, d2, qx, qy, qz);
    out[i] = scale * qx;
    out[n + i] = scale * qy;
    out[2 * n + i] = scale * qz;
}

// fast mode, pass 1: w_t = (dr s)_t = sum_k rho-hat_t(k) s_{t+k}
__global__ void k_hv_w(Grid g, const double* __restrict__ rh, const double* __restrict__ sv, double* __restrict__ w) {
    idx_t x, y, z;
    if (!coords(g, x, y, z)) return;
    const idx_t n = g.count(), i = g.lin(x, y, z);
    double acc = 0.0;
#pragma unroll
    for (int k = 0; k < 7; ++k) {
        const idx_t jx = x + dir_dx(k), jy = y + dir_dy(k), jz = z + dir_dz(k);
        if (jx < 0 || jy < 0 || jz < 0 || jx >= g.m[0] || jy >= g.m[1] || jz >= g.m[2]) continue;
        acc = fma(__ldg(&rh[k * n + i]), __ldg(&sv[g.lin(jx, jy, jz)]), acc);
    }
    w[i] = acc;
}

// fast mode, pass 2: z_i = (dr^T w)_i = sum_k rho-hat_{i+k}(-k) w_{i+k}; q_d = 2h z dT_d
__global__ void k_hv_z(Grid g, double scale, const double* __restrict__ rh, const double* __restrict__ w,
                       const double* __restrict__ dT, double* __restrict__ out) {
    idx_t x, y, z;
    if (!coords(g, x, y, z)) return;
    const idx_t n = g.count(), i = g.lin(x, y, z);
    double acc = 0.0;
#pragma unroll
    for (int k = 0; k < 7; ++k) {
        const idx_t jx = x + dir_dx(k), jy = y + dir_dy(k), jz = z + dir_dz(k);
        if (jx < 0 || jy < 0 || jz < 0 || jx >= g.m[0] || jy >= g.m[1] || jz >= g.m[2]) continue;
        const idx_t j = g.lin(jx, jy, jz);
        acc = fma(__ldg(&rh[dir_opp(k) * n + j]), __ldg(&w[j]), acc);
    }
    const double s = scale * acc;
    out[i] = s * dT[i];
    out[n + i] = s * dT[n + i];
    out[2 * n + i] = s * dT[2 * n + i];
}

__device__ __forceinline__ double sum_term(int kind, const double* __restrict__ a, const double* __restrict__ b,
                                           idx_t i) {
    const double x = __ldg(&a[i]);
    if (kind == SUM_ONE_MINUS_SQ) return 1.0 - x * x;
    if (kind == SUM_DOT) return x * __ldg(&b[i]);
    return x * x;
}

// parallel.cpp:51-73: per 4096-element chunk, the sequential partial sum. One warp per chunk:
// the lanes evaluate the chunk's terms with coalesced loads into shared memory, then lane 0
// adds them in index order (bitwise the reference's loop: the terms do not depend on the
// order, the additions are sequential). One thread per chunk left all but a few SMs idle and
// read 32 scattered lines per warp load (0.59 ms at 128^3).
template <int KIND>  // the term kind as a template parameter: branch-free batched term loads
__global__ void __launch_bounds__(32) k_chunks_warp(idx_t n, const double* __restrict__ a,
                                                    const double* __restrict__ b, double* __restrict__ partials,
                                                    idx_t nseg_chunks = 0) {
    extern __shared__ double terms[];  // [kChunk]
    idx_t c = blockIdx.x;
    if (nseg_chunks) {  // segmented: block -> (segment d, chunk c) over arrays a + d n (3 components at once)
        const idx_t d = c / nseg_chunks;
        c -= d * nseg_chunks;
        a += d * n;
        if (b) b += d * n;
        partials += d * nseg_chunks;
    }
    const idx_t lo = c * kChunk, hi = min(n, lo + kChunk);
    const int cnt = static_cast<int>(hi - lo), lane = threadIdx.x;
#pragma unroll 16
    for (int i = lane; i < cnt; i += 32) terms[i] = sum_term(KIND, a, b, lo + i);
    __syncwarp();
    if (lane != 0) return;
    double s = 0.0;
#pragma unroll 16
    for (int i = 0; i < cnt; ++i) s += terms[i];
    partials[c] = s;
}

// three segments' partials, each combined in chunk order by its own thread
__global__ void k_serial3(const double* __restrict__ partials, idx_t nch, double scale, double* __restrict__ out) {
    const int d = threadIdx.x;
    if (d >= 3) return;
    double t = 0.0;
    for (idx_t c = 0; c < nch; ++c) t += partials[d * nch + c];
    out[d] = scale * t;
}

// partials combined in chunk order (parallel.cpp:69-72), times `scale` (ngf.cpp:227)
__global__ void k_serial(const double* __restrict__ partials, idx_t nch, double scale, double* __restrict__ out) {
    if (threadIdx.x != 0) return;
    double t = 0.0;
    for (idx_t c = 0; c < nch; ++c) t += partials[c];
    *out = scale * t;
}

constexpr int kTreeThreads = 256;
constexpr int kTreePerThread = 16;
constexpr idx_t kTreeSpan = static_cast<idx_t>(kTreeThreads) * kTreePerThread;

__device__ __forceinline__ double block_sum(double v) {
    __shared__ double sh[32];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (lane == 0) sh[wid] = v;
    __syncthreads();
    v = (threadIdx.x < (blockDim.x >> 5)) ? sh[threadIdx.x] : 0.0;
    if (wid == 0) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    }
    return v;
}

__global__ void k_tree_partials(int kind, idx_t n, const double* __restrict__ a, const double* __restrict__ b,
                                double* __restrict__ partials) {
    const idx_t base = static_cast<idx_t>(blockIdx.x) * kTreeSpan;
    double s = 0.0;
#pragma unroll 4
    for (int k = 0; k < kTreePerThread; ++k) {
        const idx_t i = base + static_cast<idx_t>(k) * kTreeThreads + threadIdx.x;
        if (i < n) s += sum_term(kind, a, b, i);
    }
    s = block_sum(s);
    if (threadIdx.x == 0) partials[blockIdx.x] = s;
}

__global__ void k_tree_final(const double* __restrict__ partials, idx_t nb, double scale, double* __restrict__ out) {
    double s = 0.0;
    for (idx_t k = threadIdx.x; k < nb; k += blockDim.x) s += partials[k];
    s = block_sum(s);
    if (threadIdx.x == 0) *out = scale * s;
}

__global__ void k_inf_norm_init(double* out) { *out = 0.0; }

__global__ void k_inf_norm(idx_t n, const double* __restrict__ a, double scale, unsigned long long* out) {
    double m = 0.0;
    for (idx_t i = static_cast<idx_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<idx_t>(gridDim.x) * blockDim.x) {
        const double v = fabs(scale * a[i]);
        m = (m < v) ? v : m;  // NaN never wins, as std::max(m, |x|)
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const double v = __shfl_down_sync(0xffffffffu, m, o);
        m = (m < v) ? v : m;
    }
    if ((threadIdx.x & 31) == 0 && m > 0.0) atomicMax(out, static_cast<unsigned long long>(__double_as_longlong(m)));
}

// curvature.cpp:9-21 — ((u- - 2u) + u+) / (h*h) summed over x, y, z from 0.0.
// The quotient by h*h is the IEEE division; when every h*h is a power of two (the usual
// unit image spacing and power-of-two deformation ratios) the multiply by its exact
// reciprocal is the same correctly rounded value and replaces the division (P2).
struct LapGeo {
    int mx, my, mz, pn;
    double hh[3];   // RN(h*h) as the reference forms it
    double ihh[3];  // 1 / hh, exact when P2
};

template <bool P2>
__device__ __forceinline__ double lap_div(double v, double hh, double ihh) {
    if constexpr (P2) return v * ihh;
    else return v / hh;
}

template <bool P2>
__device__ __forceinline__ double lap_at(const double* __restrict__ u, const LapGeo& g, int x, int y, int z, int i) {
    const double ui = __ldg(&u[i]);
    const int ox0 = x > 0 ? 1 : 0, ox1 = x < g.mx - 1 ? 1 : 0;
    const int oy0 = y > 0 ? g.mx : 0, oy1 = y < g.my - 1 ? g.mx : 0;
    const int oz0 = z > 0 ? g.pn : 0, oz1 = z < g.mz - 1 ? g.pn : 0;
    double s = 0.0;
    s += lap_div<P2>(__ldg(&u[i - ox0]) - 2.0 * ui + __ldg(&u[i + ox1]), g.hh[0], g.ihh[0]);
    s += lap_div<P2>(__ldg(&u[i - oy0]) - 2.0 * ui + __ldg(&u[i + oy1]), g.hh[1], g.ihh[1]);
    s += lap_div<P2>(__ldg(&u[i - oz0]) - 2.0 * ui + __ldg(&u[i + oz1]), g.hh[2], g.ihh[2]);
    return s;
}

__device__ __forceinline__ bool lap_coords(const LapGeo& g, int& x, int& y, int& z, int& i, int zoff) {
    x = static_cast<int>(blockIdx.x) * BX + threadIdx.x;
    y = static_cast<int>(blockIdx.y) * BY + threadIdx.y;
    z = static_cast<int>(blockIdx.z) + zoff;
    i = x + y * g.mx + z * g.pn;
    return x < g.mx && y < g.my;
}

template <bool P2>
__global__ void __launch_bounds__(BX * BY) k_lap3(LapGeo g, const double* __restrict__ u, double* __restrict__ out,
                                                  int zoff) {
    int x, y, z, i;
    if (!lap_coords(g, x, y, z, i, zoff)) return;
    const long long n = static_cast<long long>(g.pn) * g.mz;
#pragma unroll
    for (int d = 0; d < 3; ++d) out[d * n + i] = lap_at<P2>(u + d * n, g, x, y, z, i);
}

// curvature.cpp:53-72 second pass (+ the alpha axpy of optimizer.cpp:84-89/98-103,
// or the gamma shift of optimizer.cpp:106-111)
template <bool P2, int MODE>
__global__ void __launch_bounds__(BX * BY) k_bilap(LapGeo g, const double* __restrict__ lu, double scale, double alpha,
                                                   double gamma, const double* __restrict__ p, double* __restrict__ out,
                                                   int zoff) {
    int x, y, z, i;
    if (!lap_coords(g, x, y, z, i, zoff)) return;
    const long long n = static_cast<long long>(g.pn) * g.mz;
#pragma unroll
    for (int d = 0; d < 3; ++d) {
        const double v = scale * lap_at<P2>(lu + d * n, g, x, y, z, i);
        const long long o = d * n + i;
        if constexpr (MODE == 0) out[o] = v;
        else if constexpr (MODE == 1) out[o] += alpha * v;
        else out[o] = v + gamma * __ldg(&p[o]);
    }
}

// alpha S = alpha (h^y sum (Lap u)^2) into a device scalar and a mapped host scalar (fast eval)
__global__ void k_curv_value(const double* __restrict__ S, double cellvol, double alpha, double* out_dev,
                             double* out_host) {
    const double v = alpha * (cellvol * S[0]);
    *out_dev = v;
    *out_host = v;
    __threadfence_system();
}

__global__ void k_curv_finalize(const double* __restrict__ S3, double cellvol, double alpha, double* out) {
    double total = 0.0;
    total += S3[0];
    total += S3[1];
    total += S3[2];
    *out = alpha * (cellvol * total);
}

__global__ void k_add_scalars(const double* a, const double* b, double* out) { *out = *a + *b; }

__global__ void k_sub(idx_t n, const double* __restrict__ a, const double* __restrict__ b, double* __restrict__ o) {
    const idx_t i = static_cast<idx_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) o[i] = a[i] - b[i];
}
__global__ void k_neg(idx_t n, const double* __restrict__ a, double* __restrict__ o) {
    const idx_t i = static_cast<idx_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) o[i] = -a[i];
}
__global__ void k_axpy_to(idx_t n, const double* __restrict__ x, double a, const double* __restrict__ y,
                          double* __restrict__ o) {
    const idx_t i = static_cast<idx_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) o[i] = x[i] + a * y[i];
}
__global__ void k_cg_update(idx_t n, double alpha, const double* __restrict__ p, const double* __restrict__ ap,
                            double* __restrict__ x, double* __restrict__ r) {
    const idx_t i = static_cast<idx_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) {
        x[i] += alpha * p[i];
        r[i] -= alpha * ap[i];
    }
}
__global__ void k_scale_to(idx_t n, double a, const double* __restrict__ x, double* __restrict__ o) {
    const idx_t i = static_cast<idx_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) o[i] = a * x[i];
}
__global__ void k_scale_inplace(idx_t n, double a, double* __restrict__ x) {
    const idx_t i = static_cast<idx_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) x[i] *= a;
}

// grid.hpp:91-101 nodal coordinates, component-major (optimizer.cpp:52-62)
__global__ void k_identity(Grid g, double* __restrict__ out) {
    idx_t x, y, z;
    if (!coords(g, x, y, z)) return;
    const idx_t n = g.count(), i = g.lin(x, y, z);
    out[i] = static_cast<double>(x) * g.h[0];
    out[n + i] = static_cast<double>(y) * g.h[1];
    out[2 * n + i] = static_cast<double>(z) * g.h[2];
}

// volume.cpp:123-160
__global__ void k_downsample(Grid f, Grid c, const double* __restrict__ v, double* __restrict__ out) {
    idx_t i, j, k;
    if (!coords(c, i, j, k)) return;
    double sum = 0.0;
    int cnt = 0;
    for (idx_t dz = 0; dz < 2; ++dz)
        for (idx_t dy = 0; dy < 2; ++dy)
            for (idx_t dx = 0; dx < 2; ++dx) {
                const idx_t fi = 2 * i + dx, fj = 2 * j + dy, fk = 2 * k + dz;
                if (fi < f.m[0] && fj < f.m[1] && fk < f.m[2]) {
                    sum += v[f.lin(fi, fj, fk)];
                    ++cnt;
                }
            }
    out[c.lin(i, j, k)] = sum / cnt;
}

// multilevel.cpp:51-115 — u = y_c - x_c, y_f = x_f + nodal_interpolate(u, x_f)
__global__ void k_prolong(Grid c, Grid f, const double* __restrict__ yc, double* __restrict__ yf) {
    idx_t x, y, z;
    if (!coords(f, x, y, z)) return;
    const idx_t nf = f.count(), nc = c.count(), i = f.lin(x, y, z);
    const double p[3] = {static_cast<double>(x) * f.h[0], static_cast<double>(y) * f.h[1],
                         static_cast<double>(z) * f.h[2]};
    idx_t b[3];
    double w[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        const idx_t ma = c.m[a];
        double s = p[a] / c.h[a];
        const double hi = static_cast<double>(ma - 1);
        s = (s < 0.0) ? 0.0 : ((hi < s) ? hi : s);
        idx_t base = static_cast<idx_t>(floor(s));
        base = base < 0 ? 0 : (base > ma - 2 ? ma - 2 : base);
        b[a] = base;
        w[a] = s - static_cast<double>(base);
    }
#pragma unroll
    for (int d = 0; d < 3; ++d) {
        double v = 0.0;
        for (int cc = 0; cc < 2; ++cc)
            for (int bb = 0; bb < 2; ++bb)
                for (int aa = 0; aa < 2; ++aa) {
                    const double weight =
                        (aa ? w[0] : 1.0 - w[0]) * (bb ? w[1] : 1.0 - w[1]) * (cc ? w[2] : 1.0 - w[2]);
                    const idx_t gx = b[0] + aa, gy = b[1] + bb, gz = b[2] + cc;
                    const double xc = d == 0 ? static_cast<double>(gx) * c.h[0]
                                             : (d == 1 ? static_cast<double>(gy) * c.h[1]
                                                       : static_cast<double>(gz) * c.h[2]);
                    const double u = yc[d * nc + c.lin(gx, gy, gz)] - xc;
                    v += weight * u;
                }
        yf[d * nf + i] = p[d] + v;
    }
}

// synthetic.cpp:15-63 (device libm: values agree with glibc to a few ulp; inputs
// are generated once and shared by every arm that consumes them)
__device__ __forceinline__ double soft_step(double x, double width) { return 1.0 / (1.0 + exp(-x / width)); }

__global__ void k_phantom(Grid g, double* __restrict__ out) {
    idx_t x, y, z;
    if (!coords(g, x, y, z)) return;
    const double p[3] = {(static_cast<double>(x) + 0.5) * g.h[0], (static_cast<double>(y) + 0.5) * g.h[1],
                         (static_cast<double>(z) + 0.5) * g.h[2]};
    const double e[3] = {static_cast<double>(g.m[0]) * g.h[0], static_cast<double>(g.m[1]) * g.h[1],
                         static_cast<double>(g.m[2]) * g.h[2]};
    const double scale = fmin(fmin(e[0], e[1]), e[2]);
    const double edge = 0.015 * scale;
    const double sc[5][3] = {{0.35, 0.4, 0.45}, {0.68, 0.62, 0.40}, {0.55, 0.30, 0.68}, {0.30, 0.70, 0.62},
                             {0.72, 0.35, 0.70}};
    const double sr[5] = {0.22, 0.14, 0.10, 0.08, 0.06};
    const double sw[5] = {1.0, -0.7, 0.8, 0.6, -0.5};
    double val = 0.1 * (p[0] / e[0]) * (p[1] / e[1]);
#pragma unroll
    for (int s = 0; s < 5; ++s) {
        double d2 = 0.0;
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            const double diff = p[a] - sc[s][a] * e[a];
            d2 += diff * diff;
        }
        val += sw[s] * soft_step(sr[s] * scale - sqrt(d2), edge);
    }
    const double plane = (p[0] / e[0] + p[1] / e[1] + p[2] / e[2]) / 3.0 - 0.55;
    val += 0.4 * soft_step(-fabs(plane) + 0.04, 0.01);
    const double pi = 3.141592653589793;
    const double tx = 2.0 * pi * p[0] / e[0];
    const double ty = 2.0 * pi * p[1] / e[1];
    const double tz = 2.0 * pi * p[2] / e[2];
    val += 0.12 * sin(3.0 * tx + 0.8 * sin(2.0 * ty)) * cos(2.0 * ty + 0.6 * sin(3.0 * tz)) +
           0.08 * cos(4.0 * tz + 0.7 * sin(2.0 * tx)) * sin(3.0 * ty + 0.5 * cos(2.0 * tx));
    out[g.lin(x, y, z)] = val;
}

// synthetic.cpp:92-108 + 145-159
__global__ void k_warp_with(Grid g, WarpTerms w, const double* __restrict__ T, double* __restrict__ out) {
    idx_t x, y, z;
    if (!coords(g, x, y, z)) return;
    double p[3] = {(static_cast<double>(x) + 0.5) * g.h[0], (static_cast<double>(y) + 0.5) * g.h[1],
                   (static_cast<double>(z) + 0.5) * g.h[2]};
    const double pi = 3.141592653589793;
    double u[3] = {0.0, 0.0, 0.0};
    for (int t = 0; t < 3; ++t)
        for (int d = 0; d < 3; ++d) {
            double v = w.amp[t][d];
            for (int a = 0; a < 3; ++a) {
                const double xx = p[a] / w.extent[a];
                v *= sin(pi * w.freq[t][a] * xx + w.phase[t][a] * xx * (1.0 - xx));
            }
            u[d] += v;
        }
    for (int d = 0; d < 3; ++d) p[d] += u[d];
    double val, gx, gy, gz;
    interpolate(T, g, p[0], p[1], p[2], val, gx, gy, gz);
    out[g.lin(x, y, z)] = val;
}

std::atomic<long long> g_launches{0};

}  // namespace

void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
long long launch_counter() { return g_launches.load(); }
void note_launches(long long n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

// ------------------------------------------------------------------ host side

HvTable make_hv_table(const Grid& g) {
    // ngf.cpp:267-300: kappa = mu(db) - mu(da), grouped; groups ordered by kappa
    // (std::map), pairs in (da outer, db inner) order. Grouping by 3-D offset
    // instead of linear kappa only separates groups that collide on degenerate
    // grids, and for every voxel at most one of a colliding set is non-zero.
    auto mu = [&](int d) -> long long {
        switch (d) {
        case NEGZ: return -g.m[0] * g.m[1];
        case NEGY: return -g.m[0];
        case NEGX: return -1;
        case CENTER: return 0;
        case POSX: return 1;
        case POSY: return g.m[0];
        default: return g.m[0] * g.m[1];
        }
    };
    struct G3 {
        int dx, dy, dz;
        long long kappa;
        int first;
        std::vector<std::pair<int, int>> pairs;
    };
    std::vector<G3> groups;
    int order = 0;
    for (int da = 0; da < 7; ++da)
        for (int db = 0; db < 7; ++db) {
            const int dx = dir_dx(db) - dir_dx(da), dy = dir_dy(db) - dir_dy(da), dz = dir_dz(db) - dir_dz(da);
            auto it = std::find_if(groups.begin(), groups.end(),
                                   [&](const G3& q) { return q.dx == dx && q.dy == dy && q.dz == dz; });
            if (it == groups.end()) {
                groups.push_back({dx, dy, dz, mu(db) - mu(da), order++, {}});
                it = groups.end() - 1;
            }
            it->pairs.emplace_back(da, db);
        }
    std::stable_sort(groups.begin(), groups.end(), [](const G3& a, const G3& b) { return a.kappa < b.kappa; });
    HvTable t{};
    t.ngroups = static_cast<int>(groups.size());
    for (int e = 0; e < t.ngroups; ++e) {
        t.dx[e] = groups[e].dx;
        t.dy[e] = groups[e].dy;
        t.dz[e] = groups[e].dz;
        t.npairs[e] = static_cast<int>(groups[e].pairs.size());
        for (int q = 0; q < t.npairs[e]; ++q) {
            t.pa[e][q] = groups[e].pairs[q].first;
            t.pb[e][q] = groups[e].pairs[q].second;
        }
    }
    return t;
}

void launch_transfer_apply(const DevPlan& P, const double* y, double* out, cudaStream_t s) {
    note_launch(), k_transfer_apply<<<grid3(P.tgt), block3(), 0, s>>>(P, y, out);
}

template <typename OutT>
__global__ void __launch_bounds__(256, MFREG_WARP_MINB) k_warp_fast(DevPlan P, const double* __restrict__ y,
                                                   const double* __restrict__ T, OutT* __restrict__ Tw,
                                                   OutT* __restrict__ dT, int zoff) {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");  // the eval pass (PDL) may queue behind
    const int mx = static_cast<int>(P.tgt.m[0]), my = static_cast<int>(P.tgt.m[1]), mz = static_cast<int>(P.tgt.m[2]);
    const int x = blockIdx.x * 32 + threadIdx.x, yy = blockIdx.y * 8 + threadIdx.y;
    const int z = blockIdx.z + zoff;
    if (x >= mx || yy >= my) return;
    const int bx = __ldg(&P.base[0][x]), by = __ldg(&P.base[1][yy]), bz = __ldg(&P.base[2][z]);
    const double rx = __ldg(&P.rem[0][x]), ry = __ldg(&P.rem[1][yy]), rz = __ldg(&P.rem[2][z]);
    const double wx[2] = {1.0 - rx, rx}, wy[2] = {1.0 - ry, ry}, wz[2] = {1.0 - rz, rz};
    double w[8];
#pragma unroll
    for (int g = 0; g < 2; ++g)
#pragma unroll
        for (int b = 0; b < 2; ++b)
#pragma unroll
            for (int a = 0; a < 2; ++a) w[(g * 2 + b) * 2 + a] = wx[a] * wy[b] * wz[g];
    // 32-bit element offsets (nodal arrays and image volumes are < 2^31 elements)
    const int ns = static_cast<int>(P.src.count());
    const int sm0 = static_cast<int>(P.src.m[0]), sm01 = static_cast<int>(P.src.m[0] * P.src.m[1]);
    // four corner-row pointers (b, g); the a = 1 corner is an immediate offset
    const double* yr[2][2];
    yr[0][0] = y + (bx + by * sm0 + bz * sm01);
    yr[0][1] = yr[0][0] + sm0;
    yr[1][0] = yr[0][0] + sm01;
    yr[1][1] = yr[1][0] + sm0;
    double pt[3];
#pragma unroll
    for (int d = 0; d < 3; ++d) {
        double acc = 0.0;
#pragma unroll
        for (int g = 0; g < 2; ++g)
#pragma unroll
            for (int b = 0; b < 2; ++b)
#pragma unroll
                for (int a = 0; a < 2; ++a) acc += w[(g * 2 + b) * 2 + a] * __ldg(yr[g][b] + d * ns + a);
        pt[d] = acc;
    }
    warp_sample_store(P, T, pt, x, yy, z, mx, my, mz, Tw, dT);
}

// z-marching fast warp: one thread per image column (x, y) over a chunk of planes. The
// column's x-y corner weights wx*wy are formed once; the nodal values of the current nodal z
// cell (two nodal planes over the block's x-y footprint, 3 components) are staged in shared
// memory once per cell (every ~ratio planes) instead of 24 global loads per voxel. Per plane,
// P y is 8 + 24 multiplies and 24 adds in the reference's operation order
// (transfer.cpp:66-81: acc += ((wx*wy)*wz)*y, (g,b,a) order from 0.0), bitwise the same as
// transfer_point / k_warp_fast.
constexpr int WZ_NXF = 34, WZ_NYF = 10;
#ifndef MFREG_WARPZ_MINB
#define MFREG_WARPZ_MINB 5  // measured at C4: 5 blocks (48 regs) 3.01 ms, 6 (40, spills) 2.96, 4 (64) 3.16; nodal values in registers, 2 blocks: 3.90; per-voxel kernel 3.52
#endif  // nodal footprint bound of a 32x8 column block (ratio >= 1)
// fastpy: P y from the column's x-y bilinear interpolants of the cell's two nodal planes and a
// z lerp (FMA; a few ulp from the reference's exact sum, i.e. the sample moves by < 1e-12 voxel),
// and the reference's exact P y and IEEE p/h only for points within 1e-9 of a cell face, where
// that difference could change the cell (and dT by O(1)): cell choice bitwise the reference's,
// T_w / dT within ~1e-15 relative (fast-mode tolerance 1e-9). On by default (MFREG_FAST_PY=0
// selects the reference-order P y): like every fast-mode reordering, the 1e-16 perturbation moves a full
// registration inside the reference's own 1-ulp envelope (C2 GN: 0.15 voxel max against the
// reference's 0.45 under +-1 ulp of the template, tests/golden/c2_envelope.json).
template <typename OutT>
__global__ void __launch_bounds__(256, MFREG_WARPZ_MINB) k_warp_z(DevPlan P, const double* __restrict__ y,
                                                   const double* __restrict__ T, OutT* __restrict__ Tw,
                                                   OutT* __restrict__ dT, int zlo, int zhi, int zc, int fastpy) {
    __shared__ double sy[3][2][WZ_NYF][WZ_NXF];
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");  // the eval pass (PDL) may queue behind
    const int mx = static_cast<int>(P.tgt.m[0]), my = static_cast<int>(P.tgt.m[1]), mz = static_cast<int>(P.tgt.m[2]);
    const int x0 = blockIdx.x * 32, y0 = blockIdx.y * 8;
    const int x = x0 + threadIdx.x, yy = y0 + threadIdx.y;
    const bool in = x < mx && yy < my;
    const int xc = min(x, mx - 1), yc = min(yy, my - 1);
    const int zb = zlo + static_cast<int>(blockIdx.z) * zc, ze = min(zhi, zb + zc);
    const int fx0 = __ldg(&P.base[0][x0]), fy0 = __ldg(&P.base[1][y0]);
    const int nxf = __ldg(&P.base[0][min(x0 + 31, mx - 1)]) - fx0 + 2;
    const int nyf = __ldg(&P.base[1][min(y0 + 7, my - 1)]) - fy0 + 2;
    const int lx = __ldg(&P.base[0][xc]) - fx0, ly = __ldg(&P.base[1][yc]) - fy0;
    const double rx = __ldg(&P.rem[0][xc]), ry = __ldg(&P.rem[1][yc]);
    const double wx[2] = {1.0 - rx, rx}, wy[2] = {1.0 - ry, ry};
    double wxy[2][2];
#pragma unroll
    for (int b = 0; b < 2; ++b)
#pragma unroll
        for (int a = 0; a < 2; ++a) wxy[b][a] = wx[a] * wy[b];
    const int ns = static_cast<int>(P.src.count());
    const int sm0 = static_cast<int>(P.src.m[0]), sm01 = static_cast<int>(P.src.m[0] * P.src.m[1]);
    const int tid = threadIdx.x + 32 * threadIdx.y, nfill = 3 * 2 * nyf * nxf;
    auto ptof = [&](double rz, double pt[3]) {
        const double wz[2] = {1.0 - rz, rz};
        double w[2][2][2];
#pragma unroll
        for (int g = 0; g < 2; ++g)
#pragma unroll
            for (int b = 0; b < 2; ++b)
#pragma unroll
                for (int a = 0; a < 2; ++a) w[g][b][a] = wxy[b][a] * wz[g];
#pragma unroll
        for (int d = 0; d < 3; ++d) {
            double acc = 0.0;
#pragma unroll
            for (int g = 0; g < 2; ++g)
#pragma unroll
                for (int b = 0; b < 2; ++b)
#pragma unroll
                    for (int a = 0; a < 2; ++a) acc += w[g][b][a] * sy[d][g][ly + b][lx + a];
            pt[d] = acc;
        }
    };
    int cur = -1;
    double Pa[3] = {0.0, 0.0, 0.0}, Pd[3] = {0.0, 0.0, 0.0};  // fastpy: bilinear at plane bz, (bz+1) - bz
#pragma unroll 1
    for (int z = zb; z < ze;) {
        const int bz = __ldg(&P.base[2][z]);
        if (bz != cur) {  // uniform across the block (same plane): restage the cell's nodal values
            cur = bz;
            __syncthreads();
            for (int t = tid; t < nfill; t += 256) {
                const int ix = t % nxf, r = t / nxf, iy = r % nyf, gd = r / nyf;  // gd = d * 2 + g
                (&sy[0][0][0][0])[(gd * WZ_NYF + iy) * WZ_NXF + ix] =
                    __ldg(y + (gd >> 1) * ns + (bz + (gd & 1)) * sm01 + (fy0 + iy) * sm0 + fx0 + ix);
            }
            __syncthreads();
            if (fastpy) {
#pragma unroll
                for (int d = 0; d < 3; ++d) {
                    double pg[2];
#pragma unroll
                    for (int g = 0; g < 2; ++g) {
                        const double c0 = fma(rx, sy[d][g][ly][lx + 1] - sy[d][g][ly][lx], sy[d][g][ly][lx]);
                        const double c1 = fma(rx, sy[d][g][ly + 1][lx + 1] - sy[d][g][ly + 1][lx], sy[d][g][ly + 1][lx]);
                        pg[g] = fma(ry, c1 - c0, c0);
                    }
                    Pa[d] = pg[0];
                    Pd[d] = pg[1] - pg[0];
                }
            }
        }
        if (in) {
            const double rz = __ldg(&P.rem[2][z]);
            double pt[3], c[3], f[3];
            bool near = true;
            if (fastpy) {
                near = false;
#pragma unroll
                for (int d = 0; d < 3; ++d) {
                    pt[d] = fma(rz, Pd[d], Pa[d]);
                    const double sa = fma(pt[d], P.tgt.ih[d], -0.5);
                    c[d] = ceil(sa);
                    f[d] = sa - (c[d] - 1.0);  // in (0, 1]: 1 at a tie
                    near = near || f[d] < 1e-9 || f[d] > 1.0 - 1e-9;
                }
            }
            if (near) {
                ptof(rz, pt);
                warp_sample_store(P, T, pt, x, yy, z, mx, my, mz, Tw, dT);
            } else {
                const long long n = static_cast<long long>(mx) * my * mz;
                warp_sample_store_c(P, T, c, f, mx, my, mz, x + static_cast<long long>(yy) * mx + static_cast<long long>(z) * mx * my,
                                    n, Tw, dT);
            }
        }
        ++z;
    }
}

// z window helpers: [lo, hi) clipped to [0, m); hi < 0 means m
static inline bool zwin(const Grid& g, dim3& gr, int& lo, int hi) {
    gr = grid3(g);
    const int m = static_cast<int>(g.m[2]);
    lo = std::max(0, lo);
    hi = hi < 0 ? m : std::min(hi, m);
    if (hi <= lo) return false;
    gr.z = static_cast<unsigned>(hi - lo);
    return true;
}
void launch_transfer_T(const DevPlan& P, const double* w, double* out, cudaStream_t s, int zlo, int zhi) {
    dim3 gr;
    if (!zwin(P.src, gr, zlo, zhi)) return;
    note_launch(), k_transfer_T<<<gr, block3(), 0, s>>>(P, w, out, zlo);
}
void launch_sample(const Grid& img0, const double* T, const double* pts, idx_t n, double* vals, double* dT,
                   cudaStream_t s) {
    Grid img = img0;
    img.set_inv();
    note_launch(), k_sample<<<blocks1(n), 256, 0, s>>>(img, T, pts, n, vals, dT);
}
void launch_warp(const DevPlan& P0, const double* y, const double* T, double* Tw, double* dT, cudaStream_t s, int zlo,
                 int zhi) {
    DevPlan P = P0;
    P.tgt.set_inv();
    if (zhi < 0) zhi = static_cast<int>(P.tgt.m[2]);
    dim3 gr = grid3(P.tgt);
    gr.z = static_cast<unsigned>(zhi - zlo);
    if (gr.z == 0) return;
    note_launch(), k_warp<<<gr, block3(), 0, s>>>(P, y, T, Tw, dT, zlo);
}
template <typename OutT>
void warp_fast_impl(const DevPlan& P0, const double* y, const double* T, OutT* Tw, OutT* dT, cudaStream_t s, int zlo,
                    int zhi) {
    DevPlan P = P0;
    P.tgt.set_inv();
    if (zhi < 0) zhi = static_cast<int>(P.tgt.m[2]);
    if (zhi <= zlo) return;
    const unsigned gx = static_cast<unsigned>((P.tgt.m[0] + 31) / 32), gy = static_cast<unsigned>((P.tgt.m[1] + 7) / 8);
    static const bool zmarch = [] {
        const char* e = std::getenv("MFREG_WARP_Z");
        return !(e && e[0] == '0');
    }();
    if (zmarch) {
        // z chunks: enough blocks for ~8 per SM, each chunk <= 64 planes
        const int nz = zhi - zlo;
        const long long cols = static_cast<long long>(gx) * gy;
        const int nch = std::max<int>((nz + 63) / 64, static_cast<int>(std::min<long long>(nz, (148LL * 8 + cols - 1) / cols)));
        const int zc = (nz + nch - 1) / nch;
        const dim3 gr(gx, gy, static_cast<unsigned>((nz + zc - 1) / zc));
        // separable fast P y (2-3% of a C4 gradient eval; the cell choice stays the
        // reference's); MFREG_FAST_PY=0 keeps the reference-order P y. Read per launch so a process
        // can compare both.
        const char* fpe = std::getenv("MFREG_FAST_PY");
        const int fastpy = (fpe && fpe[0] == '0') ? 0 : 1;
        note_launch(), k_warp_z<OutT><<<gr, dim3(32, 8, 1), 0, s>>>(P, y, T, Tw, dT, zlo, zhi, zc, fastpy);
        return;
    }
    const dim3 gr(gx, gy, static_cast<unsigned>(zhi - zlo));
    note_launch(), k_warp_fast<OutT><<<gr, dim3(32, 8, 1), 0, s>>>(P, y, T, Tw, dT, zlo);
}
__global__ void k_to_float(idx_t n, const double* __restrict__ a, float* __restrict__ o) {
    for (idx_t i = static_cast<idx_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<idx_t>(gridDim.x) * blockDim.x)
        o[i] = static_cast<float>(a[i]);
}
void launch_to_float(idx_t n, const double* a, float* o, cudaStream_t s) {
    if (n <= 0) return;
    note_launch();
    k_to_float<<<static_cast<unsigned>(std::min<idx_t>((n + 255) / 256, 148 * 16)), 256, 0, s>>>(n, a, o);
}
void launch_warp_fast(const DevPlan& P, const double* y, const double* T, double* Tw, double* dT, cudaStream_t s,
                      int zlo, int zhi) {
    warp_fast_impl(P, y, T, Tw, dT, s, zlo, zhi);
}
void launch_warp_fast(const DevPlan& P, const double* y, const double* T, float* Tw, float* dT, cudaStream_t s,
                      int zlo, int zhi) {
    warp_fast_impl(P, y, T, Tw, dT, s, zlo, zhi);
}
void launch_ngf_ws(const Grid& img0, const double* R, const double* Tw, double tau, double rho, double* r,
                   double* inv1, double* inv2, double* rh, cudaStream_t s, int zlo, int zhi) {
    Grid img = img0;
    img.set_inv();
    dim3 gr;
    if (!zwin(img, gr, zlo, zhi)) return;
    note_launch(), k_ngf_ws<<<gr, block3(), 0, s>>>(img, R, Tw, tau, rho, r, inv1, inv2, rh, zlo);
}
void launch_ngf_gradient(const Grid& img, const double* r, const double* rh, const double* dT, double* out,
                         cudaStream_t s, int zlo, int zhi) {
    const double scale = -2.0 * img.cell_volume();
    dim3 gr;
    if (!zwin(img, gr, zlo, zhi)) return;
    note_launch(), k_ngf_gradient<<<gr, block3(), 0, s>>>(img, scale, r, rh, dT, out, zlo);
}
void launch_Pp_s(const DevPlan& P, const double* p, const double* dT, double* sv, cudaStream_t s, int zlo, int zhi) {
    dim3 gr;
    if (!zwin(P.tgt, gr, zlo, zhi)) return;
    note_launch(), k_Pp_s<<<gr, block3(), 0, s>>>(P, p, dT, sv, zlo);
}
void launch_hv_closed(const Grid& img, const HvTable& tab, const double* rh, const double* sv, const double* dT,
                      double* out, cudaStream_t s, int zlo, int zhi) {
    const double scale = 2.0 * img.cell_volume();
    dim3 gr;
    if (!zwin(img, gr, zlo, zhi)) return;
    if (is_canon_hv_table(tab))
        note_launch(), k_hv_closed_canon<<<gr, block3(), 0, s>>>(img, scale, rh, sv, dT, out, zlo);
    else
        note_launch(), k_hv_closed<<<gr, block3(), 0, s>>>(img, tab, scale, rh, sv, dT, out, zlo);
}
void launch_hv_factored(const Grid& img, const double* rh, const double* sv, const double* dT, double* wbuf,
                        double* out, cudaStream_t s) {
    const double scale = 2.0 * img.cell_volume();
    note_launch(), k_hv_w<<<grid3(img), block3(), 0, s>>>(img, rh, sv, wbuf);
    note_launch(), k_hv_z<<<grid3(img), block3(), 0, s>>>(img, scale, rh, wbuf, dT, out);
}

idx_t chunk_count(idx_t n) { return (n + kChunk - 1) / kChunk; }
idx_t tree_blocks(idx_t n) { return std::max<idx_t>(1, (n + kTreeSpan - 1) / kTreeSpan); }

void launch_chunked_sum(int kind, idx_t n, const double* a, const double* b, double* partials, double* out,
                        double scale, cudaStream_t s) {
    const idx_t nch = chunk_count(n);
    if (nch > 0) {
        const unsigned g = static_cast<unsigned>(nch);
        const std::size_t sm = kChunk * sizeof(double);
        note_launch();
        if (kind == SUM_ONE_MINUS_SQ) k_chunks_warp<SUM_ONE_MINUS_SQ><<<g, 32, sm, s>>>(n, a, b, partials);
        else if (kind == SUM_DOT) k_chunks_warp<SUM_DOT><<<g, 32, sm, s>>>(n, a, b, partials);
        else k_chunks_warp<SUM_SQ><<<g, 32, sm, s>>>(n, a, b, partials);
    }
    note_launch(), k_serial<<<1, 32, 0, s>>>(partials, nch, scale, out);
}
// chunked_sum across ranks (z slabs, parity mode; DistSum in slab.cu): a rank's interior chunk
// partials (k_chunks_warp on a chunk-aligned sub-range) and the raw terms of the chunks it only
// partly owns; after the all-gather every rank rebuilds each chunk's sequential sum from the
// pieces in index order and adds the chunks in order (parallel.cpp:51-73, bitwise).
void launch_chunk_partials(int kind, idx_t n, const double* a, const double* b, double* partials, cudaStream_t s) {
    const idx_t nch = chunk_count(n);
    if (nch <= 0) return;
    const unsigned g = static_cast<unsigned>(nch);
    const std::size_t sm = kChunk * sizeof(double);
    note_launch();
    if (kind == SUM_ONE_MINUS_SQ) k_chunks_warp<SUM_ONE_MINUS_SQ><<<g, 32, sm, s>>>(n, a, b, partials);
    else if (kind == SUM_DOT) k_chunks_warp<SUM_DOT><<<g, 32, sm, s>>>(n, a, b, partials);
    else k_chunks_warp<SUM_SQ><<<g, 32, sm, s>>>(n, a, b, partials);
}
__global__ void k_sum_terms(int kind, idx_t n, const double* __restrict__ a, const double* __restrict__ b,
                            double* __restrict__ out) {
    const idx_t i = static_cast<idx_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) out[i] = sum_term(kind, a, b, i);
}
void launch_sum_terms(int kind, idx_t n, const double* a, const double* b, double* out, cudaStream_t s) {
    if (n <= 0) return;
    note_launch(), k_sum_terms<<<blocks1(n), 256, 0, s>>>(kind, n, a, b, out);
}
__global__ void k_chunk_assemble(idx_t nch, const long long* __restrict__ off, const int* __restrict__ cnt,
                                 const ChunkPiece* __restrict__ pieces, const double* __restrict__ g,
                                 double* __restrict__ vals) {
    const idx_t c = static_cast<idx_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (c >= nch) return;
    const int k = cnt[c];
    if (k == 0) {
        vals[c] = g[off[c]];
        return;
    }
    double s = 0.0;  // the chunk's terms in index order, from 0.0, across the owners' pieces
    for (int q = 0; q < k; ++q) {
        const ChunkPiece pc = pieces[off[c] + q];
        for (int t = 0; t < pc.len; ++t) s += g[pc.off + t];
    }
    vals[c] = s;
}
void launch_chunk_assemble(idx_t nch, const long long* off, const int* cnt, const ChunkPiece* pieces,
                           const double* gathered, double* vals, double scale, double* out, cudaStream_t s) {
    if (nch > 0) note_launch(), k_chunk_assemble<<<blocks1(nch, 128), 128, 0, s>>>(nch, off, cnt, pieces, gathered, vals);
    note_launch(), k_serial<<<1, 32, 0, s>>>(vals, nch, scale, out);
}
void launch_chunked_sum3(int kind, idx_t n, const double* a, const double* b, double* partials, double* out3,
                         double scale, cudaStream_t s) {
    const idx_t nch = chunk_count(n);
    if (nch > 0) {
        const unsigned g = static_cast<unsigned>(3 * nch);
        const std::size_t sm = kChunk * sizeof(double);
        note_launch();
        if (kind == SUM_ONE_MINUS_SQ) k_chunks_warp<SUM_ONE_MINUS_SQ><<<g, 32, sm, s>>>(n, a, b, partials, nch);
        else if (kind == SUM_DOT) k_chunks_warp<SUM_DOT><<<g, 32, sm, s>>>(n, a, b, partials, nch);
        else k_chunks_warp<SUM_SQ><<<g, 32, sm, s>>>(n, a, b, partials, nch);
    }
    note_launch(), k_serial3<<<1, 32, 0, s>>>(partials, nch, scale, out3);
}
void launch_tree_sum(int kind, idx_t n, const double* a, const double* b, double* partials, double* out,
                     double scale, cudaStream_t s) {
    const idx_t nb = tree_blocks(n);
    note_launch(), k_tree_partials<<<static_cast<unsigned>(nb), kTreeThreads, 0, s>>>(kind, n, a, b, partials);
    note_launch(), k_tree_final<<<1, 1024, 0, s>>>(partials, nb, scale, out);
}
void launch_inf_norm(idx_t n, const double* a, double scale, double* out, cudaStream_t s) {
    note_launch(), k_inf_norm_init<<<1, 1, 0, s>>>(out);
    const unsigned nb = static_cast<unsigned>(std::min<idx_t>(blocks1(n), 148 * 8));
    note_launch(), k_inf_norm<<<nb, 256, 0, s>>>(n, a, scale, reinterpret_cast<unsigned long long*>(out));
}

static bool lap_geo(const Grid& g, LapGeo& o) {
    o.mx = static_cast<int>(g.m[0]);
    o.my = static_cast<int>(g.m[1]);
    o.mz = static_cast<int>(g.m[2]);
    o.pn = o.mx * o.my;
    bool p2 = true;
    for (int a = 0; a < 3; ++a) {
        o.hh[a] = g.h[a] * g.h[a];
        int e = 0;
        p2 = p2 && std::frexp(o.hh[a], &e) == 0.5 && e > -1000 && e < 1000;
        o.ihh[a] = 1.0 / o.hh[a];
    }
    return p2;
}

void launch_lap3(const Grid& g, const double* u, double* out, cudaStream_t s, int zlo, int zhi, bool exact) {
    LapGeo lg;
    dim3 gr;
    if (!zwin(g, gr, zlo, zhi)) return;
    if (lap_geo(g, lg) || !exact) note_launch(), k_lap3<true><<<gr, block3(), 0, s>>>(lg, u, out, zlo);
    else note_launch(), k_lap3<false><<<gr, block3(), 0, s>>>(lg, u, out, zlo);
}

template <bool P2>
static void launch_bilap_t(dim3 gr, int zlo, const LapGeo& lg, const double* lap_u, double scale, int mode,
                           double alpha, double gamma, const double* p, double* out, cudaStream_t s) {
    if (mode == 0) k_bilap<P2, 0><<<gr, block3(), 0, s>>>(lg, lap_u, scale, alpha, gamma, p, out, zlo);
    else if (mode == 1) k_bilap<P2, 1><<<gr, block3(), 0, s>>>(lg, lap_u, scale, alpha, gamma, p, out, zlo);
    else k_bilap<P2, 2><<<gr, block3(), 0, s>>>(lg, lap_u, scale, alpha, gamma, p, out, zlo);
}

void launch_bilap(const Grid& g, const double* lap_u, double scale, int mode, double alpha, double gamma,
                  const double* p, double* out, cudaStream_t s, int zlo, int zhi, bool exact) {
    LapGeo lg;
    dim3 gr;
    if (!zwin(g, gr, zlo, zhi)) return;
    note_launch();
    if (lap_geo(g, lg) || !exact) launch_bilap_t<true>(gr, zlo, lg, lap_u, scale, mode, alpha, gamma, p, out, s);
    else launch_bilap_t<false>(gr, zlo, lg, lap_u, scale, mode, alpha, gamma, p, out, s);
}
void launch_curv_value(const double* S, double cellvol, double alpha, double* out_dev, double* out_host,
                       cudaStream_t s) {
    note_launch(), k_curv_value<<<1, 1, 0, s>>>(S, cellvol, alpha, out_dev, out_host);
}
void launch_curv_finalize(const double* S3, double cellvol, double alpha, double* out, cudaStream_t s) {
    note_launch(), k_curv_finalize<<<1, 1, 0, s>>>(S3, cellvol, alpha, out);
}
void launch_add_scalars(const double* a, const double* b, double* out, cudaStream_t s) {
    note_launch(), k_add_scalars<<<1, 1, 0, s>>>(a, b, out);
}
void launch_sub(idx_t n, const double* a, const double* b, double* out, cudaStream_t s) {
    note_launch(), k_sub<<<blocks1(n), 256, 0, s>>>(n, a, b, out);
}
void launch_neg(idx_t n, const double* a, double* out, cudaStream_t s) { note_launch(), k_neg<<<blocks1(n), 256, 0, s>>>(n, a, out); }
void launch_axpy_to(idx_t n, const double* x, double a, const double* y, double* out, cudaStream_t s) {
    note_launch(), k_axpy_to<<<blocks1(n), 256, 0, s>>>(n, x, a, y, out);
}
void launch_cg_update(idx_t n, double alpha, const double* p, const double* ap, double* x, double* r,
                      cudaStream_t s) {
    note_launch(), k_cg_update<<<blocks1(n), 256, 0, s>>>(n, alpha, p, ap, x, r);
}
void launch_scale_to(idx_t n, double a, const double* x, double* out, cudaStream_t s) {
    note_launch(), k_scale_to<<<blocks1(n), 256, 0, s>>>(n, a, x, out);
}
void launch_scale_inplace(idx_t n, double a, double* x, cudaStream_t s) {
    note_launch(), k_scale_inplace<<<blocks1(n), 256, 0, s>>>(n, a, x);
}
void launch_identity(const Grid& g, double* out, cudaStream_t s) { note_launch(), k_identity<<<grid3(g), block3(), 0, s>>>(g, out); }
void launch_downsample(const Grid& fine, const Grid& coarse, const double* v, double* out, cudaStream_t s) {
    note_launch(), k_downsample<<<grid3(coarse), block3(), 0, s>>>(fine, coarse, v, out);
}
void launch_prolong(const Grid& coarse, const Grid& fine, const double* yc, double* yf, cudaStream_t s) {
    note_launch(), k_prolong<<<grid3(fine), block3(), 0, s>>>(coarse, fine, yc, yf);
}
void launch_phantom(const Grid& g, double* out, cudaStream_t s) { note_launch(), k_phantom<<<grid3(g), block3(), 0, s>>>(g, out); }
void launch_warp_with(const Grid& g0, const WarpTerms& w, const double* T, double* out, cudaStream_t s) {
    Grid g = g0;
    g.set_inv();
    note_launch(), k_warp_with<<<grid3(g), block3(), 0, s>>>(g, w, T, out);
}

}  // namespace mfreg_b200
