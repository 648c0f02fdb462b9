// P^T collapse of a fused pass's tile (k_hv2, k_ev2): every output column keeps the
// z-weighted sums of its q^ for the two nodal z planes of its cell in registers; when a nodal plane
// completes, its sums are spread over the tile's nodes in x and y:
//  * x stage (per warp = tile row, right at the completion): the row's three components go to a
//    shared row buffer, and lane L = (d, j) sums node j's window of <= WX columns (the columns of
//    cell j-1 weighted rem_x, of cell j weighted 1 - rem_x) from a per-tile weight table, written
//    back in place at position L (two FMA chains per item);
//  * y stage (one step later, after the CTA barrier): node row lyn (a warp) sums the tile rows
//    with a per-tile weight table and writes the tile partial of that nodal plane.
// Replaces the segmented shuffle scan (fp64 shuffles are two SHFL + moves + selects per level and
// value). Tables are built once per CTA; completions are >= 2 steps apart (host guarantee).
// Bank layout (MFREG_PTC_PAD, default on): the lanes of the x stage read windows that start 4
// columns apart (ratio 4), i.e. 32 bytes apart — 8-way bank conflicts on every fp64 load (ncu:
// ~80% of both passes' excess shared wavefronts, a quarter of all their shared wavefronts). The row
// buffer therefore stores logical column c at c + c/4 (one pad word per 4 columns) and the weight
// table rows are WX + 1 long, which makes the window and weight loads of a warp conflict-free for
// ratio-4 grids; windows that start 4-aligned (every tile of a ratio-4 grid) read with immediate
// offsets, others compute the padded index per load.
#pragma once

#include "fused_dev.cuh"

#ifndef MFREG_PTC_PAD
#define MFREG_PTC_PAD 1
#endif

namespace mfreg_b200 {
namespace fdev {

constexpr int kPtcTX = FT_X;

// physical index of logical row column c (pad: one pad word per 4 columns)
__host__ __device__ constexpr int ptc_phys(int c, bool pad) { return pad ? c + (c >> 2) : c; }
__host__ __device__ constexpr int ptc_row_len(int nlx, bool pad) {
    return ptc_phys(3 * nlx > 3 * kPtcTX ? 3 * nlx : 3 * kPtcTX, pad) + (pad ? 1 : 0);
}
__host__ __device__ constexpr int ptc_win(int segw) { return 2 * segw < kPtcTX ? 2 * segw : kPtcTX; }
__host__ __device__ constexpr int ptc_wstride(int segw, bool pad) { return ptc_win(segw) + (pad ? 1 : 0); }
// shared-memory footprint: Reals (row buffers, weights) and ints (window starts, items)
__host__ __device__ constexpr int ptc_reals(int ty, int nlx, int nly, int segw, bool pad = MFREG_PTC_PAD) {
    return ty * ptc_row_len(nlx, pad) + nlx * ptc_wstride(segw, pad) + nly * ty;
}
__host__ __device__ constexpr int ptc_ints(int nlx) { return 4 * nlx; }

template <typename Real, int TY, bool PAD = MFREG_PTC_PAD>
struct Ptc {
    static __device__ __forceinline__ constexpr int ptc_phys(int c) { return fdev::ptc_phys(c, PAD); }
    Real* sA;   // [TY][XR] row buffers
    Real* sWx;  // [nlx][WXS] x weights of node j over columns xs[j] ..
    Real* sWy;  // [nly][TY] y weights of node row lyn over the tile rows
    int* sXs;   // [nlx] first column of node j's window
    int* sXi;   // [3 nlx] item L = d * nlx_t + j: window offset (logical) | weight offset << 8 | j << 20 | d << 26
    int XR, WX, WXS, nxi, nlx, nly_t;

    __device__ Ptc(Real* reals, int* ints, int nlx_, int nly_, int segw, int nlx_t, int nly_t_)
        : XR(ptc_row_len(nlx_, PAD)), WX(ptc_win(segw)), WXS(ptc_wstride(segw, PAD)), nxi(3 * nlx_t), nlx(nlx_), nly_t(nly_t_) {
        sA = reals;
        sWx = sA + TY * XR;
        sWy = sWx + nlx_ * WXS;
        sXs = ints;
        sXi = sXs + nlx_;
        (void)nly_;
    }

    // weight tables (before the CTA's first barrier)
    __device__ void build_tables(const FArgs& a, int tid, int nthreads, int x0, int y0, int nxA, int nyA, int nly) {
        const int mx = static_cast<int>(a.g.m[0]), my = static_cast<int>(a.g.m[1]);
        const int nlx_t = nxi / 3;
        if (tid < nlx_t) {
            const int j = tid;
            int lo = kPtcTX;
            for (int c = kPtcTX - 1; c >= 0; --c)
                if (x0 + c < mx && __ldg(&a.P.base[0][x0 + c]) - nxA >= j - 1) lo = c;
            const int st = max(0, min(lo, kPtcTX - WX));
            sXs[j] = st;
            for (int t = 0; t < WX; ++t) {
                const int gx = x0 + st + t;
                Real w = Real(0);
                if (gx < mx) {
                    const int b = __ldg(&a.P.base[0][gx]) - nxA;
                    const Real r = static_cast<Real>(__ldg(&a.P.rem[0][gx]));
                    w = b == j ? Real(1) - r : (b == j - 1 ? r : Real(0));
                }
                sWx[j * WXS + t] = w;
            }
        }
        for (int t = tid; t < nly * TY; t += nthreads) {
            const int lyn = t / TY, r = t % TY, gy = y0 + r;
            Real w = Real(0);
            if (gy < my && lyn < nly_t) {
                const int b = __ldg(&a.P.base[1][gy]) - nyA;
                const Real ry = static_cast<Real>(__ldg(&a.P.rem[1][gy]));
                w = b == lyn ? Real(1) - ry : (b == lyn - 1 ? ry : Real(0));
            }
            sWy[t] = w;
        }
    }
    // item table (after the first barrier: reads sXs)
    __device__ void build_items(int tid, int nthreads) {
        const int nlx_t = nxi / 3;
        for (int L = tid; L < nxi; L += nthreads) {
            const int d = L / nlx_t, j = L - d * nlx_t;
            sXi[L] = (d * kPtcTX + sXs[j]) | ((j * WXS) << 8) | (j << 20) | (d << 26);
        }
    }
    // x stage of tile row `row` (whole warp)
    __device__ void xstage(int row, int lane, Real v0, Real v1, Real v2) const {
        Real* ar = sA + row * XR;
        ar[ptc_phys(lane)] = v0;
        ar[ptc_phys(kPtcTX + lane)] = v1;
        ar[ptc_phys(2 * kPtcTX + lane)] = v2;
        __syncwarp();
        const int npx = (nxi + 31) >> 5;  // host: nlx <= 42
        Real o[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int L = lane + 32 * u;
            o[u] = Real(0);
            if (u < npx && L < nxi) {
                const int e = sXi[L];
                const int c0 = e & 0xff;  // logical first column of the window
                const Real* w = sWx + ((e >> 8) & 0xfff);
                Real acc0 = Real(0), acc1 = Real(0);  // WX is even: two chains
                if (!PAD || (c0 & 3) == 0) {
                    // 4-aligned window: the padded offsets t + t/4 are immediates
                    const Real* v = ar + ptc_phys(c0);
#pragma unroll 4
                    for (int t = 0; t < WX; t += 2) {
                        acc0 = fma(w[t], v[ptc_phys(t)], acc0);
                        acc1 = fma(w[t + 1], v[ptc_phys(t + 1)], acc1);
                    }
                } else {
#pragma unroll 2
                    for (int t = 0; t < WX; t += 2) {
                        acc0 = fma(w[t], ar[ptc_phys(c0 + t)], acc0);
                        acc1 = fma(w[t + 1], ar[ptc_phys(c0 + t + 1)], acc1);
                    }
                }
                o[u] = acc0 + acc1;
            }
        }
        __syncwarp();
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int L = lane + 32 * u;
            if (u < npx && L < nxi) ar[ptc_phys(L)] = o[u];
        }
    }
    // FAST32 alternative of the x stage: a segmented shuffle scan over the lanes of one nodal cell
    // (fp32 shuffles are single instructions and FAST32 has registers for the lane geometry);
    // writes the same in-place row layout as xstage
    struct Lane {
        Real rx;
        int bx;        // local nodal cell of the column (1024 + lane past the volume)
        int sst;       // first lane of the column's segment
        bool send, xin, xlast;
    };
    __device__ Lane lane_geom(const FArgs& a, int x0, int nxA, int lane) const {
        const int mx = static_cast<int>(a.g.m[0]);
        const int gx = x0 + lane, gxc = min(gx, mx - 1), xe = min(mx, x0 + kPtcTX);
        Lane L;
        L.xin = gx < mx;
        L.xlast = gx == xe - 1;
        L.bx = L.xin ? __ldg(&a.P.base[0][gxc]) - nxA : 1024 + lane;
        L.rx = static_cast<Real>(__ldg(&a.P.rem[0][gxc]));
        const int bx_prev = __shfl_up_sync(0xffffffffu, L.bx, 1);
        const unsigned starts = __ballot_sync(0xffffffffu, lane == 0 || bx_prev != L.bx);
        L.sst = 31 - __clz(starts & (0xffffffffu >> (31 - lane)));
        L.send = lane == 31 || ((starts >> (lane + 1)) & 1u);
        return L;
    }
    __device__ void xstage_shfl(int row, int lane, const Lane& g, int segw, Real v0, Real v1, Real v2) const {
        Real* dst = sA + row * XR;
        const int nlx_t = nxi / 3;
        Real A[3] = {(Real(1) - g.rx) * v0, (Real(1) - g.rx) * v1, (Real(1) - g.rx) * v2};
        Real B[3] = {g.rx * v0, g.rx * v1, g.rx * v2};
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            if (o >= segw) break;  // uniform
            const bool in = lane - o >= g.sst;
#pragma unroll
            for (int d = 0; d < 3; ++d) {
                const Real ua = __shfl_up_sync(0xffffffffu, A[d], o);
                const Real ub = __shfl_up_sync(0xffffffffu, B[d], o);
                A[d] = in ? A[d] + ua : A[d];
                B[d] = in ? B[d] + ub : B[d];
            }
        }
        __syncwarp();  // (the y stage of the previous completion read this row two steps ago)
#pragma unroll
        for (int d = 0; d < 3; ++d) {
            const Real bp = __shfl_sync(0xffffffffu, B[d], max(g.sst - 1, 0));
            if (g.send && g.xin) {
                dst[ptc_phys(d * nlx_t + g.bx)] = g.sst > 0 ? A[d] + bp : A[d];
                if (g.xlast) dst[ptc_phys(d * nlx_t + g.bx + 1)] = B[d];
            }
        }
    }
    // y stage into the tile partial of one nodal plane (node row lyn on warp TY-1-lyn: the halo
    // items sit on the lowest warps)
    __device__ void ystage(int row, int lane, Real* pz) const {
        for (int lyn = TY - 1 - row; lyn < nly_t; lyn += TY) {
            const Real* w = sWy + lyn * TY;
            for (int L = lane; L < nxi; L += 32) {
                const int e = sXi[L];
                const int j = (e >> 20) & 0x3f, d = e >> 26;
                Real v = Real(0);
#pragma unroll
                const Real* col = sA + ptc_phys(L);
#pragma unroll
                for (int r = 0; r < TY; ++r) v = fma(w[r], col[r * XR], v);
                pz[(lyn * nlx + j) * 3 + d] = v;
            }
        }
    }
};

}  // namespace fdev
}  // namespace mfreg_b200
