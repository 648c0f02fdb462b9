// Fused fast-mode kernels (see fused.cuh for the algebra and execution scheme).
#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <type_traits>
#include <vector>

#include <cuda.h>
#include <cudaTypedefs.h>

#include "fused.cuh"
#include "fused_dev.cuh"

namespace mfreg_b200 {

// hv_fast.cu
std::size_t hv2_smem_bytes(int nlx, int nly, int segw, int zc, int nsl, bool fp32, int ty);
int hv2_nsl_max(int ty);
int hv2_box_origin(bool fp32);
int hv2_nlx_max();
int hv2_threads(int ty);
void hv2_set_smem_cap(int bytes, int ty);
void hv2_launch(const fdev::FArgs& a, const fdev::TmaMaps& maps, dim3 grid, std::size_t smem, cudaStream_t s, bool fp32,
                int ty);
// hv3.cu
std::size_t hv3_smem_bytes(int nlx, int nsl, int zc, bool fp32, bool stored);
int hv3_tile_x();
int hv3_tile_y();
int hv3_threads();
int hv3_box_width(bool fp32);
int hv3_box_rows();
int hv3_box_origin(bool fp32);
void hv3_set_smem_cap(int bytes);
bool hv3_fp32_ok();
void hv3_launch(const fdev::FArgs& a, const fdev::TmaMaps& maps, dim3 grid, std::size_t smem, cudaStream_t s, bool fp32,
                bool stored);
// ev_fast.cu
std::size_t ev2_smem_bytes(int nlx, int nly, int segw, bool fp32);
void ev2_set_smem_cap(int bytes);
void ev_value_launch(const fdev::FArgs& a, const void* R, const void* Tw, dim3 grid, cudaStream_t s, bool fp32);
void ev2_launch(const fdev::FArgs& a, const fdev::TmaMaps& maps, dim3 grid, std::size_t smem, cudaStream_t s, bool fp32);

namespace {

using namespace fdev;

constexpr int CX = FT_X + 4, CY = FT_Y + 4, NC = CX * CY;  // halo-2 column region (36 x 12 = 432)
constexpr int C1X = FT_X + 2, C1Y = FT_Y + 2, NC1 = C1X * C1Y;  // halo-1 region (34 x 10 = 340)
constexpr int TT = FT_X * FT_Y;                              // output columns (256)
// warp-aligned thread roles: tile (warps 0-7), halo-1 ring (warps 8-10), halo-2 ring (warps 11-13)
constexpr int R1_0 = TT, R1_N = NC1 - TT;                    // 84 halo-1 ring columns
constexpr int R2_0 = 352, R2_N = NC - NC1;                   // 92 halo-2 ring columns
constexpr int NTH = 448;
constexpr int DEPTH_EV = 4;  // staging ring, eval pass (TMA, loads 2 planes ahead)
constexpr int DEPTH_HV = 5;  // Hv pass: also keeps plane k-2 (rho-hat of the Z stage, dT of q^)
constexpr int NBUF_EV = 14;  // plane buffers (NB doubles): eval R, T_w, r (x2), rho-hat in-plane (x8)
constexpr int NBUF_HV = 6;   // Hv: s, w (x2) (+2 unused)
constexpr int NSLAB = 8;                                     // nodal-slab ring (planes, power of 2)
constexpr int PAD = CX + 1;                                  // guard around the plane buffers
constexpr int NB = NC + 2 * PAD;
constexpr int kSMs = 148;
constexpr int kSmem2Cta = 115712;  // dynamic shared memory per CTA with two CTAs per SM (228 KB - 2 x 1 KB reserved)
// staging slot layouts (bytes, 128-aligned): TMA boxes land as [comp][y][x]
constexpr int HV_DT = 3 * NC;                  // doubles: dT box 36x12x3
constexpr int HV_RH = 6 * NC;                  // doubles: rho-hat box 36x12x6
constexpr int HV_SLOT = HV_DT + HV_RH;         // 3888 doubles = 31104 B
constexpr int EV_SLOT = 5 * NC;                // R, T_w, dT(3) boxes 36x12: 2160 doubles = 17280 B

template <bool EVAL, bool TMA>
__global__ void __launch_bounds__(NTH, 1) k_fused(const __grid_constant__ FArgs a, const __grid_constant__ TmaMaps maps) {
    extern __shared__ __align__(128) double sm[];
    if (a.skip && *a.skip) return;  // uniform
    const TileMeta& tm = a.tm;
    const int nlx = tm.nlx;
    // ---- shared memory carve-up (doubles); the staging ring comes first (128-byte aligned)
    constexpr int SLOT = EVAL ? EV_SLOT : HV_SLOT;
    constexpr int DEPTH = EVAL ? DEPTH_EV : DEPTH_HV;
    constexpr int NBUF = EVAL ? NBUF_EV : NBUF_HV;
    double* stg = sm;                      // [DEPTH][SLOT]
    double* sP0 = stg + DEPTH * SLOT + PAD;  // [2][NB] Hv: s; eval: R (by plane parity)
    double* sP1 = sP0 + 2 * NB;            // [2][NB] eval: T_w
    double* sW = sP1 + 2 * NB;             // [2][NB] Hv: w; eval: r
    double* sRh = sW + 2 * NB;             // [2][4][NB] in-plane rho-hat (-x,+x,-y,+y)
    double* sDq = sP0 + NBUF * NB - PAD;   // eval: [3][3][TT] dT of the tile columns (planes k, k-1, k-2)
    double* sQ = sDq + (EVAL ? 9 * TT : 0);  // [3][TT]
    double* sQx = sQ + 3 * TT;             // [3][FT_Y][nlx]
    double* sZr = sQx + 3 * FT_Y * nlx;    // [zc + 8] rem_z per plane
    double* sremx = sZr + tm.zc + 8;
    double* sremy = sremx + FT_X;
    double* slab = sremy + FT_Y;          // [NSLAB][nxf*nyf*3] nodal p (Hv)
    int* sZb = reinterpret_cast<int*>(slab + (EVAL ? 0 : NSLAB * a.nxf * a.nyf * 3));  // [zc + 8]
    int* sXr = sZb + tm.zc + 8;            // [nlx][4] x ranges of the spread tasks
    int* sYr = sXr + 4 * nlx;              // [nly][4]
    unsigned long long* bars = reinterpret_cast<unsigned long long*>(
        (reinterpret_cast<std::uintptr_t>(sYr + 4 * tm.nly) + 15) & ~static_cast<std::uintptr_t>(15));  // [DEPTH]
    double* sred = reinterpret_cast<double*>(bars + DEPTH);  // [32]

    const int tid = threadIdx.x;
    const int mx = static_cast<int>(a.g.m[0]), my = static_cast<int>(a.g.m[1]), mz = static_cast<int>(a.g.m[2]);
    const long long n = a.g.count(), plane = static_cast<long long>(mx) * my;
    const int x0 = blockIdx.x * FT_X, y0 = blockIdx.y * FT_Y;
    const int z0 = tm.zlo + static_cast<int>(blockIdx.z) * tm.zc, z1 = min(tm.zhi, z0 + tm.zc);
    const int ilo = max(z0, a.olo), ihi = min(z1, a.ohi);  // planes with outputs (D, P^T)
    const int xe = min(mx, x0 + FT_X), ye = min(my, y0 + FT_Y);
    const int nxA = __ldg(&a.P.base[0][x0]), nyA = __ldg(&a.P.base[1][y0]), nzA = __ldg(&a.P.base[2][z0]);
    const int nlx_t = __ldg(&a.P.base[0][xe - 1]) - nxA + 2;
    const int nly_t = __ldg(&a.P.base[1][ye - 1]) - nyA + 2;
    const long long tile_id = (static_cast<long long>(blockIdx.z) * tm.nty + blockIdx.y) * tm.ntx + blockIdx.x;
    double* part = a.part + tile_id * tm.part_stride;
    const std::size_t pstride = static_cast<std::size_t>(tm.nly) * nlx * 3;

    // ---- thread -> column (roles are warp-aligned, so role branches are uniform)
    const int role = tid < TT ? 0 : (tid < R2_0 ? 1 : 2);
    bool active = true;
    int lx, ly;
    if (role == 0) {
        lx = 2 + tid % FT_X;
        ly = 2 + tid / FT_X;
    } else if (role == 1) {
        const int r = tid - R1_0;  // 84 = 34 + 34 + 8 + 8
        active = r < R1_N;
        if (r < C1X) { lx = 1 + r; ly = 1; }
        else if (r < 2 * C1X) { lx = 1 + r - C1X; ly = CY - 2; }
        else if (r < 2 * C1X + FT_Y) { lx = 1; ly = 2 + r - 2 * C1X; }
        else if (r < R1_N) { lx = CX - 2; ly = 2 + r - 2 * C1X - FT_Y; }
        else { lx = 1; ly = 1; }
    } else {
        const int r = tid - R2_0;  // 92 = 36 + 36 + 10 + 10
        active = r < R2_N;
        if (r < CX) { lx = r; ly = 0; }
        else if (r < 2 * CX) { lx = r - CX; ly = CY - 1; }
        else if (r < 2 * CX + CY - 2) { lx = 0; ly = 1 + r - 2 * CX; }
        else if (r < R2_N) { lx = CX - 1; ly = 1 + r - 2 * CX - (CY - 2); }
        else { lx = 0; ly = 0; }
    }
    const int c = lx + ly * CX;                // halo-2 layout index
    const int c1 = (lx - 1) + (ly - 1) * C1X;  // halo-1 layout index (roles 0, 1)
    const int gx = x0 - 2 + lx, gy = y0 - 2 + ly;
    const bool indom = active && gx >= 0 && gx < mx && gy >= 0 && gy < my;
    const bool tile = role == 0 && gx < mx && gy < my;
    const long long col = indom ? static_cast<long long>(gx) + static_cast<long long>(gy) * mx : 0;
    // boundary masks (staged values outside the volume are zero; differences across
    // the boundary must vanish exactly, as the reference's clamped neighbours)
    const double mxm = gx > 0 ? 1.0 : 0.0, mxp = gx + 1 < mx ? 1.0 : 0.0;
    const double mym = gy > 0 ? 1.0 : 0.0, myp = gy + 1 < my ? 1.0 : 0.0;

    // ---- per-CTA tables
    for (int t = tid; t < tm.zc + 8; t += NTH) {
        const int kk = min(max(z0 - 2 + t, 0), mz - 1);
        sZb[t] = __ldg(&a.P.base[2][kk]);
        sZr[t] = __ldg(&a.P.rem[2][kk]);
    }
    if (tid < FT_X) sremx[tid] = x0 + tid < mx ? __ldg(&a.P.rem[0][x0 + tid]) : 0.0;
    if (tid < FT_Y) sremy[tid] = y0 + tid < my ? __ldg(&a.P.rem[1][y0 + tid]) : 0.0;
    {
        const int nsx = static_cast<int>(a.P.src.m[0]) - 1, nsy = static_cast<int>(a.P.src.m[1]) - 1;
        for (int t = tid; t < nlx_t; t += NTH) {  // cells nx-1 (weight r) and nx (weight 1-r), clipped to the tile
            const int nx = nxA + t;
            int lo1 = x0, hi1 = x0, lo0 = x0, hi0 = x0;
            if (nx >= 1 && nx - 1 < nsx) {
                lo1 = max(x0, __ldg(&a.P.cell_lo[0][nx - 1]));
                hi1 = max(lo1, min(xe, __ldg(&a.P.cell_hi[0][nx - 1])));
            }
            if (nx < nsx) {
                lo0 = max(x0, __ldg(&a.P.cell_lo[0][nx]));
                hi0 = max(lo0, min(xe, __ldg(&a.P.cell_hi[0][nx])));
            }
            sXr[4 * t] = lo1 - x0;
            sXr[4 * t + 1] = hi1 - x0;
            sXr[4 * t + 2] = lo0 - x0;
            sXr[4 * t + 3] = hi0 - x0;
        }
        for (int t = tid; t < nly_t; t += NTH) {
            const int ny = nyA + t;
            int lo1 = y0, hi1 = y0, lo0 = y0, hi0 = y0;
            if (ny >= 1 && ny - 1 < nsy) {
                lo1 = max(y0, __ldg(&a.P.cell_lo[1][ny - 1]));
                hi1 = max(lo1, min(ye, __ldg(&a.P.cell_hi[1][ny - 1])));
            }
            if (ny < nsy) {
                lo0 = max(y0, __ldg(&a.P.cell_lo[1][ny]));
                hi0 = max(lo0, min(ye, __ldg(&a.P.cell_hi[1][ny])));
            }
            sYr[4 * t] = lo1 - y0;
            sYr[4 * t + 1] = hi1 - y0;
            sYr[4 * t + 2] = lo0 - y0;
            sYr[4 * t + 3] = hi0 - y0;
        }
    }
    if (tid < 2 * PAD) {  // zero the guard pads of the plane buffers
        const int o = tid < PAD ? -PAD + tid : NC + (tid - PAD);
        for (int b = 0; b < NBUF; ++b) sP0[b * NB + o] = 0.0;
    }
    if (TMA && tid == 0) {
        for (int b = 0; b < DEPTH; ++b) mbar_init(&bars[b], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }

    // ---- nodal slab (Hv): x-y footprint of the halo-2 columns, ring of nodal planes
    const int fx0 = __ldg(&a.P.base[0][max(x0 - 2, 0)]);
    const int fy0 = __ldg(&a.P.base[1][max(y0 - 2, 0)]);
    const int nxf = a.nxf, nyf = a.nyf, nsl = nxf * nyf * 3;
    const long long ns = a.P.src.count(), sm0 = a.P.src.m[0], sm01 = a.P.src.m[0] * a.P.src.m[1];
    const int msx = static_cast<int>(a.P.src.m[0]), msy = static_cast<int>(a.P.src.m[1]);
    const int msz = static_cast<int>(a.P.src.m[2]);
    const int gxc = min(max(gx, 0), mx - 1), gyc = min(max(gy, 0), my - 1);
    const int bxl = __ldg(&a.P.base[0][gxc]) - fx0, byl = __ldg(&a.P.base[1][gyc]) - fy0;
    const double rx = __ldg(&a.P.rem[0][gxc]), ry = __ldg(&a.P.rem[1][gyc]);
    // per-thread slab elements (up to 4 per thread; host guarantees nsl <= 4 * NTH):
    // global offsets precomputed once (no integer division in the plane loop)
    double slab_v[4];
    long long slab_off[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        const int t = tid + u * NTH;
        slab_off[u] = -1;
        if (!EVAL && t < nsl) {
            const int ix = t % nxf, iy = (t / nxf) % nyf, d = t / (nxf * nyf);
            const int gxn = min(fx0 + ix, msx - 1), gyn = min(fy0 + iy, msy - 1);
            slab_off[u] = d * ns + gxn + gyn * sm0;
        }
    }
    auto slab_load = [&](int nz) {
#pragma unroll
        for (int u = 0; u < 4; ++u)
            if (slab_off[u] >= 0) slab_v[u] = __ldg(a.p + slab_off[u] + static_cast<long long>(nz) * sm01);
    };
    auto slab_store = [&](int nz) {
        double* dst = slab + (nz & (NSLAB - 1)) * nsl;
#pragma unroll
        for (int u = 0; u < 4; ++u)
            if (slab_off[u] >= 0) dst[tid + u * NTH] = slab_v[u];
    };
    auto slab_bilerp = [&](int nz, double& o0, double& o1, double& o2) {
        const double* q = slab + (nz & (NSLAB - 1)) * nsl + bxl + byl * nxf;
        const int pl = nxf * nyf;
        o0 = lerp(ry, lerp(rx, q[0], q[1]), lerp(rx, q[nxf], q[nxf + 1]));
        o1 = lerp(ry, lerp(rx, q[pl], q[pl + 1]), lerp(rx, q[pl + nxf], q[pl + nxf + 1]));
        o2 = lerp(ry, lerp(rx, q[2 * pl], q[2 * pl + 1]), lerp(rx, q[2 * pl + nxf], q[2 * pl + nxf + 1]));
    };

    // ---- staging of plane m into its ring slot: TMA (one thread, zero fill outside
    // the volume) or, for row strides TMA cannot address, per-thread loads with the
    // same zero-fill semantics
    auto stage_issue = [&](int m) {
        const int mr = m - (z0 - 2);
        double* st = stg + (mr % DEPTH) * SLOT;
        if (TMA) {
            if (tid < 32 && elect_one()) {  // warp 0 is converged here; one lane issues
                unsigned long long* bar = &bars[mr % DEPTH];
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                if (EVAL) {
                    mbar_expect_tx(bar, EV_SLOT * 8);
                    tma_load_3d(st, &maps.a, x0 - 2, y0 - 2, m, bar);
                    tma_load_3d(st + NC, &maps.b, x0 - 2, y0 - 2, m, bar);
                    tma_load_4d(st + 2 * NC, &maps.c, x0 - 2, y0 - 2, m, 0, bar);
                } else {
                    mbar_expect_tx(bar, HV_SLOT * 8);
                    tma_load_4d(st, &maps.a, x0 - 2, y0 - 2, m, 0, bar);
                    tma_load_4d(st + HV_DT, &maps.b, x0 - 2, y0 - 2, m, 0, bar);
                }
            }
        } else if (active) {
            const bool ok = indom && m >= 0 && m < mz;
            const long long o = col + static_cast<long long>(ok ? m : 0) * plane;
            if (EVAL) {
                st[c] = ok ? __ldg(a.R + o) : 0.0;
                st[NC + c] = ok ? __ldg(a.Tw + o) : 0.0;
                st[2 * NC + c] = ok ? __ldg(a.dT + o) : 0.0;
                st[3 * NC + c] = ok ? __ldg(a.dT + n + o) : 0.0;
                st[4 * NC + c] = ok ? __ldg(a.dT + 2 * n + o) : 0.0;
            } else {
                st[c] = ok ? __ldg(a.dT + o) : 0.0;
                st[NC + c] = ok ? __ldg(a.dT + n + o) : 0.0;
                st[2 * NC + c] = ok ? __ldg(a.dT + 2 * n + o) : 0.0;
                if (role < 2) {
#pragma unroll
                    for (int d = 0; d < 6; ++d) st[HV_DT + d * NC + c] = ok ? __ldg(a.frh + d * n + o) : 0.0;
                }
            }
        }
    };
    auto stage_wait = [&](int m) {
        if (TMA) {
            const int mr = m - (z0 - 2);
            mbar_wait(&bars[mr % DEPTH], (mr / DEPTH) & 1);
        }
    };

    __syncthreads();  // tables and barriers ready
    int pz = -1000, slab_hi = -1;
    double Pa0 = 0.0, Pa1 = 0.0, Pa2 = 0.0, Pb0 = 0.0, Pb1 = 0.0, Pb2 = 0.0;
    if (!EVAL) {  // the first two nodal planes, synchronously
        // every nodal plane the first three planes read (later steps prefetch for plane k+3)
        const int nz0 = sZb[0];
        slab_hi = min(sZb[2] + 1, msz - 1);
        for (int nz = nz0; nz <= slab_hi; ++nz) {
            slab_load(nz);
            slab_store(nz);
        }
    }
    stage_issue(z0 - 2);
    stage_issue(z0 - 1);
    __syncthreads();

    // x-y spread of one completed nodal plane: per-column z-accumulated values ->
    // sQ -> x-collapse (all threads) -> sQx -> y-collapse (all threads) -> partial
    // spread work items: x-collapse (d, row, local node x), y-collapse (d, local node y, x);
    // the first item of each thread is decomposed once here, further items (fine
    // deformation grids only) in the loop
    const int nxi = 3 * FT_Y * nlx_t, nyi = 3 * nly_t * nlx_t;
    const int x_lxn = tid % nlx_t, x_row = (tid / nlx_t) % FT_Y, x_d = tid / (nlx_t * FT_Y);
    const int y_lxn = tid % nlx_t, y_lyn = (tid / nlx_t) % nly_t, y_d = tid / (nlx_t * nly_t);
    auto xitem = [&](int lxn, int row, int d) {
        const int* xr = sXr + 4 * lxn;
        const double* q = sQ + d * TT + row * FT_X;
        double s1 = 0.0, s2 = 0.0;
        for (int x = xr[0]; x < xr[1]; ++x) s1 = fma(sremx[x], q[x], s1);
        for (int x = xr[2]; x < xr[3]; ++x) s2 = fma(1.0 - sremx[x], q[x], s2);
        sQx[(d * FT_Y + row) * nlx + lxn] = s1 + s2;
    };
    auto yitem = [&](int lxn, int lyn, int d, double* dst) {
        const int* yr = sYr + 4 * lyn;
        const double* q = sQx + d * FT_Y * nlx + lxn;
        double s1 = 0.0, s2 = 0.0;
        for (int y = yr[0]; y < yr[1]; ++y) s1 = fma(sremy[y], q[y * nlx], s1);
        for (int y = yr[2]; y < yr[3]; ++y) s2 = fma(1.0 - sremy[y], q[y * nlx], s2);
        dst[(lyn * nlx + lxn) * 3 + d] = s1 + s2;
    };
    // x-y spread of one completed nodal plane: per-column z-accumulated values ->
    // sQ -> x-collapse (all threads) -> sQx -> y-collapse (all threads) -> partial
    auto spread = [&](double v0, double v1, double v2, int nzp) {
        if (role == 0) {
            sQ[tid] = v0;
            sQ[TT + tid] = v1;
            sQ[2 * TT + tid] = v2;
        }
        __syncthreads();
        if (tid < nxi) xitem(x_lxn, x_row, x_d);
        for (int t = tid + NTH; t < nxi; t += NTH) xitem(t % nlx_t, (t / nlx_t) % FT_Y, t / (nlx_t * FT_Y));
        __syncthreads();
        double* dst = part + static_cast<std::size_t>(nzp - nzA) * pstride;
        if (tid < nyi) yitem(y_lxn, y_lyn, y_d, dst);
        for (int t = tid + NTH; t < nyi; t += NTH) yitem(t % nlx_t, (t / nlx_t) % nly_t, t / (nlx_t * nly_t), dst);
    };
    double acc00 = 0.0, acc01 = 0.0, acc02 = 0.0, acc10 = 0.0, acc11 = 0.0, acc12 = 0.0;

    // rotating buffer pointers (column position c folded in once)
    double* bA_cur = sP0 + c;          // Hv: s; eval: R  -- plane k
    double* bA_prv = sP0 + NB + c;     //                  -- plane k-1
    double* bB_cur = sP1 + c;          // eval: T_w
    double* bB_prv = sP1 + NB + c;
    double* bW_new = sW + c;           // w / r of plane k-1 (written this iteration)
    double* bW_old = sW + NB + c;      // w / r of plane k-2 (read this iteration)
    double* bR_new = sRh + c;          // in-plane rho-hat of plane k-1
    double* bR_old = sRh + 4 * NB + c; // in-plane rho-hat of plane k-2
    double* dq_w = sDq + tid;          // tile dT ring: plane k (write)
    double* dq_1 = sDq + 3 * TT + tid; //               plane k-1
    double* dq_r = sDq + 6 * TT + tid; //               plane k-2 (read)
    const double* st_k = stg + c;                        // staged plane k (dT / R,T)
    const double* st_r = stg + (DEPTH - 1) * SLOT + HV_DT + c;  // staged rho-hat of plane k-1 (Hv)
    const double hx = a.hh[0], hy = a.hh[1], hz = a.hh[2];

    // column histories (plane index relative to the current iteration k)
    double sh1 = 0.0, sh2 = 0.0;                        // Hv: s_{k-1}, s_{k-2}
    double Rh1 = 0.0, Rh2 = 0.0, Th1 = 0.0, Th2 = 0.0;  // eval: R, T_w at k-1, k-2
    double wh1 = 0.0, wh2 = 0.0;                        // w (or r) at k-2, k-3
    double sg1 = 0.0;                                   // sigma at k-2
    double pzh1 = 0.0, pzh2 = 0.0;                      // rho-hat(+z) at k-2, k-3
    double dsum = 0.0;
    int cur = nzA;  // nodal plane held in accumulator slot 0
    const bool do_z = !EVAL || a.grad;

  if constexpr (EVAL) {
#pragma unroll 1
    for (int k = z0 - 2; k <= z1 + 1; ++k) {
        const int kt = k - (z0 - 2);  // index into the per-CTA z tables
        stage_issue(k + 2);
        bool slab_pending = false;
        int slab_nz = 0;
        if (!EVAL) {  // nodal plane needed by plane k+3, loaded now, stored at the end of the iteration
            const int nzq = min(sZb[kt + 3] + 1, msz - 1);
            if (nzq > slab_hi) {  // next plane now; any further ones (cells of 1 plane) at the store
                slab_load(slab_hi + 1);
                slab_pending = true;
                slab_nz = nzq;
            }
            const int bz = sZb[kt];
            if (bz != pz) {  // uniform across the CTA: new nodal plane pair for P p
                if (bz == pz + 1) {
                    Pa0 = Pb0;
                    Pa1 = Pb1;
                    Pa2 = Pb2;
                } else {
                    slab_bilerp(bz, Pa0, Pa1, Pa2);
                }
                slab_bilerp(min(bz + 1, msz - 1), Pb0, Pb1, Pb2);
                pz = bz;
            }
        }
        const int i = k - 2, j = k - 1;
        const bool iout = do_z && i >= ilo && i < ihi;  // uniform
        const double rzk = sZr[kt];
        stage_wait(k);

        double s0 = 0.0, A0 = 0.0, B0 = 0.0;
        double wc = 0.0, sgc = 0.0, mzc = 0.0, pzc = 0.0;  // fresh values of plane j
        double q0 = 0.0, q1 = 0.0, q2 = 0.0;
        if (role < 2) {
            // ---- P: plane k
            if (!EVAL) {
                const double D0 = st_k[0], D1 = st_k[NC], D2 = st_k[2 * NC];
                s0 = fma(D0, lerp(rzk, Pa0, Pb0), fma(D1, lerp(rzk, Pa1, Pb1), D2 * lerp(rzk, Pa2, Pb2)));
                bA_cur[0] = s0;
                if (role == 0) {
                    dq_w[0] = D0;
                    dq_w[TT] = D1;
                    dq_w[2 * TT] = D2;
                }
            } else {
                A0 = st_k[0];
                B0 = st_k[NC];
                bA_cur[0] = A0;
                bB_cur[0] = B0;
                if (role == 0) {
                    dq_w[0] = st_k[2 * NC];
                    dq_w[TT] = st_k[3 * NC];
                    dq_w[2 * TT] = st_k[4 * NC];
                }
            }
            // ---- W: plane j = k-1 (reads buffers of the previous iteration)
            if (!EVAL) {
                const double r0 = st_r[0], r1 = st_r[NC], r2 = st_r[2 * NC], r3 = st_r[3 * NC], r4 = st_r[4 * NC],
                             r5 = st_r[5 * NC];
                const double sj = sh1;
                wc = r0 * (bA_prv[-1] - sj);
                wc = fma(r1, bA_prv[1] - sj, wc);
                wc = fma(r2, bA_prv[-CX] - sj, wc);
                wc = fma(r3, bA_prv[CX] - sj, wc);
                wc = fma(r4, sh2 - sj, wc);
                wc = fma(r5, s0 - sj, wc);
                sgc = ((r0 + r1) + (r2 + r3)) + (r4 + r5);
                mzc = r4;
                pzc = r5;
                bR_new[0] = r0;
                bR_new[NB] = r1;
                bR_new[2 * NB] = r2;
                bR_new[3 * NB] = r3;
            } else {
                const double Rj = Rh1, Tj = Th1;
                const double mzm = j > 0 ? 1.0 : 0.0, mzp = j + 1 < mz ? 1.0 : 0.0;
                const double dR0 = mxm * (bA_prv[-1] - Rj), dR1 = mxp * (bA_prv[1] - Rj);
                const double dR2 = mym * (bA_prv[-CX] - Rj), dR3 = myp * (bA_prv[CX] - Rj);
                const double dR4 = mzm * (Rh2 - Rj), dR5 = mzp * (A0 - Rj);
                const double dT0 = mxm * (bB_prv[-1] - Tj), dT1 = mxp * (bB_prv[1] - Tj);
                const double dT2 = mym * (bB_prv[-CX] - Tj), dT3 = myp * (bB_prv[CX] - Tj);
                const double dT4 = mzm * (Th2 - Tj), dT5 = mzp * (B0 - Tj);
                const double i0 = a.ih2[0], i1 = a.ih2[1], i2 = a.ih2[2];
                const double stt = fma(fma(dT0, dT0, dT1 * dT1), i0, fma(fma(dT2, dT2, dT3 * dT3), i1, fma(dT4, dT4, dT5 * dT5) * i2));
                const double srr = fma(fma(dR0, dR0, dR1 * dR1), i0, fma(fma(dR2, dR2, dR3 * dR3), i1, fma(dR4, dR4, dR5 * dR5) * i2));
                const double num = fma(0.5, fma(fma(dT0, dR0, dT1 * dR1), i0, fma(fma(dT2, dR2, dT3 * dR3), i1, fma(dT4, dR4, dT5 * dR5) * i2)),
                                       a.tau * a.rho);
                const double itn = rsqrt(fma(0.5, stt, a.tau * a.tau));
                const double irn = rsqrt(fma(0.5, srr, a.rho * a.rho));
                const double in1 = itn * irn;
                const double in2 = num * (itn * itn) * in1;
                const bool ok = indom && j >= 0 && j < mz;
                const double e0 = ok ? hx * fma(dR0, in1, -dT0 * in2) : 0.0;
                const double e1 = ok ? hx * fma(dR1, in1, -dT1 * in2) : 0.0;
                const double e2 = ok ? hy * fma(dR2, in1, -dT2 * in2) : 0.0;
                const double e3 = ok ? hy * fma(dR3, in1, -dT3 * in2) : 0.0;
                const double e4 = ok ? hz * fma(dR4, in1, -dT4 * in2) : 0.0;
                const double e5 = ok ? hz * fma(dR5, in1, -dT5 * in2) : 0.0;
                const double r = ok ? num * in1 : 0.0;
                wc = r;
                sgc = ((e0 + e1) + (e2 + e3)) + (e4 + e5);
                mzc = e4;
                pzc = e5;
                bR_new[0] = e0;
                bR_new[NB] = e1;
                bR_new[2 * NB] = e2;
                bR_new[3 * NB] = e3;
                if (tile && j >= z0 && j < z1) {
                    const long long gi = col + static_cast<long long>(j) * plane;
                    if (a.frh_out) {  // none when value-only lazy
                        a.frh_out[gi] = e0;
                        a.frh_out[n + gi] = e1;
                        a.frh_out[2 * n + gi] = e2;
                        a.frh_out[3 * n + gi] = e3;
                        a.frh_out[4 * n + gi] = e4;
                        a.frh_out[5 * n + gi] = e5;
                    }
                    if (j >= ilo && j < ihi) dsum += fma(-r, r, 1.0);
                }
            }
            bW_new[0] = wc;
            // ---- Z: plane i = k-2 (tile columns)
            if (role == 0 && iout) {
                // neighbour coefficient toward i: +x neighbour holds (-x), -x neighbour holds (+x), ...
                double z = bR_old[NB - 1] * bW_old[-1];
                z = fma(bR_old[1], bW_old[1], z);
                z = fma(bR_old[3 * NB - CX], bW_old[-CX], z);
                z = fma(bR_old[2 * NB + CX], bW_old[CX], z);
                z = fma(mzc, wc, z);      // rho-hat_{i+z}(-z) w_{i+z}
                z = fma(pzh2, wh2, z);    // rho-hat_{i-z}(+z) w_{i-z}
                z = fma(-sg1, wh1, z);    // -sigma_i w_i
                const double sz = tile ? a.scale * z : 0.0;
                q0 = sz * dq_r[0];
                q1 = sz * dq_r[TT];
                q2 = sz * dq_r[2 * TT];
            }
        } else {
            // halo-2 ring: P only
            if (!EVAL) {
                s0 = fma(st_k[0], lerp(rzk, Pa0, Pb0), fma(st_k[NC], lerp(rzk, Pa1, Pb1), st_k[2 * NC] * lerp(rzk, Pa2, Pb2)));
                bA_cur[0] = s0;
            } else {
                A0 = st_k[0];
                B0 = st_k[NC];
                bA_cur[0] = A0;
                bB_cur[0] = B0;
            }
        }
        if (iout) {
            const int bz = sZb[kt - 2];
            const double rz = sZr[kt - 2];
            if (bz > cur) {  // nodal plane `cur` complete: x-y spread (all threads)
                spread(acc00, acc01, acc02, cur);
                acc00 = acc10;
                acc01 = acc11;
                acc02 = acc12;
                acc10 = acc11 = acc12 = 0.0;
                cur = bz;
            }
            acc00 = fma(1.0 - rz, q0, acc00);
            acc10 = fma(rz, q0, acc10);
            acc01 = fma(1.0 - rz, q1, acc01);
            acc11 = fma(rz, q1, acc11);
            acc02 = fma(1.0 - rz, q2, acc02);
            acc12 = fma(rz, q2, acc12);
        }
        if (slab_pending) {
            slab_store(slab_hi + 1);
            for (int nz = slab_hi + 2; nz <= slab_nz; ++nz) {
                slab_load(nz);
                slab_store(nz);
            }
            slab_hi = slab_nz;
        }
        __syncthreads();
        // ---- rotate histories and buffer pointers
        sh2 = sh1;
        sh1 = s0;
        Rh2 = Rh1;
        Rh1 = A0;
        Th2 = Th1;
        Th1 = B0;
        wh2 = wh1;
        wh1 = wc;
        sg1 = sgc;
        pzh2 = pzh1;
        pzh1 = pzc;
        {
            double* t;
            t = bA_cur; bA_cur = bA_prv; bA_prv = t;
            t = bB_cur; bB_cur = bB_prv; bB_prv = t;
            t = bW_new; bW_new = bW_old; bW_old = t;
            t = bR_new; bR_new = bR_old; bR_old = t;
            t = dq_r; dq_r = dq_1; dq_1 = dq_w; dq_w = t;
            st_r = st_k + HV_DT;
            st_k = (kt & (DEPTH - 1)) == DEPTH - 1 ? st_k - (DEPTH - 1) * SLOT : st_k + SLOT;
        }
    }
  } else {
    // ---- Hv: P (plane k) -> W (plane j = k-1) -> Z (plane i = k-2), one barrier per plane.
    // The staging ring keeps planes k-2 .. k+2, so the Z stage reads its neighbours'
    // rho-hat and its own dT straight from the staged slot of plane i. The loop is
    // unrolled by two with parity-named registers / buffers (no rotation moves):
    // on entry to a step of parity P, s_{k-2} = sr[P], s_{k-1} = sr[1-P],
    // w_{k-2} = wr[P], w_{k-3} = wr[1-P], rho-hat_{k-3}(+z) = pr[1-P], sigma_{k-2} = gr[P].
    double sr[2] = {0.0, 0.0}, wr[2] = {0.0, 0.0}, pr[2] = {0.0, 0.0}, gr[2] = {0.0, 0.0};
    double* const sS = sP0 + c;  // s planes [2][NB] (by plane parity)
    double* const sWv = sW + c;  // w planes [2][NB]
    const int kfirst = z0 - 2, klast = z1 + 1;
    auto slot_of = [&](int m) { return stg + ((m - kfirst + DEPTH) % DEPTH) * SLOT + c; };  // m >= kfirst - 2
    auto step = [&](auto parc, int k) {
        constexpr int P = decltype(parc)::value;
        const int kt = k - kfirst;
        stage_issue(k + 2);
        bool slab_pending = false;
        int slab_nz = 0;
        {  // nodal plane needed by plane k+3, loaded now, stored at the end of the step
            const int nzq = min(sZb[kt + 3] + 1, msz - 1);
            if (nzq > slab_hi) {  // next plane now; any further ones (cells of 1 plane) at the store
                slab_load(slab_hi + 1);
                slab_pending = true;
                slab_nz = nzq;
            }
            const int bz = sZb[kt];
            if (bz != pz) {  // uniform: new nodal plane pair for P p
                if (bz == pz + 1) {
                    Pa0 = Pb0;
                    Pa1 = Pb1;
                    Pa2 = Pb2;
                } else {
                    slab_bilerp(bz, Pa0, Pa1, Pa2);
                }
                slab_bilerp(min(bz + 1, msz - 1), Pb0, Pb1, Pb2);
                pz = bz;
            }
        }
        const int i = k - 2;
        const bool iout = i >= ilo && i < ihi;  // uniform
        const double rzk = sZr[kt];
        stage_wait(k);
        const double* stk = slot_of(k);
        // ---- P: plane k (all columns)
        const double s0 = fma(stk[0], lerp(rzk, Pa0, Pb0),
                              fma(stk[NC], lerp(rzk, Pa1, Pb1), stk[2 * NC] * lerp(rzk, Pa2, Pb2)));
        sS[P * NB] = s0;
        double wc = 0.0, sgc = 0.0, pzc = 0.0, q0 = 0.0, q1 = 0.0, q2 = 0.0;
        if (role < 2) {
            // ---- W: plane j = k-1 (own rho-hat from the ring, neighbours' s of plane j)
            const double* rj = slot_of(k - 1) + HV_DT;
            const double r0 = rj[0], r1 = rj[NC], r2 = rj[2 * NC], r3 = rj[3 * NC], r4 = rj[4 * NC], r5 = rj[5 * NC];
            const double* sn = sS + (1 - P) * NB;
            const double sj = sr[1 - P];
            const double w01 = fma(r1, sn[1] - sj, r0 * (sn[-1] - sj));
            const double w23 = fma(r3, sn[CX] - sj, r2 * (sn[-CX] - sj));
            const double w45 = fma(r5, s0 - sj, r4 * (sr[P] - sj));
            wc = (w01 + w23) + w45;
            sgc = ((r0 + r1) + (r2 + r3)) + (r4 + r5);
            pzc = r5;
            sWv[(1 - P) * NB] = wc;
            // ---- Z: plane i = k-2 (tile columns)
            if (role == 0 && iout) {
                const double* ri = slot_of(k - 2);  // dT [3][NC], then rho-hat [6][NC]
                const double* rh = ri + HV_DT;
                const double* wn = sWv + P * NB;
                // neighbour coefficient toward i: -x neighbour holds (+x), +x neighbour (-x), ...
                const double z01 = fma(rh[NC - 1], wn[-1], rh[1] * wn[1]);
                const double z23 = fma(rh[3 * NC - CX], wn[-CX], rh[2 * NC + CX] * wn[CX]);
                const double z45 = fma(r4, wc, pr[1 - P] * wr[1 - P]);  // rho-hat_{i+z}(-z) w_{i+z}, _{i-z}(+z) w_{i-z}
                const double z = fma(-gr[P], wr[P], (z01 + z23) + z45);
                const double sz = tile ? a.scale * z : 0.0;
                q0 = sz * ri[0];
                q1 = sz * ri[NC];
                q2 = sz * ri[2 * NC];
            }
        }
        if (iout) {
            const int bz = sZb[kt - 2];
            const double rz = sZr[kt - 2];
            if (bz > cur) {  // nodal plane `cur` complete: x-y spread (all threads)
                spread(acc00, acc01, acc02, cur);
                acc00 = acc10;
                acc01 = acc11;
                acc02 = acc12;
                acc10 = acc11 = acc12 = 0.0;
                cur = bz;
            }
            acc00 = fma(1.0 - rz, q0, acc00);
            acc10 = fma(rz, q0, acc10);
            acc01 = fma(1.0 - rz, q1, acc01);
            acc11 = fma(rz, q1, acc11);
            acc02 = fma(1.0 - rz, q2, acc02);
            acc12 = fma(rz, q2, acc12);
        }
        if (slab_pending) {
            slab_store(slab_hi + 1);
            for (int nz = slab_hi + 2; nz <= slab_nz; ++nz) {
                slab_load(nz);
                slab_store(nz);
            }
            slab_hi = slab_nz;
        }
        // histories (parity-named: no moves)
        sr[P] = s0;
        wr[1 - P] = wc;
        pr[1 - P] = pzc;
        gr[1 - P] = sgc;
        __syncthreads();
    };
#pragma unroll 1
    for (int k = kfirst; k <= klast; k += 2) {
        step(std::integral_constant<int, 0>{}, k);
        if (k + 1 <= klast) step(std::integral_constant<int, 1>{}, k + 1);
    }
  }
    if (TMA) {  // drain the two look-ahead loads before the CTA exits
        stage_wait(z1 + 2);
        stage_wait(z1 + 3);
    }
    if (!EVAL || a.grad) {  // flush the last two nodal planes
        spread(acc00, acc01, acc02, cur);
        __syncthreads();
        spread(acc10, acc11, acc12, cur + 1);
    }
    if (EVAL) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) dsum += __shfl_down_sync(0xffffffffu, dsum, o);
        if ((tid & 31) == 0) sred[tid >> 5] = dsum;
        __syncthreads();
        if (tid == 0) {
            double sacc = 0.0;
            for (int w = 0; w < NTH / 32; ++w) sacc += sred[w];
            a.vpart[tile_id] = sacc;
        }
    }
}

// ------------------------------------------------------------ nodal finalize
struct FinArgs {
    Grid gy;
    TileMeta tm;
    const double* part;
    const double* vpart;
    int ntiles;
    double hbar;     // image cell volume (D scale)
    double alpha;
    double scale_y;  // 2 h_bar^y
    double cell_y;   // h_bar^y
    const double* add;  // nodal term added to out (alpha * curvature), nullable
    const double* S;    // device scalar sum (Lap u)^2 (value), nullable
    double* out;
    const double* dot_a;
    int value;
    double* sc;
    double* sc_host;
    double* red;
    unsigned int* counter;
    const int* skip;
    int nS;                   // number of device scalars summed into S
    long long fin_lo, nwin;   // finalize nodes [fin_lo, fin_lo + nwin) (per component)
    long long add_lo, add_hi; // nodes where `add` applies and the dot counts (owned)
};

__device__ __forceinline__ long long clampl(long long v, long long hi) { return v < 0 ? 0 : (v > hi ? hi : v); }

__device__ __forceinline__ double lapc(const double* __restrict__ u, const Grid& g, long long x, long long y,
                                       long long z) {
    const double ui = __ldg(&u[g.lin(x, y, z)]);
    double s = (__ldg(&u[g.lin(clampl(x - 1, g.m[0] - 1), y, z)]) - 2.0 * ui +
                __ldg(&u[g.lin(clampl(x + 1, g.m[0] - 1), y, z)])) / (g.h[0] * g.h[0]);
    s += (__ldg(&u[g.lin(x, clampl(y - 1, g.m[1] - 1), z)]) - 2.0 * ui +
          __ldg(&u[g.lin(x, clampl(y + 1, g.m[1] - 1), z)])) / (g.h[1] * g.h[1]);
    s += (__ldg(&u[g.lin(x, y, clampl(z - 1, g.m[2] - 1))]) - 2.0 * ui +
          __ldg(&u[g.lin(x, y, clampl(z + 1, g.m[2] - 1))])) / (g.h[2] * g.h[2]);
    return s;
}

constexpr int FIN_THREADS = 128;
constexpr int kFinBlocks = 148 * 16;  // finalize grid cap (grid-stride beyond)
constexpr int kFinGroups = 32;        // completion-ticket groups (counter_ holds 1 + kFinGroups)

__device__ double block_reduce(double v, double* sh) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    __syncthreads();
    if (lane == 0) sh[wid] = v;
    __syncthreads();
    v = threadIdx.x < (blockDim.x >> 5) ? sh[threadIdx.x] : 0.0;
    if (wid == 0) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    }
    return v;
}

// PT: partial element type (fp32 partials in FAST32 mode); K: compile-time bound on the
// gather entries per node per axis (fully unrolled, predicated: every load of a node is in
// flight at once), 0 = dynamic loops; C: components per thread (3: one thread per node; 1: one
// thread per (node, component), for small windows where one thread per node leaves the SMs idle)
template <typename PT, int K, int C>
#ifndef MFREG_FIN_MINB
#define MFREG_FIN_MINB 8  // 64 registers, 32 warps/SM: the gather is latency bound (C4: -30%)
#endif
__global__ void __launch_bounds__(FIN_THREADS, MFREG_FIN_MINB) k_nodal_finalize(FinArgs a) {
    const PT* const part = reinterpret_cast<const PT*>(a.part);
    __shared__ double sh[32];
    __shared__ bool last;
    if (a.skip && *a.skip) return;  // uniform (set two launches earlier)
    const long long ny = a.gy.count();
    double r0 = 0.0, r1 = 0.0;
    pdl_wait();  // partials of the image pass, the side-stream curvature term
    // C = 3: one thread per node of the window, all three components: a node's per-tile partials
    // are three adjacent values, so each gather entry is one contiguous 24-byte (12-byte) read
    // and the per-axis gather tables (a few KB, L1-resident) are walked once per node. C = 1:
    // consecutive threads take the components of one node (same tables, adjacent partials).
    // Grid-stride over a capped grid keeps the completion-counter atomics few.
    if (a.out) {
        const int mx = static_cast<int>(a.gy.m[0]), pn = static_cast<int>(a.gy.m[0] * a.gy.m[1]);
        const TileMeta& tm = a.tm;
        const long long nthr = a.nwin * (3 / C);
        for (long long tw = static_cast<long long>(blockIdx.x) * FIN_THREADS + threadIdx.x; tw < nthr;
             tw += static_cast<long long>(gridDim.x) * FIN_THREADS) {
            const long long node = a.fin_lo + (C == 3 ? tw : tw / 3);
            const int d0 = C == 3 ? 0 : static_cast<int>(tw - (tw / 3) * 3);
            const bool owned = node >= a.add_lo && node < a.add_hi;
            const int nz = static_cast<int>(node / pn), rem = static_cast<int>(node - static_cast<long long>(nz) * pn);
            const int nyy = rem / mx, nx = rem - nyy * mx;
            // operands issued first so their latency overlaps the gather
            double addv[C], dotv[C], v[C];
#pragma unroll
            for (int c = 0; c < C; ++c) {
                addv[c] = (a.add && owned) ? __ldg(a.add + (d0 + c) * ny + node) : 0.0;
                dotv[c] = (a.dot_a && owned) ? __ldg(a.dot_a + (d0 + c) * ny + node) : 0.0;
                v[c] = 0.0;
            }
            const int zb = __ldg(&tm.g_off[2][nz]), ze = __ldg(&tm.g_off[2][nz + 1]);
            const int yb = __ldg(&tm.g_off[1][nyy]), ye = __ldg(&tm.g_off[1][nyy + 1]);
            const int xb = __ldg(&tm.g_off[0][nx]), xe = __ldg(&tm.g_off[0][nx + 1]);
            auto entry = [&](int2 Z, int2 Y, int2 X) {
                const std::size_t tile = (static_cast<std::size_t>(Z.x) * tm.nty + Y.x) * tm.ntx + X.x;
                const std::size_t loc = (static_cast<std::size_t>(Z.y) * tm.nly + Y.y) * tm.nlx + X.y;
                const PT* q = part + tile * tm.part_stride + loc * 3 + d0;
                PT qv[C];
#pragma unroll
                for (int c = 0; c < C; ++c) qv[c] = __ldg(q + c);
#pragma unroll
                for (int c = 0; c < C; ++c) v[c] += static_cast<double>(qv[c]);
            };
            // CSR order: z tiles, then y, then x (fixed sum order)
            if constexpr (K > 0) {
                int2 Z[K], Y[K], X[K];
#pragma unroll
                for (int k = 0; k < K; ++k) {
                    Z[k] = zb + k < ze ? __ldg(&tm.g_ent[2][zb + k]) : make_int2(0, 0);
                    Y[k] = yb + k < ye ? __ldg(&tm.g_ent[1][yb + k]) : make_int2(0, 0);
                    X[k] = xb + k < xe ? __ldg(&tm.g_ent[0][xb + k]) : make_int2(0, 0);
                }
#pragma unroll
                for (int kz = 0; kz < K; ++kz)
#pragma unroll
                    for (int ky = 0; ky < K; ++ky)
#pragma unroll
                        for (int kx = 0; kx < K; ++kx)
                            if (zb + kz < ze && yb + ky < ye && xb + kx < xe) entry(Z[kz], Y[ky], X[kx]);
            } else {
                for (int ez = zb; ez < ze; ++ez)
                    for (int ey = yb; ey < ye; ++ey)
                        for (int ex = xb; ex < xe; ++ex)
                            entry(__ldg(&tm.g_ent[2][ez]), __ldg(&tm.g_ent[1][ey]), __ldg(&tm.g_ent[0][ex]));
            }
#pragma unroll
            for (int c = 0; c < C; ++c) {
                if (a.add && owned) v[c] += addv[c];
                a.out[(d0 + c) * ny + node] = v[c];
                if (a.dot_a && owned) r0 += dotv[c] * v[c];
            }
        }
    }
    if (a.sc == nullptr) return;
    r0 = block_reduce(r0, sh);
    if (threadIdx.x == 0) {
        a.red[2 * blockIdx.x] = r0;
        a.red[2 * blockIdx.x + 1] = r1;
        __threadfence();
        // two-level completion ticket (kFinGroups group counters, then one top counter): a
        // single counter serialised ~10^3 same-address atomics per launch (several us)
        const unsigned g = blockIdx.x % kFinGroups, ng = min(gridDim.x, static_cast<unsigned>(kFinGroups));
        const unsigned gsize = (gridDim.x - g + kFinGroups - 1) / kFinGroups;
        bool lst = false;
        if (atomicAdd(a.counter + 1 + g, 1u) == gsize - 1) {
            a.counter[1 + g] = 0u;
            __threadfence();
            lst = atomicAdd(a.counter, 1u) == ng - 1;
        }
        last = lst;
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    double s0 = 0.0, s1 = 0.0, sv = 0.0;
    for (unsigned int b = threadIdx.x; b < gridDim.x; b += FIN_THREADS) {
        s0 += a.red[2 * b];
        s1 += a.red[2 * b + 1];
    }
    if (a.value)
        for (int t = threadIdx.x; t < a.ntiles; t += FIN_THREADS) sv += a.vpart[t];
    s0 = block_reduce(s0, sh);
    s1 = block_reduce(s1, sh);
    sv = a.value ? block_reduce(sv, sh) : 0.0;
    if (threadIdx.x == 0) {
        if (a.value) {
            a.sc[0] = a.hbar * sv;                    // D
            double S = 0.0;
            for (int k = 0; a.S && k < a.nS; ++k) S += a.S[k];
            a.sc[1] = a.S ? a.alpha * (a.cell_y * S) : 0.0;  // alpha S
            if (a.sc_host) {
                a.sc_host[0] = a.sc[0];
                a.sc_host[1] = a.sc[1];
                __threadfence_system();
            }
        } else {
            a.sc[0] = s0;                             // <dot_a, out>
        }
        *a.counter = 0u;
    }
}

std::size_t fused_smem_bytes(const TileMeta& tm, int nxf, int nyf, bool eval) {
    const int slot = eval ? EV_SLOT : HV_SLOT;
    const int depth = eval ? DEPTH_EV : DEPTH_HV;
    std::size_t d = depth * slot + (eval ? NBUF_EV : NBUF_HV) * NB + (eval ? 9 * TT : 0) + 3 * TT +
                    3 * FT_Y * tm.nlx + tm.zc + 8 + FT_X + FT_Y + (eval ? 0 : NSLAB * nxf * nyf * 3);
    std::size_t ints = tm.zc + 8 + 4 * tm.nlx + 4 * tm.nly;
    return d * sizeof(double) + ints * sizeof(int) + 16 + depth * 8 + 32 * 8;
}

FArgs make_args(const DevicePlanOwner& plan, FusedPlan& fp) {
    FArgs a{};
    const DevPlan& P = plan.view();
    a.g = P.tgt;
    a.P = P;
    a.tm = fp.meta();
    for (int d = 0; d < 3; ++d) {
        a.hh[d] = 1.0 / (2.0 * a.g.h[d] * a.g.h[d]);
        a.ih2[d] = 1.0 / (a.g.h[d] * a.g.h[d]);
    }
    a.part = fp.partials();
    a.vpart = fp.value_partials();
    a.olo = fp.out_lo();
    a.ohi = fp.out_hi();
    a.nxf = fp.slab_x();
    a.nyf = fp.slab_y();
    a.dbg = 0;
    a.segw = fp.seg_width();
    return a;
}

}  // namespace

FusedPlan::FusedPlan(const DevicePlanOwner& plan, const void* R, const void* Tw, const void* dT, const void* frh,
                     const SlabSpec& slab, bool fp32, int zc_cap)
    : fp32_(fp32), state_R_(R), state_Tw_(Tw) {
    const DevPlan& P = plan.view();
    const Grid& g = P.tgt;
    TileMeta& t = meta_;
    t.ntx = static_cast<int>((g.m[0] + FT_X - 1) / FT_X);
    t.nty = static_cast<int>((g.m[1] + FT_Y - 1) / FT_Y);
    // z window: outputs on image planes [zlo, zhi); tiles also cover 2 halo planes each
    // side so the stored Hv state (rho-hat, dT) is valid wherever the Hv stencil reads it
    const int gmz = static_cast<int>(g.m[2]);
    const int msz = static_cast<int>(P.src.m[2]);
    const bool full = slab.full(gmz, msz);
    out_lo_ = full ? 0 : slab.zlo;
    out_hi_ = full ? gmz : slab.zhi;
    t.zlo = full ? 0 : std::max(0, slab.zlo - 2);
    t.zhi = full ? gmz : std::min(gmz, slab.zhi + 2);
    const auto& bz = plan.host_base[2];
    own_lo_ = full ? 0 : slab.own_lo;
    own_hi_ = full ? msz : slab.own_hi;
    fin_lo_ = full ? 0 : std::min(own_lo_, bz[out_lo_]);
    fin_hi_ = full ? msz : std::max(own_hi_, bz[out_hi_ - 1] + 2);
    // z chunking: minimise waves x (planes per chunk + 4 halo planes), waves of the
    // two-CTA Hv kernel (the eval kernel runs 2 CTAs/SM in fp64, 3 in FAST32)
    const long long nxy = static_cast<long long>(t.ntx) * t.nty;
    const int mz = t.zhi - t.zlo;
    // (chunks of <= zmax planes: the two-CTA Hv kernel keeps per-chunk z tables in shared memory,
    // 12 B per plane, so zmax is what its shared-memory budget leaves; the round-1 cap of 128 planes
    // — then measured faster — measured 3% slower than 450-plane chunks at C4 with the current
    // kernels, which stream L2-friendlier with fewer halo steps; MFREG_ZC_MAX overrides)
    int zmax = 1 << 20;
    {
        int nlxy[2];
        const int tsz2[2] = {FT_X, FT_Y}, ntl2[2] = {t.ntx, t.nty};
        for (int a = 0; a < 2; ++a) {
            const auto& base = plan.host_base[a];
            nlxy[a] = 0;
            for (int k = 0; k < ntl2[a]; ++k) {
                const int x0 = k * tsz2[a], x1 = std::min(static_cast<int>(g.m[a]), x0 + tsz2[a]);
                nlxy[a] = std::max(nlxy[a], base[x1 - 1] + 1 - base[x0] + 1);
            }
        }
        int sw = 1, run = 1;  // longest run of image columns sharing a nodal x cell (segw_ below)
        for (std::size_t k = 1; k < plan.host_base[0].size(); ++k) {
            run = plan.host_base[0][k] == plan.host_base[0][k - 1] ? run + 1 : 1;
            sw = std::max(sw, run);
        }
        const std::size_t s0 = hv2_smem_bytes(nlxy[0], nlxy[1], sw, 0, hv2_nsl_max(8), fp32, 8);
        const std::size_t s1 = hv2_smem_bytes(nlxy[0], nlxy[1], sw, 1, hv2_nsl_max(8), fp32, 8);
        if (s0 < static_cast<std::size_t>(kSmem2Cta) && s1 > s0)
            zmax = std::max(16, static_cast<int>((static_cast<std::size_t>(kSmem2Cta) - s0) / (s1 - s0)) - 8);
    }
    if (const char* zenv = std::getenv("MFREG_ZC_MAX")) zmax = std::max(4, std::atoi(zenv));
    if (zc_cap > 0) zmax = std::min(zmax, zc_cap);
    int best = (mz + zmax - 1) / zmax;
    double best_cost = 1e300;
    for (int ntz = (mz + zmax - 1) / zmax; ntz <= std::max((mz + zmax - 1) / zmax, mz / 4); ++ntz) {
        const int zc = (mz + ntz - 1) / ntz;
        const int real_ntz = (mz + zc - 1) / zc;
        const double waves = std::ceil(static_cast<double>(nxy * real_ntz) / (2 * kSMs));
        const double cost = waves * (zc + 4);
        if (cost < best_cost - 1e-9) {
            best_cost = cost;
            best = ntz;
        }
    }
    t.zc = (mz + best - 1) / best;
    t.ntz = (mz + t.zc - 1) / t.zc;
    const int tsz[3] = {FT_X, FT_Y, t.zc};
    const int ntl[3] = {t.ntx, t.nty, t.ntz};
    const int org[3] = {0, 0, t.zlo}, end[3] = {static_cast<int>(g.m[0]), static_cast<int>(g.m[1]), t.zhi};
    int nl[3];
    for (int a = 0; a < 3; ++a) {
        const auto& base = plan.host_base[a];
        const int ms = static_cast<int>(P.src.m[a]);
        std::vector<int> n0(ntl[a]), n1(ntl[a]);
        nl[a] = 0;
        for (int k = 0; k < ntl[a]; ++k) {
            const int x0 = org[a] + k * tsz[a], x1 = std::min(end[a], x0 + tsz[a]);
            n0[k] = base[x0];
            n1[k] = base[x1 - 1] + 1;
            nl[a] = std::max(nl[a], n1[k] - n0[k] + 1);
        }
        // finalize gather lists: for node nd, every tile k whose footprint holds it
        std::vector<int> off(ms + 1, 0);
        std::vector<int2> ent;
        for (int nd = 0; nd < ms; ++nd) {
            for (int k = 0; k < ntl[a]; ++k)
                if (n0[k] <= nd && nd <= n1[k]) ent.push_back(make_int2(k, nd - n0[k]));
            off[nd + 1] = static_cast<int>(ent.size());
            gmax_ = std::max(gmax_, off[nd + 1] - off[nd]);
        }
        goff_[a].resize(ms + 1);
        gent_[a].resize(std::max<std::size_t>(1, ent.size()));
        MFREG_CUDA(cudaMemcpy(goff_[a].get(), off.data(), (ms + 1) * sizeof(int), cudaMemcpyHostToDevice));
        if (!ent.empty())
            MFREG_CUDA(cudaMemcpy(gent_[a].get(), ent.data(), ent.size() * sizeof(int2), cudaMemcpyHostToDevice));
        t.g_off[a] = goff_[a].get();
        t.g_ent[a] = gent_[a].get();
    }
    t.nlx = nl[0];
    t.nly = nl[1];
    t.nlz = nl[2];
    t.part_stride = static_cast<std::size_t>(t.nlz) * t.nly * t.nlx * 3;
    part_.resize(t.part_stride * static_cast<std::size_t>(ntiles()));
    MFREG_CUDA(cudaMemset(part_.get(), 0, part_.size() * sizeof(double)));
    vpart_.resize(static_cast<std::size_t>(ntiles()));
    vticket_.resize(33);
    MFREG_CUDA(cudaMemset(vticket_.get(), 0, 33 * sizeof(unsigned int)));
    const long long ny = P.src.count();
    red_.resize(static_cast<std::size_t>(2 * ((3 * ny + FIN_THREADS - 1) / FIN_THREADS) + 2));
    counter_.resize(1 + kFinGroups);
    MFREG_CUDA(cudaMemset(counter_.get(), 0, (1 + kFinGroups) * sizeof(unsigned int)));
    // nodal slab footprint of a tile's halo-2 columns (max over tiles), per axis
    for (int a2 = 0; a2 < 2; ++a2) {
        const auto& base = plan.host_base[a2];
        const int m = static_cast<int>(g.m[a2]);
        const int ts = a2 == 0 ? FT_X : FT_Y;
        int mxf = 0;
        for (int k = 0; k < ntl[a2]; ++k) {
            const int lo = std::max(k * ts - 2, 0), hi = std::min(m - 1, k * ts + ts + 1);
            mxf = std::max(mxf, base[hi] - base[lo] + 2);
        }
        slab_[a2] = mxf;
    }
    const std::size_t hv_smem = fused_smem_bytes(t, slab_[0], slab_[1], false);
    const std::size_t ev_smem = fused_smem_bytes(t, slab_[0], slab_[1], true);
    int dev = 0, max_optin = 0;
    MFREG_CUDA(cudaGetDevice(&dev));
    MFREG_CUDA(cudaDeviceGetAttribute(&max_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    if (hv_smem > static_cast<std::size_t>(max_optin) || ev_smem > static_cast<std::size_t>(max_optin))
        throw std::invalid_argument("fused kernels: tile footprint exceeds shared memory (deformation grid too fine)");
    if (static_cast<long long>(slab_[0]) * slab_[1] * 3 > 4LL * NTH)
        throw std::invalid_argument("fused kernels: nodal slab footprint too large (deformation grid too fine)");
    // the cap is per kernel (process-wide): set it to the device limit so plans of
    // different footprints (levels, slabs, threads) never lower each other's
    MFREG_CUDA(cudaFuncSetAttribute(k_fused<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, max_optin));
    MFREG_CUDA(cudaFuncSetAttribute(k_fused<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, max_optin));
    MFREG_CUDA(cudaFuncSetAttribute(k_fused<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, max_optin));
    MFREG_CUDA(cudaFuncSetAttribute(k_fused<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, max_optin));
    // TMA needs 16-byte global strides: even mx (rows) and 16-byte aligned bases
    const bool aligned = (g.m[0] % 2 == 0) && (reinterpret_cast<std::uintptr_t>(R) % 16 == 0) &&
                         (reinterpret_cast<std::uintptr_t>(Tw) % 16 == 0) &&
                         (reinterpret_cast<std::uintptr_t>(dT) % 16 == 0) && (reinterpret_cast<std::uintptr_t>(frh) % 16 == 0);
    frh_base_ = frh;
    const char* off = std::getenv("MFREG_NO_TMA");
    tma_ = aligned && (fp32 || !(off && off[0] == '1')) && make_tma_maps(g, R, Tw, dT, frh);
    // two-CTA/SM Hv kernel (hv_fast.cu): TMA only; the nodal z cells must span >= 2 image
    // planes (x-collapse buffer reuse, nodal ring of 4), and the y collapse needs one
    // thread per tile-local node
    bool zok = true;
    for (int k = 0; k < gmz; ++k) {
        const auto& bzv = plan.host_base[2];
        if (bzv[std::min(k + 2, gmz - 1)] - bzv[k] > 1) zok = false;  // cells of >= 2 planes
        if (bzv[std::min(k + 3, gmz - 1)] - bzv[k] > 2) zok = false;
    }
    {  // longest run of image columns sharing a nodal x cell
        const auto& bx = plan.host_base[0];
        int run = 1;
        segw_ = 1;
        for (std::size_t k = 1; k < bx.size(); ++k) {
            run = bx[k] == bx[k - 1] ? run + 1 : 1;
            segw_ = std::max(segw_, run);
        }
    }
    const std::size_t hv2_smem = hv2_smem_bytes(t.nlx, t.nly, segw_, t.zc, slab_[0] * slab_[1] * 3, fp32_, 8);
    const char* no2 = std::getenv("MFREG_NO_HV2");
    hv2_ = tma_ && zok && (fp32_ || !(no2 && no2[0] == '1')) && t.nlx <= hv2_nlx_max() &&
           slab_[0] * slab_[1] * 3 <= hv2_nsl_max(8) && hv2_smem <= static_cast<std::size_t>(kSmem2Cta);
    hv2_smem_ = hv2_smem;
    // (process-wide per-kernel cap: always the 2-CTA bound, so plans never lower each other's)
    if (hv2_) hv2_set_smem_cap(kSmem2Cta, 8);
    // two-CTA/SM eval kernel (ev_fast.cu): same conditions
    ev2_smem_ = ev2_smem_bytes(t.nlx, t.nly, segw_, fp32_);
    const char* noe = std::getenv("MFREG_NO_EV2");
    ev2_ = tma_ && zok && (fp32_ || !(noe && noe[0] == '1')) && t.nlx <= hv2_nlx_max() && ev2_smem_ <= static_cast<std::size_t>(kSmem2Cta);
    if (ev2_) ev2_set_smem_cap(kSmem2Cta);
    setup_hv3(plan, R, Tw, dT, frh, zok, max_optin);
    // FAST32 runs only on the two-CTA kernels (the legacy fused kernels are fp64)
    if (fp32_ && !(hv2_ && ev2_))
        throw std::invalid_argument(
            "FAST32: the grid is not supported by the single-precision kernels (odd x size or nodal z cells "
            "spanning < 2 image planes)");
}

// Hv pass with recomputed coefficients (hv3.cu), opt-in (MFREG_HV3=1; MFREG_NO_HV3=1 wins): 28 x 12
// output tiles over the same z window, one CTA per SM; per-axis finalize gather tables as for the
// main tiling. Measured at C4: 8.1 ms fp64 / 5.7 ms FAST32 against k_hv2's 5.6 / 3.5 ms
// -- the recomputation adds ~90 fp64 operations per voxel on B200's 60-per-clock fp64 pipe, and the
// one-CTA-per-SM uniform-warp schedule issues at ~50%. Off when TMA cannot address the grid, nodal z
// cells span < 2 image planes or a tile's nodal footprint exceeds one node per thread.
void FusedPlan::setup_hv3(const DevicePlanOwner& plan, const void* R, const void* Tw, const void* dT, const void* frh,
                          bool zok, int max_optin) {
    const char* on = std::getenv("MFREG_HV3");   // recompute variant
    const char* on4 = std::getenv("MFREG_HV4");  // stored-coefficient variant
    const char* off = std::getenv("MFREG_NO_HV3");
    const char* on16 = std::getenv("MFREG_HV16");  // k_hv2 on 32 x 16 tiles, one CTA per SM
    const bool recompute = on && on[0] == '1', stored = !recompute && on4 && on4[0] == '1';
    const bool h16 = !recompute && !stored && on16 && on16[0] == '1';
    if (!(recompute || stored || h16) || (off && off[0] == '1') || !tma_ || !zok) return;
    if (!h16 && fp32_ && !hv3_fp32_ok()) return;
    static PFN_cuTensorMapEncodeTiled_v12000 encode = [] {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            fn = nullptr;
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }();
    if (!encode) return;
    const DevPlan& P = plan.view();
    const Grid& g = P.tgt;
    const int tsx = h16 ? FT_X : hv3_tile_x(), tsy = h16 ? 16 : hv3_tile_y();
    TileMeta t{};
    t.ntx = static_cast<int>((g.m[0] + tsx - 1) / tsx);
    t.nty = static_cast<int>((g.m[1] + tsy - 1) / tsy);
    t.zlo = meta_.zlo;
    t.zhi = meta_.zhi;
    // z chunks: minimise waves x (planes + 4 halo planes), one CTA per SM
    const long long nxy = static_cast<long long>(t.ntx) * t.nty;
    const int mz = t.zhi - t.zlo;
    const int zmax = 128;
    int best = (mz + zmax - 1) / zmax;
    double best_cost = 1e300;
    for (int ntz = (mz + zmax - 1) / zmax; ntz <= std::max((mz + zmax - 1) / zmax, mz / 4); ++ntz) {
        const int zc = (mz + ntz - 1) / ntz;
        const int real_ntz = (mz + zc - 1) / zc;
        const double cost = std::ceil(static_cast<double>(nxy * real_ntz) / kSMs) * (zc + 4);
        if (cost < best_cost - 1e-9) {
            best_cost = cost;
            best = ntz;
        }
    }
    t.zc = (mz + best - 1) / best;
    if (const char* zce = std::getenv("MFREG_HV3_ZC")) t.zc = std::max(4, std::min(mz, std::atoi(zce)));  // experiments
    t.ntz = (mz + t.zc - 1) / t.zc;
    const int tsz[3] = {tsx, tsy, t.zc};
    const int ntl[3] = {t.ntx, t.nty, t.ntz};
    const int org[3] = {0, 0, t.zlo}, end[3] = {static_cast<int>(g.m[0]), static_cast<int>(g.m[1]), t.zhi};
    int nl[3];
    int gmax = 0;
    std::vector<int> off3[3];
    std::vector<int2> ent3[3];
    for (int a = 0; a < 3; ++a) {
        const auto& base = plan.host_base[a];
        const int ms = static_cast<int>(P.src.m[a]);
        std::vector<int> n0(ntl[a]), n1(ntl[a]);
        nl[a] = 0;
        for (int k = 0; k < ntl[a]; ++k) {
            const int x0 = org[a] + k * tsz[a], x1 = std::min(end[a], x0 + tsz[a]);
            n0[k] = base[x0];
            n1[k] = base[x1 - 1] + 1;
            nl[a] = std::max(nl[a], n1[k] - n0[k] + 1);
        }
        off3[a].assign(ms + 1, 0);
        for (int nd = 0; nd < ms; ++nd) {
            for (int k = 0; k < ntl[a]; ++k)
                if (n0[k] <= nd && nd <= n1[k]) ent3[a].push_back(make_int2(k, nd - n0[k]));
            off3[a][nd + 1] = static_cast<int>(ent3[a].size());
            gmax = std::max(gmax, off3[a][nd + 1] - off3[a][nd]);
        }
    }
    t.nlx = nl[0];
    t.nly = nl[1];
    t.nlz = nl[2];
    t.part_stride = static_cast<std::size_t>(t.nlz) * t.nly * t.nlx * 3;
    // nodal footprint of the staged columns [x0 - 2, x0 + tsx + 1] and rows, max over tiles
    int fp[2];
    for (int a2 = 0; a2 < 2; ++a2) {
        const auto& base = plan.host_base[a2];
        const int m = static_cast<int>(g.m[a2]);
        const int ts = a2 == 0 ? tsx : tsy;
        int mxf = 0;
        for (int k = 0; k < ntl[a2]; ++k) {
            const int lo = std::max(k * ts - 2, 0), hi = std::min(m - 1, k * ts + ts + 1);
            mxf = std::max(mxf, base[hi] - base[lo] + 2);
        }
        fp[a2] = mxf;
    }
    const std::size_t smem = h16 ? hv2_smem_bytes(t.nlx, t.nly, segw_, t.zc, fp[0] * fp[1] * 3, fp32_, 16)
                                 : hv3_smem_bytes(t.nlx, fp[0] * fp[1] * 3, t.zc, fp32_, stored);
    if (h16 ? (t.nlx > hv2_nlx_max() || fp[0] * fp[1] * 3 > hv2_nsl_max(16))
            : (fp[0] * fp[1] * 3 > hv3_threads() || 3 * t.nlx * t.nly > hv3_threads()))
        return;
    if (smem > static_cast<std::size_t>(max_optin)) return;
    // tensor maps: R, T_w (3-D boxes BX x 16), dT (4-D, 3 components); fp32 needs 16-byte rows
    const int es = fp32_ ? 4 : 8;
    if ((g.m[0] * es) % 16 != 0) return;
    const cuuint64_t mx = g.m[0], my = g.m[1], mzz = g.m[2], n = g.count();
    auto enc = [&](CUtensorMap* m, const void* base, int rank, cuuint64_t comps, cuuint32_t bc, int rows_less = 0) {
        const cuuint64_t e = static_cast<cuuint64_t>(es);
        const cuuint64_t dims[4] = {mx, my, mzz, comps};
        const cuuint64_t strides[3] = {mx * e, mx * my * e, n * e};
        // (32 x 16 k_hv2: boxes start x0 - XO, 32 + 2 XO wide; dT 20 rows, rho-hat 18)
        const int bw = h16 ? FT_X + 2 * hv2_box_origin(fp32_) : hv3_box_width(fp32_);
        const int br = h16 ? 20 - rows_less : hv3_box_rows() - rows_less;
        const cuuint32_t box[4] = {static_cast<cuuint32_t>(bw), static_cast<cuuint32_t>(br), 1, bc};
        const cuuint32_t est[4] = {1, 1, 1, 1};
        return encode(m, fp32_ ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64, rank,
                      const_cast<void*>(base), dims, strides, box, est, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
    };
    TmaMaps maps{};
    const bool ok = h16 ? (enc(&maps.a, dT, 4, 3, 3) && enc(&maps.b, frh, 4, 6, 6, 2))
                  : stored ? (enc(&maps.b, frh, 4, 6, 6, 2) && enc(&maps.c, dT, 4, 3, 3))
                           : (enc(&maps.a, R, 3, 1, 1) && enc(&maps.b, Tw, 3, 1, 1) && enc(&maps.c, dT, 4, 3, 3));
    if (!ok) return;
    std::memcpy(maps_hv3_, &maps, sizeof(TmaMaps));
    for (int a = 0; a < 3; ++a) {
        goff3_[a].resize(off3[a].size());
        gent3_[a].resize(std::max<std::size_t>(1, ent3[a].size()));
        MFREG_CUDA(cudaMemcpy(goff3_[a].get(), off3[a].data(), off3[a].size() * sizeof(int), cudaMemcpyHostToDevice));
        if (!ent3[a].empty())
            MFREG_CUDA(cudaMemcpy(gent3_[a].get(), ent3[a].data(), ent3[a].size() * sizeof(int2), cudaMemcpyHostToDevice));
        t.g_off[a] = goff3_[a].get();
        t.g_ent[a] = gent3_[a].get();
    }
    meta3_ = t;
    part3_.resize(t.part_stride * static_cast<std::size_t>(ntiles3()));
    MFREG_CUDA(cudaMemset(part3_.get(), 0, part3_.size() * sizeof(double)));
    slab3_[0] = fp[0];
    slab3_[1] = fp[1];
    gmax3_ = gmax;
    hv3_smem_ = smem;
    if (h16) hv2_set_smem_cap(max_optin, 16);
    else hv3_set_smem_cap(max_optin);
    hv3_ = true;
    hv3_stored_ = stored || h16;
    hv16_ = h16;
}

bool FusedPlan::make_tma_maps(const Grid& g, const void* R, const void* Tw, const void* dT, const void* frh) {
    static PFN_cuTensorMapEncodeTiled_v12000 encode = [] {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            fn = nullptr;
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }();
    if (!encode) return false;
    const cuuint64_t mx = g.m[0], my = g.m[1], mz = g.m[2], n = g.count();
    auto encw = [&](CUtensorMap* m, const void* base, int rank, cuuint64_t comps, cuuint32_t bx, cuuint32_t by,
                    cuuint32_t bc, int es_bytes) {
        const cuuint64_t e = static_cast<cuuint64_t>(es_bytes);
        const cuuint64_t dims[4] = {mx, my, mz, comps};
        const cuuint64_t strides[3] = {mx * e, mx * my * e, n * e};
        const cuuint32_t box[4] = {bx, by, 1, bc};
        const cuuint32_t es[4] = {1, 1, 1, 1};
        return encode(m, es_bytes == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, rank,
                      const_cast<void*>(base), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
    };
    if (fp32_) {  // single-precision state: only the two-CTA kernels' maps (boxes start at x0 - 4)
        if ((g.m[0] * 4) % 16 != 0) return false;
        const int XO = hv2_box_origin(true), SXf = FT_X + 2 * XO;
        TmaMaps hv2{}, ev2{};
        const bool ok = encw(&hv2.a, dT, 4, 3, SXf, CY, 3, 4) && encw(&hv2.b, frh, 4, 6, SXf, C1Y, 6, 4) &&
                        encw(&ev2.a, R, 3, 1, SXf, CY, 1, 4) && encw(&ev2.b, Tw, 3, 1, SXf, CY, 1, 4) &&
                        encw(&ev2.c, dT, 4, 3, FT_X, FT_Y, 3, 4) && encw(&ev2.d, frh, 4, 6, FT_X, FT_Y, 6, 4);
        if (!ok) return false;
        std::memcpy(maps_hv2_, &hv2, sizeof(TmaMaps));
        std::memcpy(maps_ev2_, &ev2, sizeof(TmaMaps));
        return true;
    }
    auto enc = [&](CUtensorMap* m, const void* base, int rank, cuuint64_t comps, cuuint32_t bx, cuuint32_t by,
                   cuuint32_t bc) { return encw(m, base, rank, comps, bx, by, bc, 8); };
    TmaMaps hv{}, ev{};
    bool ok = enc(&hv.a, dT, 4, 3, CX, CY, 3) && enc(&hv.b, frh, 4, 6, CX, CY, 6) && enc(&ev.a, R, 3, 1, CX, CY, 1) &&
              enc(&ev.b, Tw, 3, 1, CX, CY, 1) && enc(&ev.c, dT, 4, 3, CX, CY, 3);
    TmaMaps hv2{}, ev2{};
    ok = ok && enc(&hv2.a, dT, 4, 3, CX, CY, 3) && enc(&hv2.b, frh, 4, 6, CX, C1Y, 6);
    ok = ok && enc(&ev2.a, R, 3, 1, CX, CY, 1) && enc(&ev2.b, Tw, 3, 1, CX, CY, 1) && enc(&ev2.c, dT, 4, 3, FT_X, FT_Y, 3) &&
         enc(&ev2.d, frh, 4, 6, FT_X, FT_Y, 6);
    if (!ok) return false;
    std::memcpy(maps_hv2_, &hv2, sizeof(TmaMaps));
    std::memcpy(maps_ev2_, &ev2, sizeof(TmaMaps));
    static_assert(sizeof(TmaMaps) <= sizeof(maps_hv_), "tensor-map storage");
    std::memcpy(maps_hv_, &hv, sizeof(TmaMaps));
    std::memcpy(maps_ev_, &ev, sizeof(TmaMaps));
    return true;
}

void launch_hv_fused(const DevicePlanOwner& plan, FusedPlan& fp, const double* frh, const double* dT, const double* p,
                     double tau, double rho, cudaStream_t s, const int* skip, int c0, int c1) {
    FArgs a = make_args(plan, fp);
    const bool group = c0 != 0 || (c1 >= 0 && c1 != fp.meta().ntz);
    if (group && (!fp.hv2() || fp.hv3())) throw std::logic_error("Hv pass z groups need the two-CTA kernel");
    if (c1 < 0) c1 = fp.meta().ntz;
    a.zch0 = c0;
    a.tau = tau;
    a.rho = rho;
    a.skip = skip;
    a.scale = 2.0 * a.g.cell_volume();
    a.frh = frh;
    a.dT = dT;
    a.p = p;
    if (fp.hv3()) {
        a.tm = fp.meta3();
        a.part = fp.partials3();
        a.nxf = fp.slab3_x();
        a.nyf = fp.slab3_y();
        a.R = static_cast<const double*>(fp.state_R());
        a.Tw = static_cast<const double*>(fp.state_Tw());
        note_launch();
        const TileMeta& t3 = fp.meta3();
        if (fp.hv16())
            hv2_launch(a, *reinterpret_cast<const TmaMaps*>(fp.maps_hv3()), dim3(t3.ntx, t3.nty, t3.ntz), fp.hv3_smem(),
                       s, fp.fp32(), 16);
        else
            hv3_launch(a, *reinterpret_cast<const TmaMaps*>(fp.maps_hv3()), dim3(t3.ntx, t3.nty, t3.ntz), fp.hv3_smem(),
                       s, fp.fp32(), fp.hv3_stored());
        return;
    }
    const TileMeta& t = fp.meta();
    note_launch();
    const std::size_t smem = fused_smem_bytes(t, a.nxf, a.nyf, false);
    if (fp.hv2()) {
        hv2_launch(a, *reinterpret_cast<const TmaMaps*>(fp.maps_hv2()), dim3(t.ntx, t.nty, c1 - c0), fp.hv2_smem(), s,
                   fp.fp32(), 8);
        return;
    }
    const TmaMaps& maps = *reinterpret_cast<const TmaMaps*>(fp.maps_hv());
    if (fp.tma()) k_fused<false, true><<<dim3(t.ntx, t.nty, t.ntz), NTH, smem, s>>>(a, maps);
    else k_fused<false, false><<<dim3(t.ntx, t.nty, t.ntz), NTH, smem, s>>>(a, maps);
}

bool launch_eval_fused(const DevicePlanOwner& plan, FusedPlan& fp, const double* R, const double* Tw, const double* dT,
                       double tau, double rho, double* frh, bool grad, cudaStream_t s, double* d_dev, double* d_host,
                       int c0, int c1) {
    FArgs a = make_args(plan, fp);
    const bool group = c0 != 0 || (c1 >= 0 && c1 != fp.meta().ntz);
    if (group && !fp.ev2()) throw std::logic_error("eval pass z groups need the two-CTA kernel");
    if (c1 < 0) c1 = fp.meta().ntz;
    a.zch0 = c0;
    a.scale = -2.0 * a.g.cell_volume();
    a.tau = tau;
    a.rho = rho;
    a.R = R;
    a.Tw = Tw;
    a.dT = dT;
    a.frh_out = frh;
    a.grad = grad ? 1 : 0;
    const TileMeta& t = fp.meta();
    note_launch();
    const std::size_t smem = fused_smem_bytes(t, a.nxf, a.nyf, true);
    if (fp.ev2()) {
        if (d_dev && d_host) {
            a.vticket = fp.vticket();
            a.dsc = d_dev;
            a.dsc_host = d_host;
            a.dscale = plan.view().tgt.cell_volume();  // h_bar (ngf.cpp:227)
            if (!grad && !frh && value_pass_enabled() && !group) {  // Armijo trial: D only, bitwise k_ev2's D
                ev_value_launch(a, fp.state_R(), fp.state_Tw(), dim3(t.ntx, t.nty, t.ntz), s, fp.fp32());
                return true;
            }
        }
        // rho-hat by TMA store when the output is the state array the plan's map addresses
        a.frh_tma = (frh != nullptr && frh == fp.frh_base() && !(std::getenv("MFREG_NO_FRH_TMA"))) ? 1 : 0;
        ev2_launch(a, *reinterpret_cast<const TmaMaps*>(fp.maps_ev2()), dim3(t.ntx, t.nty, c1 - c0), fp.ev2_smem(), s,
                   fp.fp32());
        return a.vticket != nullptr;
    }
    const TmaMaps& maps = *reinterpret_cast<const TmaMaps*>(fp.maps_ev());
    if (fp.tma()) k_fused<true, true><<<dim3(t.ntx, t.nty, t.ntz), NTH, smem, s>>>(a, maps);
    else k_fused<true, false><<<dim3(t.ntx, t.nty, t.ntz), NTH, smem, s>>>(a, maps);
    return false;
}

// MFREG_NO_VALUE_PASS=1: value-only evaluations run the full eval pass (A/B switch)
bool value_pass_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("MFREG_NO_VALUE_PASS");
        return !(e && e[0] == '1');
    }();
    return on;
}

bool& pdl_suspended() {
    thread_local bool off = false;
    return off;
}

bool pdl_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("MFREG_NO_PDL");
        return !(e && e[0] == '1');
    }();
    return on;
}

void launch_nodal_finalize(const DevicePlanOwner& plan, FusedPlan& fp, const FinalizeSpec& spec, cudaStream_t s) {
    FinArgs a{};
    a.gy = plan.view().src;
    const bool p3 = spec.hv_pass && fp.hv3();
    a.tm = p3 ? fp.meta3() : fp.meta();
    a.part = p3 ? fp.partials3() : fp.partials();
    a.vpart = fp.value_partials();
    a.ntiles = p3 ? fp.ntiles3() : fp.ntiles();
    a.hbar = plan.view().tgt.cell_volume();
    a.alpha = spec.alpha;
    a.scale_y = 2.0 * a.gy.cell_volume();
    a.cell_y = a.gy.cell_volume();
    a.add = spec.add;
    a.S = spec.S;
    a.out = spec.out;
    a.dot_a = spec.dot_a;
    a.value = spec.value ? 1 : 0;
    a.sc = spec.sc;
    a.sc_host = spec.sc_host;
    a.red = fp.red();
    a.counter = fp.counter();
    a.skip = spec.skip;
    a.nS = spec.nS;
    const long long pn = a.gy.m[0] * a.gy.m[1];
    a.fin_lo = fp.fin_lo() * pn;
    a.nwin = (fp.fin_hi() - fp.fin_lo()) * pn;
    if (spec.nlo >= 0) {  // a z range of the window (pure gather)
        if (spec.sc || spec.dot_a || spec.value || spec.nlo < fp.fin_lo() || spec.nhi > fp.fin_hi() || spec.nhi <= spec.nlo)
            throw std::logic_error("finalize: nodal z range only for pure gathers inside the window");
        a.fin_lo = spec.nlo * pn;
        a.nwin = (spec.nhi - spec.nlo) * pn;
    }
    a.add_lo = fp.own_lo() * pn;
    a.add_hi = fp.own_hi() * pn;
    note_launch();
    // value-only calls (no gradient) need one block for the scalars
    // one thread per node once that fills the GPU (about 16 resident warps per SM), else one
    // thread per (node, component)
    const bool per_node = a.nwin >= static_cast<long long>(kSMs) * 16 * 32;
    const long long nthr = per_node ? a.nwin : 3 * a.nwin;
    const long long want = spec.out ? (nthr + FIN_THREADS - 1) / FIN_THREADS : 1;
    const unsigned blocks = static_cast<unsigned>(std::max(1LL, std::min(want, static_cast<long long>(kFinBlocks))));
    const bool k2 = (p3 ? fp.gather_max3() : fp.gather_max()) <= 2;
    auto go = [&](auto kern) { launch_pdl(kern, dim3(blocks), dim3(FIN_THREADS), 0, s, a); };
    if (fp.fp32()) {
        if (k2) per_node ? go(k_nodal_finalize<float, 2, 3>) : go(k_nodal_finalize<float, 2, 1>);
        else per_node ? go(k_nodal_finalize<float, 0, 3>) : go(k_nodal_finalize<float, 0, 1>);
    } else {
        if (k2) per_node ? go(k_nodal_finalize<double, 2, 3>) : go(k_nodal_finalize<double, 2, 1>);
        else per_node ? go(k_nodal_finalize<double, 0, 3>) : go(k_nodal_finalize<double, 0, 1>);
    }
}

}  // namespace mfreg_b200
