// Gauss-Newton Hv image pass, coefficients recomputed (fast / FAST32 mode).
//
// Same operator as k_hv2 (hv_fast.cu): s = dT . P p, w = dr s, z = dr^T w, q^ = 2h z dT,
// P^T into per-tile partials, with the factored form of fused.cuh. What differs:
//  * the Hv state is the canonical one, R, T_w and dT (40 B/voxel in fp64): the six NGF
//    coefficients rho-hat_t(k) = h^_a (dR_k inv1_t - dT_k inv2_t) (ngf.cpp:39-64, 185-214)
//    are recomputed per column from the 7-point stencils of R and T_w with one reciprocal
//    square root, instead of being streamed (48 B/voxel) from the eval pass;
//  * overlapped tiles, uniform warps: a CTA is 16 warps, warp r = image row y0 - 2 + r,
//    lane l = image column x0 - 2 + l, and every stage runs on whole warps: P (s) on all
//    16 rows and 32 lanes, the coefficients and w on rows 1..14 (lanes 1..30 valid), the
//    dr^T stage and P^T on rows 2..13 (lanes 2..29 = the 28 x 12 output tile). No halo
//    work items, no divergent second columns; the halo lanes just compute unused values;
//  * neighbour exchange: x neighbours by warp shuffles, y neighbours through shared
//    memory (s and the y fluxes by plane parity, R / T_w from the staged box), z
//    neighbours in the column's registers (histories named by step parity);
//  * staging: one TMA box per field and plane (R, T_w: 32 x 16, dT: 32 x 16 x 3; fp32
//    boxes are 36 wide and start 4 columns left, 16-byte alignment), a ring of 5 planes
//    with 4 in flight; one CTA per SM (512 threads, <= 128 registers).
// Boundary semantics as the reference's clamped neighbours: differences across the
// volume boundary are masked to zero, columns outside the volume have zero coefficients,
// dT vanishes outside (TMA zero fill) so q does.
#include <cstdint>

#include "fused_dev.cuh"

namespace mfreg_b200 {

namespace {

using namespace fdev;

constexpr int LX = 32;         // lanes = staged columns per row
constexpr int OX = LX - 4;     // output columns per tile (lanes 2..29)
#ifndef MFREG_HV3_OY
#define MFREG_HV3_OY 12
#endif
constexpr int OY = MFREG_HV3_OY;  // output rows per tile
constexpr int NR = OY + 4;     // warps = staged rows
constexpr int NT = LX * NR;    // 512 threads
constexpr int NSL = 4;         // nodal plane ring (power of 2)

// STORED = false (recompute): slot of plane m = R, T_w, dT of plane m; the coefficients of
//   plane j read R / T_w of planes j-1 .. j+1 -> ring of 5, 4 planes in flight.
// STORED = true: slot of plane m = dT of plane m and the stored rho-hat of plane m-1 (rows
//   1..14 only), i.e. exactly what step m reads -> ring of 3, each slot refilled as soon as its
//   step ends (hv2's staging rule).
template <typename Real, bool STORED>
struct Geo3 {
    static constexpr int XO = sizeof(Real) == 8 ? 0 : 2;  // lane l <-> box column l + XO
    static constexpr int BX = LX + 2 * XO;                // box width (fp32 boxes start x0 - 4: 16-B aligned)
    static constexpr int BOX = BX * NR;                   // one field, one plane (the 4-D dT box lands its
                                                          // components BOX apart)
    static constexpr int BOXR = BX * (NR - 2);            // one rho-hat component (rows 1..NR-2)
    static constexpr int SR = 0, ST = BOX;                // recompute: R, T_w
    static constexpr int SD = STORED ? 0 : 2 * BOX;       // dT[3]
    static constexpr int SRH = 3 * BOX;                   // stored: rho-hat[6]
    static constexpr int TX_ELEMS = STORED ? 3 * BOX + 6 * BOXR : 5 * BOX;  // bytes / sizeof(Real) per plane
    static constexpr int SLOT = static_cast<int>((TX_ELEMS * sizeof(Real) + 127) / 128 * 128 / sizeof(Real));
    static constexpr int RING = STORED ? 3 : 5;
    static constexpr int LAG = STORED ? 0 : 1;            // the slot freed after step k holds plane k - LAG
    static_assert((BOX * sizeof(Real)) % 128 == 0, "TMA destinations 128-byte aligned");
};

template <int P_>
struct Par {
    static constexpr int P = P_;
};

__device__ __forceinline__ double rsq3(double v) { return rsqrt(v); }
__device__ __forceinline__ float rsq3(float v) { return rsqrtf(v); }

template <typename Real, bool STORED>
__global__ void __launch_bounds__(NT, 1) k_hv3(const __grid_constant__ FArgs a, const __grid_constant__ TmaMaps maps) {
    using G = Geo3<Real, STORED>;
    constexpr int XO = G::XO, BX = G::BX, SR = G::SR, ST = G::ST, SD = G::SD, SLOT = G::SLOT, BOX = G::BOX;
    constexpr int SRH = G::SRH, BOXR = G::BOXR, RING = G::RING, LAG = G::LAG;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    if (a.skip && *a.skip) return;  // uniform
    const TileMeta& tm = a.tm;
    const int nlx = tm.nlx;
    const int tid = threadIdx.x, lane = tid & 31, row = tid >> 5;
    const int mx = static_cast<int>(a.g.m[0]), my = static_cast<int>(a.g.m[1]), mz = static_cast<int>(a.g.m[2]);
    const int xb = blockIdx.x * OX, yb = blockIdx.y * OY;
    const int z0 = tm.zlo + static_cast<int>(blockIdx.z) * tm.zc, z1 = min(tm.zhi, z0 + tm.zc);
    const int ilo = max(z0, a.olo), ihi = min(z1, a.ohi);
    const int xe = min(mx, xb + OX), ye = min(my, yb + OY);
    const int nxA = __ldg(&a.P.base[0][xb]), nyA = __ldg(&a.P.base[1][yb]), nzA = __ldg(&a.P.base[2][z0]);
    const int nlx_t = __ldg(&a.P.base[0][xe - 1]) - nxA + 2;
    const int nly_t = __ldg(&a.P.base[1][ye - 1]) - nyA + 2;
    const long long tile_id = (static_cast<long long>(blockIdx.z) * tm.nty + blockIdx.y) * tm.ntx + blockIdx.x;
    Real* const part = reinterpret_cast<Real*>(a.part) + tile_id * tm.part_stride;
    const std::size_t pstride = static_cast<std::size_t>(tm.nly) * nlx * 3;
    const int msx = static_cast<int>(a.P.src.m[0]), msy = static_cast<int>(a.P.src.m[1]);
    const int msz = static_cast<int>(a.P.src.m[2]);
    const int nxf = a.nxf, nyf = a.nyf, nsl = nxf * nyf * 3, segw = a.segw;

    // ---- shared memory: ring | barriers | z tables (double) | nodal ring, s, fluxes, x-collapsed rows,
    // row table (Real / double) | ints
    Real* const stg = reinterpret_cast<Real*>(smem_raw);
    unsigned long long* const bars = reinterpret_cast<unsigned long long*>(stg + RING * SLOT);  // [RING], 64 B
    double* const sZr = reinterpret_cast<double*>(bars + 8);   // [zc + 8] rem_z of planes kfirst ..
    double* const sry = sZr + tm.zc + 8;                        // [OY]
    Real* const nod = reinterpret_cast<Real*>(sry + OY);        // [NSL][nsl] nodal p
    Real* const sS = nod + NSL * nsl;                           // [2][NR][LX] s by step parity
    Real* const sF = sS + 2 * NR * LX;                          // [2][2][NR][LX] y fluxes (+y, -y) by step parity
    Real* const sQx = sF + 4 * NR * LX;                         // [3][OY][nlx]
    int* const sZb = reinterpret_cast<int*>(sQx + 3 * OY * nlx);  // [zc + 8]
    int* const sby = sZb + tm.zc + 8;                           // [OY]
    const unsigned bar0 = smem_u32(bars);

    // ---- my column
    const int gx = xb - 2 + lane, gy = yb - 2 + row;
    const bool inx = gx >= 0 && gx < mx, iny = gy >= 0 && gy < my;
    const bool cw = row >= 1 && row <= NR - 2;  // coefficient / w rows (warp-uniform)
    const bool zw = row >= 2 && row <= NR - 3;  // output rows
    const int cb = row * BX + lane + XO;        // my box index
    const bool mxm = gx > 0, mxp = gx + 1 < mx, mym = gy > 0, myp = gy + 1 < my;  // in-volume neighbours

    // P p geometry: nodal footprint of the staged region, my bilinear weights
    const int fx0 = __ldg(&a.P.base[0][max(xb - 2, 0)]);
    const int fy0 = __ldg(&a.P.base[1][max(yb - 2, 0)]);
    const int gxc = min(max(gx, 0), mx - 1), gyc = min(max(gy, 0), my - 1);
    const int poff = (__ldg(&a.P.base[0][gxc]) - fx0) + (__ldg(&a.P.base[1][gyc]) - fy0) * nxf;
    const Real prx = static_cast<Real>(__ldg(&a.P.rem[0][gxc])), pry = static_cast<Real>(__ldg(&a.P.rem[1][gyc]));

    // nodal p element this thread loads (host guarantees nsl <= NT); highest threads first
    const long long ns = a.P.src.count(), sm0 = a.P.src.m[0], sm01 = sm0 * a.P.src.m[1];
    const int rt = NT - 1 - tid;
    int sl_off = -1, sl_d = 0;
    if (rt < nsl) {
        const int ix = rt % nxf, iy = (rt / nxf) % nyf;
        sl_d = rt / (nxf * nyf);
        sl_off = min(fx0 + ix, msx - 1) + min(fy0 + iy, msy - 1) * static_cast<int>(sm0);
    }
    Real sl_v = Real(0);
    auto slab_load = [&](int nz) {
        if (sl_off >= 0) sl_v = static_cast<Real>(__ldg(a.p + sl_d * ns + static_cast<long long>(nz) * sm01 + sl_off));
    };
    auto slab_store = [&](int nz) {
        if (sl_off >= 0) nod[(nz & (NSL - 1)) * nsl + rt] = sl_v;
    };
    auto bilerp = [&](int nz, Real& o0, Real& o1, Real& o2) {
        const Real* q = nod + (nz & (NSL - 1)) * nsl + poff;
        const int pl = nxf * nyf;
        o0 = lerp(pry, lerp(prx, q[0], q[1]), lerp(prx, q[nxf], q[nxf + 1]));
        o1 = lerp(pry, lerp(prx, q[pl], q[pl + 1]), lerp(prx, q[pl + nxf], q[pl + nxf + 1]));
        o2 = lerp(pry, lerp(prx, q[2 * pl], q[2 * pl + 1]), lerp(prx, q[2 * pl + nxf], q[2 * pl + nxf + 1]));
    };

    // P^T x collapse geometry: output lanes 2..29 inside the volume; the others form
    // one-lane segments of their own and never write
    const bool xo = lane >= 2 && lane < 2 + OX && gx < mx;
    const int bxc = __ldg(&a.P.base[0][gxc]) - nxA;
    const int bx = xo ? bxc : 1024 + lane;
    const Real rxq = static_cast<Real>(__ldg(&a.P.rem[0][gxc]));
    const bool xlast = xo && gx == xe - 1;
    const int bx_prev = __shfl_up_sync(0xffffffffu, bx, 1);
    const unsigned starts = __ballot_sync(0xffffffffu, lane == 0 || bx_prev != bx);
    const int sst = 31 - __clz(starts & (0xffffffffu >> (31 - lane)));  // first lane of my segment
    const bool send = lane == 31 || ((starts >> (lane + 1)) & 1u);
    const bool pcarry = sst >= 3;  // the previous segment is an output nodal cell (lane sst-1 >= 2)

    if (tid < OY) {
        const int gyr = min(yb + tid, my - 1);
        sby[tid] = __ldg(&a.P.base[1][gyr]) - nyA;
        sry[tid] = __ldg(&a.P.rem[1][gyr]);
    }
    for (int t = tid; t < tm.zc + 8; t += NT) {
        const int kk = min(max(z0 - 2 + t, 0), mz - 1);
        sZb[t] = __ldg(&a.P.base[2][kk]);
        sZr[t] = __ldg(&a.P.rem[2][kk]);
    }
    if (tid == 0) {
        for (int b = 0; b < RING; ++b) mbar_init(&bars[b], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }

    const int kfirst = z0 - 2, klast = z1 + 1;
    // plane m -> slot (m - kfirst) % RING: R, T_w, dT boxes of plane m (one thread; inlined so
    // the tensor maps stay in the kernel's parameter space)
#define HV3_ISSUE(m_)                                                                      \
    do {                                                                                   \
        if (tid == 0) {                                                                    \
            const int rr_ = ((m_) - kfirst) % RING;                                        \
            Real* st_ = stg + rr_ * SLOT;                                                  \
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");                  \
            mbar_expect_tx(&bars[rr_], G::TX_ELEMS * sizeof(Real));                        \
            if constexpr (STORED) {                                                        \
                tma_load_4d(st_ + SRH, &maps.b, xb - 2 - XO, yb - 1, (m_) - 1, 0, &bars[rr_]); \
            } else {                                                                       \
                tma_load_3d(st_ + SR, &maps.a, xb - 2 - XO, yb - 2, (m_), &bars[rr_]);      \
                tma_load_3d(st_ + ST, &maps.b, xb - 2 - XO, yb - 2, (m_), &bars[rr_]);      \
            }                                                                              \
            tma_load_4d(st_ + SD, &maps.c, xb - 2 - XO, yb - 2, (m_), 0, &bars[rr_]);       \
        }                                                                                  \
    } while (0)
    auto zbase = [&](int k) { return sZb[k - kfirst]; };  // k in [kfirst, klast + 3]
    auto zrem = [&](int k) { return static_cast<Real>(sZr[k - kfirst]); };

    auto xcollapse = [&](Real v0, Real v1, Real v2) {
        Real* dst = sQx + (row - 2) * nlx;
        Real A[3] = {(Real(1) - rxq) * v0, (Real(1) - rxq) * v1, (Real(1) - rxq) * v2};
        Real B[3] = {rxq * v0, rxq * v1, rxq * v2};
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            if (o >= segw) break;  // uniform
            const bool in = lane - o >= sst;
#pragma unroll
            for (int d = 0; d < 3; ++d) {
                const Real ua = __shfl_up_sync(0xffffffffu, A[d], o);
                const Real ub = __shfl_up_sync(0xffffffffu, B[d], o);
                A[d] = in ? A[d] + ua : A[d];
                B[d] = in ? B[d] + ub : B[d];
            }
        }
#pragma unroll
        for (int d = 0; d < 3; ++d) {
            const Real bp = __shfl_sync(0xffffffffu, B[d], max(sst - 1, 0));
            if (send && xo) {
                dst[d * OY * nlx + bx] = pcarry ? A[d] + bp : A[d];
                if (xlast) dst[d * OY * nlx + bx + 1] = B[d];
            }
        }
    };
    const int nyi = 3 * nly_t * nlx_t;
    auto ycollapse = [&](int nzp) {
        if (rt < nyi) {
            const int lxn = rt % nlx_t, lyn = (rt / nlx_t) % nly_t, d = rt / (nlx_t * nly_t);
            const Real* q = sQx + d * OY * nlx + lxn;
            Real v = Real(0);
#pragma unroll
            for (int r = 0; r < OY; ++r) {
                const int b = sby[r];
                const Real ry = static_cast<Real>(sry[r]);
                const Real wgt = b == lyn ? Real(1) - ry : (b == lyn - 1 ? ry : Real(0));
                v = fma(wgt, q[r * nlx], v);
            }
            part[static_cast<std::size_t>(nzp - nzA) * pstride + (lyn * nlx + lxn) * 3 + d] = v;
        }
    };

    // coefficient constants
    const Real i0 = static_cast<Real>(a.ih2[0]), i1 = static_cast<Real>(a.ih2[1]), i2 = static_cast<Real>(a.ih2[2]);
    const Real hx = static_cast<Real>(a.hh[0]), hy = static_cast<Real>(a.hh[1]), hz = static_cast<Real>(a.hh[2]);
    const Real taurho = static_cast<Real>(a.tau * a.rho), tau2 = static_cast<Real>(a.tau * a.tau),
               rho2 = static_cast<Real>(a.rho * a.rho);
    const Real scale = static_cast<Real>(a.scale);

    pdl_wait();       // p (the CG update before this launch) from here on
    __syncthreads();  // tables, barriers
    int slab_hi;
    {
        const int nz0 = zbase(kfirst);
        slab_hi = min(zbase(kfirst + 2) + 1, msz - 1);
        for (int nz = nz0; nz <= slab_hi; ++nz) {
            slab_load(nz);
            slab_store(nz);
        }
    }
    for (int m = 0; m < RING - LAG; ++m)
        if (kfirst + m <= klast) HV3_ISSUE(kfirst + m);
    int slot = 0;        // ring slot of plane k
    unsigned phase = 0;  // its mbarrier parity
    __syncthreads();

    // ---- loop state, histories named by step parity P = (k - kfirst) & 1
    int pz = -1000;
    Real Pa0 = 0, Pa1 = 0, Pa2 = 0, Pb0 = 0, Pb1 = 0, Pb2 = 0;  // P p at nodal planes bz, bz+1
    Real Rh[2] = {0, 0}, Th[2] = {0, 0};                        // own R, T_w of planes k-1 / k-2 by parity
    Real sh[2] = {0, 0};                                        // own s
    Real dq[2][3] = {{0, 0, 0}, {0, 0, 0}};                     // own dT
    Real fzp[2] = {0, 0};                                       // rho-hat(+z) w of plane k-3 (for Z of k-2)
    Real swv[2] = {0, 0}, gxv[2] = {0, 0};                      // sigma w and x inflow of plane k-2
    Real acc00 = 0, acc01 = 0, acc02 = 0, acc10 = 0, acc11 = 0, acc12 = 0;
    int cur = nzA, ypend = -1;

    auto step = [&](auto parc, int k) {
        constexpr int P = decltype(parc)::P;
        if (ypend >= 0) {  // y collapse of the plane completed last step (sQx published by the barrier)
            ycollapse(ypend);
            ypend = -1;
        }
        bool slab_pending = false;
        int slab_nz = 0;
        {
            const int nzq = min(zbase(k + 3) + 1, msz - 1);
            if (nzq > slab_hi) {
                slab_load(nzq);
                slab_pending = true;
                slab_nz = nzq;
                slab_hi = nzq;
            }
        }
        const int bzk = zbase(k);
        if (bzk != pz) {  // uniform: new nodal plane pair
            if (bzk == pz + 1) {
                Pa0 = Pb0;
                Pa1 = Pb1;
                Pa2 = Pb2;
            } else {
                bilerp(bzk, Pa0, Pa1, Pa2);
            }
            bilerp(min(bzk + 1, msz - 1), Pb0, Pb1, Pb2);
            pz = bzk;
        }
        mbar_wait_at(bar0 + 8 * slot, phase);
        const Real* st = stg + slot * SLOT;                                  // plane k
        const Real* sp = stg + (slot == 0 ? RING - 1 : slot - 1) * SLOT;     // plane k-1
        // ---- P: plane k (all rows, all lanes)
        const Real rzk = zrem(k);
        const Real D0 = st[SD + cb], D1 = st[SD + BOX + cb], D2 = st[SD + 2 * BOX + cb];
        const Real s_k = fma(D0, lerp(rzk, Pa0, Pb0), fma(D1, lerp(rzk, Pa1, Pb1), D2 * lerp(rzk, Pa2, Pb2)));
        sS[P * NR * LX + tid] = s_k;
        Real R_k = Real(0), T_k = Real(0);
        if constexpr (!STORED) {
            R_k = st[SR + cb];
            T_k = st[ST + cb];
        }
        // ---- coefficients and w at plane j = k-1 (rows 1..14)
        const int j = k - 1;
        Real fzm = 0, fzp_new = 0, sw_new = 0, gx_new = 0;
        if (STORED && cw && k >= kfirst + 2) {  // uniform; the coefficients as the eval pass stored them
            const Real* rh = st + SRH + (row - 1) * BX + lane + XO;  // (zero across the boundary / outside)
            const Real c0 = rh[0], c1 = rh[BOXR], c2 = rh[2 * BOXR], c3 = rh[3 * BOXR], c4 = rh[4 * BOXR],
                       c5 = rh[5 * BOXR];
            const Real sj = sh[1 - P];
            const Real* sn = sS + (1 - P) * NR * LX + tid;  // plane j (written last step)
            const Real sxm = __shfl_up_sync(0xffffffffu, sj, 1), sxp = __shfl_down_sync(0xffffffffu, sj, 1);
            const Real wa = fma(c1, sxp - sj, c0 * (sxm - sj));
            const Real wb = fma(c3, sn[LX] - sj, c2 * (sn[-LX] - sj));
            const Real wc = fma(c5, s_k - sj, c4 * (sh[P] - sj));
            const Real w = (wa + wb) + wc;
            const Real fpx = __shfl_up_sync(0xffffffffu, c1 * w, 1);    // from lane - 1 (its +x)
            const Real fmx = __shfl_down_sync(0xffffffffu, c0 * w, 1);  // from lane + 1 (its -x)
            gx_new = fpx + fmx;
            Real* const Fj = sF + P * 2 * NR * LX + tid;
            Fj[0] = c3 * w;        // +y flux (row + 1 reads it)
            Fj[NR * LX] = c2 * w;  // -y flux (row - 1 reads it)
            fzm = c4 * w;
            fzp_new = c5 * w;
            sw_new = (((c0 + c1) + (c2 + c3)) + (c4 + c5)) * w;
        }
        if (!STORED && cw && k >= kfirst + 2) {  // uniform
            const Real Rj = Rh[1 - P], Tj = Th[1 - P];
            const bool ok = inx && iny && j >= 0 && j < mz;
            const bool mzm = j > 0, mzp = j + 1 < mz;
            // in-plane neighbours: x by shuffle, y from the staged box of plane j
            const Real Rxm = __shfl_up_sync(0xffffffffu, Rj, 1), Rxp = __shfl_down_sync(0xffffffffu, Rj, 1);
            const Real Txm = __shfl_up_sync(0xffffffffu, Tj, 1), Txp = __shfl_down_sync(0xffffffffu, Tj, 1);
            const Real Rym = sp[SR + cb - BX], Ryp = sp[SR + cb + BX];
            const Real Tym = sp[ST + cb - BX], Typ = sp[ST + cb + BX];
            const Real dR0 = mxm ? Rxm - Rj : Real(0), dR1 = mxp ? Rxp - Rj : Real(0);
            const Real dR2 = mym ? Rym - Rj : Real(0), dR3 = myp ? Ryp - Rj : Real(0);
            const Real dR4 = mzm ? Rh[P] - Rj : Real(0), dR5 = mzp ? R_k - Rj : Real(0);
            const Real dT0 = mxm ? Txm - Tj : Real(0), dT1 = mxp ? Txp - Tj : Real(0);
            const Real dT2 = mym ? Tym - Tj : Real(0), dT3 = myp ? Typ - Tj : Real(0);
            const Real dT4 = mzm ? Th[P] - Tj : Real(0), dT5 = mzp ? T_k - Tj : Real(0);
            const Real stt = fma(fma(dT0, dT0, dT1 * dT1), i0, fma(fma(dT2, dT2, dT3 * dT3), i1, fma(dT4, dT4, dT5 * dT5) * i2));
            const Real srr = fma(fma(dR0, dR0, dR1 * dR1), i0, fma(fma(dR2, dR2, dR3 * dR3), i1, fma(dR4, dR4, dR5 * dR5) * i2));
            const Real num = fma(Real(0.5), fma(fma(dT0, dR0, dT1 * dR1), i0, fma(fma(dT2, dR2, dT3 * dR3), i1, fma(dT4, dR4, dT5 * dR5) * i2)),
                                 taurho);
            const Real nt2 = fma(Real(0.5), stt, tau2);
            const Real nr2 = fma(Real(0.5), srr, rho2);
            const Real in1 = rsq3(nt2 * nr2);
            const Real in2 = num * ((in1 * in1) * (in1 * nr2));
            // hat-h folded into the two factors per axis
            const Real ax = ok ? hx * in1 : Real(0), bx2 = ok ? hx * in2 : Real(0);
            const Real ay = ok ? hy * in1 : Real(0), by2 = ok ? hy * in2 : Real(0);
            const Real az = ok ? hz * in1 : Real(0), bz2 = ok ? hz * in2 : Real(0);
            const Real c0 = fma(dR0, ax, -dT0 * bx2), c1 = fma(dR1, ax, -dT1 * bx2);
            const Real c2 = fma(dR2, ay, -dT2 * by2), c3 = fma(dR3, ay, -dT3 * by2);
            const Real c4 = fma(dR4, az, -dT4 * bz2), c5 = fma(dR5, az, -dT5 * bz2);
            // w = sum_k c_k (s_{t+k} - s_t)
            const Real sj = sh[1 - P];
            const Real* sn = sS + (1 - P) * NR * LX + tid;  // plane j (written last step)
            const Real sxm = __shfl_up_sync(0xffffffffu, sj, 1), sxp = __shfl_down_sync(0xffffffffu, sj, 1);
            const Real wa = fma(c1, sxp - sj, c0 * (sxm - sj));
            const Real wb = fma(c3, sn[LX] - sj, c2 * (sn[-LX] - sj));
            const Real wc = fma(c5, s_k - sj, c4 * (sh[P] - sj));
            const Real w = (wa + wb) + wc;
            // fluxes: x by shuffle, y through shared memory, z and sigma w in registers
            const Real fpx = __shfl_up_sync(0xffffffffu, c1 * w, 1);    // from lane - 1 (its +x)
            const Real fmx = __shfl_down_sync(0xffffffffu, c0 * w, 1);  // from lane + 1 (its -x)
            gx_new = fpx + fmx;
            Real* const Fj = sF + P * 2 * NR * LX + tid;
            Fj[0] = c3 * w;        // +y flux (row + 1 reads it)
            Fj[NR * LX] = c2 * w;  // -y flux (row - 1 reads it)
            fzm = c4 * w;
            fzp_new = c5 * w;
            sw_new = (((c0 + c1) + (c2 + c3)) + (c4 + c5)) * w;
        }
        // ---- dr^T and P^T: plane i = k-2 (rows 2..13)
        const int i = k - 2;
        const bool zact = i >= ilo && i < ihi;  // CTA-uniform
        const int bz = zact ? zbase(i) : cur;
        if (zw && zact) {  // warp-uniform
            const Real* Fi = sF + (1 - P) * 2 * NR * LX + tid;
            const Real z = ((gxv[1 - P] + fzp[P]) + (Fi[-LX] + Fi[NR * LX + LX])) + (fzm - swv[1 - P]);
            const Real sz = scale * z;  // dT (TMA zero fill) makes q vanish outside the volume
            const Real q0 = sz * dq[P][0], q1 = sz * dq[P][1], q2 = sz * dq[P][2];
            const Real rz = zrem(i);
            if (bz > cur) {  // nodal plane `cur` complete: x collapse now, y collapse after the barrier
                xcollapse(acc00, acc01, acc02);
                acc00 = acc10;
                acc01 = acc11;
                acc02 = acc12;
                acc10 = acc11 = acc12 = Real(0);
            }
            acc00 = fma(Real(1) - rz, q0, acc00);
            acc10 = fma(rz, q0, acc10);
            acc01 = fma(Real(1) - rz, q1, acc01);
            acc11 = fma(rz, q1, acc11);
            acc02 = fma(Real(1) - rz, q2, acc02);
            acc12 = fma(rz, q2, acc12);
        }
        if (bz > cur) {  // every thread tracks the completed plane (the y collapse runs on rows 14-15)
            ypend = cur;
            cur = bz;
        }
        // ---- histories (parity P slots now hold plane k)
        if constexpr (!STORED) {
            Rh[P] = R_k;
            Th[P] = T_k;
        }
        sh[P] = s_k;
        dq[P][0] = D0;
        dq[P][1] = D1;
        dq[P][2] = D2;
        fzp[P] = fzp_new;
        swv[P] = sw_new;
        gxv[P] = gx_new;
        if (slab_pending) slab_store(slab_nz);
        __syncthreads();
        // the slot of plane k - LAG is free: refill it with plane k - LAG + RING
        if (k - LAG + RING <= klast) HV3_ISSUE(k - LAG + RING);
        if (++slot == RING) {
            slot = 0;
            phase ^= 1u;
        }
    };
#pragma unroll 1
    for (int k = kfirst; k <= klast; k += 2) {
        step(Par<0>{}, k);
        if (k + 1 <= klast) step(Par<1>{}, k + 1);
    }
    pdl_trigger();  // the finalize may be scheduled while the tiles flush
    // ---- flush: pending y collapse, then the last two nodal planes
    if (ypend >= 0) ycollapse(ypend);
    __syncthreads();
    if (zw) xcollapse(acc00, acc01, acc02);
    __syncthreads();
    ycollapse(cur);
    __syncthreads();
    if (zw) xcollapse(acc10, acc11, acc12);
    __syncthreads();
    ycollapse(cur + 1);
#undef HV3_ISSUE
}

template <typename Real>
std::size_t smem3(int nlx, int nsl, int zc, bool stored) {
    const std::size_t bx = sizeof(Real) == 8 ? LX : LX + 4;
    const std::size_t slot = ((stored ? 3 * bx * NR + 6 * bx * (NR - 2) : 5 * bx * NR) * sizeof(Real) + 127) / 128 * 128;
    return static_cast<std::size_t>(stored ? 3 : 5) * slot + 64 +
           (static_cast<std::size_t>(zc) + 8 + OY) * sizeof(double) +
           (static_cast<std::size_t>(NSL) * nsl + 2 * NR * LX + 4 * NR * LX + 3 * OY * static_cast<std::size_t>(nlx)) *
               sizeof(Real) +
           (static_cast<std::size_t>(zc) + 8 + OY) * sizeof(int);
}

}  // namespace

std::size_t hv3_smem_bytes(int nlx, int nsl, int zc, bool fp32, bool stored) {
    return fp32 ? smem3<float>(nlx, nsl, zc, stored) : smem3<double>(nlx, nsl, zc, stored);
}
int hv3_tile_x() { return OX; }
int hv3_tile_y() { return OY; }
int hv3_threads() { return NT; }
int hv3_box_width(bool fp32) { return fp32 ? LX + 4 : LX; }
int hv3_box_rows() { return NR; }
int hv3_box_origin(bool fp32) { return fp32 ? 4 : 2; }  // box x0 = tile x0 - this

#if (MFREG_HV3_OY + 4) * 36 * 4 % 128 == 0
#define MFREG_HV3_F32 1  // fp32 boxes (36 wide) stay 128-byte aligned for this tile height
#else
#define MFREG_HV3_F32 0
#endif
bool hv3_fp32_ok() { return MFREG_HV3_F32 != 0; }

void hv3_set_smem_cap(int bytes) {
    MFREG_CUDA(cudaFuncSetAttribute(k_hv3<double, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    MFREG_CUDA(cudaFuncSetAttribute(k_hv3<double, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
#if MFREG_HV3_F32
    MFREG_CUDA(cudaFuncSetAttribute(k_hv3<float, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    MFREG_CUDA(cudaFuncSetAttribute(k_hv3<float, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
#endif
}

void hv3_launch(const FArgs& a, const TmaMaps& maps, dim3 grid, std::size_t smem, cudaStream_t s, bool fp32,
                bool stored) {
#if MFREG_HV3_F32
    if (fp32) {
        if (stored) launch_pdl(k_hv3<float, true>, grid, dim3(NT), smem, s, a, maps);
        else launch_pdl(k_hv3<float, false>, grid, dim3(NT), smem, s, a, maps);
        return;
    }
#endif
    if (stored) launch_pdl(k_hv3<double, true>, grid, dim3(NT), smem, s, a, maps);
    else launch_pdl(k_hv3<double, false>, grid, dim3(NT), smem, s, a, maps);
}

}  // namespace mfreg_b200
