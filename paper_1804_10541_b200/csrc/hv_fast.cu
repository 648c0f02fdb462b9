// Gauss-Newton Hv image pass, two CTAs per SM (fast mode).
//
// Same algebra as k_fused<false> (fused.cuh): s = dT . P p, w = dr s,
// z = dr^T w, q^ = 2h z dT, P^T into per-tile partials. What differs is the
// execution scheme, built so that two 256-thread CTAs fit one SM (113 KB of
// shared memory and 128 registers per thread each), so one CTA's barrier and
// TMA waits are covered by the other CTA's arithmetic:
//  * one thread per output column of the 32x8 tile; the halo columns are extra
//    work items of threads 0..163 (ring-1 edges: P and W, ring-1 corners and
//    ring-2 edges: P only) instead of dedicated halo warps; their geometry is
//    packed into one word per item in shared memory (re-read per use in fp64);
//  * TMA staging per step: dT of plane k (36x12 s region, read by P) in a ring of
//    3 and rho-hat of plane k-1 (36x10 w rows, read by W of plane k-1 in the same
//    step) in a ring of 3, both 2 steps ahead, so a slot is consumed in exactly one
//    step and no coefficient is carried in registers;
//  * the dr^T stage reads fluxes instead of (coefficient, w) pairs: W of
//    column t forms rho-hat_t(k) w_t for its in-plane neighbours; x fluxes move
//    inside the warp (a warp is one tile row) by shuffles, y fluxes through two
//    consumer-indexed shared arrays, the z fluxes and sigma_t w_t stay in the
//    column's registers, so z_i is 2-3 shared loads + a few adds;
//  * nodal interpolants: item 0's in registers, the halo items' in shared memory;
//    fp64 reads the nodes at a plane change from L1/L2, FAST32 from a shared ring
//    of the tile's nodal footprint filled one step ahead;
//  * P^T: per-column z weights in registers; on a completed nodal plane each warp
//    (one tile row) collapses x through its shared row and the per-tile weight
//    tables (ptc.cuh; FAST32: a segmented shuffle scan) and the y collapse runs one
//    step later, after the regular barrier — no extra barriers in the plane loop
//    (the host guarantees nodal z cells of >= 2 image planes, so completions are
//    >= 2 steps apart).
// Boundary semantics are those of the TMA zero fill: rho-hat and dT vanish
// outside the volume, and the eval pass stores zero coefficients across it.
// Tile height 16 (512 threads, one CTA per SM) is instantiated too (MFREG_HV16=1).
// Compile-time switches: MFREG_HV2_SLAB (fp64 shared nodal ring), MFREG_HV2_RRING
// (rho-hat ring depth), MFREG_HV2_EXP (timing experiments with wrong results:
// scripts/variants.py builds only).
#include <cstdint>

#include "ptc.cuh"

#ifndef MFREG_REVMAP
#define MFREG_REVMAP 1
#endif
#ifndef MFREG_HV2_EXP
#define MFREG_HV2_EXP 0  // timing experiments only (wrong results): 1 no P^T collapse, 2 no halo items
#endif
#ifndef MFREG_HV2_PAD
#define MFREG_HV2_PAD 1  // conflict-free P^T x stage (ptc.cuh): +1.7 KB of shared memory
#endif
#ifndef MFREG_HV2_SPLIT
#define MFREG_HV2_SPLIT 0  // split (arrive / wait) step barrier on an mbarrier
#endif
#ifndef MFREG_HV2_BF
#define MFREG_HV2_BF 1  // branch-free y flux stores (padded flux arrays: the last / first tile row writes a junk row)
#endif
#ifndef MFREG_HV2_WF
#define MFREG_HV2_WF 1  // w = sum_k rho_k s_{t+k} - sigma s_t (FMA chains) instead of sum_k rho_k (s_{t+k} - s_t)
#endif

namespace mfreg_b200 {

namespace {

using namespace fdev;

constexpr int TX = FT_X;                               // 32-column output tiles
constexpr int DRING = 3;                               // dT staging slots (2 planes ahead)
#ifndef MFREG_HV2_RRING
#define MFREG_HV2_RRING 2  // one plane ahead (3: 17 KB more shared memory, which the padded P^T rows need)
#endif
#ifndef MFREG_HV2_SLAB
#define MFREG_HV2_SLAB 0   // nodal footprint in shared memory (1) or the interpolants read from L1/L2 (0)
#endif
// per precision: the shared-memory-bound switches apply to fp64 (FAST32 measured 1.3% slower with
// them: its 4-byte rows conflict less and its rho-hat ring of 3 fits anyway)
template <typename Real>
struct Cfg {
    static constexpr bool F64 = sizeof(Real) == 8;
    static constexpr int RRING = F64 ? MFREG_HV2_RRING : 3;  // rho-hat staging slots (RRING - 1 planes ahead)
    static constexpr bool PAD = F64 && MFREG_HV2_PAD, BF = F64 && MFREG_HV2_BF, WF = F64 && MFREG_HV2_WF;
};
constexpr int NSL = 4;                                 // nodal plane ring (power of 2)

// Tile height variants: 32 x 8 (256 threads, two CTAs per SM; shares the eval pass's tiling) and
// 32 x 16 (512 threads, one CTA per SM, own tiling): the halo columns per output column drop
// from 0.64 (P) / 0.31 (W) to 0.38 / 0.19
template <int TY_>
struct Tl {
    static constexpr int TY = TY_;
    static constexpr int SY = TY + 4, WY = TY + 2;          // s region rows / rho-hat rows
    static constexpr int NT = TX * TY;                      // threads
    static constexpr int NX_W = 2 * TX + 2 * TY;            // extra items [0, NX_W): ring-1 edges (P + W)
    static constexpr int NX_P = NX_W + 4 + 2 * TX + 2 * TY;  // then ring-1 corners, ring-2 edges (P only)
    static constexpr int MINB = TY == 8 ? 2 : 1;            // CTAs per SM
    // consumer-indexed y flux arrays of one plane parity: +y at 0, -y at FM; branch-free stores pad
    // each with a junk row (+y: after, written by the last tile row; -y: before, by the first)
    template <bool BF>
    static constexpr int FM = BF ? NT + 2 * TX : NT;
    template <bool BF>
    static constexpr int FPAR = BF ? 2 * NT + 2 * TX : 2 * NT;
};

// Box geometry per state precision: a TMA box must start 16-byte aligned in x, so the
// boxes start XO columns left of the tile (x0 - 2 for fp64, x0 - 4 for fp32) and are
// SX = 32 + 2 XO wide; the s frame is SX x 12, the rho-hat box SX x 10 (one row lower).
template <typename Real, int TY_>
struct Geo {
    static constexpr int SY = Tl<TY_>::SY, WY = Tl<TY_>::WY;
    static constexpr int XO = sizeof(Real) == 8 ? 2 : 4;
    static constexpr int SX = TX + 2 * XO, NS = SX * SY, NW = SX * WY;
    static constexpr int SLOT_DT = 3 * NS;              // dT box [3][12][SX]
    static constexpr int SLOT_RH = 6 * NW;              // rho-hat box [6][10][SX]
    static_assert((SLOT_DT * sizeof(Real)) % 128 == 0 && (SLOT_RH * sizeof(Real)) % 128 == 0, "TMA boxes 128-byte aligned");
};

// extra work item e -> column (lx, ly) in the s frame (tile columns at lx = XO .. XO+31);
// `dir` = consumer flux array of a ring-1 edge item (0: +x, 1: -x, 2: +y, 3: -y)
template <int XO, int TY_>
__device__ __forceinline__ void extra_item(int e, int& lx, int& ly, int& dir) {
    constexpr int TY = TY_, SY = Tl<TY_>::SY, NX_W = Tl<TY_>::NX_W;
    dir = -1;
    if (e < TX) { lx = XO + e; ly = 1; dir = 2; }                               // ring-1, y = -1 row: feeds +y
    else if (e < 2 * TX) { lx = XO + e - TX; ly = SY - 2; dir = 3; }            // ring-1, y = TY row: feeds -y
    else if (e < 2 * TX + TY) { lx = XO - 1; ly = 2 + e - 2 * TX; dir = 0; }   // ring-1, x = -1: feeds +x
    else if (e < NX_W) { lx = XO + TX; ly = 2 + e - 2 * TX - TY; dir = 1; }     // ring-1, x = TX: feeds -x
    else if (e < NX_W + 4) {                                                    // ring-1 corners
        const int q = e - NX_W;
        lx = (q & 1) ? XO + TX : XO - 1;
        ly = (q & 2) ? SY - 2 : 1;
    } else {                                                                    // ring-2 edges
        const int r = e - NX_W - 4;
        if (r < TX) { lx = XO + r; ly = 0; }
        else if (r < 2 * TX) { lx = XO + r - TX; ly = SY - 1; }
        else if (r < 2 * TX + TY) { lx = XO - 2; ly = 2 + r - 2 * TX; }
        else { lx = XO + TX + 1; ly = 2 + r - 2 * TX - TY; }
    }
}

template <int P_>
struct Par {
    static constexpr int P = P_;
};

template <typename Real, int TY_>
__global__ void __launch_bounds__(Tl<TY_>::NT, Tl<TY_>::MINB) k_hv2(const __grid_constant__ FArgs a, const __grid_constant__ TmaMaps maps) {
    using G = Geo<Real, TY_>;
    using C = Cfg<Real>;
    constexpr int RRING = C::RRING;
    // FAST32 keeps the nodal footprint in shared memory (its smem has room; the L1/L2 reads of the
    // interpolants at a plane change stall it); fp64 reads them from L1/L2 (no room for the ring)
    constexpr bool SLAB = MFREG_HV2_SLAB || sizeof(Real) == 4;
    constexpr int TY = TY_, SY = Tl<TY_>::SY, NT = Tl<TY_>::NT, NX_W = Tl<TY_>::NX_W, NX_P = Tl<TY_>::NX_P;
    (void)SY;
    constexpr int XO = G::XO, SX = G::SX, NS = G::NS, NW = G::NW, SLOT_DT = G::SLOT_DT, SLOT_RH = G::SLOT_RH;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    if (a.skip && *a.skip) return;  // uniform
    const TileMeta& tm = a.tm;
    const int nlx = tm.nlx;
    const int tid = threadIdx.x, lane = tid & 31, row = tid >> 5;
    const int mx = static_cast<int>(a.g.m[0]), my = static_cast<int>(a.g.m[1]), mz = static_cast<int>(a.g.m[2]);
    const int x0 = blockIdx.x * TX, y0 = blockIdx.y * TY;
    const int bzc = static_cast<int>(blockIdx.z) + a.zch0;  // z tile chunk
    const int z0 = tm.zlo + bzc * tm.zc, z1 = min(tm.zhi, z0 + tm.zc);
    const int ilo = max(z0, a.olo), ihi = min(z1, a.ohi);
    const int xe = min(mx, x0 + TX), ye = min(my, y0 + TY);
    const int nxA = __ldg(&a.P.base[0][x0]), nyA = __ldg(&a.P.base[1][y0]), nzA = __ldg(&a.P.base[2][z0]);
    const int nlx_t = __ldg(&a.P.base[0][xe - 1]) - nxA + 2;
    const int nly_t = __ldg(&a.P.base[1][ye - 1]) - nyA + 2;
    const long long tile_id = (static_cast<long long>(bzc) * tm.nty + blockIdx.y) * tm.ntx + blockIdx.x;
    Real* const part = reinterpret_cast<Real*>(a.part) + tile_id * tm.part_stride;
    const std::size_t pstride = static_cast<std::size_t>(tm.nly) * nlx * 3;
    const int msx = static_cast<int>(a.P.src.m[0]), msy = static_cast<int>(a.P.src.m[1]);
    const int msz = static_cast<int>(a.P.src.m[2]);
    const int segw = a.segw;

    // ---- shared memory: dT ring | rho-hat ring | barriers | z table (fp64) | nodal ring, s planes,
    // fluxes, item-1 interpolants, P^T rows (Real) | int tables
    Real* const stgD = reinterpret_cast<Real*>(smem_raw);       // [DRING][SLOT_DT]
    Real* const stgR = stgD + DRING * SLOT_DT;                   // [RRING][SLOT_RH]
    unsigned long long* const bars = reinterpret_cast<unsigned long long*>(stgR + RRING * SLOT_RH);  // [DRING + RRING]
    double* const sZr = reinterpret_cast<double*>(bars + 8);  // [zc + 8] rem_z of the planes kfirst ..
    const int nxf = a.nxf, nyf = a.nyf, pl = nxf * nyf, nsl = 3 * pl;
    Real* const slab = reinterpret_cast<Real*>(sZr + tm.zc + 8);  // [NSL][3][nyf][nxf] nodal p footprint
    Real* const sS = slab + (SLAB ? NSL * nsl : 0);  // [2][NS] by plane parity
    constexpr int FM = Tl<TY_>::template FM<C::BF>, FPAR = Tl<TY_>::template FPAR<C::BF>;
    Real* const sF = sS + 2 * NS;               // [2][FPAR] consumer-indexed y fluxes by plane parity
    Real* const sE = sF + 2 * FPAR;             // [2][2][TY] x fluxes from the ring-1 x edges by plane parity,
                                                // then 2 zero entries (the edge-flux slot of inner lanes)
    Real* const sQ1 = sE + 2 * 2 * TY + 2;      // [6][NX_P] item-1 P p at nodal planes bz, bz+1
    // P^T collapse buffers and tables (ptc.cuh)
    Real* const sPt = sQ1 + 6 * NX_P;
    int* const sZb = reinterpret_cast<int*>(sPt + ptc_reals(TY, nlx, tm.nly, segw, C::PAD));  // [zc + 8] base_z of planes kfirst ..
    int* const sI1 = sZb + tm.zc + 8;           // [NX_P] packed item-1 geometry
    Ptc<Real, TY, C::PAD> ptc(sPt, sI1 + NX_P, nlx, tm.nly, segw, nlx_t, nly_t);
    const unsigned barD = smem_u32(bars), barR = barD + 8 * DRING;
    // split step barrier (fp64, MFREG_HV2_SPLIT): threads arrive on an mbarrier at the end of a
    // step and wait for it only after the next step's TMA wait, nodal interpolants and P values,
    // which touch nothing another thread writes (FAST32's shared nodal ring would)
    constexpr bool SPLIT = MFREG_HV2_SPLIT && sizeof(Real) == 8 && !SLAB;
    const unsigned barS = barD + 8 * 7;

    // ---- per-thread columns: item 0 = tile column (tx, ty) = (lane, row); item 1 = extra halo column
    const int tx = lane, ty = row;
    const int c0 = (tx + XO) + (ty + 2) * SX, w0 = c0 - SX;  // s frame / rho-hat frame (one row lower)
    const int gx0 = x0 + tx, gy0 = y0 + ty;
    const bool has1 = (MFREG_HV2_EXP & 2) ? false : tid < NX_P, w1 = (MFREG_HV2_EXP & 2) ? false : tid < NX_W;  // warp-aligned except warp 2 (split P+W / P) and warp 5
    // item-1 geometry, packed once into shared memory and re-read where it is used (keeping it
    // live in registers across the plane loop costs more than the loads): bits 0-9 the s-frame
    // index c1, 10-20 the flux slot f1, 21-22 the coefficient toward the tile, 23 x edge
    if (has1) {
        int lx1 = 0, ly1 = 0, dir1 = -1;
        extra_item<XO, TY>(tid, lx1, ly1, dir1);
        // where the ring-1 edge flux goes: y edges -> consumer-indexed sF (+y: 0, -y: 1), x edges -> sE
        const bool xedge = dir1 == 0 || dir1 == 1;
        const int f1 = xedge ? dir1 * TY + min(max(ly1 - 2, 0), TY - 1)
                             : (dir1 - 2) * FM + min(max(lx1 - XO, 0), TX - 1) + (dir1 == 2 ? 0 : TY - 1) * TX;
        const int ci = dir1 == 0 ? 1 : (dir1 == 1 ? 0 : (dir1 == 2 ? 3 : 2));
        static_assert(G::NS <= 1024 && FPAR <= 2048, "item-1 packing");
        sI1[tid] = (lx1 + ly1 * SX) | (max(f1, 0) << 10) | (ci << 21) | (xedge ? 1 << 23 : 0);
    }
    // (FAST32 has registers to spare: it keeps the packed word in one instead of reloading it)
    const int e1r = has1 ? sI1[tid] : 0;
    auto item1 = [&]() { return sizeof(Real) == 8 ? lds_v(sI1 + tid) : e1r; };

    // P p: the tile's nodal footprint (nxf x nyf nodes from (fx0, fy0), clamped at the last node)
    // of four nodal planes in shared memory, each plane loaded one step before its first use (<= 2
    // elements per thread, held in registers across the step); a column's bilinear interpolant
    // reads its cell's four nodes from there
    const long long ns = a.P.src.count(), sm0 = a.P.src.m[0], sm01 = sm0 * a.P.src.m[1];
    const int fx0 = __ldg(&a.P.base[0][max(x0 - 2, 0)]), fy0 = __ldg(&a.P.base[1][max(y0 - 2, 0)]);
    auto col_geom = [&](int gx, int gy, int& off, double& rx, double& ry) {
        const int gxc = min(max(gx, 0), mx - 1), gyc = min(max(gy, 0), my - 1);
        const int bx = __ldg(&a.P.base[0][gxc]), by = __ldg(&a.P.base[1][gyc]);
        off = SLAB ? (bx - fx0) + (by - fy0) * nxf : bx + by * static_cast<int>(sm0);
        rx = __ldg(&a.P.rem[0][gxc]);
        ry = __ldg(&a.P.rem[1][gyc]);
    };
    auto bilerp = [&](int nz, int off, Real rx, Real ry, Real& o0, Real& o1, Real& o2) {
        if constexpr (SLAB) {
            const Real* q = slab + (nz & (NSL - 1)) * nsl + off;
            o0 = lerp(ry, lerp(rx, q[0], q[1]), lerp(rx, q[nxf], q[nxf + 1]));
            o1 = lerp(ry, lerp(rx, q[pl], q[pl + 1]), lerp(rx, q[pl + nxf], q[pl + nxf + 1]));
            o2 = lerp(ry, lerp(rx, q[2 * pl], q[2 * pl + 1]), lerp(rx, q[2 * pl + nxf], q[2 * pl + nxf + 1]));
        } else {
            // one row pointer per component and y, +1 for x (the transfer plan clamps base to
            // [0, m-2], transfer.cpp:30-33, so the +x / +y neighbours exist)
            const double* q0 = a.p + (static_cast<long long>(nz) * sm01 + off);
            const double* q1 = q0 + ns;
            const double* q2 = q1 + ns;
            auto v = [](const double* q) { return static_cast<Real>(__ldg(q)); };
            o0 = lerp(ry, lerp(rx, v(q0), v(q0 + 1)), lerp(rx, v(q0 + sm0), v(q0 + sm0 + 1)));
            o1 = lerp(ry, lerp(rx, v(q1), v(q1 + 1)), lerp(rx, v(q1 + sm0), v(q1 + sm0 + 1)));
            o2 = lerp(ry, lerp(rx, v(q2), v(q2 + 1)), lerp(rx, v(q2 + sm0), v(q2 + sm0 + 1)));
        }
    };
    // footprint elements of this thread (highest threads first: the halo items sit on the lowest)
    const int rt = NT - 1 - tid;
    int sl_off[2];  // element index within nodal plane 0 (component included), -1: none
    Real sl_v[2] = {Real(0), Real(0)};
#pragma unroll
    for (int u = 0; u < 2; ++u) {
        const int t = rt + u * NT;
        sl_off[u] = -1;
        if (t < nsl) {
            const int d = t / pl, r = t - d * pl, iy = r / nxf, ix = r - iy * nxf;
            sl_off[u] = static_cast<int>(d * ns + min(fy0 + iy, msy - 1) * sm0 + min(fx0 + ix, msx - 1));
        }
    }
    auto slab_load = [&](int nz) {
        if constexpr (!SLAB) return;
        const double* q = a.p + static_cast<long long>(nz) * sm01;
#pragma unroll
        for (int u = 0; u < 2; ++u)
            if (sl_off[u] >= 0) sl_v[u] = static_cast<Real>(__ldg(q + sl_off[u]));
    };
    auto slab_store = [&](int nz) {
        if constexpr (!SLAB) return;
        Real* dst = slab + (nz & (NSL - 1)) * nsl;
#pragma unroll
        for (int u = 0; u < 2; ++u)
            if (sl_off[u] >= 0) dst[rt + u * NT] = sl_v[u];
    };

    // edge-flux slot of the tile column (lanes 0 / 31 read a ring-1 x edge, the others a zero
    // slot past both parity halves); in-row x flux masks
    const int eoff = tx == 0 ? ty : (tx == TX - 1 ? TY + ty : -1);
    const Real mpx = tx > 0 ? Real(1) : Real(0), mmx = tx + 1 < TX ? Real(1) : Real(0);

    if (tid < 2) sE[4 * TY + tid] = Real(0);
    ptc.build_tables(a, tid, NT, x0, y0, nxA, nyA, tm.nly);
    for (int t = tid; t < tm.zc + 8; t += NT) {
        const int kk = min(max(z0 - 2 + t, 0), mz - 1);
        sZb[t] = __ldg(&a.P.base[2][kk]);
        sZr[t] = __ldg(&a.P.rem[2][kk]);
    }
    if (tid == 0) {
        for (int b = 0; b < DRING + RRING; ++b) mbar_init(&bars[b], 1);
        if (SPLIT) mbar_init(&bars[7], NT);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }

    const int kfirst = z0 - 2, klast = z1 + 1;
    // dT of plane m into dT slot r (read by P of step m); rho-hat of plane m into rho-hat slot r
    // (read by W of step m + 1). One thread; inlined so the tensor maps stay in the kernel's
    // parameter space.
#define HV2_ISSUE_D(m_, r_)                                                               \
    do {                                                                                  \
        if (tid == 0) {                                                                   \
            const int rr_ = (r_);                                                         \
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");                 \
            mbar_expect_tx(&bars[rr_], SLOT_DT * sizeof(Real));                            \
            tma_load_4d(stgD + rr_ * SLOT_DT, &maps.a, x0 - XO, y0 - 2, (m_), 0, &bars[rr_]); \
        }                                                                                 \
    } while (0)
#define HV2_ISSUE_R(m_, r_)                                                               \
    do {                                                                                  \
        if (tid == 0) {                                                                   \
            const int rr_ = (r_);                                                         \
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");                 \
            mbar_expect_tx(&bars[DRING + rr_], SLOT_RH * sizeof(Real));                    \
            tma_load_4d(stgR + rr_ * SLOT_RH, &maps.b, x0 - XO, y0 - 1, (m_), 0, &bars[DRING + rr_]); \
        }                                                                                 \
    } while (0)
    auto zbase = [&](int k) { return sZb[k - kfirst]; };  // k in [kfirst, klast + 3]
    auto zrem = [&](int k) { return sZr[k - kfirst]; };

    // (FAST32: the shuffle scan, whose lane geometry fits its registers)
    const auto plane_geom = ptc.lane_geom(a, x0, nxA, lane);
    auto xstage = [&](Real v0, Real v1, Real v2) {
        if constexpr (sizeof(Real) == 4) ptc.xstage_shfl(row, lane, plane_geom, segw, v0, v1, v2);
        else ptc.xstage(row, lane, v0, v1, v2);
    };
    auto ystage = [&](int nzp) { ptc.ystage(row, lane, part + static_cast<std::size_t>(nzp - nzA) * pstride); };

    pdl_wait();       // p (the CG update before this launch) from here on
    __syncthreads();  // tables, barriers
    // first two nodal planes, synchronously; first two staged planes
    // (the planes steps kfirst .. kfirst+2 read; later steps prefetch one plane each,
    // the host guarantees base_z advances by <= 1 per plane and <= 2 per 3 planes)
    ptc.build_items(tid, NT);
    int slab_hi;
    {
        const int nz0 = zbase(kfirst);
        slab_hi = min(zbase(kfirst + 2) + 1, msz - 1);
        for (int nz = nz0; nz <= slab_hi; ++nz) {
            slab_load(nz);
            slab_store(nz);
        }
    }
    HV2_ISSUE_D(kfirst, 0);
    if (kfirst + 1 <= klast) HV2_ISSUE_D(kfirst + 1, 1);
    for (int m = 0; m < RRING - 1; ++m)
        if (kfirst + m <= klast) HV2_ISSUE_R(kfirst - 1 + m, m);
    int dslot = 0, rslot = 0;        // ring slots of the current step
    unsigned dphase = 0, rphase = 0;  // their mbarrier phase parities
    __syncthreads();

    // ---- loop state (parity-named histories, P = (k - kfirst) & 1)
    int pz = -1000;
    Real Pa0 = 0.0, Pa1 = 0.0, Pa2 = 0.0, Pb0 = 0.0, Pb1 = 0.0, Pb2 = 0.0;  // item 0: P p at nodal planes bz, bz+1
    Real sh0[2] = {0.0, 0.0}, sh1[2] = {0.0, 0.0};   // s history (item 0, item 1)
    Real dq[2][3] = {{0.0, 0.0, 0.0}, {0.0, 0.0, 0.0}};  // dT of planes k-1, k-2 (item 0)
    Real fzp[2] = {0.0, 0.0};                        // rho-hat(+z) w of planes k-2, k-3
    Real gx = 0.0;                                   // in-row x fluxes into the column, plane k-2
    Real sw = 0.0;                                   // sigma w of plane k-2
    Real acc00 = 0.0, acc01 = 0.0, acc02 = 0.0, acc10 = 0.0, acc11 = 0.0, acc12 = 0.0;
    int cur = nzA, ypend = -1;
    const Real scale = a.scale;

#define STEP_END()                                               \
    do {                                                         \
        if constexpr (SPLIT) mbar_arrive_at(barS);               \
        else __syncthreads();                                    \
    } while (0)
    auto step = [&](auto parc, int k) {
        constexpr int P = decltype(parc)::P;
        if constexpr (!SPLIT) {
        // refill the slots step k-1 read (free since the barrier)
        if (k + 2 <= klast) HV2_ISSUE_D(k + 2, dslot == 0 ? DRING - 1 : dslot - 1);
        if (k + RRING - 1 <= klast) HV2_ISSUE_R(k + RRING - 2, rslot == 0 ? RRING - 1 : rslot - 1);
        }
        bool slab_pending = false;
        int slab_nz = 0;
        {
            const int nzq = min(zbase(k + 3) + 1, msz - 1);
            if (SLAB && nzq > slab_hi) {  // uniform
                slab_load(nzq);
                slab_pending = true;
                slab_nz = nzq;
                slab_hi = nzq;
            }
        }
        if constexpr (!SPLIT) {
        if (ypend >= 0) {  // y collapse of the plane completed last step (sA published by the barrier)
            ystage(ypend);
            ypend = -1;
        }
        }
        const int bzk = zbase(k);
        const Real rzk = zrem(k);
        if (bzk != pz) {  // uniform: new nodal plane pair
            Real* q1 = sQ1 + tid;  // item 1: [0..2] plane bz, [3..5] plane bz+1 (own entries only)
            int off0, off1 = 0;
            double rx0d, ry0d, rx1 = 0.0, ry1 = 0.0;
            col_geom(gx0, gy0, off0, rx0d, ry0d);
            if (has1) {
                const int c1 = item1() & 0x3ff;
                col_geom(x0 - XO + c1 % SX, y0 - 2 + c1 / SX, off1, rx1, ry1);
            }
            const Real rxq = static_cast<Real>(rx0d), ry0 = static_cast<Real>(ry0d);
            const Real rx1r = static_cast<Real>(rx1), ry1r = static_cast<Real>(ry1);
            if (bzk == pz + 1) {
                Pa0 = Pb0; Pa1 = Pb1; Pa2 = Pb2;
                if (has1) {
                    q1[0] = q1[3 * NX_P];
                    q1[NX_P] = q1[4 * NX_P];
                    q1[2 * NX_P] = q1[5 * NX_P];
                }
            } else {
                bilerp(bzk, off0, rxq, ry0, Pa0, Pa1, Pa2);
                if (has1) bilerp(bzk, off1, rx1r, ry1r, q1[0], q1[NX_P], q1[2 * NX_P]);
            }
            const int bz1 = min(bzk + 1, msz - 1);
            bilerp(bz1, off0, rxq, ry0, Pb0, Pb1, Pb2);
            if (has1) bilerp(bz1, off1, rx1r, ry1r, q1[3 * NX_P], q1[4 * NX_P], q1[5 * NX_P]);
            pz = bzk;
        }
        mbar_wait_at(barD + 8 * dslot, dphase);
        mbar_wait_at(barR + 8 * rslot, rphase);
        const Real* st = stgD + dslot * SLOT_DT;
        const Real* sr = stgR + rslot * SLOT_RH;
        // ---- P: plane k
        const Real pp0 = lerp(rzk, Pa0, Pb0), pp1 = lerp(rzk, Pa1, Pb1), pp2 = lerp(rzk, Pa2, Pb2);
        auto zl = [&](Real a0, Real b0) { return lerp(rzk, a0, b0); };
        const Real D0 = st[c0], D1 = st[NS + c0], D2 = st[2 * NS + c0];
        const Real s0 = fma(D0, pp0, fma(D1, pp1, D2 * pp2));
        Real s1 = 0.0;
        auto halo_s = [&]() {  // s of the halo item (stored by the caller)
            if (has1) {
                const int c1 = item1() & 0x3ff;
                const Real* q1 = sQ1 + tid;
                s1 = fma(st[c1], zl(q1[0], q1[3 * NX_P]),
                         fma(st[NS + c1], zl(q1[NX_P], q1[4 * NX_P]), st[2 * NS + c1] * zl(q1[2 * NX_P], q1[5 * NX_P])));
            }
        };
        if constexpr (SPLIT) {
        halo_s();
        // the previous step's barrier: everything above only read this step's TMA slots and
        // own registers / sQ1 entries; from here on the shared buffers of the previous step
        if (k != kfirst) mbar_wait_at(barS, (k - kfirst - 1) & 1);
        // refill the slots step k-1 read (free since the barrier)
        if (k + 2 <= klast) HV2_ISSUE_D(k + 2, dslot == 0 ? DRING - 1 : dslot - 1);
        if (k + RRING - 1 <= klast) HV2_ISSUE_R(k + RRING - 2, rslot == 0 ? RRING - 1 : rslot - 1);
        if (ypend >= 0) {  // y collapse of the plane completed last step (sA published by the barrier)
            ystage(ypend);
            ypend = -1;
        }
        }
        sS[P * NS + c0] = s0;
        if (SPLIT && has1) sS[P * NS + (item1() & 0x3ff)] = s1;
        // ---- W: plane j = k-1 (in-plane neighbours' s from the other parity buffer)
        const Real* sn = sS + (1 - P) * NS;
        const Real* rh = sr + w0;  // rho-hat of plane j, [6][NW]
        Real* const Fj = sF + (1 - P) * FPAR;
        Real fzm, fzp_new, sw_new, gx_new;
        {
            const Real sj = sh0[1 - P];
            const Real sg = ((rh[0] + rh[1 * NW]) + (rh[2 * NW] + rh[3 * NW])) + (rh[4 * NW] + rh[5 * NW]);
            Real w;
            if constexpr (C::WF) {
                const Real wa = fma(rh[1 * NW], sn[c0 + 1], rh[0] * sn[c0 - 1]);
                const Real wb = fma(rh[3 * NW], sn[c0 + SX], rh[2 * NW] * sn[c0 - SX]);
                const Real wc = fma(rh[5 * NW], s0, rh[4 * NW] * sh0[P]);
                w = fma(-sg, sj, (wa + wb) + wc);
            } else {
                const Real wa = fma(rh[1 * NW], sn[c0 + 1] - sj, rh[0] * (sn[c0 - 1] - sj));
                const Real wb = fma(rh[3 * NW], sn[c0 + SX] - sj, rh[2 * NW] * (sn[c0 - SX] - sj));
                const Real wc = fma(rh[5 * NW], s0 - sj, rh[4 * NW] * (sh0[P] - sj));
                w = (wa + wb) + wc;
            }
            // x fluxes stay in the warp (one tile row): from lane-1 (+x) and lane+1 (-x)
            const Real fpx = __shfl_up_sync(0xffffffffu, rh[1 * NW] * w, 1);
            const Real fmx = __shfl_down_sync(0xffffffffu, rh[0] * w, 1);
            gx_new = fma(mpx, fpx, mmx * fmx);
            if (C::BF || ty + 1 < TY) Fj[tid + TX] = rh[3 * NW] * w;  // +y flux -> (tx, ty+1)
            if (C::BF || ty > 0) Fj[FM + tid - TX] = rh[2 * NW] * w;  // -y flux -> (tx, ty-1)
            fzm = rh[4 * NW] * w;
            fzp_new = rh[5 * NW] * w;
            sw_new = sg * w;
        }
        // ---- Z: plane i = k-2 (tile columns)
        const int i = k - 2;
        if (i >= ilo && i < ihi) {  // uniform
            const Real* Fi = sF + P * FPAR;
            const Real ex = sE[eoff >= 0 ? P * 2 * TY + eoff : 4 * TY];  // ring-1 x edge flux (or zero)
            const Real z = ((gx + ex) + (Fi[tid] + Fi[FM + tid])) + ((fzm + fzp[P]) - sw);
            const Real sz = scale * z;  // dT (TMA zero fill) makes q vanish outside the volume
            const Real q0 = sz * dq[P][0], q1 = sz * dq[P][1], q2 = sz * dq[P][2];
            const int bz = zbase(i);
            const Real rz = zrem(i);
            if (bz > cur) {  // nodal plane `cur` complete: x collapse now, y collapse after the barrier
                xstage(acc00, acc01, acc02);
                ypend = cur;
                acc00 = acc10;
                acc01 = acc11;
                acc02 = acc12;
                acc10 = acc11 = acc12 = 0.0;
                cur = bz;
            }
            acc00 = fma(Real(1) - rz, q0, acc00);
            acc10 = fma(rz, q0, acc10);
            acc01 = fma(Real(1) - rz, q1, acc01);
            acc11 = fma(rz, q1, acc11);
            acc02 = fma(Real(1) - rz, q2, acc02);
            acc12 = fma(rz, q2, acc12);
        }
        // ---- halo items (after the tile column's P, W and Z: one basic block the compiler can
        // interleave; their s and fluxes are read in the next step)
        if constexpr (!SPLIT) {  // (halo items after the tile column's P, W and Z: one basic block)
            halo_s();
            if (has1) sS[P * NS + (item1() & 0x3ff)] = s1;
        }
        if (w1) {  // ring-1 edge column: only the flux toward the tile
            const int e1 = item1(), c1 = e1 & 0x3ff, f1 = (e1 >> 10) & 0x7ff;
            const Real* rg = sr + c1 - SX;
            const Real sj = sh1[1 - P];
            const Real wa = fma(rg[1 * NW], sn[c1 + 1] - sj, rg[0] * (sn[c1 - 1] - sj));
            const Real wb = fma(rg[3 * NW], sn[c1 + SX] - sj, rg[2 * NW] * (sn[c1 - SX] - sj));
            const Real wc = fma(rg[5 * NW], s1 - sj, rg[4 * NW] * (sh1[P] - sj));
            const Real w = (wa + wb) + wc;
            const Real cf = rg[((e1 >> 21) & 3) * NW];
            if constexpr (C::BF) {
                Real* const dst = (e1 & (1 << 23)) ? sE + (1 - P) * 2 * TY : Fj;
                dst[f1] = cf * w;
            } else {
                if (e1 & (1 << 23)) sE[(1 - P) * 2 * TY + f1] = cf * w;
                else Fj[f1] = cf * w;
            }
        }
        // ---- histories
        dq[P][0] = D0;
        dq[P][1] = D1;
        dq[P][2] = D2;
        sh0[P] = s0;
        sh1[P] = s1;
        fzp[P] = fzp_new;
        sw = sw_new;
        gx = gx_new;
        if (++dslot == DRING) {
            dslot = 0;
            dphase ^= 1u;
        }
        if (++rslot == RRING) {
            rslot = 0;
            rphase ^= 1u;
        }
        if (slab_pending) slab_store(slab_nz);
        STEP_END();
    };
    // pairs of steps without a conditional second step (no register moves on the back edge),
    // then the odd last step
    int k = kfirst;
#pragma unroll 1
    for (; k + 1 <= klast; k += 2) {
        step(Par<0>{}, k);
        step(Par<1>{}, k + 1);
    }
    if (k <= klast) step(Par<0>{}, k);
    pdl_trigger();  // the finalize may be scheduled while the tiles flush
    if constexpr (SPLIT) __syncthreads();  // (the last step only arrived)
    // ---- flush: pending y collapse, then the last two nodal planes
    if (ypend >= 0) ystage(ypend);
    __syncthreads();
    xstage(acc00, acc01, acc02);
    __syncthreads();
    ystage(cur);
    __syncthreads();
    xstage(acc10, acc11, acc12);
    __syncthreads();
    ystage(cur + 1);
#undef HV2_ISSUE_D
#undef HV2_ISSUE_R
}

}  // namespace

namespace {
template <typename Real, int TY_>
std::size_t smem_bytes(int nlx, int nly, int segw, int zc, int nsl) {
    using G = Geo<Real, TY_>;
    using T = Tl<TY_>;
    using C = Cfg<Real>;
    const std::size_t ring = (static_cast<std::size_t>(DRING) * G::SLOT_DT + C::RRING * G::SLOT_RH) * sizeof(Real) + 64;
    const std::size_t dbl = (zc + 8) * sizeof(double);
    constexpr bool SLAB = MFREG_HV2_SLAB || sizeof(Real) == 4;
    const std::size_t real = (static_cast<std::size_t>(SLAB ? NSL * nsl : 0) + 2 * static_cast<std::size_t>(G::NS) + 2 * T::template FPAR<C::BF> + 2 * 2 * T::TY + 2 + 6 * T::NX_P +
                              ptc_reals(T::TY, nlx, nly, segw, C::PAD)) *
                             sizeof(Real);
    return ring + dbl + real + (zc + 8 + ptc_ints(nlx) + T::NX_P) * sizeof(int);
}
}  // namespace

// fp32 = true: the Hv state (dT, rho-hat) and the arithmetic in single precision (FAST32 mode);
// ty = tile height (8: two CTAs per SM, 16: one)
std::size_t hv2_smem_bytes(int nlx, int nly, int segw, int zc, int nsl, bool fp32, int ty) {
    if (ty == 16)
        return fp32 ? smem_bytes<float, 16>(nlx, nly, segw, zc, nsl) : smem_bytes<double, 16>(nlx, nly, segw, zc, nsl);
    return fp32 ? smem_bytes<float, 8>(nlx, nly, segw, zc, nsl) : smem_bytes<double, 8>(nlx, nly, segw, zc, nsl);
}
int hv2_nsl_max(int ty) { return 2 * TX * ty; }  // footprint elements: <= 2 per thread

int hv2_nlx_max() { return 42; }  // x items of a row in <= 4 warp passes
int hv2_threads(int ty) { return TX * ty; }
int hv2_box_origin(bool fp32) { return fp32 ? Geo<float, 8>::XO : Geo<double, 8>::XO; }

void hv2_set_smem_cap(int bytes, int ty) {
    if (ty == 16) {
        MFREG_CUDA(cudaFuncSetAttribute(k_hv2<double, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
        MFREG_CUDA(cudaFuncSetAttribute(k_hv2<float, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
        return;
    }
    MFREG_CUDA(cudaFuncSetAttribute(k_hv2<double, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    MFREG_CUDA(cudaFuncSetAttribute(k_hv2<float, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
}

void hv2_launch(const FArgs& a, const TmaMaps& maps, dim3 grid, std::size_t smem, cudaStream_t s, bool fp32, int ty) {
    if (ty == 16) {
        if (fp32) launch_pdl(k_hv2<float, 16>, grid, dim3(TX * 16), smem, s, a, maps);
        else launch_pdl(k_hv2<double, 16>, grid, dim3(TX * 16), smem, s, a, maps);
        return;
    }
    if (fp32) launch_pdl(k_hv2<float, 8>, grid, dim3(TX * 8), smem, s, a, maps);
    else launch_pdl(k_hv2<double, 8>, grid, dim3(TX * 8), smem, s, a, maps);
}

}  // namespace mfreg_b200
