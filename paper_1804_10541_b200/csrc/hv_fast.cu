// Gauss-Newton Hv image pass, two CTAs per SM (fast mode).
//
// Same algebra as k_fused<false> (fused.cuh): s = dT . P p, w = dr s,
// z = dr^T w, q^ = 2h z dT, P^T into per-tile partials. What differs is the
// execution scheme, built so that two 256-thread CTAs fit one SM (113 KB of
// shared memory and 128 registers per thread each), so one CTA's barrier and
// TMA waits are covered by the other CTA's arithmetic:
//  * one thread per output column of the 32x8 tile; the halo columns are extra
//    work items of threads 0..163 (ring-1 edges: P and W, ring-1 corners and
//    ring-2 edges: P only) instead of dedicated halo warps;
//  * the staging ring holds one TMA slot per step: step k stages dT of plane k
//    (36x12 s region, read by P) and rho-hat of plane k-1 (36x10 w rows, read
//    by W of plane k-1 in the same step), so a slot is consumed in exactly one
//    step and no coefficient is carried in registers (ring of 3: 2 steps ahead);
//  * the dr^T stage reads fluxes instead of (coefficient, w) pairs: W of
//    column t forms rho-hat_t(k) w_t for its in-plane neighbours; x fluxes move
//    inside the warp (a warp is one tile row) by shuffles, y fluxes through two
//    consumer-indexed shared arrays, the z fluxes and sigma_t w_t stay in the
//    column's registers, so z_i is 2-3 shared loads + a few adds;
//  * the halo columns' nodal interpolants live in shared memory (each thread
//    reads back only its own entries), keeping the plane loop within 128
//    registers;
//  * P^T: per-column z weights in registers; on a completed nodal plane each
//    warp (one tile row) collapses x with a segmented shuffle scan over the
//    nodal cells and the y collapse runs one step later, after the regular
//    barrier — no extra barriers in the plane loop (the host guarantees nodal
//    z cells of >= 2 image planes, so completions are >= 2 steps apart).
// Boundary semantics are those of the TMA zero fill: rho-hat and dT vanish
// outside the volume, and the eval pass stores zero coefficients across it.
#include <cstdint>

#include "fused_dev.cuh"

#ifndef MFREG_REVMAP
#define MFREG_REVMAP 1
#endif

namespace mfreg_b200 {

namespace {

using namespace fdev;

constexpr int TX = FT_X, TY = FT_Y;                    // 32 x 8 output tile
constexpr int SY = TY + 4, WY = TY + 2;                // s region rows / rho-hat rows
constexpr int NT = TX * TY;                            // 256 threads
constexpr int RING = 3;                                // staging slots (2 planes ahead)
constexpr int NX_W = 80;                               // extra items [0, 80): ring-1 edges (P + W)
constexpr int NX_P = 164;                              // extra items [80, 164): P only
constexpr int NSL = 4;                                 // nodal plane ring (power of 2)

// Box geometry per state precision: a TMA box must start 16-byte aligned in x, so the
// boxes start XO columns left of the tile (x0 - 2 for fp64, x0 - 4 for fp32) and are
// SX = 32 + 2 XO wide; the s frame is SX x 12, the rho-hat box SX x 10 (one row lower).
template <typename Real>
struct Geo {
    static constexpr int XO = sizeof(Real) == 8 ? 2 : 4;
    static constexpr int SX = TX + 2 * XO, NS = SX * SY, NW = SX * WY;
    static constexpr int SLOT_DT = 3 * NS;              // dT box [3][12][SX]
    static constexpr int SLOT_RH = 6 * NW;              // rho-hat box [6][10][SX]
    static constexpr int SLOT = static_cast<int>(((SLOT_DT + SLOT_RH) * sizeof(Real) + 127) / 128 * 128 / sizeof(Real));
    static_assert((SLOT_DT * sizeof(Real)) % 128 == 0, "rho-hat box must land 128-byte aligned");
};

// extra work item e -> column (lx, ly) in the s frame (tile columns at lx = XO .. XO+31);
// `dir` = consumer flux array of a ring-1 edge item (0: +x, 1: -x, 2: +y, 3: -y)
template <int XO>
__device__ __forceinline__ void extra_item(int e, int& lx, int& ly, int& dir) {
    dir = -1;
    if (e < 32) { lx = XO + e; ly = 1; dir = 2; }                       // ring-1, y = -1 row: feeds +y
    else if (e < 64) { lx = XO + e - 32; ly = SY - 2; dir = 3; }        // ring-1, y = TY row: feeds -y
    else if (e < 72) { lx = XO - 1; ly = 2 + e - 64; dir = 0; }         // ring-1, x = -1: feeds +x
    else if (e < 80) { lx = XO + TX; ly = 2 + e - 72; dir = 1; }        // ring-1, x = TX: feeds -x
    else if (e < 84) {                                                  // ring-1 corners
        const int q = e - 80;
        lx = (q & 1) ? XO + TX : XO - 1;
        ly = (q & 2) ? SY - 2 : 1;
    } else {                                                            // ring-2 edges
        const int r = e - 84;
        if (r < 32) { lx = XO + r; ly = 0; }
        else if (r < 64) { lx = XO + r - 32; ly = SY - 1; }
        else if (r < 72) { lx = XO - 2; ly = 2 + r - 64; }
        else { lx = XO + TX + 1; ly = 2 + r - 72; }
    }
}

template <int P_>
struct Par {
    static constexpr int P = P_;
};

template <typename Real>
__global__ void __launch_bounds__(NT, 2) k_hv2(const __grid_constant__ FArgs a, const __grid_constant__ TmaMaps maps) {
    using G = Geo<Real>;
    constexpr int XO = G::XO, SX = G::SX, NS = G::NS, NW = G::NW, SLOT_DT = G::SLOT_DT, SLOT_RH = G::SLOT_RH,
                  SLOT = G::SLOT;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    if (a.skip && *a.skip) return;  // uniform
    const TileMeta& tm = a.tm;
    const int nlx = tm.nlx;
    const int tid = threadIdx.x, lane = tid & 31, row = tid >> 5;
    const int mx = static_cast<int>(a.g.m[0]), my = static_cast<int>(a.g.m[1]), mz = static_cast<int>(a.g.m[2]);
    const int x0 = blockIdx.x * TX, y0 = blockIdx.y * TY;
    const int z0 = tm.zlo + static_cast<int>(blockIdx.z) * tm.zc, z1 = min(tm.zhi, z0 + tm.zc);
    const int ilo = max(z0, a.olo), ihi = min(z1, a.ohi);
    const int xe = min(mx, x0 + TX), ye = min(my, y0 + TY);
    const int nxA = __ldg(&a.P.base[0][x0]), nyA = __ldg(&a.P.base[1][y0]), nzA = __ldg(&a.P.base[2][z0]);
    const int nlx_t = __ldg(&a.P.base[0][xe - 1]) - nxA + 2;
    const int nly_t = __ldg(&a.P.base[1][ye - 1]) - nyA + 2;
    const long long tile_id = (static_cast<long long>(blockIdx.z) * tm.nty + blockIdx.y) * tm.ntx + blockIdx.x;
    Real* const part = reinterpret_cast<Real*>(a.part) + tile_id * tm.part_stride;
    const std::size_t pstride = static_cast<std::size_t>(tm.nly) * nlx * 3;
    const int msx = static_cast<int>(a.P.src.m[0]), msy = static_cast<int>(a.P.src.m[1]);
    const int msz = static_cast<int>(a.P.src.m[2]);
    const int nxf = a.nxf, nyf = a.nyf, nsl = nxf * nyf * 3, segw = a.segw;

    // ---- shared memory: ring | barriers | nodal ring, row/z tables (fp64) | s planes, fluxes,
    // item-1 interpolants, x-collapsed rows (Real) | int tables
    Real* const stg = reinterpret_cast<Real*>(smem_raw);
    unsigned long long* const bars = reinterpret_cast<unsigned long long*>(stg + RING * SLOT);  // [RING] (32 B)
    Real* const slab = reinterpret_cast<Real*>(bars + 4);  // [NSL][nsl] nodal p (NSL * nsl is a multiple of 4)
    double* const sry = reinterpret_cast<double*>(slab + NSL * nsl);  // [TY]
    double* const sZr = sry + TY;               // [zc + 8] rem_z of the planes kfirst ..
    Real* const sS = reinterpret_cast<Real*>(sZr + tm.zc + 8);  // [2][NS] by plane parity
    Real* const sF = sS + 2 * NS;               // [2][2][NT] consumer-indexed y fluxes by plane parity
    Real* const sE = sF + 2 * 2 * NT;           // [2][2][TY] x fluxes from the ring-1 x edges by plane parity,
                                                // then 2 zero entries (the edge-flux slot of inner lanes)
    Real* const sQ1 = sE + 2 * 2 * TY + 2;      // [6][NX_P] item-1 P p at nodal planes bz, bz+1
    Real* const sQx = sQ1 + 6 * NX_P;           // [3][TY][nlx] (completions >= 2 steps apart)
    int* const sby = reinterpret_cast<int*>(sQx + 3 * TY * nlx);  // [TY]
    int* const sZb = sby + TY;                  // [zc + 8] base_z of the planes kfirst ..
    const unsigned bar0 = smem_u32(bars);

    // ---- per-thread columns: item 0 = tile column (tx, ty) = (lane, row); item 1 = extra halo column
    const int tx = lane, ty = row;
    const int c0 = (tx + XO) + (ty + 2) * SX, w0 = c0 - SX;  // s frame / rho-hat frame (one row lower)
    const int gx0 = x0 + tx, gy0 = y0 + ty;
    const bool has1 = tid < NX_P, w1 = tid < NX_W;  // warp-aligned except warp 2 (split P+W / P) and warp 5
    int lx1 = 0, ly1 = 0, dir1 = -1;
    if (has1) extra_item<XO>(tid, lx1, ly1, dir1);
    const int c1 = lx1 + ly1 * SX, w1i = c1 - SX;
    // where the ring-1 edge flux goes: y edges -> consumer-indexed sF (+y: 0, -y: 1), x edges -> sE
    const bool xedge = dir1 == 0 || dir1 == 1;
    const int f1 = xedge ? dir1 * TY + min(max(ly1 - 2, 0), TY - 1)
                         : (dir1 - 2) * NT + min(max(lx1 - XO, 0), TX - 1) + (dir1 == 2 ? 0 : TY - 1) * TX;

    // nodal slab geometry (P p): x-y footprint of the s region, bilinear weights per column
    const int fx0 = __ldg(&a.P.base[0][max(x0 - 2, 0)]);
    const int fy0 = __ldg(&a.P.base[1][max(y0 - 2, 0)]);
    auto col_geom = [&](int gx, int gy, int& off, double& rx, double& ry) {
        const int gxc = min(max(gx, 0), mx - 1), gyc = min(max(gy, 0), my - 1);
        off = (__ldg(&a.P.base[0][gxc]) - fx0) + (__ldg(&a.P.base[1][gyc]) - fy0) * nxf;
        rx = __ldg(&a.P.rem[0][gxc]);
        ry = __ldg(&a.P.rem[1][gyc]);
    };
    const int gx1 = x0 - XO + lx1, gy1 = y0 - 2 + ly1;
    // edge-flux slot of the tile column (lanes 0 / 31 read a ring-1 x edge, the others a zero
    // slot past both parity halves) and the ring-1 item's coefficient offset toward the tile
    const int eoff = tx == 0 ? ty : (tx == TX - 1 ? TY + ty : -1);
    const int cfo = dir1 == 0 ? 1 * NW : (dir1 == 1 ? 0 : (dir1 == 2 ? 3 * NW : 2 * NW));
    const Real mpx = tx > 0 ? Real(1) : Real(0), mmx = tx + 1 < TX ? Real(1) : Real(0);

    // nodal p elements this thread loads (<= 2 per thread; host guarantees nsl <= 2 * NT)
    const long long ns = a.P.src.count(), sm0 = a.P.src.m[0], sm01 = sm0 * a.P.src.m[1];
    // (offsets within one component plane; component d adds d * ns)
    int slab_off[2], slab_d[2];
    Real slab_v[2] = {Real(0), Real(0)};
#pragma unroll
    for (int u = 0; u < 2; ++u) {
        const int t = (MFREG_REVMAP ? NT - 1 - tid : tid) + u * NT;
        slab_off[u] = -1;
        slab_d[u] = 0;
        if (t < nsl) {
            const int ix = t % nxf, iy = (t / nxf) % nyf;
            slab_d[u] = t / (nxf * nyf);
            slab_off[u] = min(fx0 + ix, msx - 1) + min(fy0 + iy, msy - 1) * static_cast<int>(sm0);
        }
    }
    auto slab_load = [&](int nz) {
#pragma unroll
        for (int u = 0; u < 2; ++u)
            if (slab_off[u] >= 0)
                slab_v[u] = static_cast<Real>(__ldg(a.p + slab_d[u] * ns + static_cast<long long>(nz) * sm01 + slab_off[u]));
    };
    auto slab_store = [&](int nz) {
        Real* dst = slab + (nz & (NSL - 1)) * nsl;
#pragma unroll
        for (int u = 0; u < 2; ++u)
            if (slab_off[u] >= 0) dst[(MFREG_REVMAP ? NT - 1 - tid : tid) + u * NT] = slab_v[u];
    };
    auto bilerp = [&](int nz, int off, Real rx, Real ry, Real& o0, Real& o1, Real& o2) {
        const Real* q = slab + (nz & (NSL - 1)) * nsl + off;
        const int pl = nxf * nyf;
        auto v = [&](int i) { return static_cast<Real>(q[i]); };
        o0 = lerp(ry, lerp(rx, v(0), v(1)), lerp(rx, v(nxf), v(nxf + 1)));
        o1 = lerp(ry, lerp(rx, v(pl), v(pl + 1)), lerp(rx, v(pl + nxf), v(pl + nxf + 1)));
        o2 = lerp(ry, lerp(rx, v(2 * pl), v(2 * pl + 1)), lerp(rx, v(2 * pl + nxf), v(2 * pl + nxf + 1)));
    };

    // x collapse geometry of the tile column: nodal cell, weight, segment of equal cells in the warp
    // (columns past the volume form one-lane segments of their own and write nothing)
    const int gxc0 = min(gx0, mx - 1);
    const bool xin = gx0 < mx, xlast = gx0 == xe - 1;
    const int bxc = __ldg(&a.P.base[0][gxc0]) - nxA;
    const int bx = xin ? bxc : 1024 + lane;
    const Real rxq = __ldg(&a.P.rem[0][gxc0]);
    const int bx_prev = __shfl_up_sync(0xffffffffu, bx, 1);
    const unsigned starts = __ballot_sync(0xffffffffu, lane == 0 || bx_prev != bx);
    const int sst = 31 - __clz(starts & (0xffffffffu >> (31 - lane)));  // first lane of my segment
    const bool send = lane == 31 || ((starts >> (lane + 1)) & 1u);

    if (tid < 2) sE[4 * TY + tid] = Real(0);
    if (tid < TY) {
        const int gyc = min(y0 + tid, my - 1);
        sby[tid] = __ldg(&a.P.base[1][gyc]) - nyA;
        sry[tid] = __ldg(&a.P.rem[1][gyc]);
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
    // step m: dT of plane m, rho-hat of plane m-1 (one thread; inlined so the tensor
    // maps stay in the kernel's parameter space)
#define HV2_ISSUE(m_, r_)                                                               \
    do {                                                                                \
        if (tid == 0) {                                                                 \
            const int rr_ = (r_);                                                       \
            Real* st_ = stg + rr_ * SLOT;                                              \
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");               \
            mbar_expect_tx(&bars[rr_], (SLOT_DT + SLOT_RH) * sizeof(Real));              \
            tma_load_4d(st_, &maps.a, x0 - XO, y0 - 2, (m_), 0, &bars[rr_]);             \
            tma_load_4d(st_ + SLOT_DT, &maps.b, x0 - XO, y0 - 1, (m_) - 1, 0, &bars[rr_]); \
        }                                                                               \
    } while (0)
    auto zbase = [&](int k) { return sZb[k - kfirst]; };  // k in [kfirst, klast + 3]
    auto zrem = [&](int k) { return sZr[k - kfirst]; };

    // x collapse of one completed nodal plane (tile row = warp) into sQx[par]
    auto xcollapse = [&](Real v0, Real v1, Real v2) {
        Real* dst = sQx + row * nlx;
        Real A[3] = {(Real(1) - rxq) * v0, (Real(1) - rxq) * v1, (Real(1) - rxq) * v2};
        Real B[3] = {rxq * v0, rxq * v1, rxq * v2};
        // segmented inclusive scan over the lanes of equal nodal cell (segments <= segw lanes)
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
            if (send && xin) {
                dst[d * TY * nlx + bx] = sst > 0 ? A[d] + bp : A[d];
                if (xlast) dst[d * TY * nlx + bx + 1] = B[d];
            }
        }
    };
    // y collapse of sQx into the tile partial of nodal plane nzp
    const int nyi = 3 * nly_t * nlx_t;
    // the y collapse (and the nodal-plane loads) run on the highest threads: the halo items sit on
    // the lowest ones, so this evens out the warps' work between barriers
    const int rtid = MFREG_REVMAP ? NT - 1 - tid : tid;
    auto ycollapse = [&](int nzp) {
        if (rtid < nyi) {
            const int lxn = rtid % nlx_t, lyn = (rtid / nlx_t) % nly_t, d = rtid / (nlx_t * nly_t);
            const Real* q = sQx + d * TY * nlx + lxn;
            Real v = 0.0;
#pragma unroll
            for (int r = 0; r < TY; ++r) {
                const int b = sby[r];
                const Real ry = sry[r];
                const Real wgt = b == lyn ? Real(1) - ry : (b == lyn - 1 ? ry : Real(0));
                v = fma(wgt, q[r * nlx], v);
            }
            part[static_cast<std::size_t>(nzp - nzA) * pstride + (lyn * nlx + lxn) * 3 + d] = v;
        }
    };

    pdl_wait();       // p (the CG update before this launch) from here on
    __syncthreads();  // tables, barriers
    // first two nodal planes, synchronously; first two staged planes
    // (the planes steps kfirst .. kfirst+2 read; later steps prefetch one plane each,
    // the host guarantees base_z advances by <= 1 per plane and <= 2 per 3 planes)
    int slab_hi;
    {
        const int nz0 = zbase(kfirst);
        slab_hi = min(zbase(kfirst + 2) + 1, msz - 1);
        for (int nz = nz0; nz <= slab_hi; ++nz) {
            slab_load(nz);
            slab_store(nz);
        }
    }
    HV2_ISSUE(kfirst, 0);
    if (kfirst + 1 <= klast) HV2_ISSUE(kfirst + 1, 1);
    int slot = 0;         // ring slot of the current step
    unsigned phase = 0;   // its mbarrier phase parity
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

    auto step = [&](auto parc, int k) {
        constexpr int P = decltype(parc)::P;
        if (k + 2 <= klast) HV2_ISSUE(k + 2, slot == 0 ? 2 : slot - 1);
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
        const Real rzk = zrem(k);
        if (bzk != pz) {  // uniform: new nodal plane pair
            Real* q1 = sQ1 + tid;  // item 1: [0..2] plane bz, [3..5] plane bz+1 (own entries only)
            // item 0 geometry from the x-collapse registers and the row tables; item 1 from global
            const int off0 = (bxc + nxA - fx0) + (sby[row] + nyA - fy0) * nxf;
            const Real ry0 = sry[row];
            int off1 = 0;
            double rx1 = 0.0, ry1 = 0.0;
            if (has1) col_geom(gx1, gy1, off1, rx1, ry1);
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
        mbar_wait_at(bar0 + 8 * slot, phase);
        const Real* st = stg + slot * SLOT;
        // ---- P: plane k
        const Real pp0 = lerp(rzk, Pa0, Pb0), pp1 = lerp(rzk, Pa1, Pb1), pp2 = lerp(rzk, Pa2, Pb2);
        const Real D0 = st[c0], D1 = st[NS + c0], D2 = st[2 * NS + c0];
        const Real s0 = fma(D0, pp0, fma(D1, pp1, D2 * pp2));
        sS[P * NS + c0] = s0;
        Real s1 = 0.0;
        if (has1) {
            const Real* q1 = sQ1 + tid;
            s1 = fma(st[c1], lerp(rzk, q1[0], q1[3 * NX_P]),
                     fma(st[NS + c1], lerp(rzk, q1[NX_P], q1[4 * NX_P]), st[2 * NS + c1] * lerp(rzk, q1[2 * NX_P], q1[5 * NX_P])));
            sS[P * NS + c1] = s1;
        }
        // ---- W: plane j = k-1 (in-plane neighbours' s from the other parity buffer)
        const Real* sn = sS + (1 - P) * NS;
        const Real* rh = st + SLOT_DT + w0;  // rho-hat of plane j, [6][NW]
        Real* const Fj = sF + (1 - P) * 2 * NT;
        Real fzm, fzp_new, sw_new, gx_new;
        {
            const Real sj = sh0[1 - P];
            const Real wa = fma(rh[1 * NW], sn[c0 + 1] - sj, rh[0] * (sn[c0 - 1] - sj));
            const Real wb = fma(rh[3 * NW], sn[c0 + SX] - sj, rh[2 * NW] * (sn[c0 - SX] - sj));
            const Real wc = fma(rh[5 * NW], s0 - sj, rh[4 * NW] * (sh0[P] - sj));
            const Real w = (wa + wb) + wc;
            const Real sg = ((rh[0] + rh[1 * NW]) + (rh[2 * NW] + rh[3 * NW])) + (rh[4 * NW] + rh[5 * NW]);
            // x fluxes stay in the warp (one tile row): from lane-1 (+x) and lane+1 (-x)
            const Real fpx = __shfl_up_sync(0xffffffffu, rh[1 * NW] * w, 1);
            const Real fmx = __shfl_down_sync(0xffffffffu, rh[0] * w, 1);
            gx_new = fma(mpx, fpx, mmx * fmx);
            if (ty + 1 < TY) Fj[tid + TX] = rh[3 * NW] * w;       // +y flux -> (tx, ty+1)
            if (ty > 0) Fj[NT + tid - TX] = rh[2 * NW] * w;       // -y flux -> (tx, ty-1)
            fzm = rh[4 * NW] * w;
            fzp_new = rh[5 * NW] * w;
            sw_new = sg * w;
        }
        if (w1) {  // ring-1 edge column: only the flux toward the tile
            const Real* rg = st + SLOT_DT + w1i;
            const Real sj = sh1[1 - P];
            const Real wa = fma(rg[1 * NW], sn[c1 + 1] - sj, rg[0] * (sn[c1 - 1] - sj));
            const Real wb = fma(rg[3 * NW], sn[c1 + SX] - sj, rg[2 * NW] * (sn[c1 - SX] - sj));
            const Real wc = fma(rg[5 * NW], s1 - sj, rg[4 * NW] * (sh1[P] - sj));
            const Real w = (wa + wb) + wc;
            const Real cf = rg[cfo];
            if (xedge) sE[(1 - P) * 2 * TY + f1] = cf * w;
            else Fj[f1] = cf * w;
        }
        // ---- Z: plane i = k-2 (tile columns)
        const int i = k - 2;
        if (i >= ilo && i < ihi) {  // uniform
            const Real* Fi = sF + P * 2 * NT;
            const Real ex = sE[eoff >= 0 ? P * 2 * TY + eoff : 4 * TY];  // ring-1 x edge flux (or zero)
            const Real z = ((gx + ex) + (Fi[tid] + Fi[NT + tid])) + ((fzm + fzp[P]) - sw);
            const Real sz = scale * z;  // dT (TMA zero fill) makes q vanish outside the volume
            const Real q0 = sz * dq[P][0], q1 = sz * dq[P][1], q2 = sz * dq[P][2];
            const int bz = zbase(i);
            const Real rz = zrem(i);
            if (bz > cur) {  // nodal plane `cur` complete: x collapse now, y collapse after the barrier
                xcollapse(acc00, acc01, acc02);
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
        // ---- histories
        dq[P][0] = D0;
        dq[P][1] = D1;
        dq[P][2] = D2;
        sh0[P] = s0;
        sh1[P] = s1;
        fzp[P] = fzp_new;
        sw = sw_new;
        gx = gx_new;
        if (++slot == RING) {
            slot = 0;
            phase ^= 1u;
        }
        if (slab_pending) slab_store(slab_nz);
        __syncthreads();
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
    xcollapse(acc00, acc01, acc02);
    __syncthreads();
    ycollapse(cur);
    __syncthreads();
    xcollapse(acc10, acc11, acc12);
    __syncthreads();
    ycollapse(cur + 1);
#undef HV2_ISSUE
}

}  // namespace

namespace {
template <typename Real>
std::size_t smem_bytes(int nlx, int nsl, int zc) {
    using G = Geo<Real>;
    const std::size_t ring = static_cast<std::size_t>(RING) * G::SLOT * sizeof(Real) + 32;
    const std::size_t dbl = static_cast<std::size_t>(NSL) * nsl * sizeof(Real) + (TY + zc + 8) * sizeof(double);
    const std::size_t real = (2 * static_cast<std::size_t>(G::NS) + 2 * 2 * NT + 2 * 2 * TY + 2 + 6 * NX_P +
                              3 * static_cast<std::size_t>(TY) * nlx) * sizeof(Real);
    return ring + dbl + real + (TY + zc + 8) * sizeof(int);
}
}  // namespace

// fp32 = true: the Hv state (dT, rho-hat) and the arithmetic in single precision (FAST32 mode)
std::size_t hv2_smem_bytes(int nlx, int nsl, int zc, bool fp32) {
    return fp32 ? smem_bytes<float>(nlx, nsl, zc) : smem_bytes<double>(nlx, nsl, zc);
}

int hv2_nsl_max() { return 2 * NT; }
int hv2_ring_planes() { return NSL; }
int hv2_threads() { return NT; }
int hv2_box_origin(bool fp32) { return fp32 ? Geo<float>::XO : Geo<double>::XO; }

void hv2_set_smem_cap(int bytes) {
    MFREG_CUDA(cudaFuncSetAttribute(k_hv2<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    MFREG_CUDA(cudaFuncSetAttribute(k_hv2<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
}

void hv2_launch(const FArgs& a, const TmaMaps& maps, dim3 grid, std::size_t smem, cudaStream_t s, bool fp32) {
    if (fp32) launch_pdl(k_hv2<float>, grid, dim3(NT), smem, s, a, maps);
    else launch_pdl(k_hv2<double>, grid, dim3(NT), smem, s, a, maps);
}

}  // namespace mfreg_b200
