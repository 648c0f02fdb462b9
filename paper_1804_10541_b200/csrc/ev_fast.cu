// NGF eval image pass, two CTAs per SM (fast mode).
//
// Same algebra and outputs as k_fused<true> (fused.cu): per voxel the six
// coefficients rho-hat (ngf.cpp:39-64, stored as the Hv state), the residual
// r = num inv1 (ngf.cpp:204-211), the per-tile sums of (1 - r^2) (ngf_value,
// ngf.cpp:225-231) and, when `grad`, the NGF gradient -2h dT (dr^T r)
// (ngf.cpp:66-103) spread by P^T into per-tile partials. Execution mirrors
// k_hv2 (hv_fast.cu):
//  * one thread per tile column (32x8 tile) plus the 80 ring-1 edge columns as
//    second items of threads 0..79 (their coefficients only feed the fluxes
//    toward the tile);
//  * the staging ring (5 slots, 3 steps ahead) holds per step k the R and T_w
//    boxes of plane k (36x12) and the tile's dT of plane k-2 (32x8x3): stage A
//    of plane j = k-1 reads its in-plane neighbours from the previous step's
//    slot, its z neighbours from this slot and a register, and the dr^T stage
//    of plane i = k-2 reads dT from this slot;
//  * dr^T r: x fluxes by warp shuffles, y fluxes through consumer-indexed
//    shared arrays, z fluxes and sigma r in registers;
//  * P^T: z weights in registers, segmented-scan x collapse per warp, y
//    collapse one step later (no extra barriers in the plane loop).
// Boundary handling as the reference's clamped neighbours: differences across
// the volume boundary are masked to zero, coefficients outside are zero.
#include <cstdint>

#include "ptc.cuh"

#ifndef MFREG_EV2_EXP
#define MFREG_EV2_EXP 0  // timing experiment only (wrong Hv state): 1 = no rho-hat stores
#endif
#ifndef MFREG_REVMAP
#define MFREG_REVMAP 1
#endif

namespace mfreg_b200 {

namespace {

using namespace fdev;

constexpr int TX = FT_X, TY = FT_Y;                    // 32 x 8 output tile
constexpr int SY = TY + 4;                             // R / T_w box rows
constexpr int NT = TX * TY;                            // 256 threads
constexpr int RING = 5;                                // staging slots (3 steps ahead)
constexpr int NX_A = 80;                               // extra items: ring-1 edge columns

// Box geometry per state precision (TMA boxes start 16-byte aligned in x: x0 - XO)
template <typename Real>
struct Geo {
    static constexpr int XO = sizeof(Real) == 8 ? 2 : 4;
    static constexpr int SX = TX + 2 * XO, NS = SX * SY;
    static constexpr int SLOT_R = 0, SLOT_T = NS, SLOT_D = 2 * NS;  // R, T_w [12][SX], dT [3][8][32]
    static constexpr int SLOT = 2 * NS + 3 * NT;
    static_assert((SLOT * sizeof(Real)) % 128 == 0 && (SLOT_T * sizeof(Real)) % 128 == 0 &&
                      (SLOT_D * sizeof(Real)) % 128 == 0, "TMA alignment");
};

// extra item e in [0, 80) -> ring-1 edge column (lx, ly) in the box frame (tile columns at
// lx = XO .. XO+31) and the consumer flux array (0: +x, 1: -x, 2: +y, 3: -y)
template <int XO>
__device__ __forceinline__ void edge_item(int e, int& lx, int& ly, int& dir) {
    if (e < 32) { lx = XO + e; ly = 1; dir = 2; }
    else if (e < 64) { lx = XO + e - 32; ly = SY - 2; dir = 3; }
    else if (e < 72) { lx = XO - 1; ly = 2 + e - 64; dir = 0; }
    else { lx = XO + TX; ly = 2 + e - 72; dir = 1; }
}

template <int P_>
struct Par {
    static constexpr int P = P_;
};

__device__ __forceinline__ double rsq(double v) { return rsqrt(v); }
__device__ __forceinline__ float rsq(float v) { return rsqrtf(v); }

// NGF coefficients of one column at plane j from the six clamped differences
template <typename Real>
struct Coef {
    Real e[6];  // rho-hat: -x, +x, -y, +y, -z, +z
    Real r;     // residual
};

// the normalisation of one column: inv1, inv2 (ngf.cpp:204-209) and the residual
template <typename Real>
struct Norm {
    Real in1, in2, r;
};
template <typename Real>
__device__ __forceinline__ Norm<Real> ngf_norm(const FArgs& a, Real dR0, Real dR1, Real dR2, Real dR3, Real dR4,
                                               Real dR5, Real dT0, Real dT1, Real dT2, Real dT3, Real dT4, Real dT5) {
    const Real i0 = static_cast<Real>(a.ih2[0]), i1 = static_cast<Real>(a.ih2[1]), i2 = static_cast<Real>(a.ih2[2]);
    const Real stt = fma(fma(dT0, dT0, dT1 * dT1), i0, fma(fma(dT2, dT2, dT3 * dT3), i1, fma(dT4, dT4, dT5 * dT5) * i2));
    const Real srr = fma(fma(dR0, dR0, dR1 * dR1), i0, fma(fma(dR2, dR2, dR3 * dR3), i1, fma(dR4, dR4, dR5 * dR5) * i2));
    const Real num = fma(Real(0.5), fma(fma(dT0, dR0, dT1 * dR1), i0, fma(fma(dT2, dR2, dT3 * dR3), i1, fma(dT4, dR4, dT5 * dR5) * i2)),
                         static_cast<Real>(a.tau * a.rho));
    const Real nt2 = fma(Real(0.5), stt, static_cast<Real>(a.tau * a.tau));
    const Real nr2 = fma(Real(0.5), srr, static_cast<Real>(a.rho * a.rho));
    Norm<Real> o;
    o.in1 = rsq(nt2 * nr2);
    o.in2 = num * ((o.in1 * o.in1) * (o.in1 * nr2));
    o.r = num * o.in1;
    return o;
}

template <typename Real>
__device__ __forceinline__ Coef<Real> ngf_coef(const FArgs& a, Real dR0, Real dR1, Real dR2, Real dR3, Real dR4,
                                               Real dR5, Real dT0, Real dT1, Real dT2, Real dT3, Real dT4, Real dT5,
                                               bool ok) {
    const Real i0 = static_cast<Real>(a.ih2[0]), i1 = static_cast<Real>(a.ih2[1]), i2 = static_cast<Real>(a.ih2[2]);
    const Real stt = fma(fma(dT0, dT0, dT1 * dT1), i0, fma(fma(dT2, dT2, dT3 * dT3), i1, fma(dT4, dT4, dT5 * dT5) * i2));
    const Real srr = fma(fma(dR0, dR0, dR1 * dR1), i0, fma(fma(dR2, dR2, dR3 * dR3), i1, fma(dR4, dR4, dR5 * dR5) * i2));
    const Real num = fma(Real(0.5), fma(fma(dT0, dR0, dT1 * dR1), i0, fma(fma(dT2, dR2, dT3 * dR3), i1, fma(dT4, dR4, dT5 * dR5) * i2)),
                         static_cast<Real>(a.tau * a.rho));
    // one reciprocal square root: in1 = 1/(|T| |R|) = rsqrt(|T|^2 |R|^2) and
    // in2 = num / (|T|^3 |R|) = num in1^3 |R|^2
    const Real nt2 = fma(Real(0.5), stt, static_cast<Real>(a.tau * a.tau));
    const Real nr2 = fma(Real(0.5), srr, static_cast<Real>(a.rho * a.rho));
    const Real in1 = rsq(nt2 * nr2);
    const Real in2 = num * ((in1 * in1) * (in1 * nr2));
    const Real hx = static_cast<Real>(a.hh[0]), hy = static_cast<Real>(a.hh[1]), hz = static_cast<Real>(a.hh[2]);
    Coef<Real> c;
    c.e[0] = ok ? hx * fma(dR0, in1, -dT0 * in2) : Real(0);
    c.e[1] = ok ? hx * fma(dR1, in1, -dT1 * in2) : Real(0);
    c.e[2] = ok ? hy * fma(dR2, in1, -dT2 * in2) : Real(0);
    c.e[3] = ok ? hy * fma(dR3, in1, -dT3 * in2) : Real(0);
    c.e[4] = ok ? hz * fma(dR4, in1, -dT4 * in2) : Real(0);
    c.e[5] = ok ? hz * fma(dR5, in1, -dT5 * in2) : Real(0);
    c.r = ok ? num * in1 : Real(0);
    return c;
}

template <typename Real>
__global__ void __launch_bounds__(NT, sizeof(Real) == 4 ? 3 : 2) k_ev2(const __grid_constant__ FArgs a, const __grid_constant__ TmaMaps maps) {
    using G = Geo<Real>;
    constexpr int XO = G::XO, SX = G::SX, NS = G::NS, SLOT_R = G::SLOT_R, SLOT_T = G::SLOT_T, SLOT_D = G::SLOT_D,
                  SLOT = G::SLOT;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const TileMeta& tm = a.tm;
    const int nlx = tm.nlx;
    const int tid = threadIdx.x, lane = tid & 31, row = tid >> 5;
    const int mx = static_cast<int>(a.g.m[0]), my = static_cast<int>(a.g.m[1]), mz = static_cast<int>(a.g.m[2]);
    const long long n = a.g.count(), plane = static_cast<long long>(mx) * my;
    const int x0 = blockIdx.x * TX, y0 = blockIdx.y * TY;
    const int bzc = static_cast<int>(blockIdx.z) + a.zch0;  // z tile chunk (z-group launches)
    const int z0 = tm.zlo + bzc * tm.zc, z1 = min(tm.zhi, z0 + tm.zc);
    const int ilo = max(z0, a.olo), ihi = min(z1, a.ohi);
    const int xe = min(mx, x0 + TX), ye = min(my, y0 + TY);
    const int nxA = __ldg(&a.P.base[0][x0]), nyA = __ldg(&a.P.base[1][y0]), nzA = __ldg(&a.P.base[2][z0]);
    const int nlx_t = __ldg(&a.P.base[0][xe - 1]) - nxA + 2;
    const int nly_t = __ldg(&a.P.base[1][ye - 1]) - nyA + 2;
    const long long tile_id = (static_cast<long long>(bzc) * tm.nty + blockIdx.y) * tm.ntx + blockIdx.x;
    Real* const part = reinterpret_cast<Real*>(a.part) + tile_id * tm.part_stride;
    Real* const frh_out = reinterpret_cast<Real*>(a.frh_out);
    const std::size_t pstride = static_cast<std::size_t>(tm.nly) * nlx * 3;
    const int segw = a.segw;
    const bool grad = a.grad != 0;

    // ---- shared memory: ring | barriers | reduction (fp64) | fluxes, P^T buffers (Real) | ints
    Real* const stg = reinterpret_cast<Real*>(smem_raw);
    Real* const sOut = stg + RING * SLOT;       // [2][6][TY][TX] rho-hat of the tile plane (TMA store)
    unsigned long long* const bars = reinterpret_cast<unsigned long long*>(sOut + 2 * 6 * NT);  // [RING] (48 B)
    double* const sred = reinterpret_cast<double*>(bars + 6);  // [NT / 32]
    Real* const sF = reinterpret_cast<Real*>(sred + NT / 32);  // [2][2][NT] consumer-indexed y fluxes
    Real* const sE = sF + 2 * 2 * NT;           // [2][2][TY] x fluxes from the ring-1 x edges by plane parity
    Real* const sPt = sE + 2 * 2 * TY;          // P^T collapse buffers and tables (ptc.cuh)
    // (conflict-free padded P^T rows for fp64; FAST32 measured faster without them)
    constexpr bool PAD = MFREG_PTC_PAD && sizeof(Real) == 8;
    int* const sI1 = reinterpret_cast<int*>(sPt + ptc_reals(TY, nlx, tm.nly, segw, PAD));  // [NX_A] packed item 1
    Ptc<Real, TY, PAD> ptc(sPt, sI1 + NX_A, nlx, tm.nly, segw, nlx_t, nly_t);
    const unsigned bar0 = smem_u32(bars);

    // ---- columns: item 0 = tile column (lane, row); item 1 (threads < 80) = ring-1 edge column
    const int tx = lane, ty = row;
    const int c0 = (tx + XO) + (ty + 2) * SX;
    const int gx0 = x0 + tx, gy0 = y0 + ty;
    const bool w1 = tid < NX_A;
    // item-1 geometry packed once into shared memory and re-read per step (cheaper than keeping it
    // live across the plane loop): bits 0-9 the box index c1, 10-19 the flux slot f1, 20-21 the
    // direction toward the tile, 22 x edge, 23-26 the in-volume neighbour masks (-x, +x, -y, +y),
    // 27 the column inside the volume
    if (w1) {
        int lx1 = XO, ly1 = 2, dir1 = 0;
        edge_item<XO>(tid, lx1, ly1, dir1);
        const int gx1 = x0 - XO + lx1, gy1 = y0 - 2 + ly1;
        const bool xedge = dir1 == 0 || dir1 == 1;
        const int f1 = xedge ? dir1 * TY + min(max(ly1 - 2, 0), TY - 1)
                             : (dir1 - 2) * NT + min(max(lx1 - XO, 0), TX - 1) + (dir1 == 2 ? 0 : TY - 1) * TX;
        static_assert(NS <= 1024 && 2 * NT <= 1024, "item-1 packing");
        sI1[tid] = (lx1 + ly1 * SX) | (f1 << 10) | (dir1 << 20) | (xedge ? 1 << 22 : 0) | (gx1 > 0 ? 1 << 23 : 0) |
                   (gx1 + 1 < mx ? 1 << 24 : 0) | (gy1 > 0 ? 1 << 25 : 0) | (gy1 + 1 < my ? 1 << 26 : 0) |
                   (gx1 >= 0 && gx1 < mx && gy1 >= 0 && gy1 < my ? 1 << 27 : 0);
    }
    // in-plane neighbours of the tile column, clamped at the volume boundary like the reference's
    // neighbours (the difference with itself is an exact zero: no mask multiplies), and its
    // "inside the volume" flag
    const int cxm0 = c0 - (gx0 > 0 ? 1 : 0), cxp0 = c0 + (gx0 + 1 < mx ? 1 : 0);
    const int cym0 = c0 - (gy0 > 0 ? SX : 0), cyp0 = c0 + (gy0 + 1 < my ? SX : 0);
    const bool in0 = gx0 < mx && gy0 < my;
    const long long col0 = in0 ? static_cast<long long>(gx0) + static_cast<long long>(gy0) * mx : 0;

    ptc.build_tables(a, tid, NT, x0, y0, nxA, nyA, tm.nly);
    if (tid == 0) {
        for (int b = 0; b < RING; ++b) mbar_init(&bars[b], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }

    const int kfirst = z0 - 2, klast = z1 + 1;
    // step m: R, T_w of plane m, the tile's dT of plane m-2 (one thread)
#define EV2_ISSUE(m_, r_)                                                          \
    do {                                                                           \
        if (tid == 0) {                                                            \
            const int rr_ = (r_);                                                  \
            Real* st_ = stg + rr_ * SLOT;                                         \
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");          \
            mbar_expect_tx(&bars[rr_], SLOT * sizeof(Real));                       \
            tma_load_3d(st_ + SLOT_R, &maps.a, x0 - XO, y0 - 2, (m_), &bars[rr_]);  \
            tma_load_3d(st_ + SLOT_T, &maps.b, x0 - XO, y0 - 2, (m_), &bars[rr_]);  \
            tma_load_4d(st_ + SLOT_D, &maps.c, x0, y0, (m_) - 2, 0, &bars[rr_]);    \
        }                                                                          \
    } while (0)

    auto xcollapse = [&](Real v0, Real v1, Real v2) { ptc.xstage(row, lane, v0, v1, v2); };
    auto ycollapse = [&](int nzp) { ptc.ystage(row, lane, part + static_cast<std::size_t>(nzp - nzA) * pstride); };
    auto zbase = [&](int k) { return __ldg(&a.P.base[2][min(max(k, 0), mz - 1)]); };
    auto zrem = [&](int k) { return __ldg(&a.P.rem[2][min(max(k, 0), mz - 1)]); };

    pdl_wait();       // T_w, dT (the warp kernel before this launch) from here on
    __syncthreads();  // tables, barriers
    ptc.build_items(tid, NT);
    for (int m = 0; m < RING - 2; ++m)
        if (kfirst + m <= klast) EV2_ISSUE(kfirst + m, m);
    int slot = 0, slot_prev = RING - 1;  // ring slots of this step and the previous one
    unsigned phase = 0;

    // ---- loop state (P = (k - kfirst) & 1)
    Real Rm0 = 0.0, Tm0 = 0.0, Rm1 = 0.0, Tm1 = 0.0;  // own R, T_w at plane k-2 (items 0, 1)
    Real fzp[2] = {0.0, 0.0};                        // rho-hat(+z) r of planes k-2, k-3
    Real sw = 0.0;                                   // sigma r of plane k-2
    Real gx = 0.0;                                   // in-row x fluxes into the column, plane k-2
    double dsum = 0.0;
    Real acc00 = 0.0, acc01 = 0.0, acc02 = 0.0, acc10 = 0.0, acc11 = 0.0, acc12 = 0.0;
    int cur = nzA, ypend = -1;
    const Real scale = a.scale;

    auto step = [&](auto parc, int k) {
        constexpr int P = decltype(parc)::P;
        if (k + RING - 2 <= klast) EV2_ISSUE(k + RING - 2, slot >= 2 ? slot - 2 : slot + RING - 2);
        if (ypend >= 0) {  // y collapse of the plane completed last step
            ycollapse(ypend);
            ypend = -1;
        }
        // rho-hat of plane k-2 (staged last step, published by the barrier) -> global by TMA
        if (a.frh_tma && tid == 0 && k - 2 >= z0 && k - 2 < z1)
            tma_store_4d(&maps.d, sOut + (1 - P) * 6 * NT, x0, y0, k - 2, 0);
        mbar_wait_at(bar0 + 8 * slot, phase);
        const Real* st = stg + slot * SLOT;       // plane k (R, T_w), dT of plane k-2
        const Real* sp = stg + slot_prev * SLOT;  // plane k-1 (R, T_w)
        // ---- A: plane j = k-1
        const int j = k - 1;
        const Real mzm = j > 0 ? Real(1) : Real(0), mzp = j + 1 < mz ? Real(1) : Real(0);
        const bool jin = j >= 0 && j < mz;
        Real fzm, fzp_new, sw_new, gx_new;
        {
            const Real Rj = sp[SLOT_R + c0], Tj = sp[SLOT_T + c0];
            const Real Rp = st[SLOT_R + c0], Tp = st[SLOT_T + c0];
            const Coef cf = ngf_coef(a, sp[SLOT_R + cxm0] - Rj, sp[SLOT_R + cxp0] - Rj, sp[SLOT_R + cym0] - Rj,
                                     sp[SLOT_R + cyp0] - Rj, mzm * (Rm0 - Rj), mzp * (Rp - Rj), sp[SLOT_T + cxm0] - Tj,
                                     sp[SLOT_T + cxp0] - Tj, sp[SLOT_T + cym0] - Tj, sp[SLOT_T + cyp0] - Tj,
                                     mzm * (Tm0 - Tj), mzp * (Tp - Tj), in0 && jin);
            Rm0 = Rj;
            Tm0 = Tj;
            if (j >= z0 && j < z1) {  // Hv state of the tile plane (none when value-only lazy)
                if (a.frh_tma) {  // staged for the TMA store next step (it clips columns past the volume)
                    Real* o = sOut + P * 6 * NT + tid;
#pragma unroll
                    for (int d = 0; d < 6; ++d) o[d * NT] = cf.e[d];
                    tma_store_fence();
                } else if (frh_out && in0) {
                    const long long gi = col0 + static_cast<long long>(j) * plane;
#pragma unroll
                    for (int d = 0; d < 6; ++d) frh_out[d * n + gi] = cf.e[d];
                }
                if (in0 && j >= ilo && j < ihi) dsum += fma(-static_cast<double>(cf.r), static_cast<double>(cf.r), 1.0);
            }
            const Real r = cf.r;
            const Real fpx = __shfl_up_sync(0xffffffffu, cf.e[1] * r, 1);
            const Real fmx = __shfl_down_sync(0xffffffffu, cf.e[0] * r, 1);
            gx_new = (tx > 0 ? fpx : Real(0)) + (tx + 1 < TX ? fmx : Real(0));
            Real* const Fj = sF + (1 - P) * 2 * NT;
            if (ty + 1 < TY) Fj[tid + TX] = cf.e[3] * r;  // +y flux -> (tx, ty+1)
            if (ty > 0) Fj[NT + tid - TX] = cf.e[2] * r;  // -y flux -> (tx, ty-1)
            fzm = cf.e[4] * r;
            fzp_new = cf.e[5] * r;
            sw_new = (((cf.e[0] + cf.e[1]) + (cf.e[2] + cf.e[3])) + (cf.e[4] + cf.e[5])) * r;
        }
        if (w1) {  // ring-1 edge column: the flux toward the tile
            const int e1 = lds_v(sI1 + tid), c1 = e1 & 0x3ff, f1 = (e1 >> 10) & 0x3ff, dir1 = (e1 >> 20) & 3;
            // clamped in-plane neighbours (exact-zero differences at the volume boundary)
            const int cxm = c1 - ((e1 >> 23) & 1), cxp = c1 + ((e1 >> 24) & 1);
            const int cym = c1 - ((e1 >> 25) & 1) * SX, cyp = c1 + ((e1 >> 26) & 1) * SX;
            const bool in1c = (e1 >> 27) & 1;
            const Real Rj = sp[SLOT_R + c1], Tj = sp[SLOT_T + c1];
            const Real Rp = st[SLOT_R + c1], Tp = st[SLOT_T + c1];
            const Real dR0 = sp[SLOT_R + cxm] - Rj, dR1 = sp[SLOT_R + cxp] - Rj, dR2 = sp[SLOT_R + cym] - Rj,
                       dR3 = sp[SLOT_R + cyp] - Rj;
            const Real dT0 = sp[SLOT_T + cxm] - Tj, dT1 = sp[SLOT_T + cxp] - Tj, dT2 = sp[SLOT_T + cym] - Tj,
                       dT3 = sp[SLOT_T + cyp] - Tj;
            const Norm<Real> nm = ngf_norm(a, dR0, dR1, dR2, dR3, mzm * (Rm1 - Rj), mzp * (Rp - Rj), dT0, dT1, dT2, dT3,
                                           mzm * (Tm1 - Tj), mzp * (Tp - Tj));
            Rm1 = Rj;
            Tm1 = Tj;
            // only the coefficient toward the tile: the +x flux comes from e[1] (x = -1 column), -x
            // from e[0], +y from e[3], -y from e[2]
            const Real dRs = dir1 == 0 ? dR1 : (dir1 == 1 ? dR0 : (dir1 == 2 ? dR3 : dR2));
            const Real dTs = dir1 == 0 ? dT1 : (dir1 == 1 ? dT0 : (dir1 == 2 ? dT3 : dT2));
            const Real hs = static_cast<Real>(dir1 < 2 ? a.hh[0] : a.hh[1]);
            const bool ok = in1c && jin;
            const Real e = ok ? hs * fma(dRs, nm.in1, -dTs * nm.in2) : Real(0), r1 = ok ? nm.r : Real(0);
            if ((e1 >> 22) & 1) sE[(1 - P) * 2 * TY + f1] = e * r1;
            else sF[(1 - P) * 2 * NT + f1] = e * r1;
        }
        // ---- Z: plane i = k-2 (tile columns): gradient -2h dT (dr^T r) -> P^T
        const int i = k - 2;
        if (grad && i >= ilo && i < ihi) {  // uniform
            const Real* Fi = sF + P * 2 * NT;
            const Real* Ei = sE + P * 2 * TY + ty;
            const Real ex = tx == 0 ? Ei[0] : (tx == TX - 1 ? Ei[TY] : Real(0));
            const Real z = ((gx + ex) + (Fi[tid] + Fi[NT + tid])) + ((fzm + fzp[P]) - sw);
            const Real sz = scale * z;  // dT vanishes outside the volume (TMA zero fill)
            const Real* dq = st + SLOT_D + tid;
            const Real q0 = sz * dq[0], q1 = sz * dq[NT], q2 = sz * dq[2 * NT];
            const int bz = zbase(i);
            const Real rz = zrem(i);
            if (bz > cur) {
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
        fzp[P] = fzp_new;
        sw = sw_new;
        gx = gx_new;
        if (a.frh_tma && tid == 0) tma_store_wait_read();  // the staging buffer is rewritten next step
        slot_prev = slot;
        if (++slot == RING) {
            slot = 0;
            phase ^= 1u;
        }
        __syncthreads();
    };
    // pairs of steps without a conditional second step, then the odd last step
    int k = kfirst;
#pragma unroll 1
    for (; k + 1 <= klast; k += 2) {
        step(Par<0>{}, k);
        step(Par<1>{}, k + 1);
    }
    if (k <= klast) step(Par<0>{}, k);
#undef EV2_ISSUE
    if (a.frh_tma && tid == 0) tma_store_wait_all();  // rho-hat complete before the grid ends
    pdl_trigger();  // the finalize may be scheduled while the tiles flush
    if (grad) {  // flush: pending y collapse, then the last two nodal planes
        if (ypend >= 0) ycollapse(ypend);
        __syncthreads();
        xcollapse(acc00, acc01, acc02);
        __syncthreads();
        ycollapse(cur);
        __syncthreads();
        xcollapse(acc10, acc11, acc12);
        __syncthreads();
        ycollapse(cur + 1);
    }
    // per-tile sum of (1 - r^2), fixed order
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) dsum += __shfl_down_sync(0xffffffffu, dsum, o);
    if (lane == 0) sred[row] = dsum;
    __syncthreads();
    // (the last-CTA flag goes to sred[0] once thread 0 has read sred: no static shared memory,
    // which would push two CTAs past an SM's shared memory at the dynamic-size cap)
    unsigned int* const s_last = reinterpret_cast<unsigned int*>(sred);
    if (tid == 0) {
        double s = 0.0;
        for (int w = 0; w < NT / 32; ++w) s += sred[w];
        a.vpart[tile_id] = s;
        if (a.vticket) {  // two-level completion ticket over the CTAs (32 group counters, then one)
            __threadfence();
            // (over all tiles: a pass launched in z groups counts every group's CTAs)
            const unsigned nct = static_cast<unsigned>(tm.ntx * tm.nty * tm.ntz), id = static_cast<unsigned>(tile_id);
            const unsigned g = id % 32u, ng = min(nct, 32u), gsize = (nct - g + 31u) / 32u;
            unsigned lst = 0;
            if (atomicAdd(a.vticket + 1 + g, 1u) == gsize - 1) {
                a.vticket[1 + g] = 0u;
                __threadfence();
                lst = atomicAdd(a.vticket, 1u) == ng - 1 ? 1u : 0u;
            }
            *s_last = lst;
        }
    }
    if (!a.vticket) return;
    __syncthreads();
    if (!*s_last) return;
    // last CTA: D = h_bar * sum over tiles in tile order per thread, then a fixed tree
    __threadfence();
    const unsigned nct = static_cast<unsigned>(tm.ntx * tm.nty * tm.ntz);
    double v = 0.0;
    for (unsigned t = tid; t < nct; t += NT) v += a.vpart[t];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    __syncthreads();  // sred reuse
    if (lane == 0) sred[row] = v;
    __syncthreads();
    if (tid == 0) {
        double t = 0.0;
        for (int w = 0; w < NT / 32; ++w) t += sred[w];
        const double d = a.dscale * t;
        a.dsc[0] = d;
        a.dsc_host[0] = d;
        __threadfence_system();
        a.vticket[0] = 0u;
    }
}

// Value-only NGF pass (the Armijo trial evaluations): D = h_bar sum (1 - r^2) with r computed
// exactly as k_ev2 computes it (same clamped differences with the TMA zero fill, ngf_coef) and
// summed in k_ev2's order (per column over its planes, per tile by the same warp and row tree,
// over tiles in the same last-CTA order), so D is bitwise the gradient evaluation's D. It reads
// R and T_w only (16 B/voxel at fp64) and writes nothing per voxel: no TMA ring, no P^T, no
// coefficient stores. One thread per tile column marching z; neighbours from L1.
template <typename Real>
__global__ void __launch_bounds__(NT) k_ev_value(const __grid_constant__ FArgs a, const Real* __restrict__ R,
                                                 const Real* __restrict__ Tw) {
    __shared__ double sred[NT / 32];
    __shared__ unsigned int s_last;
    const TileMeta& tm = a.tm;
    const int tid = threadIdx.x, lane = tid & 31, row = tid >> 5;
    const int mx = static_cast<int>(a.g.m[0]), my = static_cast<int>(a.g.m[1]), mz = static_cast<int>(a.g.m[2]);
    const long long plane = static_cast<long long>(mx) * my;
    const int x0 = blockIdx.x * TX, y0 = blockIdx.y * TY;
    const int bzc = static_cast<int>(blockIdx.z) + a.zch0;  // z tile chunk (z-group launches)
    const int z0 = tm.zlo + bzc * tm.zc, z1 = min(tm.zhi, z0 + tm.zc);
    const int ilo = max(z0, a.olo), ihi = min(z1, a.ohi);
    const long long tile_id = (static_cast<long long>(bzc) * tm.nty + blockIdx.y) * tm.ntx + blockIdx.x;
    const int gx0 = x0 + lane, gy0 = y0 + row;
    const bool in0 = gx0 < mx && gy0 < my;
    const Real m0xm = gx0 > 0 ? Real(1) : Real(0), m0xp = gx0 + 1 < mx ? Real(1) : Real(0);
    const Real m0ym = gy0 > 0 ? Real(1) : Real(0), m0yp = gy0 + 1 < my ? Real(1) : Real(0);
    const bool hxm = gx0 > 0, hxp = gx0 + 1 < mx, hym = gy0 > 0, hyp = gy0 + 1 < my;
    const long long col = static_cast<long long>(min(gx0, mx - 1)) + static_cast<long long>(min(gy0, my - 1)) * mx;
    // a neighbour outside the volume reads 0 (the TMA zero fill k_ev2 sees)
    auto ld = [&](const Real* f, long long i, bool ok) { return ok ? __ldg(f + i) : Real(0); };
    double dsum = 0.0;
    if (in0 && ilo < ihi) {
        Real Rm = ld(R, col + (ilo - 1) * plane, ilo > 0), Tm = ld(Tw, col + (ilo - 1) * plane, ilo > 0);
        Real Rj = __ldg(R + col + ilo * plane), Tj = __ldg(Tw + col + ilo * plane);
#pragma unroll 1
        for (int j = ilo; j < ihi; ++j) {
            const long long o = col + j * plane;
            const bool hzp = j + 1 < mz;
            const Real Rp = ld(R, o + plane, hzp), Tp = ld(Tw, o + plane, hzp);
            const Real mzm = j > 0 ? Real(1) : Real(0), mzp = hzp ? Real(1) : Real(0);
            const Coef<Real> cf = ngf_coef(
                a, m0xm * (ld(R, o - 1, hxm) - Rj), m0xp * (ld(R, o + 1, hxp) - Rj), m0ym * (ld(R, o - mx, hym) - Rj),
                m0yp * (ld(R, o + mx, hyp) - Rj), mzm * (Rm - Rj), mzp * (Rp - Rj), m0xm * (ld(Tw, o - 1, hxm) - Tj),
                m0xp * (ld(Tw, o + 1, hxp) - Tj), m0ym * (ld(Tw, o - mx, hym) - Tj), m0yp * (ld(Tw, o + mx, hyp) - Tj),
                mzm * (Tm - Tj), mzp * (Tp - Tj), true);
            dsum += fma(-static_cast<double>(cf.r), static_cast<double>(cf.r), 1.0);
            Rm = Rj;
            Tm = Tj;
            Rj = Rp;
            Tj = Tp;
        }
    }
    // per-tile sum, then the last CTA: k_ev2's reduction order exactly
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) dsum += __shfl_down_sync(0xffffffffu, dsum, o);
    if (lane == 0) sred[row] = dsum;
    __syncthreads();
    if (tid == 0) {
        double t = 0.0;
        for (int w = 0; w < NT / 32; ++w) t += sred[w];
        a.vpart[tile_id] = t;
        __threadfence();
        const unsigned nct = gridDim.x * gridDim.y * gridDim.z, id = static_cast<unsigned>(tile_id);
        const unsigned g = id % 32u, ng = min(nct, 32u), gsize = (nct - g + 31u) / 32u;
        unsigned lst = 0;
        if (atomicAdd(a.vticket + 1 + g, 1u) == gsize - 1) {
            a.vticket[1 + g] = 0u;
            __threadfence();
            lst = atomicAdd(a.vticket, 1u) == ng - 1 ? 1u : 0u;
        }
        s_last = lst;
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    const unsigned nct = gridDim.x * gridDim.y * gridDim.z;
    double v = 0.0;
    for (unsigned t = tid; t < nct; t += NT) v += a.vpart[t];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    __syncthreads();
    if (lane == 0) sred[row] = v;
    __syncthreads();
    if (tid == 0) {
        double t = 0.0;
        for (int w = 0; w < NT / 32; ++w) t += sred[w];
        const double d = a.dscale * t;
        a.dsc[0] = d;
        a.dsc_host[0] = d;
        __threadfence_system();
        a.vticket[0] = 0u;
    }
}

}  // namespace

namespace {
template <typename Real>
std::size_t smem_bytes(int nlx, int nly, int segw) {
    using G = Geo<Real>;
    return static_cast<std::size_t>(RING) * G::SLOT * sizeof(Real) + 2 * 6 * NT * sizeof(Real) + 48 +
           (NT / 32) * sizeof(double) +
           (2 * 2 * NT + 2 * 2 * TY + static_cast<std::size_t>(ptc_reals(TY, nlx, nly, segw, MFREG_PTC_PAD && sizeof(Real) == 8))) * sizeof(Real) +
           (NX_A + ptc_ints(nlx)) * sizeof(int);
}
}  // namespace

std::size_t ev2_smem_bytes(int nlx, int nly, int segw, bool fp32) {
    return fp32 ? smem_bytes<float>(nlx, nly, segw) : smem_bytes<double>(nlx, nly, segw);
}

void ev2_set_smem_cap(int bytes) {
    MFREG_CUDA(cudaFuncSetAttribute(k_ev2<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    MFREG_CUDA(cudaFuncSetAttribute(k_ev2<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
}

void ev_value_launch(const FArgs& a, const void* R, const void* Tw, dim3 grid, cudaStream_t s, bool fp32) {
    if (fp32) k_ev_value<float><<<grid, NT, 0, s>>>(a, static_cast<const float*>(R), static_cast<const float*>(Tw));
    else k_ev_value<double><<<grid, NT, 0, s>>>(a, static_cast<const double*>(R), static_cast<const double*>(Tw));
}

void ev2_launch(const FArgs& a, const TmaMaps& maps, dim3 grid, std::size_t smem, cudaStream_t s, bool fp32) {
    if (fp32) launch_pdl(k_ev2<float>, grid, dim3(NT), smem, s, a, maps);
    else launch_pdl(k_ev2<double>, grid, dim3(NT), smem, s, a, maps);
}

}  // namespace mfreg_b200
