// Fused fast-mode kernels (see fused.cuh for the algebra and execution scheme).
#include <algorithm>
#include <cstdlib>
#include <vector>

#include "fused.cuh"

namespace mfreg_b200 {

namespace {

constexpr int CX = FT_X + 4, CY = FT_Y + 4, NC = CX * CY;  // columns incl. 2-voxel halo (432)
constexpr int NTH = 448;                                     // threads per CTA (>= NC, multiple of 32)
constexpr int TT = FT_X * FT_Y;                              // output columns (256)
constexpr int NH1 = (FT_X + 2) * (FT_Y + 2);                 // columns incl. 1-voxel halo (340)
constexpr int kSMs = 148;

struct FArgs {
    Grid g;
    DevPlan P;
    TileMeta tm;
    double hh[3];   // h^_a = 1 / (2 h_a^2)
    double ih2[3];  // 1 / h_a^2
    double scale;   // Hv: 2 h_bar; eval gradient: -2 h_bar
    double tau, rho;
    const double* R;    // eval
    const double* Tw;   // eval
    const double* dT;
    const double* frh;  // Hv input: rho-hat [6][n]
    const double* p;    // Hv nodal operand
    double* frh_out;    // eval output
    double* part;
    double* vpart;
    int grad;
};

__device__ __forceinline__ double lerp(double t, double a, double b) { return fma(t, b - a, a); }

// bilinear x-y interpolation of the 3 nodal components on nodal plane nz at a fixed column
__device__ __forceinline__ void bilerp3(const double* __restrict__ p, long long ns, long long sm0, long long sm01,
                                        int bx, int by, int nz, double rx, double ry, double out[3]) {
    const long long c = bx + by * sm0 + nz * sm01;
#pragma unroll
    for (int d = 0; d < 3; ++d) {
        const double* q = p + d * ns + c;
        const double v0 = lerp(rx, __ldg(q), __ldg(q + 1));
        const double v1 = lerp(rx, __ldg(q + sm0), __ldg(q + sm0 + 1));
        out[d] = lerp(ry, v0, v1);
    }
}

// Per-CTA precomputed task of the x-y spread (P^T in x then y): which local
// node / row a thread reduces and the clipped voxel ranges of its two cells.
struct SpreadTask {
    int xrow, xl, xlo1, xhi1, xlo0, xhi0;  // x-collapse: row, local node, ranges for cells nx-1 (w = r), nx (w = 1-r)
    int yl, yx, ylo1, yhi1, ylo0, yhi0;    // y-collapse: local node y, local node x, ranges
    bool xon, yon;
};

__device__ SpreadTask make_spread_task(const DevPlan& P, int x0, int y0, int xe, int ye, int nxA, int nyA, int nlx_t,
                                       int nly_t) {
    SpreadTask t{};
    const int tid = threadIdx.x;
    const int nsx = static_cast<int>(P.src.m[0]) - 1, nsy = static_cast<int>(P.src.m[1]) - 1;
    t.xon = tid < FT_Y * nlx_t;
    if (t.xon) {
        t.xrow = tid / nlx_t;
        t.xl = tid % nlx_t;
        const int nx = nxA + t.xl;
        t.xlo1 = t.xhi1 = t.xlo0 = t.xhi0 = x0;
        if (nx >= 1 && nx - 1 < nsx) {
            t.xlo1 = max(x0, __ldg(&P.cell_lo[0][nx - 1]));
            t.xhi1 = max(t.xlo1, min(xe, __ldg(&P.cell_hi[0][nx - 1])));
        }
        if (nx < nsx) {
            t.xlo0 = max(x0, __ldg(&P.cell_lo[0][nx]));
            t.xhi0 = max(t.xlo0, min(xe, __ldg(&P.cell_hi[0][nx])));
        }
        if (y0 + t.xrow >= ye) t.xhi1 = t.xlo1, t.xhi0 = t.xlo0;
    }
    t.yon = tid < nly_t * nlx_t;
    if (t.yon) {
        t.yl = tid / nlx_t;
        t.yx = tid % nlx_t;
        const int ny = nyA + t.yl;
        t.ylo1 = t.yhi1 = t.ylo0 = t.yhi0 = y0;
        if (ny >= 1 && ny - 1 < nsy) {
            t.ylo1 = max(y0, __ldg(&P.cell_lo[1][ny - 1]));
            t.yhi1 = max(t.ylo1, min(ye, __ldg(&P.cell_hi[1][ny - 1])));
        }
        if (ny < nsy) {
            t.ylo0 = max(y0, __ldg(&P.cell_lo[1][ny]));
            t.yhi0 = max(t.ylo0, min(ye, __ldg(&P.cell_hi[1][ny])));
        }
    }
    return t;
}

// x-y spread of the per-column nodal-plane accumulators into the tile partial
// (P^T in x and y; z weights were applied per column). Called by all threads.
__device__ __noinline__ void spread_plane(const SpreadTask& st, const double* sremx, const double* sremy, double* sQ,
                                             double* sQx, int nlx, const double acc[3], bool tile, int tcol, int x0,
                                             int y0, double* dst) {
    if (tile) {
        sQ[tcol] = acc[0];
        sQ[TT + tcol] = acc[1];
        sQ[2 * TT + tcol] = acc[2];
    }
    __syncthreads();
    if (st.xon) {
#pragma unroll
        for (int d = 0; d < 3; ++d) {
            const double* q = sQ + d * TT + st.xrow * FT_X;
            double s = 0.0;
            for (int x = st.xlo1; x < st.xhi1; ++x) s = fma(sremx[x - x0], q[x - x0], s);
            for (int x = st.xlo0; x < st.xhi0; ++x) s = fma(1.0 - sremx[x - x0], q[x - x0], s);
            sQx[(d * FT_Y + st.xrow) * nlx + st.xl] = s;
        }
    }
    __syncthreads();
    if (st.yon) {
#pragma unroll
        for (int d = 0; d < 3; ++d) {
            const double* q = sQx + d * FT_Y * nlx + st.yx;
            double s = 0.0;
            for (int y = st.ylo1; y < st.yhi1; ++y) s = fma(sremy[y - y0], q[(y - y0) * nlx], s);
            for (int y = st.ylo0; y < st.yhi0; ++y) s = fma(1.0 - sremy[y - y0], q[(y - y0) * nlx], s);
            dst[(st.yl * nlx + st.yx) * 3 + d] = s;
        }
    }
    __syncthreads();
}

// Shared-memory plane buffers are padded by PAD doubles on both sides so that
// every active column may read its +-1 / +-CX neighbours without a guard.
constexpr int PAD = CX + 1;
constexpr int NB = NC + 2 * PAD;

template <bool EVAL, int MINB>
__global__ void __launch_bounds__(NTH, MINB) k_fused(FArgs a) {
    extern __shared__ double sm[];
    double* sP0 = sm + PAD;            // [2][NB] Hv: s; eval: R (by plane parity)
    double* sP1 = sP0 + 2 * NB;        // [2][NB] eval: T_w
    double* sW = sP1 + 2 * NB;         // [2][NB] Hv: w; eval: r
    double* sRh = sW + 2 * NB;         // [2][4][NB] in-plane rho-hat (-x,+x,-y,+y)
    double* sDq = sRh + 8 * NB - PAD;  // [3][3][TT] dT of the tile columns
    double* sQ = sDq + 9 * TT;         // [3][TT]
    double* sQx = sQ + 3 * TT;         // [3][FT_Y][nlx]
    double* sremx = sQx + 3 * FT_Y * a.tm.nlx;
    double* sremy = sremx + FT_X;
    __shared__ double sred[32];

    const TileMeta& tm = a.tm;
    const int tid = threadIdx.x;
    const int mx = static_cast<int>(a.g.m[0]), my = static_cast<int>(a.g.m[1]), mz = static_cast<int>(a.g.m[2]);
    const long long n = a.g.count(), plane = static_cast<long long>(mx) * my;
    const int x0 = blockIdx.x * FT_X, y0 = blockIdx.y * FT_Y;
    const int z0 = blockIdx.z * tm.zc, z1 = min(mz, z0 + tm.zc);
    const int xe = min(mx, x0 + FT_X), ye = min(my, y0 + FT_Y);
    const int nxA = __ldg(&a.P.base[0][x0]), nyA = __ldg(&a.P.base[1][y0]), nzA = __ldg(&a.P.base[2][z0]);
    const int nlx_t = __ldg(&a.P.base[0][xe - 1]) - nxA + 2;
    const int nly_t = __ldg(&a.P.base[1][ye - 1]) - nyA + 2;
    const long long tile_id = (static_cast<long long>(blockIdx.z) * tm.nty + blockIdx.y) * tm.ntx + blockIdx.x;
    double* part = a.part + tile_id * tm.part_stride;
    const std::size_t pstride = static_cast<std::size_t>(tm.nly) * tm.nlx * 3;

    // thread -> column: tile columns first (warps 0-7 run every phase), then the
    // halo-1 ring (phase W), then the halo-2 ring (loads only)
    const bool active = tid < NC;
    int lx, ly;
    if (tid < TT) {
        lx = 2 + tid % FT_X;
        ly = 2 + tid / FT_X;
    } else if (tid < NH1) {
        const int r = tid - TT;  // 84 = 34 + 34 + 8 + 8
        if (r < CX - 2) { lx = 1 + r; ly = 1; }
        else if (r < 2 * (CX - 2)) { lx = 1 + r - (CX - 2); ly = CY - 2; }
        else if (r < 2 * (CX - 2) + FT_Y) { lx = 1; ly = 2 + r - 2 * (CX - 2); }
        else { lx = CX - 2; ly = 2 + r - 2 * (CX - 2) - FT_Y; }
    } else {
        const int r = tid < NC ? tid - NH1 : 0;  // 92 = 36 + 36 + 10 + 10
        if (r < CX) { lx = r; ly = 0; }
        else if (r < 2 * CX) { lx = r - CX; ly = CY - 1; }
        else if (r < 2 * CX + CY - 2) { lx = 0; ly = 1 + r - 2 * CX; }
        else { lx = CX - 1; ly = 1 + r - 2 * CX - (CY - 2); }
    }
    const int c = lx + ly * CX;  // position in the plane buffers
    const bool inW = tid < NH1;
    const bool inZ = tid < TT;
    const int gx = x0 - 2 + lx, gy = y0 - 2 + ly;
    const bool indom = active && gx >= 0 && gx < mx && gy >= 0 && gy < my;
    const bool tile = inZ && gx < mx && gy < my;
    // clamped column (out-of-domain halo columns replicate the boundary column:
    // differences across the boundary vanish exactly, as the reference's clamps)
    const int gxc = min(max(gx, 0), mx - 1), gyc = min(max(gy, 0), my - 1);
    const long long col = static_cast<long long>(gxc) + static_cast<long long>(gyc) * mx;

    if (tid < FT_X) sremx[tid] = x0 + tid < mx ? __ldg(&a.P.rem[0][x0 + tid]) : 0.0;
    if (tid < FT_Y) sremy[tid] = y0 + tid < my ? __ldg(&a.P.rem[1][y0 + tid]) : 0.0;
    if (tid < 2 * PAD) {  // zero the guard pads of every padded buffer
        const int o = tid < PAD ? -PAD + tid : NC + (tid - PAD);
        for (int b = 0; b < 14; ++b) sP0[b * NB + o] = 0.0;
    }
    const SpreadTask st = make_spread_task(a.P, x0, y0, xe, ye, nxA, nyA, nlx_t, nly_t);

    // separable P p (Hv): fixed x-y weights per column, z blend per plane
    int pz = -1000;
    double Pa0 = 0.0, Pa1 = 0.0, Pa2 = 0.0, Pb0 = 0.0, Pb1 = 0.0, Pb2 = 0.0;
    const long long ns = a.P.src.count(), sm0 = a.P.src.m[0], sm01 = a.P.src.m[0] * a.P.src.m[1];
    const int bx = __ldg(&a.P.base[0][gxc]), by = __ldg(&a.P.base[1][gyc]);
    const double rx = __ldg(&a.P.rem[0][gxc]), ry = __ldg(&a.P.rem[1][gyc]);

    // column histories (plane index relative to the current iteration k)
    double sh1 = 0.0, sh2 = 0.0;              // Hv: s_{k-1}, s_{k-2}
    double Rh1 = 0.0, Rh2 = 0.0, Th1 = 0.0, Th2 = 0.0;  // eval: R, T_w at k-1, k-2
    double wh1 = 0.0, wh2 = 0.0;              // w (or r) at k-2, k-3
    double sg1 = 0.0;                          // sigma at k-2
    double pzh1 = 0.0, pzh2 = 0.0;             // rho-hat(+z) at k-2, k-3
    double acc00 = 0.0, acc01 = 0.0, acc02 = 0.0, acc10 = 0.0, acc11 = 0.0, acc12 = 0.0;
    double dsum = 0.0;
    int cur = nzA;

    // prefetch registers: plane k+1 (clamped) streams, rho-hat of plane k (Hv)
    double nA = 0.0, nB = 0.0, nD0 = 0.0, nD1 = 0.0, nD2 = 0.0;
    double nr0 = 0.0, nr1 = 0.0, nr2 = 0.0, nr3 = 0.0, nr4 = 0.0, nr5 = 0.0;
    const bool need_dT = EVAL ? inZ : active;
    {
        const long long o = col + static_cast<long long>(min(max(z0 - 2, 0), mz - 1)) * plane;
        if (EVAL && active) {
            nA = __ldg(a.R + o);
            nB = __ldg(a.Tw + o);
        }
        if (need_dT) {
            nD0 = __ldg(a.dT + o);
            nD1 = __ldg(a.dT + n + o);
            nD2 = __ldg(a.dT + 2 * n + o);
        }
        const int kr = z0 - 3;
        if (!EVAL && inW && indom && kr >= 0 && kr < mz) {
            const long long oi = col + static_cast<long long>(kr) * plane;
            nr0 = __ldg(a.frh + oi);
            nr1 = __ldg(a.frh + n + oi);
            nr2 = __ldg(a.frh + 2 * n + oi);
            nr3 = __ldg(a.frh + 3 * n + oi);
            nr4 = __ldg(a.frh + 4 * n + oi);
            nr5 = __ldg(a.frh + 5 * n + oi);
        }
    }
    __syncthreads();

#pragma unroll 1
    for (int k = z0 - 2; k <= z1 + 1; ++k) {
        const int kc = min(max(k, 0), mz - 1);
        // ---- rotate prefetched values in, issue the next loads
        const double A0 = nA, B0 = nB, D0 = nD0, D1 = nD1, D2 = nD2;
        const double r0 = nr0, r1 = nr1, r2 = nr2, r3 = nr3, r4 = nr4, r5 = nr5;  // Hv: rho-hat of plane k-1
        {
            const long long o = col + static_cast<long long>(min(k + 1, mz - 1) < 0 ? 0 : min(k + 1, mz - 1)) * plane;
            if (EVAL && active) {
                nA = __ldg(a.R + o);
                nB = __ldg(a.Tw + o);
            }
            if (need_dT) {
                nD0 = __ldg(a.dT + o);
                nD1 = __ldg(a.dT + n + o);
                nD2 = __ldg(a.dT + 2 * n + o);
            }
            if (!EVAL && inW) {
                const bool ok = indom && k >= 0 && k < mz;
                const long long oi = col + static_cast<long long>(kc) * plane;
                nr0 = ok ? __ldg(a.frh + oi) : 0.0;
                nr1 = ok ? __ldg(a.frh + n + oi) : 0.0;
                nr2 = ok ? __ldg(a.frh + 2 * n + oi) : 0.0;
                nr3 = ok ? __ldg(a.frh + 3 * n + oi) : 0.0;
                nr4 = ok ? __ldg(a.frh + 4 * n + oi) : 0.0;
                nr5 = ok ? __ldg(a.frh + 5 * n + oi) : 0.0;
            }
        }

        // ---- phase P: plane k into shared memory
        double s0 = 0.0;
        if (!EVAL) {
            const int bz = __ldg(&a.P.base[2][kc]);
            const double rz = __ldg(&a.P.rem[2][kc]);
            if (bz != pz) {  // uniform across the CTA
                double t[3];
                if (bz == pz + 1) {
                    Pa0 = Pb0;
                    Pa1 = Pb1;
                    Pa2 = Pb2;
                } else {
                    bilerp3(a.p, ns, sm0, sm01, bx, by, bz, rx, ry, t);
                    Pa0 = t[0];
                    Pa1 = t[1];
                    Pa2 = t[2];
                }
                bilerp3(a.p, ns, sm0, sm01, bx, by, bz + 1, rx, ry, t);
                Pb0 = t[0];
                Pb1 = t[1];
                Pb2 = t[2];
                pz = bz;
            }
            s0 = fma(D0, lerp(rz, Pa0, Pb0), fma(D1, lerp(rz, Pa1, Pb1), D2 * lerp(rz, Pa2, Pb2)));
            if (active) sP0[(k & 1) * NB + c] = s0;
            if (inW) {  // in-plane coefficients of plane k-1 for the neighbours' phase Z
                double* rb = sRh + ((k - 1) & 1) * 4 * NB + c;
                rb[0] = r0;
                rb[NB] = r1;
                rb[2 * NB] = r2;
                rb[3 * NB] = r3;
            }
        } else if (active) {
            sP0[(k & 1) * NB + c] = A0;
            sP1[(k & 1) * NB + c] = B0;
        }
        if (inZ) {
            double* dq = sDq + ((k + 3) % 3) * 3 * TT + tid;
            dq[0] = D0;
            dq[TT] = D1;
            dq[2 * TT] = D2;
        }
        __syncthreads();

        // ---- phase W: w (Hv) or rho-hat and r (eval) of plane j = k-1
        const int j = k - 1;
        double wc = 0.0, sgc = 0.0, mzc = 0.0, pzc = 0.0;  // fresh values of plane j
        if (inW) {
            if (!EVAL) {
                const double* cs = sP0 + (j & 1) * NB;
                const double sj = sh1;
                wc = r0 * (cs[c - 1] - sj);
                wc = fma(r1, cs[c + 1] - sj, wc);
                wc = fma(r2, cs[c - CX] - sj, wc);
                wc = fma(r3, cs[c + CX] - sj, wc);
                wc = fma(r4, sh2 - sj, wc);
                wc = fma(r5, s0 - sj, wc);
                sgc = ((r0 + r1) + (r2 + r3)) + (r4 + r5);
                mzc = r4;
                pzc = r5;
            } else {
                const double* cR = sP0 + (j & 1) * NB;
                const double* cT = sP1 + (j & 1) * NB;
                const double Rj = Rh1, Tj = Th1;
                const double dR0 = cR[c - 1] - Rj, dR1 = cR[c + 1] - Rj, dR2 = cR[c - CX] - Rj, dR3 = cR[c + CX] - Rj;
                const double dR4 = Rh2 - Rj, dR5 = A0 - Rj;
                const double dT0 = cT[c - 1] - Tj, dT1 = cT[c + 1] - Tj, dT2 = cT[c - CX] - Tj, dT3 = cT[c + CX] - Tj;
                const double dT4 = Th2 - Tj, dT5 = B0 - Tj;
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
                const double hx = a.hh[0], hy = a.hh[1], hz = a.hh[2];
                const double q0 = ok ? hx * fma(dR0, in1, -dT0 * in2) : 0.0;
                const double q1 = ok ? hx * fma(dR1, in1, -dT1 * in2) : 0.0;
                const double q2 = ok ? hy * fma(dR2, in1, -dT2 * in2) : 0.0;
                const double q3 = ok ? hy * fma(dR3, in1, -dT3 * in2) : 0.0;
                const double q4 = ok ? hz * fma(dR4, in1, -dT4 * in2) : 0.0;
                const double q5 = ok ? hz * fma(dR5, in1, -dT5 * in2) : 0.0;
                const double r = ok ? num * in1 : 0.0;
                wc = r;
                sgc = ((q0 + q1) + (q2 + q3)) + (q4 + q5);
                mzc = q4;
                pzc = q5;
                double* rb = sRh + (j & 1) * 4 * NB + c;
                rb[0] = q0;
                rb[NB] = q1;
                rb[2 * NB] = q2;
                rb[3 * NB] = q3;
                if (tile && j >= z0 && j < z1) {
                    const long long gi = col + static_cast<long long>(j) * plane;
                    a.frh_out[gi] = q0;
                    a.frh_out[n + gi] = q1;
                    a.frh_out[2 * n + gi] = q2;
                    a.frh_out[3 * n + gi] = q3;
                    a.frh_out[4 * n + gi] = q4;
                    a.frh_out[5 * n + gi] = q5;
                    dsum += fma(-r, r, 1.0);
                }
            }
            sW[(j & 1) * NB + c] = wc;
        }
        __syncthreads();

        // ---- phase Z: divergence at plane i = k-2, P^T accumulation
        if (!EVAL || a.grad) {
            const int i = k - 2;
            double q0 = 0.0, q1 = 0.0, q2 = 0.0;
            if (inZ) {
                const double* cw = sW + (i & 1) * NB;
                const double* cr = sRh + (i & 1) * 4 * NB;
                // neighbour coefficient toward i: +x neighbour holds (-x), -x neighbour holds (+x), ...
                double z = cr[NB + c - 1] * cw[c - 1];
                z = fma(cr[c + 1], cw[c + 1], z);
                z = fma(cr[3 * NB + c - CX], cw[c - CX], z);
                z = fma(cr[2 * NB + c + CX], cw[c + CX], z);
                z = fma(mzc, wc, z);      // rho-hat_{i+z}(-z) w_{i+z}
                z = fma(pzh2, wh2, z);    // rho-hat_{i-z}(+z) w_{i-z}
                z = fma(-sg1, wh1, z);    // -sigma_i w_i
                const double sz = a.scale * z;
                const double* dq = sDq + ((k + 1) % 3) * 3 * TT + tid;  // plane k-2
                q0 = sz * dq[0];
                q1 = sz * dq[TT];
                q2 = sz * dq[2 * TT];
            }
            if (i >= z0 && i < z1) {  // uniform
                const int bz = __ldg(&a.P.base[2][i]);
                const double rz = __ldg(&a.P.rem[2][i]);
                if (bz > cur) {  // nodal plane `cur` complete: spread in x-y (all threads)
                    const double acc[3] = {acc00, acc01, acc02};
                    spread_plane(st, sremx, sremy, sQ, sQx, tm.nlx, acc, tile, tid, x0, y0,
                                 part + static_cast<std::size_t>(cur - nzA) * pstride);
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
        }
        __syncthreads();
        // ---- rotate the column histories
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
    }
    if (!EVAL || a.grad) {
        const double acc0[3] = {acc00, acc01, acc02}, acc1[3] = {acc10, acc11, acc12};
        spread_plane(st, sremx, sremy, sQ, sQx, tm.nlx, acc0, tile, tid, x0, y0,
                     part + static_cast<std::size_t>(cur - nzA) * pstride);
        spread_plane(st, sremx, sremy, sQ, sQx, tm.nlx, acc1, tile, tid, x0, y0,
                     part + static_cast<std::size_t>(cur + 1 - nzA) * pstride);
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
    const double* v;
    double* out;
    const double* dot_a;
    int value;
    double* sc;
    double* red;
    unsigned int* counter;
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

constexpr int FIN_THREADS = 256;

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

__global__ void __launch_bounds__(FIN_THREADS) k_nodal_finalize(FinArgs a) {
    __shared__ double sh[32];
    __shared__ bool last;
    const long long ny = a.gy.count();
    const long long node = static_cast<long long>(blockIdx.x) * FIN_THREADS + threadIdx.x;
    double r0 = 0.0, r1 = 0.0;  // reduction terms (dot or S)
    if (node < ny) {
        const long long mx = a.gy.m[0], my = a.gy.m[1], mzn = a.gy.m[2];
        const long long nx = node % mx, nyy = (node / mx) % my, nz = node / (mx * my);
        double acc[3] = {0.0, 0.0, 0.0};
        if (a.out) {
            const TileMeta& tm = a.tm;
            const int tz0 = tm.node_tlo[2][nz], tz1 = tm.node_thi[2][nz];
            const int ty0 = tm.node_tlo[1][nyy], ty1 = tm.node_thi[1][nyy];
            const int tx0 = tm.node_tlo[0][nx], tx1 = tm.node_thi[0][nx];
            for (int tz = tz0; tz <= tz1; ++tz) {
                const int lz = static_cast<int>(nz) - tm.tile_n0[2][tz];
                for (int ty = ty0; ty <= ty1; ++ty) {
                    const int lyn = static_cast<int>(nyy) - tm.tile_n0[1][ty];
                    for (int tx = tx0; tx <= tx1; ++tx) {
                        const int lxn = static_cast<int>(nx) - tm.tile_n0[0][tx];
                        const double* pp = a.part + ((static_cast<std::size_t>(tz) * tm.nty + ty) * tm.ntx + tx) *
                                                        tm.part_stride +
                                           ((static_cast<std::size_t>(lz) * tm.nly + lyn) * tm.nlx + lxn) * 3;
                        acc[0] += pp[0];
                        acc[1] += pp[1];
                        acc[2] += pp[2];
                    }
                }
            }
        }
#pragma unroll
        for (int d = 0; d < 3; ++d) {
            double v = acc[d];
            if (a.v != nullptr && (a.alpha != 0.0 || a.value)) {
                const double* u = a.v + d * ny;
                const double li = lapc(u, a.gy, nx, nyy, nz);
                if (a.value) r1 = fma(li, li, r1);
                if (a.out && a.alpha != 0.0) {
                    const Grid& g = a.gy;
                    double s = (lapc(u, g, clampl(nx - 1, mx - 1), nyy, nz) - 2.0 * li + lapc(u, g, clampl(nx + 1, mx - 1), nyy, nz)) /
                               (g.h[0] * g.h[0]);
                    s += (lapc(u, g, nx, clampl(nyy - 1, my - 1), nz) - 2.0 * li + lapc(u, g, nx, clampl(nyy + 1, my - 1), nz)) /
                         (g.h[1] * g.h[1]);
                    s += (lapc(u, g, nx, nyy, clampl(nz - 1, mzn - 1)) - 2.0 * li + lapc(u, g, nx, nyy, clampl(nz + 1, mzn - 1))) /
                         (g.h[2] * g.h[2]);
                    v = fma(a.alpha * a.scale_y, s, v);
                }
            }
            if (a.out) a.out[d * ny + node] = v;
            if (a.dot_a) r0 = fma(a.dot_a[d * ny + node], v, r0);
        }
    }
    if (a.sc == nullptr) return;
    r0 = block_reduce(r0, sh);
    r1 = a.value ? block_reduce(r1, sh) : 0.0;
    if (threadIdx.x == 0) {
        a.red[2 * blockIdx.x] = r0;
        a.red[2 * blockIdx.x + 1] = r1;
        __threadfence();
        const unsigned int t = atomicAdd(a.counter, 1u);
        last = (t == gridDim.x - 1);
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
            a.sc[1] = a.alpha * (a.cell_y * s1);      // alpha S
        } else {
            a.sc[0] = s0;                             // <dot_a, out>
        }
        *a.counter = 0u;
    }
}

std::size_t fused_smem_bytes(const TileMeta& tm) {
    return sizeof(double) * (14 * NB + 9 * TT + 3 * TT + 3 * FT_Y * tm.nlx + FT_X + FT_Y);
}

int fused_occupancy() {
    static const int occ = [] {
        const char* e = std::getenv("MFREG_FUSED_OCC");
        return (e && e[0] == '2') ? 2 : 1;
    }();
    return occ;
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
    return a;
}

}  // namespace

FusedPlan::FusedPlan(const DevicePlanOwner& plan) {
    const DevPlan& P = plan.view();
    const Grid& g = P.tgt;
    TileMeta& t = meta_;
    t.ntx = static_cast<int>((g.m[0] + FT_X - 1) / FT_X);
    t.nty = static_cast<int>((g.m[1] + FT_Y - 1) / FT_Y);
    // z chunking: minimise waves(1 CTA/SM) x (planes per chunk + 4 halo planes)
    const long long nxy = static_cast<long long>(t.ntx) * t.nty;
    const int mz = static_cast<int>(g.m[2]);
    int best = 1;
    double best_cost = 1e300;
    for (int ntz = 1; ntz <= std::max(1, mz / 4); ++ntz) {
        const int zc = (mz + ntz - 1) / ntz;
        const int real_ntz = (mz + zc - 1) / zc;
        const double waves = std::ceil(static_cast<double>(nxy * real_ntz) / kSMs);
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
    int nl[3];
    for (int a = 0; a < 3; ++a) {
        const auto& base = plan.host_base[a];
        const int ms = static_cast<int>(P.src.m[a]);
        const int m = static_cast<int>(g.m[a]);
        std::vector<int> n0(ntl[a]), n1(ntl[a]);
        nl[a] = 0;
        for (int k = 0; k < ntl[a]; ++k) {
            const int x0 = k * tsz[a], x1 = std::min(m, x0 + tsz[a]);
            n0[k] = base[x0];
            n1[k] = base[x1 - 1] + 1;
            nl[a] = std::max(nl[a], n1[k] - n0[k] + 1);
        }
        std::vector<int> lo(ms, 0), hi(ms, -1);
        for (int nd = 0; nd < ms; ++nd)
            for (int k = 0; k < ntl[a]; ++k)
                if (n0[k] <= nd && nd <= n1[k]) {
                    if (hi[nd] < 0) lo[nd] = k;
                    hi[nd] = k;
                }
        tlo_[a].resize(ms);
        thi_[a].resize(ms);
        n0_[a].resize(ntl[a]);
        MFREG_CUDA(cudaMemcpy(tlo_[a].get(), lo.data(), ms * sizeof(int), cudaMemcpyHostToDevice));
        MFREG_CUDA(cudaMemcpy(thi_[a].get(), hi.data(), ms * sizeof(int), cudaMemcpyHostToDevice));
        MFREG_CUDA(cudaMemcpy(n0_[a].get(), n0.data(), ntl[a] * sizeof(int), cudaMemcpyHostToDevice));
        t.node_tlo[a] = tlo_[a].get();
        t.node_thi[a] = thi_[a].get();
        t.tile_n0[a] = n0_[a].get();
    }
    t.nlx = nl[0];
    t.nly = nl[1];
    t.nlz = nl[2];
    t.part_stride = static_cast<std::size_t>(t.nlz) * t.nly * t.nlx * 3;
    part_.resize(t.part_stride * static_cast<std::size_t>(ntiles()));
    MFREG_CUDA(cudaMemset(part_.get(), 0, part_.size() * sizeof(double)));
    vpart_.resize(static_cast<std::size_t>(ntiles()));
    const long long ny = P.src.count();
    red_.resize(static_cast<std::size_t>(2 * ((ny + FIN_THREADS - 1) / FIN_THREADS) + 2));
    counter_.resize(1);
    MFREG_CUDA(cudaMemset(counter_.get(), 0, sizeof(unsigned int)));
    const int smem = static_cast<int>(fused_smem_bytes(t));
    MFREG_CUDA(cudaFuncSetAttribute(k_fused<false, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    MFREG_CUDA(cudaFuncSetAttribute(k_fused<true, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    MFREG_CUDA(cudaFuncSetAttribute(k_fused<false, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    MFREG_CUDA(cudaFuncSetAttribute(k_fused<true, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
}

void launch_hv_fused(const DevicePlanOwner& plan, FusedPlan& fp, const double* frh, const double* dT, const double* p,
                     cudaStream_t s) {
    FArgs a = make_args(plan, fp);
    a.scale = 2.0 * a.g.cell_volume();
    a.frh = frh;
    a.dT = dT;
    a.p = p;
    const TileMeta& t = fp.meta();
    note_launch();
    if (fused_occupancy() == 2) k_fused<false, 2><<<dim3(t.ntx, t.nty, t.ntz), NTH, fused_smem_bytes(t), s>>>(a);
    else k_fused<false, 1><<<dim3(t.ntx, t.nty, t.ntz), NTH, fused_smem_bytes(t), s>>>(a);
}

void launch_eval_fused(const DevicePlanOwner& plan, FusedPlan& fp, const double* R, const double* Tw, const double* dT,
                       double tau, double rho, double* frh, bool grad, cudaStream_t s) {
    FArgs a = make_args(plan, fp);
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
    if (fused_occupancy() == 2) k_fused<true, 2><<<dim3(t.ntx, t.nty, t.ntz), NTH, fused_smem_bytes(t), s>>>(a);
    else k_fused<true, 1><<<dim3(t.ntx, t.nty, t.ntz), NTH, fused_smem_bytes(t), s>>>(a);
}

void launch_nodal_finalize(const DevicePlanOwner& plan, FusedPlan& fp, const FinalizeSpec& spec, cudaStream_t s) {
    FinArgs a{};
    a.gy = plan.view().src;
    a.tm = fp.meta();
    a.part = fp.partials();
    a.vpart = fp.value_partials();
    a.ntiles = fp.ntiles();
    a.hbar = plan.view().tgt.cell_volume();
    a.alpha = spec.alpha;
    a.scale_y = 2.0 * a.gy.cell_volume();
    a.cell_y = a.gy.cell_volume();
    a.v = spec.v;
    a.out = spec.out;
    a.dot_a = spec.dot_a;
    a.value = spec.value ? 1 : 0;
    a.sc = spec.sc;
    a.red = fp.red();
    a.counter = fp.counter();
    const long long ny = a.gy.count();
    note_launch();
    k_nodal_finalize<<<static_cast<unsigned>((ny + FIN_THREADS - 1) / FIN_THREADS), FIN_THREADS, 0, s>>>(a);
}

}  // namespace mfreg_b200
