// Kernel launchers for the B200 NGF + curvature hot path (implemented in kernels.cu).
// Each launcher names the reference function it replaces (file:line under
// /root/reference/proj).
#pragma once

#include "common.cuh"

namespace mfreg_b200 {

// Closed-form GN Hv offset table (reference make_offset_table, ngf.cpp:267-300),
// regrouped by 3-D offset and ordered by the linear offset kappa of the grid.
struct HvTable {
    int ngroups;
    int dx[25], dy[25], dz[25];
    int npairs[25];
    int pa[25][7], pb[25][7];
};
HvTable make_hv_table(const Grid& g);

// launch accounting (mfreg_cu_launch_count)
void note_launch();
void note_launches(long long n);
long long launch_counter();

// ---- grid transfer and warp (transfer.cpp:49-150, volume.cpp:29-94)
void launch_transfer_apply(const DevPlan& P, const double* y, double* out, cudaStream_t s);
// (zlo, zhi): z window of the outputs (nodal planes for P^T / curvature, image planes otherwise);
// the default is the whole grid
void launch_transfer_T(const DevPlan& P, const double* w, double* out, cudaStream_t s, int zlo = 0, int zhi = -1);
void launch_sample(const Grid& img, const double* T, const double* pts, idx_t n, double* vals, double* dT,
                   cudaStream_t s);
// Fused P*y + trilinear sample: T_w and dT/dP (32 B/voxel) without materialising P*y.
// image planes [zlo, zhi) (zhi < 0: all)
void launch_warp_fast(const DevPlan& P, const double* y, const double* T, double* Tw, double* dT, cudaStream_t s,
                      int zlo = 0, int zhi = -1);
// FAST32 state: single-precision copies / T_w, dT
void launch_to_float(idx_t n, const double* a, float* o, cudaStream_t s);
void launch_warp_fast(const DevPlan& P, const double* y, const double* T, float* Tw, float* dT, cudaStream_t s,
                      int zlo = 0, int zhi = -1);
void launch_warp(const DevPlan& P, const double* y, const double* T, double* Tw, double* dT, cudaStream_t s,
                 int zlo = 0, int zhi = -1);

// ---- NGF workspace (ngf.cpp:185-214) + rho-hat table (ngf.cpp:39-64)
void launch_ngf_ws(const Grid& img, const double* R, const double* Tw, double tau, double rho, double* r,
                   double* inv1, double* inv2, double* rh, cudaStream_t s, int zlo = 0, int zhi = -1);
void launch_ngf_gradient(const Grid& img, const double* r, const double* rh, const double* dT, double* out,
                         cudaStream_t s, int zlo = 0, int zhi = -1);
// s_i = dT_i . (P p)_i  (the inner product inside ngf.cpp:145-148)
void launch_Pp_s(const DevPlan& P, const double* p, const double* dT, double* sv, cudaStream_t s, int zlo = 0,
                 int zhi = -1);
// parity: closed form (ngf.cpp:105-163), bit-identical
void launch_hv_closed(const Grid& img, const HvTable& tab, const double* rh, const double* sv, const double* dT,
                      double* out, cudaStream_t s, int zlo = 0, int zhi = -1);
// fast: factored 2h dT^T dr^T (dr (dT p))
void launch_hv_factored(const Grid& img, const double* rh, const double* sv, const double* dT, double* wbuf,
                        double* out, cudaStream_t s);

// ---- reductions (parallel.cpp:51-73 chunked_sum; exact order) and fast tree sums
enum SumKind { SUM_ONE_MINUS_SQ = 0, SUM_DOT = 1, SUM_SQ = 2 };
// exact: per-4096-chunk sequential partials, then `out = scale * sum_in_order(partials)`
void launch_chunked_sum(int kind, idx_t n, const double* a, const double* b, double* partials, double* out,
                        double scale, cudaStream_t s);
// fast: deterministic two-level tree sum (fixed block partition, fixed order)
// three equal-length segments (a + d n, d = 0..2), each summed as launch_chunked_sum into out3[d]
void launch_chunked_sum3(int kind, idx_t n, const double* a, const double* b, double* partials, double* out3,
                         double scale, cudaStream_t s);
// distributed chunked_sum pieces (slab.cu DistSum)
struct ChunkPiece {
    long long off;  // first term in the gathered blocks
    int len;
};
void launch_chunk_partials(int kind, idx_t n, const double* a, const double* b, double* partials, cudaStream_t s);
void launch_sum_terms(int kind, idx_t n, const double* a, const double* b, double* out, cudaStream_t s);
void launch_chunk_assemble(idx_t nch, const long long* off, const int* cnt, const ChunkPiece* pieces,
                           const double* gathered, double* vals, double scale, double* out, cudaStream_t s);
void launch_tree_sum(int kind, idx_t n, const double* a, const double* b, double* partials, double* out,
                     double scale, cudaStream_t s);
idx_t chunk_count(idx_t n);
idx_t tree_blocks(idx_t n);
// max |x| (exact; order independent), NaN ignored as std::max does (optimizer.cpp:23-29)
void launch_inf_norm(idx_t n, const double* a, double scale, double* out, cudaStream_t s);

// ---- curvature (curvature.cpp:9-98), nodal grid, 3 components
// exact = false (fast modes): the quotient by h*h is the product with its reciprocal (within 1 ulp)
void launch_lap3(const Grid& g, const double* u, double* out, cudaStream_t s, int zlo = 0, int zhi = -1,
                 bool exact = true);
// mode 0: out = scale*Lap(in); 1: out += alpha*(scale*Lap(in)); 2: out = scale*Lap(in) + gamma*p
void launch_bilap(const Grid& g, const double* lap_u, double scale, int mode, double alpha, double gamma,
                  const double* p, double* out, cudaStream_t s, int zlo = 0, int zhi = -1, bool exact = true);
// curvature value finalize: out = alpha * (cellvol * ((S0 + S1) + S2))
void launch_curv_finalize(const double* S3, double cellvol, double alpha, double* out, cudaStream_t s);
void launch_curv_value(const double* S, double cellvol, double alpha, double* out_dev, double* out_host,
                       cudaStream_t s);
void launch_add_scalars(const double* a, const double* b, double* out, cudaStream_t s);

// ---- BLAS-1 (exact, element-parallel)
void launch_sub(idx_t n, const double* a, const double* b, double* out, cudaStream_t s);          // a - b
void launch_neg(idx_t n, const double* a, double* out, cudaStream_t s);                           // -a
void launch_axpy_to(idx_t n, const double* x, double a, const double* y, double* out, cudaStream_t s);  // x + a*y
void launch_cg_update(idx_t n, double alpha, const double* p, const double* ap, double* x, double* r,
                      cudaStream_t s);
void launch_scale_to(idx_t n, double a, const double* x, double* out, cudaStream_t s);            // a*x
void launch_identity(const Grid& g, double* out, cudaStream_t s);

// ---- pyramid / prolongation (volume.cpp:123-160, multilevel.cpp:51-115)
void launch_downsample(const Grid& fine, const Grid& coarse, const double* v, double* out, cudaStream_t s);
void launch_prolong(const Grid& coarse, const Grid& fine, const double* yc, double* yf, cudaStream_t s);

// ---- synthetic inputs (synthetic.cpp:15-175)
struct WarpTerms {
    double extent[3];
    double amp[3][3];
    int freq[3][3];
    double phase[3][3];
};
void launch_phantom(const Grid& g, double* out, cudaStream_t s);
void launch_warp_with(const Grid& g, const WarpTerms& w, const double* T, double* out, cudaStream_t s);
void launch_scale_inplace(idx_t n, double a, double* x, cudaStream_t s);

}  // namespace mfreg_b200
