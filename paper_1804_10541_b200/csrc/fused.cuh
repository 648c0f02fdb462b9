// Fused `fast`-mode kernels: one pass over the image grid per operator, with the
// grid transfer P / P^T folded in, plus one small nodal finalize kernel.
//
// Factored Gauss-Newton product. With the directional
// coefficients rho-hat_t(k) = h^_a (dR_k inv1_t - dT_k inv2_t), dX_k = X_{t+k} - X_t
// (ngf.cpp:39-64; zero across the domain boundary, clamped neighbours) and
// rho-hat_t(0) = -sum_k rho-hat_t(k) =: -sigma_t, the reference's closed-form
// H^ p^ = 2h dT dr^T dr (dT . p^) (ngf.cpp:105-163) factors as
//   w_t = (dr s)_t   = sum_k rho-hat_t(k) (s_{t+k} - s_t),           s = dT . P p
//   z_i = (dr^T w)_i = sum_k rho-hat_{i+k}(-k) w_{i+k} - sigma_i w_i
// and the NGF gradient (ngf.cpp:66-103) is -2h dT (dr^T r). The eval pass stores
// the six rho-hat per voxel (48 B) next to dT (24 B); every Hv then streams
// 72 B/voxel and needs ~40 flops/voxel.
//
// Execution: 2.5D column marching. A CTA owns a 32x8 output tile and a z range;
// threads map to the tile columns first (warps 0-7), then the 1-voxel halo ring,
// then the 2-voxel halo ring. Each thread marches its column in z with the
// column's history in registers; only the in-plane neighbour data lives in
// shared memory. Loads of plane k+1 are issued before plane k is processed.
// P p is separable per column (x-y weights fixed, z blend per plane). P^T
// accumulates z weights per column in registers and spreads over x-y in
// shared memory once per completed nodal plane; per-tile partials are summed
// per node in a fixed order by the finalize kernel (deterministic, no atomics).
#pragma once

#include <utility>

#include "objective.cuh"

namespace mfreg_b200 {

constexpr int FT_X = 32;  // output tile (x) per CTA
constexpr int FT_Y = 8;   // output tile (y) per CTA

// Host-computed tiling of the image grid and the per-tile nodal footprints.
struct TileMeta {
    int ntx, nty, ntz;          // tiles per axis
    int zc;                     // z planes per tile
    int zlo, zhi;               // image planes the tiles cover
    int nlx, nly, nlz;          // max local nodes per tile per axis
    std::size_t part_stride;    // doubles per tile partial (nlz*nly*nlx*3)
    const int* g_off[3];        // per axis, CSR over nodes: entries [g_off[n], g_off[n+1])
    const int2* g_ent[3];       //   entry = (tile index along the axis, local node index in that tile)
};

class FusedPlan {
public:
    // R, Tw, dT, frh: the device arrays the fused kernels stream (tensor maps are
    // built over them when TMA can address the grid)
    // `slab`: z window; the full domain when slab.full()
    // fp32: the state arrays are single precision (FAST32 mode; two-CTA kernels only)
    // zc_cap > 0: z tile chunks of at most that many planes (the host-buffer pipeline's plan);
    // 0: as the shared-memory budget of the z tables allows (MFREG_ZC_MAX overrides)
    FusedPlan(const DevicePlanOwner& plan, const void* R, const void* Tw, const void* dT, const void* frh,
              const SlabSpec& slab, bool fp32 = false, int zc_cap = 0);
    bool fp32() const { return fp32_; }
    const void* state_R() const { return state_R_; }    // the arrays the passes read (fp64 or FAST32)
    const void* state_Tw() const { return state_Tw_; }
    bool tma() const { return tma_; }
    bool hv2() const { return hv2_; }  // two-CTA/SM Hv kernel (hv_fast.cu)
    std::size_t hv2_smem() const { return hv2_smem_; }
    int seg_width() const { return segw_; }
    int gather_max() const { return gmax_; }
    unsigned int* vticket() { return vticket_.get(); }  // max finalize gather entries per node per axis
    bool ev2() const { return ev2_; }  // two-CTA/SM eval kernel (ev_fast.cu)
    std::size_t ev2_smem() const { return ev2_smem_; }
    const void* maps_ev2() const { return maps_ev2_; }
    const void* frh_base() const { return frh_base_; }  // the rho-hat array the eval TMA store addresses
    const void* maps_hv2() const { return maps_hv2_; }
    const void* maps_hv() const { return maps_hv_; }
    const void* maps_ev() const { return maps_ev_; }
    // uniform-warp Hv pass (hv3.cu): own tiling (28 x 12 output tiles), own partials; it streams
    // the stored rho-hat (hv3_stored) or recomputes it from R and T_w (then the Hv state is R,
    // T_w, dT and the eval pass stores no rho-hat)
    bool hv3() const { return hv3_; }
    bool hv3_stored() const { return hv3_stored_; }
    bool hv16() const { return hv16_; }  // the own-tiling Hv pass is k_hv2 on 32 x 16 tiles (default)
    bool hv3_recompute() const { return hv3_ && !hv3_stored_; }
    const TileMeta& meta3() const { return meta3_; }
    double* partials3() { return part3_.get(); }
    int ntiles3() const { return meta3_.ntx * meta3_.nty * meta3_.ntz; }
    int slab3_x() const { return slab3_[0]; }
    int slab3_y() const { return slab3_[1]; }
    int gather_max3() const { return gmax3_; }
    std::size_t hv3_smem() const { return hv3_smem_; }
    const void* maps_hv3() const { return maps_hv3_; }
    const TileMeta& meta() const { return meta_; }
    double* partials() { return part_.get(); }
    double* value_partials() { return vpart_.get(); }
    double* red() { return red_.get(); }
    unsigned int* counter() { return counter_.get(); }
    int ntiles() const { return meta_.ntx * meta_.nty * meta_.ntz; }
    int slab_x() const { return slab_[0]; }
    int slab_y() const { return slab_[1]; }
    int out_lo() const { return out_lo_; }   // image planes with outputs
    int out_hi() const { return out_hi_; }
    int fin_lo() const { return fin_lo_; }   // nodal planes the finalize writes
    int fin_hi() const { return fin_hi_; }
    int own_lo() const { return own_lo_; }   // owned nodal planes (curvature term, dots)
    int own_hi() const { return own_hi_; }

private:
    TileMeta meta_{};
    DevArray<int> goff_[3];
    DevArray<int2> gent_[3];
    DVec part_, vpart_, red_;
    DevArray<unsigned int> counter_;
    int slab_[2] = {0, 0};
    int out_lo_ = 0, out_hi_ = 0, fin_lo_ = 0, fin_hi_ = 0, own_lo_ = 0, own_hi_ = 0;
    bool tma_ = false;
    bool hv2_ = false;
    std::size_t hv2_smem_ = 0;
    int segw_ = 32;
    int gmax_ = 0;
    DevArray<unsigned int> vticket_;
    bool ev2_ = false;
    const void* frh_base_ = nullptr;
    std::size_t ev2_smem_ = 0;
    alignas(64) unsigned char maps_ev2_[4 * 128];
    alignas(64) unsigned char maps_hv2_[4 * 128];
    alignas(64) unsigned char maps_hv_[4 * 128];  // TmaMaps (4 CUtensorMap)
    alignas(64) unsigned char maps_ev_[4 * 128];
    bool hv3_ = false;
    bool hv3_stored_ = false;
    bool hv16_ = false;
    TileMeta meta3_{};
    DevArray<int> goff3_[3];
    DevArray<int2> gent3_[3];
    DVec part3_;
    int slab3_[2] = {0, 0};
    int gmax3_ = 0;
    std::size_t hv3_smem_ = 0;
    alignas(64) unsigned char maps_hv3_[4 * 128];
    void setup_hv3(const DevicePlanOwner& plan, const void* R, const void* Tw, const void* dT, const void* frh, bool zok,
                   int max_optin);
    bool fp32_ = false;
    const void* state_R_ = nullptr;
    const void* state_Tw_ = nullptr;
    bool make_tma_maps(const Grid& g, const void* R, const void* Tw, const void* dT, const void* frh);
};

// Direction order of the stored coefficients: -x, +x, -y, +y, -z, +z.
constexpr int kRhoDirs = 6;

// Gauss-Newton Hv image pass: s = dT . P p -> w -> z -> q^ = 2h z dT -> P^T partials.
// (tau, rho: the NGF parameters, used when the pass recomputes the coefficients, hv3)
// [c0, c1): the z tile chunks of this launch (a z group of the two-CTA kernel; c1 < 0: all)
void launch_hv_fused(const DevicePlanOwner& plan, FusedPlan& fp, const double* frh, const double* dT, const double* p,
                     double tau, double rho, cudaStream_t s, const int* skip = nullptr, int c0 = 0, int c1 = -1);

// Eval image pass on the warped state (T_w, dT from launch_warp): rho-hat (6 per
// voxel, stored as Hv state), per-tile sums of (1 - r^2) and, when `grad`, the
// NGF gradient -2h dT (dr^T r) spread by P^T into per-tile partials.
// d_dev / d_host (optional): with the two-CTA kernel, its last CTA writes D there (returns
// true); otherwise (legacy kernel) D is left to the finalize (returns false)
// [c0, c1): z tile chunks of this launch (two-CTA kernel; the D ticket counts every group's CTAs)
bool launch_eval_fused(const DevicePlanOwner& plan, FusedPlan& fp, const double* R, const double* Tw, const double* dT,
                       double tau, double rho, double* frh, bool grad, cudaStream_t s, double* d_dev = nullptr,
                       double* d_host = nullptr, int c0 = 0, int c1 = -1);

// Nodal finalize (one launch):
//   out != null: out = gather(P^T partials) [+ add];
//   dot_a != null: sc[0] = <dot_a, out>;
//   value: sc[0] = h * sum over tiles of (1 - r^2) partials, sc[1] = alpha h^y S;
// all reductions fixed-order (last-block pattern).
struct FinalizeSpec {
    const double* add = nullptr;  // nodal term added to out (alpha * curvature gradient / Hv)
    const double* S = nullptr;    // device scalars: sum (Lap u)^2 (value), nS partial sums added in order
    int nS = 1;
    double alpha = 0.0;
    double* out = nullptr;        // nodal result
    const double* dot_a = nullptr;
    bool value = false;           // eval: D and alpha S into sc[0], sc[1]
    double* sc = nullptr;         // device scalars
    double* sc_host = nullptr;    // device view of mapped host scalars: value mode also writes D, alpha S there
    const int* skip = nullptr;    // device flag: skip the launch when set
    bool hv_pass = false;         // the partials come from the Hv pass (hv3 tiling when on)
    int nlo = -1, nhi = -1;       // nodal z planes [nlo, nhi) only (pure gathers: out without sc); -1: the plan's window
};
// cudaLaunchKernelEx with programmatic stream serialisation (MFREG_NO_PDL=1: plain launch)
bool pdl_enabled();
// (host pipeline: the z groups launch without PDL, so a group's CTAs are not placed on the SMs
// ahead of the previous group's finalize; per host thread)
bool& pdl_suspended();
bool value_pass_enabled();
template <typename... KArgs, typename... Args>
void launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, std::size_t smem, cudaStream_t s, Args&&... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() && !pdl_suspended() ? 1 : 0;
    MFREG_CUDA(cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...));
}

void launch_nodal_finalize(const DevicePlanOwner& plan, FusedPlan& fp, const FinalizeSpec& spec, cudaStream_t s);

}  // namespace mfreg_b200
