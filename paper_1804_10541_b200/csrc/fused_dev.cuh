// Device-side building blocks shared by the fused fast-mode kernels (fused.cu,
// hv_fast.cu): kernel arguments, tensor maps, mbarrier / TMA wrappers.
#pragma once

#include <cuda.h>
#include <cudaTypedefs.h>

#include "fused.cuh"

namespace mfreg_b200 {
namespace fdev {

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
    int olo, ohi;       // output image planes (z slab); the tiles may extend 2 planes beyond
    int nxf, nyf;       // nodal slab footprint (max over tiles) per plane, x and y
    int dbg;            // profiling switches (0 in production)
    int segw;           // max image columns per nodal x cell (segmented-scan length)
    int frh_tma;        // eval: frh_out is the array TmaMaps::d addresses (rho-hat stored by TMA)
    const int* skip;    // device flag: return immediately when set (CG already converged)
    // eval (two-CTA kernel): when set, the last CTA to finish sums the per-tile (1 - r^2) in tile
    // order and writes D = dscale * sum to dsc[0] and the mapped host scalar dsc_host[0]
    unsigned int* vticket;  // [1 + 32] completion counters
    double* dsc;
    double* dsc_host;
    double dscale;
    int zch0;  // first z tile chunk of this launch (a pass launched in z groups; blockIdx.z + zch0)
};

struct TmaMaps {
    CUtensorMap a, b, c;  // Hv: dT, rho-hat; eval: R, T_w, dT
    CUtensorMap d;        // eval (two-CTA kernel): rho-hat output, one tile x 6 components (TMA store)
};

__device__ __forceinline__ double lerp(double t, double a, double b) { return fma(t, b - a, a); }
__device__ __forceinline__ float lerp(float t, float a, float b) { return fmaf(t, b - a, a); }

__device__ __forceinline__ unsigned smem_u32(const void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }
// shared-memory load the compiler may neither hoist nor merge (per-use reload of packed tables,
// cheaper than keeping the values live across a long loop)
__device__ __forceinline__ int lds_v(const int* p) {
    int v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(smem_u32(p)));
    return v;
}

// Programmatic dependent launch: kernels launched with launch_pdl() may start while the
// previous kernel in the stream drains; everything that reads that kernel's output must
// follow pdl_wait() (a no-op for an ordinary launch).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
// lets the next (PDL) launch in the stream be scheduled once every CTA of this grid got here
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
// wait on an mbarrier given by its shared-window address
__device__ __forceinline__ void mbar_wait_at(unsigned bar, unsigned parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tWAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(bar),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void mbar_arrive_at(unsigned bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tWAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// one elected lane of a converged warp (TMA must be issued from warp-uniform control flow)
__device__ __forceinline__ bool elect_one() {
    unsigned pred = 0;
    asm volatile(
        "{\n\t.reg .pred P;\n\t.reg .b32 r;\n\telect.sync r|P, 0xffffffff;\n\tselp.u32 %0, 1, 0, P;\n\t}"
        : "=r"(pred));
    return pred != 0;
}

__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int x, int y, int z,
                                            unsigned long long* bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::
            "r"(smem_u32(dst)),
        "l"(map), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, int x, int y, int z, int w,
                                            unsigned long long* bar) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];" ::
            "r"(smem_u32(dst)),
        "l"(map), "r"(x), "r"(y), "r"(z), "r"(w), "r"(smem_u32(bar))
        : "memory");
}

// TMA store of a shared-memory box (bulk group of the issuing thread); the writers of the box
// execute tma_store_fence() before the barrier that precedes the issue
__device__ __forceinline__ void tma_store_fence() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void tma_store_4d(const CUtensorMap* map, const void* src, int x, int y, int z, int w) {
    asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%2, %3, %4, %5}], [%1];" ::"l"(map),
                 "r"(smem_u32(src)), "r"(x), "r"(y), "r"(z), "r"(w)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
// the issuing thread's stores have finished reading shared memory / are complete
__device__ __forceinline__ void tma_store_wait_read() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void tma_store_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

}  // namespace fdev
}  // namespace mfreg_b200
