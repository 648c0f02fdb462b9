// Probe: TMA 4D boxes of various shapes (debugging aid; not part of the library).
#include <cstdio>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include "../../paper_1804_10541_b200/csrc/fused_dev.cuh"
using namespace mfreg_b200::fdev;
__global__ void k(const __grid_constant__ TmaMaps maps, int off_b, int bytes, double* out, int nout, int variant) {
    extern __shared__ __align__(128) double sm[];
    unsigned long long& bar = *reinterpret_cast<unsigned long long*>(sm + 8000);
    if (threadIdx.x == 0) { mbar_init(&bar, 1); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
    __syncthreads();
    const bool go = variant & 1 ? (threadIdx.x < 32 && elect_one()) : threadIdx.x == 0;
    if (go) {
        mbar_expect_tx(&bar, bytes);
        tma_load_4d(sm, &maps.a, (variant & 2) ? 0 : -2, (variant & 2) ? 0 : -2, (variant & 2) ? 0 : -3, 0, &bar);
        if (!(variant & 4)) tma_load_4d(sm + off_b, &maps.b, (variant & 8) ? 0 : -1, (variant & 8) ? 0 : -1, (variant & 16) ? 0 : ((variant & 32) ? -2 : -4), 0, &bar);
    }
    mbar_wait(&bar, 0);
    for (int i = threadIdx.x; i < nout; i += blockDim.x) out[i] = sm[i];
}
int main(int argc, char** argv) {
    int bx = argc > 1 ? atoi(argv[1]) : 34, by = argc > 2 ? atoi(argv[2]) : 10;
    const int mx = 64, my = 48, mz = 40; const size_t n = (size_t)mx * my * mz;
    double *dT, *frh, *out; cudaMalloc(&dT, 3 * n * 8); cudaMalloc(&frh, 6 * n * 8); cudaMalloc(&out, 1 << 20);
    void* fn = nullptr; cudaDriverEntryPointQueryResult q{};
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    auto encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    auto enc = [&](CUtensorMap* m, double* base, cuuint64_t comps, cuuint32_t bxx, cuuint32_t byy, cuuint32_t bc) {
        const cuuint64_t dims[4] = {mx, my, mz, comps};
        const cuuint64_t strides[3] = {mx * 8ull, mx * my * 8ull, n * 8};
        const cuuint32_t box[4] = {bxx, byy, 1, bc};
        const cuuint32_t es[4] = {1, 1, 1, 1};
        return (int)encode(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    };
    TmaMaps maps{};
    int e1 = enc(&maps.a, dT, 3, 36, 12, 3), e2 = enc(&maps.b, frh, 6, bx, by, 6);
    int variant = argc > 3 ? atoi(argv[3]) : 0;
    int bytes = (36 * 12 * 3 + ((variant & 4) ? 0 : bx * by * 6)) * 8;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
    k<<<1, 128, 80000>>>(maps, 36 * 12 * 3, bytes, out, 100, variant);
    cudaError_t e = cudaDeviceSynchronize();
    printf("variant %d box %dx%d enc %d %d -> %s\n", variant, bx, by, e1, e2, cudaGetErrorString(e));
    return 0;
}
