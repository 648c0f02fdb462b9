// fp64 pipe peak on this GPU (the fp64 ridge of the Hv kernel). Each thread runs
// 8 independent DFMA chains (enough ILP to cover the DFMA latency), 148 x 8 blocks of 256
// threads; flops = 2 per DFMA. Also the DADD/DMUL issue rate. Prints one JSON line.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu && ./fp64_peak
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void k_chain(double* out, int iters, double a, double b) {
    double x[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-3 + k;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            if (OP == 0) x[k] = fma(x[k], a, b);
            else if (OP == 1) x[k] = x[k] + b;
            else x[k] = x[k] * a;
        }
    }
    double s = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += x[k];
    if (s == 12345.678) out[0] = s;  // keep the chains alive
}

int main() {
    double* out;
    cudaMalloc(&out, 8);
    int dev = 0, sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
    const int iters = 1 << 14, blocks = sms * 8, threads = 256;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    double res[3];
    for (int op = 0; op < 3; ++op) {
        float best = 1e30f;
        for (int rep = 0; rep < 5; ++rep) {
            cudaEventRecord(e0);
            if (op == 0) k_chain<0><<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
            else if (op == 1) k_chain<1><<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
            else k_chain<2><<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (ms < best) best = ms;
        }
        const double ops = double(blocks) * threads * iters * 8;
        res[op] = ops / (best * 1e-3);  // instructions per second (one lane op each)
    }
    std::printf("{\"sms\": %d, \"clock_khz\": %d, \"dfma_tflops\": %.3f, \"dadd_tops\": %.3f, \"dmul_tops\": %.3f, "
                "\"dfma_per_sm_per_clk\": %.2f}\n",
                sms, clk, 2 * res[0] / 1e12, res[1] / 1e12, res[2] / 1e12, res[0] / (sms * (clk * 1e3)));
    return 0;
}
