// tools/smem_step_bench.cu -- latency/throughput of one accumulate "k-step" of the row kernel:
// each lane does U read-modify-writes (LDS.64, DFMA, STS.64) on a shared FP64 window, then
// __syncwarp. Variants: random vs conflict-free addresses, with/without __syncwarp, and
// warps per SM. Prints cycles per step per warp and updates per cycle per SM.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/smem_step_bench tools/smem_step_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int U, bool RANDOM, bool SYNC>
__global__ void step_kernel(const int* __restrict__ idx, int S, int steps, double a, double* out,
                            long long* cyc) {
    extern __shared__ double win[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    double* acc = win + wid * (S + 2);
    for (int j = lane; j < S; j += 32) acc[j] = 0;
    __syncwarp();
    const uint32_t base = (uint32_t)__cvta_generic_to_shared(acc);
    int off[U];
    const int* ip = idx + ((blockIdx.x * 131 + wid * 17) & 4095) * 32 * U;
#pragma unroll
    for (int u = 0; u < U; ++u) off[u] = RANDOM ? (ip[u * 32 + lane] % S) : ((u * 32 + lane) % S);
    long long t0 = clock64();
    for (int s = 0; s < steps; ++s) {
        uint32_t ad[U];
        double v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            ad[u] = base + 8u * (uint32_t)((off[u] + s * 97) % S);
            asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v[u]) : "r"(ad[u]) : "memory");
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            double r = __fma_rn(a, 1.0000001, v[u]);
            asm volatile("st.shared.f64 [%0], %1;" ::"r"(ad[u]), "d"(r) : "memory");
        }
        if (SYNC) __syncwarp();
    }
    long long t1 = clock64();
    double sum = 0;
    for (int j = lane; j < S; j += 32) sum += acc[j];
    if (sum == 1234.5) out[0] = sum;
    if (lane == 0) atomicAdd((unsigned long long*)cyc, (unsigned long long)(t1 - t0));
}

template <int U, bool RANDOM, bool SYNC>
void run(const int* idx, int S, int wps, int sms, double* out, long long* cyc) {
    const int wpc = wps < 4 ? wps : 4, ctas_per_sm = (wps + wpc - 1) / wpc;
    const size_t smem = (size_t)wpc * (S + 2) * 8;
    cudaFuncSetAttribute(step_kernel<U, RANDOM, SYNC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int steps = 2000, grid = sms * ctas_per_sm;
    cudaMemset(cyc, 0, 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    step_kernel<U, RANDOM, SYNC><<<grid, wpc * 32, smem>>>(idx, S, steps, 0.5, out, cyc);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    long long c;
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    const double warps = (double)grid * wpc;
    const double cps = (double)c / warps / steps;
    const double upd = warps * steps * 32.0 * U;
    printf("{\"U\":%d,\"random\":%d,\"sync\":%d,\"S\":%d,\"warps_per_sm\":%d,\"cycles_per_step\":%.1f,"
           "\"upd_per_clk_per_sm\":%.2f,\"Gupd_s\":%.1f,\"err\":\"%s\"}\n",
           U, (int)RANDOM, (int)SYNC, S, ctas_per_sm * wpc, cps, 32.0 * U * ctas_per_sm * wpc / cps,
           upd / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int n = 4096 * 32 * 8;
    int* h = new int[n];
    uint64_t s = 7;
    for (int i = 0; i < n; ++i) {
        s = s * 6364136223846793005ull + 1442695040888963407ull;
        h[i] = (int)(s >> 33);
    }
    int* idx;
    cudaMalloc(&idx, n * 4);
    cudaMemcpy(idx, h, n * 4, cudaMemcpyHostToDevice);
    double* out;
    long long* cyc;
    cudaMalloc(&out, 64);
    cudaMalloc(&cyc, 64);
    for (int wps : {1, 4, 8, 16}) {
        run<2, true, true>(idx, 2080, wps, sms, out, cyc);
        run<2, true, false>(idx, 2080, wps, sms, out, cyc);
        run<2, false, true>(idx, 2080, wps, sms, out, cyc);
        run<6, true, true>(idx, 2080, wps, sms, out, cyc);
        run<6, false, true>(idx, 2080, wps, sms, out, cyc);
    }
    return 0;
}
