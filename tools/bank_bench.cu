// tools/bank_bench.cu -- shared-memory 64-bit access conflict model on B200 (tuning aid).
// Each pattern gives a slot index (double) per lane; every warp issues 8 independent LDS.64
// (or STS.64) per iteration at base + 8*slot (+ a per-iteration 128-byte-aligned offset that
// keeps banks). Pipe-bound cycles per warp-instruction ~= wavefronts per instruction.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__constant__ int c_pat[32];

template <bool STORE>
__global__ void bank_kernel(int iters, double* out, long long* cyc) {
    extern __shared__ double win[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    double* w = win + wid * 1024;
    for (int j = lane; j < 1024; j += 32) w[j] = j;
    __syncwarp();
    const uint32_t base = (uint32_t)__cvta_generic_to_shared(w) + 8u * (uint32_t)c_pat[lane];
    double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const uint32_t a = base + 128u * (uint32_t)(u + 8 * (it & 3));
            if (STORE) {
                asm volatile("st.shared.f64 [%0], %1;" ::"r"(a), "d"(acc[u]) : "memory");
            } else {
                double v;
                asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a) : "memory");
                acc[u] += v;
            }
        }
    }
    long long t1 = clock64();
    double s = 0;
    for (int u = 0; u < 8; ++u) s += acc[u];
    if (s == 1234.5) out[0] = s;
    if (threadIdx.x == 0) atomicMax((unsigned long long*)cyc, (unsigned long long)(t1 - t0));
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* out;
    long long* cyc;
    cudaMalloc(&out, 64);
    cudaMalloc(&cyc, 64);
    const int wpb = 16, iters = 4000;
    const size_t smem = (size_t)wpb * 1024 * 8;
    cudaFuncSetAttribute(bank_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(bank_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    struct P { const char* name; int s[32]; };
    P pats[16];
    int np = 0;
    auto add = [&](const char* nm, auto f) { pats[np].name = nm; for (int l = 0; l < 32; ++l) pats[np].s[l] = f(l); ++np; };
    add("consecutive l", [](int l) { return l; });
    add("same bankpair 16l", [](int l) { return 16 * l; });
    add("halves distinct, pair twice (l%16 + 16*(l/16))", [](int l) { return l % 16 + 16 * (l / 16); });
    add("half0 pairs 0..7 x2, half1 pairs 8..15 x2", [](int l) { int h = l / 16, m = l % 16; return (8 * h + m / 2) + 16 * (m % 2) + 32 * h; });
    add("every pair twice, mixed halves (l/2 + 16*(l%2))", [](int l) { return (l / 2) + 16 * (l % 2); });
    add("pair = l%16, distinct addr (l + 16*(l/16)*3)", [](int l) { return (l % 16) + 16 * ((l / 16) * 3); });
    add("each pair 4x over warp (l%8 + 16*(l/8))", [](int l) { return (l % 8) + 16 * (l / 8); });
    add("only lanes 0-15 distinct pairs, 16-31 broadcast slot0", [](int l) { return l < 16 ? l : 0; });
    add("2 lanes same address per pair (l%16)", [](int l) { return l % 16; });
    add("half0 distinct; half1 all pair 0 distinct addr", [](int l) { return l < 16 ? l : 16 * (l - 15); });
    for (int st = 0; st < 2; ++st)
        for (int p = 0; p < np; ++p) {
            cudaMemcpyToSymbol(c_pat, pats[p].s, sizeof(int) * 32);
            cudaMemset(cyc, 0, 8);
            if (st) bank_kernel<true><<<sms, wpb * 32, smem>>>(iters, out, cyc);
            else bank_kernel<false><<<sms, wpb * 32, smem>>>(iters, out, cyc);
            cudaDeviceSynchronize();
            long long c;
            cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
            printf("%s %-55s cycles/warp-inst %.2f  (%s)\n", st ? "STS" : "LDS", pats[p].name,
                   (double)c / ((double)iters * 8 * wpb), cudaGetErrorString(cudaGetLastError()));
        }
    return 0;
}
