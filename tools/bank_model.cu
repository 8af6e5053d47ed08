// tools/bank_model.cu -- does the per-16-lane-half "most repeated bank pair" model predict the cost
// of 64-bit shared loads/stores on B200 for irregular (random) lane->slot patterns? (tuning aid)
// For each random pattern: model = sum over the two halves of max multiplicity of (slot mod 16)
// among distinct slots (same slot = broadcast); measured = pipe cycles per warp-instruction.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
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
    const int wpb = 16, iters = 2000;
    const size_t smem = (size_t)wpb * 1024 * 8;
    cudaFuncSetAttribute(bank_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(bank_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    srand(12345);
    double se_l = 0, se_s = 0;
    for (int p = 0; p < 48; ++p) {
        int s[32];
        // slots in [0, 512): a random window, distinct slots (as a B row's columns are distinct)
        for (int l = 0; l < 32; ++l) {
            for (;;) {
                s[l] = rand() % 512;
                bool dup = false;
                for (int q = 0; q < l; ++q) dup |= s[q] == s[l];
                if (!dup) break;
            }
        }
        if (p >= 32) for (int l = 0; l < 32; ++l) s[l] = 16 * (rand() % 32) + (rand() % (p - 28));  // skewed residues
        int model = 0, model_q = 0;
        for (int h = 0; h < 2; ++h) {
            int cnt[16] = {0};
            for (int l = 16 * h; l < 16 * h + 16; ++l) {
                bool seen = false;
                for (int q = 16 * h; q < l; ++q) seen |= s[q] == s[l];
                if (!seen) cnt[s[l] & 15]++;
            }
            int mx = 0;
            for (int r = 0; r < 16; ++r) mx = cnt[r] > mx ? cnt[r] : mx;
            model += mx;
        }
        for (int qq = 0; qq < 4; ++qq) {  // alternative: quarter-warp groups of 8 lanes
            int cnt[16] = {0};
            for (int l = 8 * qq; l < 8 * qq + 8; ++l) cnt[s[l] & 15]++;
            int mx = 0;
            for (int r = 0; r < 16; ++r) mx = cnt[r] > mx ? cnt[r] : mx;
            model_q += mx;
        }
        double m[2];
        for (int st = 0; st < 2; ++st) {
            cudaMemcpyToSymbol(c_pat, s, sizeof(int) * 32);
            cudaMemset(cyc, 0, 8);
            if (st) bank_kernel<true><<<sms, wpb * 32, smem>>>(iters, out, cyc);
            else bank_kernel<false><<<sms, wpb * 32, smem>>>(iters, out, cyc);
            cudaDeviceSynchronize();
            long long c;
            cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
            m[st] = (double)c / ((double)iters * 8 * wpb);
        }
        printf("pattern %2d model(halves) %2d model(quarters) %2d  LDS %.2f (x2 %.2f)  STS %.2f\n", p, model, model_q,
               m[0], 2 * m[0], m[1]);
        se_l += 2 * m[0] - model;
        se_s += m[1] - model;
    }
    printf("mean (2*LDS - model) %.3f, mean (STS - model) %.3f\n", se_l / 48, se_s / 48);
    return 0;
}
