// tools/dmma_order.cu -- is an sm_100a FP64 MMA (mma.sync.m8n8k4 f64) a sequential fma chain over k?
// For random and adversarial inputs (cancellations, mixed magnitudes) compare the 8x8 result of one
// DMMA (D = A B + C, k = 4) bit for bit with (a) fma(a3,b3,fma(a2,b2,fma(a1,b1,fma(a0,b0,c)))) and
// (b) the same chain in descending k, (c) c + (exactly rounded dot product). Prints mismatch counts.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/dmma_order tools/dmma_order.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t rng(uint64_t& s) {
    s += 0x9e3779b97f4a7c15ull;
    uint64_t z = s;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}
__device__ double rnd(uint64_t& s, int mode) {
    const double u = (double)(rng(s) >> 11) * 0x1p-53 * 2.0 - 1.0;
    if (mode == 0) return u;
    const int e = (int)(rng(s) % 60) - 30;  // mixed magnitudes
    return ldexp(u, e);
}

__global__ void test(int trials, int mode, unsigned long long* bad) {
    const int lane = threadIdx.x & 31;
    uint64_t s = 1234567ull + 7919ull * (blockIdx.x * blockDim.x + threadIdx.x) + 104729ull * mode;
    __shared__ double A[8][4], B[4][8], C[8][8];
    unsigned long long nb[3] = {0, 0, 0};
    for (int t = 0; t < trials; ++t) {
        // lane fills part of A, B, C
        if (lane < 32) { A[lane >> 2][lane & 3] = rnd(s, mode); B[lane >> 3][lane & 7] = rnd(s, mode); }
        for (int q = lane; q < 64; q += 32) C[q >> 3][q & 7] = rnd(s, mode);
        __syncwarp();
        if (mode == 2) {  // planted cancellation: c = -(sum of products) approximately
            if (lane < 64) {
                for (int q = lane; q < 64; q += 32) {
                    const int i = q >> 3, j = q & 7;
                    double sum = 0;
                    for (int k = 0; k < 4; ++k) sum += A[i][k] * B[k][j];
                    C[i][j] = -sum * (1.0 + ldexp((double)((int)(rng(s) % 7) - 3), -50));
                }
            }
            __syncwarp();
        }
        // fragments (PTX ISA m8n8k4 f64: A row: lane -> row lane/4, col lane%4; B col: lane -> row lane%4, col lane/4;
        // C/D: lane -> row lane/4, cols 2*(lane%4), +1)
        const double a = A[lane >> 2][lane & 3];
        const double b = B[lane & 3][lane >> 2];
        const double c0 = C[lane >> 2][2 * (lane & 3)], c1 = C[lane >> 2][2 * (lane & 3) + 1];
        double d0, d1;
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%4,%5};"
                     : "=d"(d0), "=d"(d1) : "d"(a), "d"(b), "d"(c0), "d"(c1));
        const int i = lane >> 2;
        for (int h = 0; h < 2; ++h) {
            const int j = 2 * (lane & 3) + h;
            const double d = h ? d1 : d0;
            double up = C[i][j], dn = C[i][j];
            for (int k = 0; k < 4; ++k) up = __fma_rn(A[i][k], B[k][j], up);
            for (int k = 3; k >= 0; --k) dn = __fma_rn(A[i][k], B[k][j], dn);
            if (__double_as_longlong(d) != __double_as_longlong(up)) nb[0]++;
            if (__double_as_longlong(d) != __double_as_longlong(dn)) nb[1]++;
            // products summed first (pairwise, exact-ish) then added to c: a "fused dot" proxy
            double p01 = __fma_rn(A[i][1], B[1][j], A[i][0] * B[0][j]);
            double p23 = __fma_rn(A[i][3], B[3][j], A[i][2] * B[2][j]);
            double fd = (p01 + p23) + C[i][j];
            if (__double_as_longlong(d) != __double_as_longlong(fd)) nb[2]++;
        }
        __syncwarp();
    }
    for (int q = 0; q < 3; ++q) atomicAdd(bad + q, nb[q]);
}

int main() {
    unsigned long long* bad;
    cudaMalloc(&bad, 24);
    for (int mode = 0; mode < 3; ++mode) {
        cudaMemset(bad, 0, 24);
        const int trials = 2000;
        test<<<148 * 8, 32>>>(trials, mode, bad);
        unsigned long long h[3];
        cudaMemcpy(h, bad, 24, cudaMemcpyDeviceToHost);
        const double total = 148.0 * 8 * 32 * 2 * trials;
        printf("{\"mode\": %d, \"outputs\": %.0f, \"mismatch_ascending_chain\": %llu, \"mismatch_descending_chain\": %llu, \"mismatch_pairwise_dot\": %llu}\n",
               mode, total, h[0], h[1], h[2]);
    }
    return 0;
}
