// tools/microbench.cu -- B200 co-bound microbenchmarks for the ELLPACK X^2 roofline:
//   (1) L2-resident gather of 12 B records (8 B value + 4 B column) at random rows
//   (2) shared-memory FP64 read-modify-write at random addresses (the dense-window accumulator)
//   (3) FP64 FMA throughput (CUDA cores)
//   (4) HBM streaming write bandwidth (the output stream)
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/microbench tools/microbench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e) { printf("CUDA %s line %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__global__ void gather12(const double* __restrict__ v, const int* __restrict__ c, const int* __restrict__ rows,
                         int nrows_idx, int rowlen, int reps, double* out) {
    // each warp reads rows[k] (random), 32 consecutive records of `rowlen` (coalesced), like a B-row gather
    int lane = threadIdx.x & 31;
    long w = (blockIdx.x * (long)blockDim.x + threadIdx.x) >> 5;
    long nw = (gridDim.x * (long)blockDim.x) >> 5;
    double acc = 0;
    for (int r = 0; r < reps; ++r)
        for (long k = w; k < nrows_idx; k += nw) {
            long base = (long)rows[(k * 7 + r * 131) % nrows_idx] * rowlen;
            #pragma unroll 4
            for (int q = lane; q < rowlen; q += 32) acc += __ldg(v + base + q) * (double)__ldg(c + base + q);
        }
    if (acc == 1234.5) out[0] = acc;
}

// mode 0: random addresses (the accumulator of a sparse row: bank-pair collisions at random);
// mode 1: 32 consecutive doubles per instruction (conflict-free: 2 wavefronts per 32 lanes)
__global__ void smem_rmw(const int* __restrict__ idx, int nidx, int S, int reps, int mode, double* out) {
    extern __shared__ double win[];
    int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    double* a = win + wid * S;
    for (int j = lane; j < S; j += 32) a[j] = 0;
    __syncwarp();
    int base = (blockIdx.x * 977 + wid * 131) % (nidx - 4 * 32 * reps);
    for (int r = 0; r < reps; ++r) {
        #pragma unroll
        for (int u = 0; u < 4; ++u) {
            int j = mode ? (((r * 4 + u) * 32 + lane) & (S - 1)) : (idx[base + (r * 4 + u) * 32 + lane] % S);
            a[j] = __fma_rn(1.0000001, 0.5, a[j]);
        }
        __syncwarp();
    }
    double s = 0;
    for (int j = lane; j < S; j += 32) s += a[j];
    if (s == 1234.5) out[0] = s;
}

__global__ void fma64(int reps, double* out) {
    double a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
    const double m = 0.999999, c = 1e-7;
    for (int r = 0; r < reps; ++r) {
        a0 = __fma_rn(a0, m, c); a1 = __fma_rn(a1, m, c); a2 = __fma_rn(a2, m, c); a3 = __fma_rn(a3, m, c);
        a4 = __fma_rn(a4, m, c); a5 = __fma_rn(a5, m, c); a6 = __fma_rn(a6, m, c); a7 = __fma_rn(a7, m, c);
    }
    double s = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
    if (s == 1234.5) out[0] = s;
}

__global__ void hbm_write(double* p, long n) {
    long i = blockIdx.x * (long)blockDim.x + threadIdx.x, st = gridDim.x * (long)blockDim.x;
    for (; i < n; i += st) p[i] = (double)i;
}

int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1); float ms;
    double* out; CK(cudaMalloc(&out, 64));
    // (1) L2 gather: 8 MB-ish resident table of rows (values+cols), random row order
    for (int rowlen : {32, 128}) {
        int nrows = (8 << 20) / (12 * rowlen);
        double* v; int* c; int* rows;
        CK(cudaMalloc(&v, (size_t)nrows * rowlen * 8)); CK(cudaMalloc(&c, (size_t)nrows * rowlen * 4));
        CK(cudaMemset(v, 0, (size_t)nrows * rowlen * 8)); CK(cudaMemset(c, 0, (size_t)nrows * rowlen * 4));
        int nidx = 1 << 20; int* h = new int[nidx];
        uint64_t s = 12345; for (int i = 0; i < nidx; ++i) { s = s * 6364136223846793005ull + 1442695040888963407ull; h[i] = (int)((s >> 33) % nrows); }
        CK(cudaMalloc(&rows, nidx * 4)); CK(cudaMemcpy(rows, h, nidx * 4, cudaMemcpyHostToDevice));
        int reps = 4;
        gather12<<<sms * 8, 256>>>(v, c, rows, nidx, rowlen, 1, out);
        CK(cudaDeviceSynchronize());
        cudaEventRecord(e0);
        gather12<<<sms * 8, 256>>>(v, c, rows, nidx, rowlen, reps, out);
        cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
        double bytes = (double)reps * nidx * rowlen * 12.0;
        printf("{\"bench\":\"l2_gather12\",\"rowlen\":%d,\"GBps\":%.1f,\"ms\":%.3f}\n", rowlen, bytes / ms / 1e6, ms);
        cudaFree(v); cudaFree(c); cudaFree(rows); delete[] h;
    }
    // (2) smem random FP64 RMW, windows of S doubles per warp
    {
        int nidx = 1 << 22; int* h = new int[nidx]; uint64_t s = 99;
        for (int i = 0; i < nidx; ++i) { s = s * 6364136223846793005ull + 1442695040888963407ull; h[i] = (int)(s >> 33); }
        int* idx; CK(cudaMalloc(&idx, nidx * 4)); CK(cudaMemcpy(idx, h, nidx * 4, cudaMemcpyHostToDevice));
        for (int mode : {0, 1}) for (int S : {512, 1024, 2048, 4096}) for (int wpc : {1, 2, 4, 8}) {
            size_t smem = (size_t)wpc * S * 8;
            if (smem > 227 * 1024) continue;
            cudaFuncSetAttribute(smem_rmw, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            int bps = 0; cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, smem_rmw, wpc * 32, smem);
            if (bps < 1) continue;
            int grid = sms * bps * 4, reps = 2048;
            smem_rmw<<<grid, wpc * 32, smem>>>(idx, nidx, S, 16, mode, out); CK(cudaDeviceSynchronize());
            cudaEventRecord(e0);
            smem_rmw<<<grid, wpc * 32, smem>>>(idx, nidx, S, reps, mode, out);
            cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
            double upd = (double)grid * wpc * 32 * 4 * reps;
            printf("{\"bench\":\"smem_rmw_f64\",\"addresses\":\"%s\",\"S\":%d,\"warps_per_sm\":%d,\"Gupd_per_s\":%.1f,\"ms\":%.3f}\n",
                   mode ? "conflict_free" : "random", S, bps * wpc, upd / ms / 1e6, ms);
        }
        cudaFree(idx); delete[] h;
    }
    // (3) FP64 FMA
    {
        int reps = 1 << 14, grid = sms * 16;
        fma64<<<grid, 256>>>(16, out); CK(cudaDeviceSynchronize());
        cudaEventRecord(e0); fma64<<<grid, 256>>>(reps, out); cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
        double flops = 2.0 * 8 * reps * (double)grid * 256;
        printf("{\"bench\":\"fp64_fma\",\"TFLOPs\":%.2f,\"ms\":%.3f}\n", flops / ms / 1e9, ms);
    }
    // (4) HBM write
    {
        long n = 1L << 31; double* p; CK(cudaMalloc(&p, n * 8));
        hbm_write<<<sms * 8, 512>>>(p, n); CK(cudaDeviceSynchronize());
        cudaEventRecord(e0); hbm_write<<<sms * 8, 512>>>(p, n); cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
        printf("{\"bench\":\"hbm_write\",\"GBps\":%.1f,\"ms\":%.3f}\n", n * 8.0 / ms / 1e6, ms);
        cudaFree(p);
    }
    return 0;
}
