// devutil.cuh -- small device helpers shared by the row kernels of libellpack (sm_100a):
// warp reductions, explicit 32-bit shared-memory accesses, predicated stores, L2-policy gathers.
#pragma once
#include "internal.cuh"

namespace ell {

__device__ __forceinline__ int warp_min(int v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v = min(v, __shfl_xor_sync(FULL, v, o));
    return v;
}
__device__ __forceinline__ int warp_max(int v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v = max(v, __shfl_xor_sync(FULL, v, o));
    return v;
}
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v = __dadd_rn(v, __shfl_xor_sync(FULL, v, o));
    return v;
}

// 32-bit shared-window accesses (no generic->shared conversion per access)
__device__ __forceinline__ double lds64(uint32_t a) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ void sts64(uint32_t a, double v) {
    asm volatile("st.shared.f64 [%0], %1;" ::"r"(a), "d"(v) : "memory");
}
__device__ __forceinline__ void lds128(uint32_t a, double& x, double& y) {
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(x), "=d"(y) : "r"(a) : "memory");
}
__device__ __forceinline__ void sts128(uint32_t a, double x, double y) {
    asm volatile("st.shared.v2.f64 [%0], {%1, %2};" ::"r"(a), "d"(x), "d"(y) : "memory");
}
__device__ __forceinline__ uint32_t lds8(uint32_t a) {
    uint32_t v;
    asm volatile("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ void sts8(uint32_t a, uint32_t v) {
    asm volatile("st.shared.u8 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t lds16u(uint32_t a) {
    uint32_t v;
    asm volatile("ld.shared.u16 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ void sts16u(uint32_t a, uint32_t v) {
    asm volatile("st.shared.u16 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}

// Branch-free predicated store of one output entry (value + column).
__device__ __forceinline__ void st_entry(bool pred, double* pv, int32_t* pc, double x, int32_t c) {
    asm volatile(
        "{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %0, 0;\n\t"
        "@q st.global.cs.f64 [%1], %2;\n\t@q st.global.cs.b32 [%3], %4;\n\t}" ::"r"((int)pred),
        "l"(pv), "d"(x), "l"(pc), "r"(c)
        : "memory");
}

__device__ __forceinline__ int lds32i(uint32_t a) {
    int v;
    asm volatile("ld.shared.s32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ void sts32i(uint32_t a, int v) {
    asm volatile("st.shared.s32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
// Gathers of the balanced B copy: read-only, no L1 allocation (each is used once per SM), L2
// evict_last (every record is re-read by the ~2 hB rows around it while the output stream,
// written with .cs, passes through L2).
__device__ __forceinline__ uint64_t l2_evict_last_policy() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
// predicated forms with an immediate byte offset: the address is formed once per B row
template <int OFF>
__device__ __forceinline__ void ldg_keep_i2_if(bool pr, const void* p, uint64_t pol, int2& v) {
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t"
                 "@q ld.global.nc.L1::no_allocate.L2::cache_hint.v2.s32 {%0, %1}, [%3+%5], %4;\n\t}"
                 : "+r"(v.x), "+r"(v.y) : "r"((int)pr), "l"(p), "l"(pol), "n"(OFF));
}
template <int OFF>
__device__ __forceinline__ void ldg_keep_d2_if(bool pr, const void* p, uint64_t pol, double2& v) {
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t"
                 "@q ld.global.nc.L1::no_allocate.L2::cache_hint.v2.f64 {%0, %1}, [%3+%5], %4;\n\t}"
                 : "+d"(v.x), "+d"(v.y) : "r"((int)pr), "l"(p), "l"(pol), "n"(OFF));
}
__device__ __forceinline__ int2 ldg_keep_i2(const void* p, uint64_t pol) {
    int2 v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.s32 {%0, %1}, [%2], %3;"
                 : "=r"(v.x), "=r"(v.y) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ double2 ldg_keep_d2(const void* p, uint64_t pol) {
    double2 v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;"
                 : "=d"(v.x), "=d"(v.y) : "l"(p), "l"(pol));
    return v;
}

// read-and-clear of an accumulator slot: shared 64-bit atomic exchange with +0.0
__device__ __forceinline__ double lds64_clear(uint32_t a) {
    unsigned long long v;
    asm volatile("atom.shared.exch.b64 %0, [%1], 0;" : "=l"(v) : "r"(a) : "memory");
    return __longlong_as_double((long long)v);
}

// predicated shared accesses (padding lanes issue no request and cost no wavefront)
__device__ __forceinline__ double lds64_if(bool pr, uint32_t a) {
    double v;  // undefined when !pr (the predicated store discards the result)
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %1, 0;\n\t@q ld.shared.f64 %0, [%2];\n\t}"
                 : "=d"(v) : "r"((int)pr), "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ void sts64_if(bool pr, uint32_t a, double v) {
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %0, 0;\n\t@q st.shared.f64 [%1], %2;\n\t}"
                 ::"r"((int)pr), "r"(a), "d"(v) : "memory");
}

__device__ __forceinline__ uint64_t opaque_u64(uint64_t x) {
    asm volatile("mov.b64 %0, %0;" : "+l"(x));  // keeps the row base a plain 64-bit register
    return x;
}


}  // namespace ell
