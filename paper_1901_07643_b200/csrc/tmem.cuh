// tmem.cuh -- sm_100a helpers shared by the walk kernels (walk_kernel.cuh: 8 workers
// per warp; walk7_kernel.cuh: 32 workers per warp): tensor-memory loads/stores
// (tcgen05.ld/st 32x32b: each lane its own TMEM lane), predicated global/shared
// stores and shared loads written in PTX so they stay predicated and ordered.
#pragma once
#include <cstdint>

namespace bnr {

// ---------------------------------------------------------------- tensor memory
__device__ __forceinline__ void tm_ld4(uint32_t a, uint32_t* r)
{
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(a));
}
__device__ __forceinline__ void tm_ld8(uint32_t a, uint32_t* r)
{
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(a));
}
__device__ __forceinline__ void tm_ld16(uint32_t a, uint32_t* r)
{
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                   "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                 : "r"(a));
}
__device__ __forceinline__ void tm_ld32(uint32_t a, uint32_t* r)
{
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                 "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                   "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
                   "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]),
                   "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]),
                   "=r"(r[30]), "=r"(r[31])
                 : "r"(a));
}
__device__ __forceinline__ void tm_st4(uint32_t a, const uint32_t* r)
{
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};" ::"r"(a), "r"(r[0]), "r"(r[1]),
                 "r"(r[2]), "r"(r[3]));
}
__device__ __forceinline__ void tm_st8(uint32_t a, const uint32_t* r)
{
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(a), "r"(r[0]),
                 "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]));
}
__device__ __forceinline__ void tm_st16(uint32_t a, const uint32_t* r)
{
    asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(a),
                 "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
                 "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]));
}
__device__ __forceinline__ void tm_st32(uint32_t a, const uint32_t* r)
{
    asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
                 "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(a),
                 "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
                 "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]),
                 "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]),
                 "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31]));
}
// N consecutive 32-bit columns of the lane's TMEM lane (N a multiple of 4)
template <int N>
__device__ __forceinline__ void tm_ld(uint32_t a, uint32_t* r)
{
    if constexpr (N >= 32) { tm_ld32(a, r); tm_ld<N - 32>(a + 32, r + 32); }
    else if constexpr (N >= 16) { tm_ld16(a, r); tm_ld<N - 16>(a + 16, r + 16); }
    else if constexpr (N >= 8) { tm_ld8(a, r); tm_ld<N - 8>(a + 8, r + 8); }
    else if constexpr (N >= 4) { tm_ld4(a, r); tm_ld<N - 4>(a + 4, r + 4); }
}
template <int N>
__device__ __forceinline__ void tm_st(uint32_t a, const uint32_t* r)
{
    if constexpr (N >= 32) { tm_st32(a, r); tm_st<N - 32>(a + 32, r + 32); }
    else if constexpr (N >= 16) { tm_st16(a, r); tm_st<N - 16>(a + 16, r + 16); }
    else if constexpr (N >= 8) { tm_st8(a, r); tm_st<N - 8>(a + 8, r + 8); }
    else if constexpr (N >= 4) { tm_st4(a, r); tm_st<N - 4>(a + 4, r + 4); }
}
// wait for the lane's outstanding tcgen05.ld.  BNREG_TM_PIN: also pin the destination
// registers behind the wait with empty asm (the front end does not know the wait defines
// them); without it -- the default since round 2, 2.5% fewer walk instructions -- the SASS
// LDTM's scoreboard orders every use of its registers behind the load (parity-tested)
template <int N>
__device__ __forceinline__ void tm_wait_ld(uint32_t* r)
{
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#ifdef BNREG_TM_PIN
#pragma unroll
    for (int q = 0; q < N; ++q) asm volatile("" : "+r"(r[q]));
#else
    (void)r;
#endif
}
// pin more destination registers behind an already issued wait
template <int N>
__device__ __forceinline__ void tm_pin(uint32_t* r)
{
#ifdef BNREG_TM_PIN
#pragma unroll
    for (int q = 0; q < N; ++q) asm volatile("" : "+r"(r[q]));
#else
    (void)r;
#endif
}
__device__ __forceinline__ void tm_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ double tm_f64(const uint32_t* r) { return __hiloint2double((int)r[1], (int)r[0]); }
__device__ __forceinline__ void tm_put(uint32_t* r, double x)
{
    r[0] = (uint32_t)__double2loint(x);
    r[1] = (uint32_t)__double2hiint(x);
}

// Predicated stores that stay predicated (no branch around them, so the
// entries of a step remain one basic block the scheduler can interleave).
// BNREG_K8 debug builds: count a violated bounds condition in k8[k8_n]
#ifdef BNREG_K8
#define K8_CHECK(L, cond)                                                                           \
    do {                                                                                            \
        if ((L).k8 && !(cond)) atomicAdd((L).k8 + (L).k8_n, 1u);                                     \
    } while (0)
#define K8_COUNT(L, ok, ix)                                                                         \
    do {                                                                                            \
        if ((L).k8 && (ok)) atomicAdd((L).k8 + ((ix) < (L).k8_n ? (unsigned long long)(ix) : (L).k8_n), 1u); \
    } while (0)
#else
#define K8_CHECK(L, cond) do { } while (0)
#define K8_COUNT(L, ok, ix) do { } while (0)
#endif

#ifndef BNREG_ST_POLICY
#define BNREG_ST_POLICY ".cs"   // the record stores' cache operator (A/B: "", ".cg", ".cs")
#endif
__device__ __forceinline__ void stg2_cs_if(double* p, double a, double b, bool q)
{
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %3, 0;\n\t@q st.global" BNREG_ST_POLICY ".v2.f64 [%0], {%1, %2};\n\t}" ::"l"(p),
                 "d"(a), "d"(b), "r"((unsigned)q));
}
__device__ __forceinline__ void stg_cs_if(double* p, double v, bool q)
{
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q st.global.cs.f64 [%0], %1;\n\t}" ::"l"(p), "d"(v),
                 "r"((unsigned)q));
}
__device__ __forceinline__ void sts_pair_if(unsigned a, double x, double u, double y, int rs, bool q)
{
    // E_i = (x, u) at a, E_{i+1}.x = y at a + rs
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %5, 0;\n\t@q st.shared.v2.f64 [%0], {%1, %2};\n\t"
                 "@q st.shared.f64 [%3], %4;\n\t}" ::"r"(a), "d"(x), "d"(u), "r"(a + rs), "d"(y), "r"((unsigned)q)
                 : "memory");
}
__device__ __forceinline__ double lds1(unsigned a)
{
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ double2 lds2(unsigned a)
{
    double2 v;
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(a));
    return v;
}

}  // namespace bnr
