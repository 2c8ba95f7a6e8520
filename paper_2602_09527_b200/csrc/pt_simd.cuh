// Packed float32x2 arithmetic for sm_100a (PTX add/sub/mul/fma .f32x2 ->
// SASS FADD2 / FMUL2 / FFMA2): two independent lanes per instruction.
#pragma once
#include <cuda_runtime.h>

namespace pt {

// Packed float32x2 arithmetic (sm_100a FFMA2 / FADD2): two Joseph samples or
// two pixels per instruction, halving the FP issue slots of the hot loops.
struct f2 {
    unsigned long long v;
};
__device__ __forceinline__ f2 pk(float a, float b)
{
    f2 r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r.v) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ void upk(f2 r, float& a, float& b)
{
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(r.v));
}
__device__ __forceinline__ f2 fma2(f2 a, f2 b, f2 c)
{
    f2 r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r.v) : "l"(a.v), "l"(b.v), "l"(c.v));
    return r;
}
__device__ __forceinline__ f2 add2(f2 a, f2 b)
{
    f2 r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r.v) : "l"(a.v), "l"(b.v));
    return r;
}
__device__ __forceinline__ f2 add2_rm(f2 a, f2 b)
{
    f2 r;
    asm("add.rm.f32x2 %0, %1, %2;" : "=l"(r.v) : "l"(a.v), "l"(b.v));
    return r;
}
__device__ __forceinline__ f2 sub2(f2 a, f2 b)
{
    f2 r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r.v) : "l"(a.v), "l"(b.v));
    return r;
}
__device__ __forceinline__ f2 mul2(f2 a, f2 b)
{
    f2 r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r.v) : "l"(a.v), "l"(b.v));
    return r;
}
__device__ __forceinline__ float lo_of(f2 a)
{
    float x, y;
    upk(a, x, y);
    return x;
}
__device__ __forceinline__ float hi_of(f2 a)
{
    float x, y;
    upk(a, x, y);
    return y;
}

}  // namespace pt
