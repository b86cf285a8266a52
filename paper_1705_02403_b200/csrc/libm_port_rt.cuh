// Runtime of the generated libm restatements (libm_port.cuh, written by
// tools/libm_port.py): register bit-casts, the IEEE operations each machine
// instruction performs (one rounding, round to nearest even), the frame and
// the read-only tables.  Compiles as CUDA (host and device) and as plain
// C++ (the host build that tests/test_libm_port.py pins against the libm).
#pragma once
#include <cstdint>
#include <cstring>

#if defined(__CUDACC__)
// (out of line: each restated routine is a few hundred operations, called
// from several sites of one kernel)
#define LM_FN static __host__ __device__ __noinline__
#if defined(__CUDA_ARCH__)
#define LM_DATA __device__ const
#else
#define LM_DATA static const
#endif
#else
#include <cmath>
#define LM_FN static inline
#define LM_DATA static const
#endif

namespace lmport {

typedef unsigned long long u64;
typedef unsigned int u32;
typedef unsigned short u16;
typedef unsigned char u8;

constexpr int LM_STK = 128;  // frame bytes: rbp offsets -0x40 .. +0x3f
constexpr u64 LM_FRAME = 0x7ff000000000ull;  // the frame's (rbp's) address

LM_FN double lm_f(u64 b) {
  double d;
  memcpy(&d, &b, 8);
  return d;
}
LM_FN u64 lm_b(double d) {
  u64 b;
  memcpy(&b, &d, 8);
  return b;
}
#if defined(__CUDA_ARCH__)
LM_FN double lm_add(double a, double b) { return __dadd_rn(a, b); }
LM_FN double lm_sub(double a, double b) { return __dsub_rn(a, b); }
LM_FN double lm_mul(double a, double b) { return __dmul_rn(a, b); }
LM_FN double lm_div(double a, double b) { return __ddiv_rn(a, b); }
LM_FN double lm_fma(double a, double b, double c) { return __fma_rn(a, b, c); }
LM_FN double lm_sqrt(double a) { return __dsqrt_rn(a); }
#else
LM_FN double lm_add(double a, double b) { return a + b; }
LM_FN double lm_sub(double a, double b) { return a - b; }
LM_FN double lm_mul(double a, double b) { return a * b; }
LM_FN double lm_div(double a, double b) { return a / b; }
LM_FN double lm_fma(double a, double b, double c) { return std::fma(a, b, c); }
LM_FN double lm_sqrt(double a) { return std::sqrt(a); }
#endif
LM_FN double lm_nan() { return lm_f(0x7ff8000000000000ull); }

LM_FN u64 lm_stk_ld64(const unsigned char* s, long long off) {
  u64 v;
  memcpy(&v, s + off + 64, 8);
  return v;
}
LM_FN u64 lm_stk_ld32(const unsigned char* s, long long off) {
  u32 v;
  memcpy(&v, s + off + 64, 4);
  return v;
}
LM_FN void lm_stk_st64(unsigned char* s, long long off, u64 v) { memcpy(s + off + 64, &v, 8); }
LM_FN void lm_stk_st32(unsigned char* s, long long off, u64 v) {
  const u32 w = static_cast<u32>(v);
  memcpy(s + off + 64, &w, 4);
}

}  // namespace lmport

#define LM_LD64(a) lm_ld64_impl(a)
#define LM_LD32(a) lm_ld32_impl(a)
