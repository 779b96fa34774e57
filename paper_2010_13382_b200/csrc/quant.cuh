// quant.cuh -- the Q8row quantizer (DESIGN R6-R8) shared by every kernel that
// emits s8 activation rows, so the result does not depend on where the
// quantizer is fused (R12):
//   scale = amax / 127 (IEEE division; 1.0 for an all-zero row)
//   q     = clamp(RNE(x / scale), -127, 127)
// x is always the fp16-rounded activation value.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "ptx.cuh"

namespace ff {

__device__ __forceinline__ float q8_scale(float amax) { return amax > 0.0f ? __fdiv_rn(amax, 127.0f) : 1.0f; }

__device__ __forceinline__ int8_t q8_quant1(float x, float s) {
  float v = rintf(__fdiv_rn(x, s));  // rintf = round-half-to-even
  v = fminf(fmaxf(v, -127.0f), 127.0f);
  return static_cast<int8_t>(static_cast<int>(v));
}

// q8_quant1 for 4 values without division or branches, packed s8x4 (byte i
// = value i), on packed fp32 pairs; rs = __frcp_rn(s).
//   t = x * rs, r = x - t * s (exact, FMA), q = t + r * rs
// is the correctly rounded quotient fl(x / s) (Markstein's correction with a
// correctly rounded reciprocal); RNE(q) is read off the 1.5 * 2^23 magic add
// (exact for |q| < 2^22), whose low mantissa byte is RNE(q) in two's
// complement.  No clamp: |q| <= 127 since |x| <= amax.  Verified against
// rintf(x / s) for every (x, amax) pair of fp16 values with |x| <= amax
// (tests/test_quant_identity.py).
__device__ __forceinline__ uint32_t q8_quant4(float2 x01, float2 x23, float s, float rs) {
  const float2 kMagic = make_float2(12582912.0f, 12582912.0f);  // 1.5 * 2^23
  const float2 r2 = make_float2(rs, rs), ns2 = make_float2(-s, -s);
  const float2 t01 = mul2(x01, r2), t23 = mul2(x23, r2);
  const float2 q01 = fma2(fma2(t01, ns2, x01), r2, t01), q23 = fma2(fma2(t23, ns2, x23), r2, t23);
  const float2 m01 = add2(q01, kMagic), m23 = add2(q23, kMagic);
  return __byte_perm(__byte_perm(__float_as_uint(m01.x), __float_as_uint(m01.y), 0x0040),
                     __byte_perm(__float_as_uint(m23.x), __float_as_uint(m23.y), 0x0040), 0x5410);
}

// Softmax normalisation p = e / l as the correctly rounded IEEE quotient
// (DESIGN R9) without a division per element: with rl = __frcp_rn(l) (once per
// row), q = e * rl, r = e - q * l (exact, FMA), p = q + r * rl (Markstein's
// correction, as in q8_quant4).  Checked against IEEE e / l on 2e7 random
// pairs e in (0, 1], l in [1, 512] (DESIGN R9); e = 0 (masked key) gives 0.
__device__ __forceinline__ float2 div2_cr(float2 e, float2 l2, float2 rl2) {
  const float2 q = mul2(e, rl2);
  const float2 r = fma2(make_float2(-q.x, -q.y), l2, e);
  return fma2(r, rl2, q);
}
__device__ __forceinline__ float div_cr(float e, float l, float rl) {
  const float q = __fmul_rn(e, rl);
  return __fmaf_rn(__fmaf_rn(-q, l, e), rl, q);
}

}  // namespace ff
