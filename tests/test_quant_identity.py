"""The division-free int8 quantizer the kernels use (csrc/quant.cuh
q8_quant4) equals the Q8row definition (DESIGN R6-R8: q = RNE(fl(x / s)),
s = fl(amax / 127)) on its whole input domain.

x is always an fp16-rounded activation and amax = max |x| of its row, so the
domain is every pair of fp16 values (x, amax) with |x| <= amax: ~1e9 pairs,
enumerated exhaustively by a small C program that restates the kernel's
arithmetic (t = x * rcp(s); r = fma(-t, s, x); q = fma(r, rcp(s), t); RNE(q)
via the 1.5 * 2^23 magic add) next to the definition (rintf(x / s)).
This checks an arithmetic identity the CUDA path relies on; it shares no code
with the oracle.
"""
import os
import shutil
import subprocess
import tempfile

import pytest

SRC = r"""
#include <stdio.h>
#include <math.h>
#include <stdint.h>
#include <string.h>
static float h2f(uint16_t h) {
  uint32_t e = (h >> 10) & 31, m = h & 1023;
  return e == 0 ? ldexpf((float)m, -24) : ldexpf((float)(m | 1024), (int)e - 25);
}
int main(void) {
  static float pos[31743];
  int np = 0;
  for (uint32_t h = 1; h < 0x7C00; ++h) pos[np++] = h2f((uint16_t)h);  /* positive finite fp16 */
  long long bad = 0, tot = 0;
  for (int ia = 0; ia < np; ++ia) {
    const float amax = pos[ia];
    const float s = amax / 127.0f;      /* R6: IEEE division */
    const float rs = 1.0f / s;          /* __frcp_rn */
    for (int ix = -1; ix <= ia; ++ix)
      for (int sg = 0; sg < 2; ++sg) {
        float x = ix < 0 ? 0.0f : pos[ix];
        if (sg) x = -x;
        const float def = rintf(x / s);  /* R8: RNE of the IEEE quotient */
        const float t = x * rs;
        const float r = fmaf(-t, s, x);
        const float q = fmaf(r, rs, t);
        const float m = q + 12582912.0f;
        uint32_t mb;
        memcpy(&mb, &m, 4);
        const int8_t k = (int8_t)(mb & 0xFF);  /* the byte the kernel stores */
        ++tot;
        if ((float)k != def || fabsf(def) > 127.0f) {
          if (bad < 5) printf("amax %a x %a def %g got %d\n", amax, x, def, k);
          ++bad;
        }
      }
  }
  printf("%lld %lld\n", tot, bad);
  return bad != 0;
}
"""


@pytest.mark.skipif(shutil.which("gcc") is None, reason="needs gcc")
def test_division_free_quantizer_exhaustive():
    with tempfile.TemporaryDirectory() as d:
        src, exe = os.path.join(d, "q.c"), os.path.join(d, "q")
        with open(src, "w") as f:
            f.write(SRC)
        # IEEE single precision, no contraction: the C statements are the
        # kernel's individual fp32 operations
        subprocess.run(["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-o", exe, src, "-lm"], check=True)
        r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
        tot, bad = map(int, r.stdout.split()[-2:])
        assert tot > 1_000_000_000 and bad == 0, r.stdout


SRC_U8 = r"""
#include <stdio.h>
#include <math.h>
#include <stdint.h>
#include <string.h>
#include <stdlib.h>
static float h2f(uint16_t h) {
  uint32_t e = (h >> 10) & 31, m = h & 1023;
  return e == 0 ? ldexpf((float)m, -24) : ldexpf((float)(m | 1024), (int)e - 25);
}
static uint64_t st = 0x9E3779B97F4A7C15ull;
static uint32_t rnd(void) { st ^= st << 13; st ^= st >> 7; st ^= st << 17; return (uint32_t)st; }
int main(void) {
  static float pos[31744];
  int np = 0;
  pos[np++] = 0.0f;
  for (uint32_t h = 1; h < 0x7C00; ++h) pos[np++] = h2f((uint16_t)h);
  long long bad = 0, tot = 0;
  for (int pair = 0; pair < 3000; ++pair) {
    /* (hi, nlo) = (max(0, max x), max(0, -min x)) of an fp16 tensor; the
       first pairs are edge cases (one side 0, equal sides, extremes) */
    int ih, il;
    if (pair < 64) { ih = pair * 491 % np; il = pair % 4 == 0 ? 0 : (pair % 4 == 1 ? ih : (np - 1 - pair)); }
    else { ih = rnd() % np; il = rnd() % np; }
    const float hi = pos[ih], nlo = pos[il];
    float sc = (hi + nlo) / 255.0f;          /* R22: IEEE division */
    if (sc == 0.0f) sc = 1.0f;
    const float zp = fminf(fmaxf(rintf(nlo / sc), 0.0f), 255.0f);
    const float rs = 1.0f / sc;              /* __frcp_rn */
    for (int ix = 0; ix < np; ++ix)
      for (int sg = 0; sg < 2; ++sg) {
        const float x = sg ? -pos[ix] : pos[ix];
        if (x > hi || -x > nlo) continue;
        const float def = fminf(fmaxf(rintf(x / sc) + zp, 0.0f), 255.0f);
        const float t = x * rs;
        const float r = fmaf(-t, sc, x);
        const float q = fmaf(r, rs, t);
        const float rn = (q + 12582912.0f) - 12582912.0f;
        const float got = fminf(fmaxf(rn + zp, 0.0f), 255.0f);
        ++tot;
        if ((uint32_t)got != (uint32_t)def) {
          if (bad < 5) printf("hi %a nlo %a x %a def %g got %g\n", hi, nlo, x, def, got);
          ++bad;
        }
      }
  }
  printf("%lld %lld\n", tot, bad);
  return bad != 0;
}
"""


@pytest.mark.skipif(shutil.which("gcc") is None, reason="needs gcc")
def test_division_free_per_tensor_u8_quantizer():
    """The per-tensor u8 quantizer (rowops.cu tensor_quant_kernel, DESIGN
    R22: q = clamp(RNE(x / scale) + zp, 0, 255)) computed without a division
    equals the definition for every fp16 x of 3000 (max, -min) range pairs
    (edge pairs first, then random), ~1e8 values."""
    with tempfile.TemporaryDirectory() as d:
        src, exe = os.path.join(d, "q.c"), os.path.join(d, "q")
        with open(src, "w") as f:
            f.write(SRC_U8)
        subprocess.run(["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-o", exe, src, "-lm"], check=True)
        r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
        tot, bad = map(int, r.stdout.split()[-2:])
        assert tot > 10_000_000 and bad == 0, r.stdout
