/* TEST INFRASTRUCTURE ONLY — part of the CPU oracle, never linked into the product.
 *
 * Correctly-rounded single-precision transcendentals for the "oracle-CR" build of the
 * reference (see oracle/Makefile) and for the C restatement in tgs_oracle.c.
 *
 * Why: the reference's float path calls glibc's expf / sincosf (rasterizer.cpp:38-39 via
 * gaussian.hpp:47-49, gaussian.hpp:72-75, rasterizer.cpp:328-331). glibc 2.39 is not
 * correctly rounded for those, and the GPU cannot reproduce glibc's
 * internal polynomial bit-for-bit. Both sides therefore agree on the contract
 * "float f(float x) = round_to_float(f_double((double)x))": the double result is accurate
 * to <1 ulp(double), so rounding it to float gives the correctly-rounded float except when
 * the exact value lies within ~2^-29 relative of a float rounding midpoint (≈4e-9 per call).
 * The GPU side (csrc/tgsx_math.cuh) evaluates exactly the same expression in FP64.
 *
 * Linked with -Wl,-Bsymbolic so calls from the reference objects inside the same .so bind
 * here instead of to libm (which the host python process has already loaded).
 */
#define _GNU_SOURCE
#include <math.h>

float expf(float x) { return (float)exp((double)x); }
float sinf(float x) { return (float)sin((double)x); }
float cosf(float x) { return (float)cos((double)x); }
void sincosf(float x, float* s, float* c) {
    *s = (float)sin((double)x);
    *c = (float)cos((double)x);
}
float logf(float x) { return (float)log((double)x); }
