/* TEST INFRASTRUCTURE ONLY — transcendental policy for the C oracle (tgs_oracle.c).
 *
 * mode 1 (default, "CR"): f(float x) := (float) f_double((double)x) — the contract the GPU
 *   kernels implement (see cr_libm.c for the rationale).
 * mode 0 ("native"): glibc's own expf / sinf / cosf / logf — reproduces the unmodified
 *   reference build (oracle/_ref/libtgs_ref_native.so) bit for bit.
 */
#ifndef TGS_ORACLE_CR_MATH_H
#define TGS_ORACLE_CR_MATH_H
#include <math.h>

extern int or_math_cr;

static inline float m_expf(float x) { return or_math_cr ? (float)exp((double)x) : expf(x); }
static inline float m_logf(float x) { return or_math_cr ? (float)log((double)x) : logf(x); }
static inline float m_cosf(float x) { return or_math_cr ? (float)cos((double)x) : cosf(x); }
static inline float m_sinf(float x) { return or_math_cr ? (float)sin((double)x) : sinf(x); }

#endif
