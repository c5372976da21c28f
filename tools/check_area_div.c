#include <math.h>
#include <stdio.h>
#include <stdint.h>
// The AREA converter's division (R10: one f32 RN division of a bin sum by its pixel count): K4
// computes it as q' = fma(fma(-q, b, a), y, q) with y = RN(1/b) and q = RN(a * y) (Markstein's
// correction step).  This program checks q' == RN(a / b) for EVERY integer a < 2^18 + 1 and
// b <= 1100 (bins of at most 21 x 13 pixels of 255 fit: a <= 69615, b <= 273).  Exit code 1 on
// any mismatch.  Built and run by tests/test_oracle.py (gcc -mfma, contraction off).
int main(void) {
  long bad = 0, tot = 0;
  for (int b = 1; b <= 1100; ++b) {
    const float fb = (float)b;
    const float y = 1.0f / fb;  // correctly rounded (IEEE division)
    for (int a = 0; a <= (1 << 18); ++a) {
      const float fa = (float)a;
      const float q = fa * y;
      const float r = fmaf(-q, fb, fa);
      const float q1 = fmaf(r, y, q);
      const float ref = fa / fb;
      ++tot;
      if (q1 != ref) { if (bad < 5) printf("a=%d b=%d q1=%.9g ref=%.9g\n", a, b, q1, ref); ++bad; }
    }
  }
  printf("bad %ld of %ld\n", bad, tot);
  return bad ? 1 : 0;
}
