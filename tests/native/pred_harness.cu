// Host harness for the CUDA path's exact predicates (rpd_internal.cuh compiled as host code).
// stdin: lines of 4 planes "rad a0 a1 a2 a3 n0 n1 n2 rank" (x4); stdout per line:
// "det4_sign sos_sign det4_is_zero"
#include <stdio.h>
#include "../../paper_2403_18761_b200/csrc/rpd_internal.cuh"
using namespace rpd;
int main() {
  XPlane P[4];
  while (true) {
    for (int k = 0; k < 4; ++k) {
      int rad;
      if (scanf("%d %lld %lld %lld %lld %lld %lld %lld %lld", &rad, &P[k].a[0], &P[k].a[1],
                &P[k].a[2], &P[k].a[3], &P[k].n[0], &P[k].n[1], &P[k].n[2], &P[k].rank) != 9)
        return 0;
      P[k].radical = rad;
    }
    const XPlane* r[4] = {&P[0], &P[1], &P[2], &P[3]};
    int zh = 0;
    int d = det4_sign(r);
    int s = sos_sign_exact(P[0], P[1], P[2], P[3], &zh);
    int z = det4_is_zero(P[0], P[1], P[2], P[3]);
    printf("%d %d %d\n", d, s, z);
  }
}
