/* gen_edgelist.c — synthetic weighted edge list for ingestion benchmarks:
 * n lines "src dst weight\n", ids from a 64-bit mix of the line index over
 * [0, 2^scale), weights U[1,5) printed with 6 decimals.
 *   gcc -O2 -o tools/gen_edgelist tools/gen_edgelist.c && tools/gen_edgelist 22 69000000 > g.txt */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

static uint64_t mix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

static char* put_u(char* p, uint64_t v) {
  char tmp[24];
  int n = 0;
  do { tmp[n++] = (char)('0' + v % 10); v /= 10; } while (v);
  while (n) *p++ = tmp[--n];
  return p;
}

int main(int argc, char** argv) {
  const int scale = argc > 1 ? atoi(argv[1]) : 22;
  const uint64_t n = argc > 2 ? strtoull(argv[2], 0, 10) : 1000000;
  const uint64_t mask = (1ull << scale) - 1;
  static char buf[1 << 20];
  char* p = buf;
  for (uint64_t i = 0; i < n; i++) {
    const uint64_t a = mix(2 * i + 1), b = mix(2 * i + 2);
    p = put_u(p, a & mask);
    *p++ = ' ';
    p = put_u(p, (a >> 32) & mask);
    *p++ = ' ';
    const uint64_t w = 1000000 + (b % 4000000);  /* 1.000000 .. 4.999999 */
    p = put_u(p, w / 1000000);
    *p++ = '.';
    char frac[6];
    uint64_t f = w % 1000000;
    for (int k = 5; k >= 0; k--) { frac[k] = (char)('0' + f % 10); f /= 10; }
    for (int k = 0; k < 6; k++) *p++ = frac[k];
    *p++ = '\n';
    if (p - buf > (1 << 20) - 64) { fwrite(buf, 1, p - buf, stdout); p = buf; }
  }
  fwrite(buf, 1, p - buf, stdout);
  return 0;
}
