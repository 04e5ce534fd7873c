#include <cstdio>
#include <cstdlib>
#include <cstdint>
#define QUALIFIERS static inline
#include <vector_types.h>
#include <curand_philox4x32_x.h>
int main(int argc, char** argv) {
  // reads lines "c0 c1 c2 c3 k0 k1" (hex) from stdin, prints 4 words
  unsigned a,b,c,d,e,f;
  while (scanf("%x %x %x %x %x %x", &a,&b,&c,&d,&e,&f) == 6) {
    uint4 ctr; ctr.x=a; ctr.y=b; ctr.z=c; ctr.w=d; uint2 key; key.x=e; key.y=f;
    uint4 o = curand_Philox4x32_10(ctr, key);
    printf("%08x %08x %08x %08x\n", o.x, o.y, o.z, o.w);
  }
}
