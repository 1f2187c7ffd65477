// Exhaustive check of colour_avg (csrc/rf_volume.cu): floor((2n + d) / (2d)) as
// the high word of (2n + d) * ceil(2^32 / (2d)) for every colour, weight and
// input the fused update can see. gcc -O2 colour_magic.c && ./a.out
#include <stdio.h>
#include <stdint.h>
int main(){
  for (uint32_t d=1; d<=256; ++d){
    uint64_t D=2ull*d; uint32_t M=(uint32_t)(((1ull<<32)+D-1)/D);
    for (uint32_t c=0;c<=255;++c) for(uint32_t in=0; in<=255; ++in){
      uint32_t w=d-1; uint32_t num=2u*(c*w+in)+d;
      uint32_t q=(uint32_t)(((uint64_t)num*M)>>32);
      uint32_t ref=num/(2*d);
      if(q!=ref){printf("FAIL d=%u c=%u in=%u\n",d,c,in);return 1;}
    }
  }
  printf("ok\n");return 0;}
