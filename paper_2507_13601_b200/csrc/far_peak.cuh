// far_peak.cuh — integer-issue microbenchmark for the roofline denominator (SURVEY.md §8(d):
// "the peak integer-issue and smem rates should be confirmed on the box with a tiny
// microbenchmark ... Do not hard-code them").  Eight independent 32-bit chains per thread,
// 16 unrolled steps per loop trip, enough warps per SMSP to cover the 4-cycle latency.
//   mode 0: alu pipe only        (shf -> SHF, xor -> LOP3; ptxas moves plain adds to the fma pipe)
//   mode 1: alu + fma pipes      (add.u32 alternating with mad.lo.u32 a*a+b -> IMAD): the issue limit
//   mode 2: shared-memory loads  (ld.shared.u32, 32 distinct banks per warp instruction)
// Each PTX instruction counts one lane-op (mode 2: 4 bytes).
#pragma once
#include <cstdint>

namespace farb {

template <int MODE>
__global__ void __launch_bounds__(1024) far_peak_kernel(unsigned* out, int iters) {
  __shared__ unsigned sm[4096];
  for (int q = threadIdx.x; q < 4096; q += blockDim.x) sm[q] = q * 2654435761u;
  __syncthreads();
  const unsigned sbase = (unsigned)__cvta_generic_to_shared(sm + (threadIdx.x & 31));
  unsigned a[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) a[c] = threadIdx.x * (c + 1) + blockIdx.x;
  const unsigned b = threadIdx.x | 1u;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        if (MODE == 0) {
          if (u & 1) asm volatile("xor.b32 %0, %0, %1;" : "+r"(a[c]) : "r"(b));
          else asm volatile("shf.l.wrap.b32 %0, %0, %0, 5;" : "+r"(a[c]));
        } else if (MODE == 1) {
          if (u & 1) asm volatile("mad.lo.u32 %0, %0, %0, %1;" : "+r"(a[c]) : "r"(b));
          else asm volatile("add.u32 %0, %0, %1;" : "+r"(a[c]) : "r"(b));
        } else {
          unsigned v;
          asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(sbase + 4u * 32u * (unsigned)(c + 8 * u)));
          a[c] ^= v;
        }
      }
    }
  }
  unsigned s = 0;
#pragma unroll
  for (int c = 0; c < 8; ++c) s ^= a[c];
  if (s == 0x12345678u) out[0] = s;  // keeps the chains live
}

}  // namespace farb
