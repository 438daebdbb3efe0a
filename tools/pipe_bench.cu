// pipe_bench.cu -- issue throughput of the integer instructions the transcode
// kernels are built from (perf helper; not part of the library).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/pipe_bench tools/pipe_bench.cu
// Each thread runs 8 independent chains of one instruction kind; the result is
// warp-instructions per cycle per SM (4 = one per SMSP per cycle).
#include <cstdio>
#include <cstdint>

template <int KIND>
__device__ __forceinline__ uint32_t op(uint32_t x, uint32_t k) {
  uint32_t r;
  if (KIND == 0) asm volatile("lop3.b32 %0, %1, %2, %1, 0x96;" : "=r"(r) : "r"(x), "r"(k));
  if (KIND == 1) asm volatile("shf.r.wrap.b32 %0, %1, %1, %2;" : "=r"(r) : "r"(x), "r"(k));
  if (KIND == 2) asm volatile("mad.lo.u32 %0, %1, %2, %1;" : "=r"(r) : "r"(x), "r"(k));
  if (KIND == 3) asm volatile("mad.hi.u32 %0, %1, %2, %1;" : "=r"(r) : "r"(x), "r"(k));
  if (KIND == 4) asm volatile("prmt.b32 %0, %1, %2, 0x5140;" : "=r"(r) : "r"(x), "r"(k));
  if (KIND == 5) asm volatile("add.u32 %0, %1, %2;" : "=r"(r) : "r"(x), "r"(k));
  if (KIND == 6) asm volatile("mul.hi.u32 %0, %1, %2;" : "=r"(r) : "r"(x), "r"(k));
  if (KIND == 7) asm volatile("popc.b32 %0, %1;" : "=r"(r) : "r"(x));
  if (KIND == 8) {  // half ALU, half IMAD
    uint32_t t;
    asm volatile("lop3.b32 %0, %1, %2, %1, 0x96;" : "=r"(t) : "r"(x), "r"(k));
    asm volatile("mad.lo.u32 %0, %1, %2, %1;" : "=r"(r) : "r"(t), "r"(k));
  }
  if (KIND == 9) {  // half ALU, half IMAD.HI
    uint32_t t;
    asm volatile("lop3.b32 %0, %1, %2, %1, 0x96;" : "=r"(t) : "r"(x), "r"(k));
    asm volatile("mad.hi.u32 %0, %1, %2, %1;" : "=r"(r) : "r"(t), "r"(k));
  }
  if (KIND == 10) {  // mad.wide
    uint64_t w;
    asm volatile("mad.wide.u32 %0, %1, %2, %3;" : "=l"(w) : "r"(x), "r"(k), "l"((uint64_t)x));
    r = (uint32_t)w ^ (uint32_t)(w >> 32);
  }

  if (KIND == 11) asm volatile("add.u32 %0, %1, %2;" : "=r"(r) : "r"(x), "r"(k));
  if (KIND == 12) { uint32_t t; asm volatile("lop3.b32 %0, %1, %2, %1, 0x96;" : "=r"(t) : "r"(x), "r"(k));
                    asm volatile("add.u32 %0, %1, %2;" : "=r"(r) : "r"(t), "r"(k)); }
  if (KIND == 13) { asm volatile("{.reg .pred p; setp.lt.u32 p, %1, %2; selp.u32 %0, %1, %2, p;}" : "=r"(r) : "r"(x), "r"(k)); }
  if (KIND == 14) { uint32_t t; asm volatile("lop3.b32 %0, %1, %2, %1, 0x96;" : "=r"(t) : "r"(x), "r"(k));
                    asm volatile("mad.lo.u32 %0, %1, 16, %2;" : "=r"(r) : "r"(t), "r"(k)); }
  if (KIND == 15) { asm volatile("{.reg .u32 t; shl.b32 t, %1, 4; add.u32 %0, t, %2;}" : "=r"(r) : "r"(x), "r"(k)); }
  // shr + add: ptxas fuses into LEA.HI; alone, and beside a LOP3
  if (KIND == 16) { asm volatile("{.reg .u32 t; shr.u32 t, %1, 7; add.u32 %0, t, %2;}" : "=r"(r) : "r"(x), "r"(k)); }
  if (KIND == 17) { uint32_t t; asm volatile("lop3.b32 %0, %1, %2, %1, 0x96;" : "=r"(t) : "r"(x), "r"(k));
                    asm volatile("{.reg .u32 u; shr.u32 u, %1, 7; add.u32 %0, u, %2;}" : "=r"(r) : "r"(t), "r"(k)); }
  if (KIND == 18) asm volatile("{.reg .u32 t; shl.b32 t, %1, 8; add.u32 %0, t, %2;}" : "=r"(r) : "r"(x), "r"(k));
  if (KIND == 19) { uint32_t t; asm volatile("lop3.b32 %0, %1, %2, %1, 0x96;" : "=r"(t) : "r"(x), "r"(k));
                    asm volatile("{.reg .pred p; setp.ne.u32 p, %1, 0; selp.u32 %0, %1, %2, p;}" : "=r"(r) : "r"(t), "r"(k)); }
  if (KIND == 20) { uint32_t t; asm volatile("lop3.b32 %0, %1, %2, %1, 0x96;" : "=r"(t) : "r"(x), "r"(k));
                    asm volatile("{.reg .u32 u; add.u32 u, %1, %2; add.u32 %0, u, %1;}" : "=r"(r) : "r"(t), "r"(k)); }  // LOP3 + IADD3?
  if (KIND == 21) { asm volatile("{.reg .u32 u; add.u32 u, %1, %2; add.u32 %0, u, %1;}" : "=r"(r) : "r"(x), "r"(k)); }  // IADD3 alone
  if (KIND == 22) { uint32_t t; asm volatile("lop3.b32 %0, %1, %2, %1, 0x96;" : "=r"(t) : "r"(x), "r"(k));
                    asm volatile("{.reg .pred p; setp.ne.u32 p, %2, 0; selp.u32 %0, %1, %2, p;}" : "=r"(r) : "r"(t), "r"(k)); }  // LOP3 + SEL (fixed pred)
  if (KIND == 23) { uint32_t t; asm volatile("lop3.b32 %0, %1, %2, %1, 0x96;" : "=r"(t) : "r"(x), "r"(k));
                    asm volatile("{.reg .pred p; setp.lt.u32 p, %1, %2; @p add.u32 %0, %1, 7; @!p add.u32 %0, %1, 9;}" : "=r"(r) : "r"(t), "r"(k)); }  // LOP3 + ISETP + 2 pred add
  if (KIND == 24) { uint32_t t; asm volatile("lop3.b32 %0, %1, %2, %1, 0x96;" : "=r"(t) : "r"(x), "r"(k));
                    asm volatile("mul.hi.u32 %0, %1, 0x4000000;" : "=r"(r) : "r"(t)); }  // LOP3 + IMAD.HI as shift
  if (KIND == 25) { uint32_t t, u; asm volatile("lop3.b32 %0, %1, %2, %1, 0x96;" : "=r"(t) : "r"(x), "r"(k));
                    asm volatile("lop3.b32 %0, %1, %2, %1, 0x6a;" : "=r"(u) : "r"(t), "r"(k));
                    asm volatile("mul.hi.u32 %0, %1, 0x4000000;" : "=r"(r) : "r"(u)); }  // 2 LOP3 + 1 IMAD.HI
  if (KIND == 26) { uint32_t t; asm volatile("lop3.b32 %0, %1, %2, %1, 0x96;" : "=r"(t) : "r"(x), "r"(k));
                    asm volatile("mul.lo.u32 %0, %1, 64;" : "=r"(r) : "r"(t)); }  // LOP3 + IMAD.SHL
  if (KIND == 27) { uint32_t t; asm volatile("lop3.b32 %0, %1, %2, %1, 0x96;" : "=r"(t) : "r"(x), "r"(k));
                    asm volatile("add.u32 %0, %1, 0x1234;" : "=r"(r) : "r"(t)); }  // LOP3 + VIADD (imm)
  if (KIND == 28) { asm volatile("add.u32 %0, %1, 0x1234;" : "=r"(r) : "r"(x)); }  // VIADD alone
  if (KIND == 29) { uint32_t t; asm volatile("prmt.b32 %0, %1, %2, 0x5140;" : "=r"(t) : "r"(x), "r"(k));
                    asm volatile("mad.lo.u32 %0, %1, %2, %1;" : "=r"(r) : "r"(t), "r"(k)); }  // PRMT + IMAD
  if (KIND == 30) { uint32_t t; asm volatile("shf.r.wrap.b32 %0, %1, %1, %2;" : "=r"(t) : "r"(x), "r"(k));
                    asm volatile("mad.lo.u32 %0, %1, %2, %1;" : "=r"(r) : "r"(t), "r"(k)); }  // SHF + IMAD
  if (KIND == 31) { uint32_t t; asm volatile("lop3.b32 %0, %1, %2, %1, 0x96;" : "=r"(t) : "r"(x), "r"(k));
                    asm volatile("{.reg .pred p; setp.lt.u32 p, %1, %2; selp.u32 %0, 5, 9, p;}" : "=r"(r) : "r"(t), "r"(k)); }  // LOP3 + ISETP + SEL
  if (KIND == 32) { uint32_t t; asm volatile("lop3.b32 %0, %1, %2, %1, 0x96;" : "=r"(t) : "r"(x), "r"(k));
                    asm volatile("fma.rn.f32 %0, %1, %1, %1;" : "=f"(*(float*)&r) : "f"(__uint_as_float(t))); }  // LOP3 + FFMA
  if (KIND == 33) { uint32_t t; asm volatile("lop3.b32 %0, %1, %2, %1, 0x96;" : "=r"(t) : "r"(x), "r"(k));
                    asm volatile("{.reg .b64 w; mad.wide.u32 w, %1, %2, 0; cvt.u32.u64 %0, w;}" : "=r"(r) : "r"(t), "r"(k)); }  // LOP3 + IMAD.WIDE
  if (KIND == 34) { uint32_t t; asm volatile("lop3.b32 %0, %1, %2, %1, 0x96;" : "=r"(t) : "r"(x), "r"(k));
                    asm volatile("bfe.u32 %0, %1, 6, 6;" : "=r"(r) : "r"(t)); }  // LOP3 + BFE (what SASS?)
  if (KIND == 35) { uint32_t t, u; asm volatile("mad.lo.u32 %0, %1, %2, %1;" : "=r"(t) : "r"(x), "r"(k));
                    asm volatile("mad.lo.u32 %0, %1, %2, %1;" : "=r"(u) : "r"(t), "r"(k));
                    asm volatile("lop3.b32 %0, %1, %2, %1, 0x96;" : "=r"(r) : "r"(u), "r"(k)); }  // 2 IMAD + LOP3
  return r;
}

template <int KIND>
__global__ void kern(uint32_t* out, uint32_t k, int iters, long long* cyc) {
  uint32_t a[8];
#pragma unroll
  for (int i = 0; i < 8; i++) a[i] = threadIdx.x * 7 + i;
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int u = 0; u < 16; u++)
#pragma unroll
      for (int i = 0; i < 8; i++) a[i] = op<KIND>(a[i], KIND >= 11 ? a[(i + 1) & 7] : k);
  }
  __syncthreads();
  const long long t1 = clock64();
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < 8; i++) s ^= a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) atomicMax((unsigned long long*)cyc, (unsigned long long)(t1 - t0));
}

template <int KIND>
void run(const char* name, int opsPerStep) {
  uint32_t* out;
  long long* cyc;
  cudaMalloc(&out, 148 * 1024 * 4);
  cudaMalloc(&cyc, 8);
  const int iters = 2000;
  for (int rep = 0; rep < 2; rep++) {
    cudaMemset(cyc, 0, 8);
    kern<KIND><<<148, 1024>>>(out, 0x12345u, iters, cyc);
    cudaDeviceSynchronize();
  }
  long long c;
  cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  const double warp_inst = 32.0 /*warps*/ * iters * 16 * 8 * opsPerStep;
  printf("%-28s %.3f warp-inst/cycle/SM  (%.3f per SMSP)\n", name, warp_inst / c, warp_inst / c / 4);
  cudaFree(out);
  cudaFree(cyc);
}

int main() {
  run<0>("LOP3", 1);
  run<1>("SHF", 1);
  run<2>("IMAD", 1);
  run<3>("IMAD.HI (mad.hi)", 1);
  run<4>("PRMT", 1);
  run<5>("IADD (add.u32)", 1);
  run<6>("mul.hi", 1);
  run<7>("POPC", 1);
  run<8>("LOP3+IMAD", 2);
  run<9>("LOP3+IMAD.HI", 2);
  run<10>("mad.wide (+2 ops)", 3);
  run<11>("add (cross-chain)", 1);
  run<12>("LOP3+add", 2);
  run<13>("setp+selp", 2);
  run<14>("LOP3+mad x16 imm", 2);
  run<15>("shl4+add (LEA?)", 2);
  run<16>("shr7+add (LEA.HI)", 1);
  run<17>("LOP3+LEA.HI", 2);
  run<18>("shl8+add", 1);
  run<19>("LOP3+setp+selp", 3);
  run<20>("LOP3+IADD3", 2);
  run<21>("IADD3 alone", 1);
  run<22>("LOP3+SEL", 2);
  run<23>("LOP3+ISETP+2 pred add", 4);
  run<24>("LOP3+IMAD.HI shift", 2);
  run<25>("2 LOP3+IMAD.HI", 3);
  run<26>("LOP3+IMAD.SHL", 2);
  run<27>("LOP3+VIADD", 2);
  run<28>("VIADD alone", 1);
  run<29>("PRMT+IMAD", 2);
  run<30>("SHF+IMAD", 2);
  run<31>("LOP3+ISETP+SEL", 3);
  run<32>("LOP3+FFMA", 2);
  run<33>("LOP3+IMAD.WIDE", 2);
  run<34>("LOP3+BFE", 2);
  run<35>("2 IMAD+LOP3", 3);
  return 0;
}
