// pipe_probe.cu -- which pipe each integer instruction issues to on sm_100a,
// and at what cost (perf helper; not part of the library).  Run under
//   ncu --metrics sm__inst_executed_pipe_alu.sum,sm__inst_executed_pipe_fma.sum,
//       sm__inst_executed_pipe_fmaheavy.sum,sm__pipe_alu_cycles_active.sum,
//       sm__pipe_fma_cycles_active.sum,sm__pipe_fmaheavy_cycles_active.sum,
//       smsp__inst_executed.sum,sm__cycles_elapsed.max ./pipe_probe
// and on its own for the issue rates it prints.  Each kernel runs 8
// independent chains of one instruction per thread.
#include <cstdint>
#include <cstdio>

template <int K>
__device__ __forceinline__ void op(uint32_t& x, uint64_t& w, uint32_t k) {
  if (K == 0) asm volatile("lop3.b32 %0, %0, %1, %0, 0x96;" : "+r"(x) : "r"(k));
  if (K == 1) asm volatile("shf.r.wrap.b32 %0, %0, %0, %1;" : "+r"(x) : "r"(k));
  if (K == 2) asm volatile("prmt.b32 %0, %0, %1, 0x5140;" : "+r"(x) : "r"(k));
  if (K == 3) asm volatile("mad.lo.u32 %0, %0, %1, %0;" : "+r"(x) : "r"(k));
  if (K == 4) asm volatile("mad.hi.u32 %0, %0, %1, %0;" : "+r"(x) : "r"(k));
  if (K == 5) {  // full 64-bit product, both halves live in the chain
    asm volatile("mad.wide.u32 %0, %1, %2, %0;" : "+l"(w) : "r"(x), "r"(k));
    x = (uint32_t)(w >> 32);
  }
  if (K == 6) asm volatile("add.u32 %0, %0, %1;" : "+r"(x) : "r"(k));          // IADD / IMAD.IADD?
  if (K == 7) asm volatile("{.reg .u32 t; add.u32 t, %0, %1; add.u32 %0, t, %0;}" : "+r"(x) : "r"(k));  // IADD3
  if (K == 8) asm volatile("shl.b32 %0, %0, 5;" : "+r"(x));                     // SHF or IMAD.SHL
  if (K == 9) asm volatile("{.reg .pred p; setp.lt.u32 p, %0, %1; selp.u32 %0, %1, 7, p;}" : "+r"(x) : "r"(k));  // ISETP+SEL
  if (K == 10) asm volatile("{.reg .u32 t; shr.u32 t, %0, 7; add.u32 %0, t, %1;}" : "+r"(x) : "r"(k));  // LEA.HI
  if (K == 11) asm volatile("{.reg .u32 t; shl.b32 t, %0, 3; add.u32 %0, t, %1;}" : "+r"(x) : "r"(k));  // LEA / IMAD
  if (K == 12) asm volatile("bfe.u32 %0, %0, 6, 6;" : "+r"(x));
  if (K == 13) asm volatile("min.u32 %0, %0, %1;" : "+r"(x) : "r"(k));
  if (K == 14) asm volatile("{.reg .pred p; setp.ne.u32 p, %0, 0; @p add.u32 %0, %0, %1;}" : "+r"(x) : "r"(k));
  if (K == 15) {  // two LOP3 + one full IMAD.WIDE: does the wide multiply take ALU cycles?
    asm volatile("lop3.b32 %0, %0, %1, %0, 0x96;" : "+r"(x) : "r"(k));
    asm volatile("lop3.b32 %0, %0, %1, %0, 0x6a;" : "+r"(x) : "r"(k));
    asm volatile("mad.wide.u32 %0, %1, %2, %0;" : "+l"(w) : "r"(x), "r"(k));
    x = (uint32_t)(w >> 32);
  }
  if (K == 16) {  // two LOP3 + one IMAD.HI
    asm volatile("lop3.b32 %0, %0, %1, %0, 0x96;" : "+r"(x) : "r"(k));
    asm volatile("lop3.b32 %0, %0, %1, %0, 0x6a;" : "+r"(x) : "r"(k));
    asm volatile("mad.hi.u32 %0, %0, %1, %0;" : "+r"(x) : "r"(k));
  }
  if (K == 17) {  // two LOP3 + two IMAD
    asm volatile("lop3.b32 %0, %0, %1, %0, 0x96;" : "+r"(x) : "r"(k));
    asm volatile("lop3.b32 %0, %0, %1, %0, 0x6a;" : "+r"(x) : "r"(k));
    asm volatile("mad.lo.u32 %0, %0, %1, %0;" : "+r"(x) : "r"(k));
    asm volatile("mad.lo.u32 %0, %0, %1, 77;" : "+r"(x) : "r"(k));
  }
  if (K == 18) asm volatile("fma.rn.f32 %0, %0, %0, %0;" : "+f"(*reinterpret_cast<float*>(&x)));
  if (K == 19) {  // LOP3 + FFMA
    asm volatile("lop3.b32 %0, %0, %1, %0, 0x96;" : "+r"(x) : "r"(k));
    asm volatile("fma.rn.f32 %0, %0, %0, %0;" : "+f"(*reinterpret_cast<float*>(&x)));
  }
  if (K == 20) asm volatile("{.reg .b16 a, b; mov.b32 {a, b}, %0; mov.b32 %0, {b, a};}" : "+r"(x));  // PRMT/?
  if (K == 21) asm volatile("{.reg .b16 a, b; mov.b32 {a, b}, %0; add.u16 a, a, b; mov.b32 %0, {a, b};}" : "+r"(x));
  if (K == 22) asm volatile("vadd2.u32.u32.u32 %0, %0, %1, %0;" : "+r"(x) : "r"(k));  // VIADD2?
  if (K == 23) asm volatile("{.reg .b32 t; add.rn.f16x2 t, %0, %1; mov.b32 %0, t;}" : "+r"(x) : "r"(k));  // HADD2
}

template <int K>
__global__ void kern(uint32_t* out, uint32_t k, int iters, long long* cyc) {
  uint32_t a[8];
  uint64_t w[8];
#pragma unroll
  for (int i = 0; i < 8; i++) {
    a[i] = threadIdx.x * 7 + i + k;
    w[i] = a[i];
  }
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int u = 0; u < 8; u++)
#pragma unroll
      for (int i = 0; i < 8; i++) op<K>(a[i], w[i], k + i);
  }
  __syncthreads();
  const long long t1 = clock64();
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < 8; i++) s ^= a[i] ^ (uint32_t)w[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) atomicMax((unsigned long long*)cyc, (unsigned long long)(t1 - t0));
}

static const char* kNames[] = {"LOP3", "SHF", "PRMT", "IMAD", "IMAD.HI", "IMAD.WIDE(hi+lo)", "add", "add3",
                               "shl5", "setp+selp", "shr7+add", "shl3+add", "bfe", "min", "setp+@p add",
                               "2LOP3+IMAD.WIDE", "2LOP3+IMAD.HI", "2LOP3+2IMAD", "FFMA", "LOP3+FFMA",
                               "swap halves", "add.u16", "vadd2", "hadd2"};
static const int kOps[] = {1, 1, 1, 1, 1, 1, 1, 2, 1, 2, 2, 2, 1, 1, 2, 3, 3, 4, 1, 2, 1, 3, 1, 1};

template <int K>
void run() {
  uint32_t* out;
  long long* cyc;
  cudaMalloc(&out, 148 * 1024 * 4);
  cudaMalloc(&cyc, 8);
  const int iters = 1000;
  cudaMemset(cyc, 0, 8);
  kern<K><<<148, 1024>>>(out, 0x12345u, iters, cyc);
  cudaDeviceSynchronize();
  long long c;
  cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  const double warp_steps = 32.0 * iters * 8 * 8;  // per SM: 32 warps x steps
  printf("%2d %-22s %.3f cycles per step per SMSP (%.3f instr/cycle/SMSP at %d ops/step)\n", K, kNames[K],
         c / (warp_steps / 4), warp_steps / 4 * kOps[K] / c, kOps[K]);
  cudaFree(out);
  cudaFree(cyc);
}

template <int... Ks>
void run_all(std::integer_sequence<int, Ks...>) {
  (run<Ks>(), ...);
}

int main() {
  run_all(std::make_integer_sequence<int, 24>{});
  return 0;
}
