// Scratch microbenchmark: FP32 pipe throughput per SMSP on sm_100a.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false ubench_fp.cu -o ubench_fp
#include <cstdio>
#include <cuda_runtime.h>

#define NCH 8
#define ITERS 4096

__device__ __forceinline__ unsigned long long pk(float a, float b) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}

template <int V>
__global__ void kern(float* out, float c0, float c1, float nz, long long* cyc) {
  float a[NCH], b[NCH];
  unsigned long long p[NCH], q[NCH];
  for (int i = 0; i < NCH; ++i) {
    a[i] = threadIdx.x * 1e-3f + i;
    b[i] = a[i] * 0.5f;
    p[i] = pk(a[i], b[i]);
    q[i] = pk(b[i], a[i]);
  }
  const unsigned long long cc = pk(c0, c0), zz = pk(nz, nz);
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < NCH; ++i) {
      if constexpr (V == 0) {   // FFMA reg-reg-reg
        asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(a[i]) : "f"(c0), "f"(b[i]));
      } else if constexpr (V == 1) {   // FFMA with immediate
        asm volatile("fma.rn.f32 %0, %0, 0f3F800347, %1;" : "+f"(a[i]) : "f"(b[i]));
      } else if constexpr (V == 2) {   // FFMA2
        asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(p[i]) : "l"(cc), "l"(q[i]));
      } else if constexpr (V == 3) {   // FADD2
        asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(p[i]) : "l"(q[i]));
      } else if constexpr (V == 4) {   // FMUL + FADD scalar (bit-exact tap), 2 instrs
        float t;
        asm volatile("mul.rn.f32 %0, %1, %2;" : "=f"(t) : "f"(c0), "f"(a[i]));
        asm volatile("add.rn.f32 %0, %0, %1;" : "+f"(a[i]) : "f"(t));
      } else if constexpr (V == 5) {   // FFMA2(c,u,-0) + FADD2 (paired bit-exact tap)
        unsigned long long t;
        asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(t) : "l"(cc), "l"(p[i]), "l"(zz));
        asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(p[i]) : "l"(t));
      } else if constexpr (V == 6) {   // FMUL imm + FADD
        float t;
        asm volatile("mul.rn.f32 %0, %1, 0f3F800347;" : "=f"(t) : "f"(a[i]));
        asm volatile("add.rn.f32 %0, %0, %1;" : "+f"(a[i]) : "f"(t));
      } else if constexpr (V == 7) {   // FADD scalar
        asm volatile("add.rn.f32 %0, %0, %1;" : "+f"(a[i]) : "f"(b[i]));
      } else if constexpr (V == 8) {   // FMUL scalar reg
        asm volatile("mul.rn.f32 %0, %0, %1;" : "+f"(a[i]) : "f"(c0));
      } else if constexpr (V == 9) {   // FFMA2 + IMAD.MOV-ish move (mov.b32 via integer add 0)
        asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(p[i]) : "l"(cc), "l"(q[i]));
        unsigned u = __float_as_uint(b[i]);
        asm volatile("mad.lo.u32 %0, %0, 3, 1;" : "+r"(u));
        b[i] = __uint_as_float(u);
      } else if constexpr (V == 10) {   // FFMA scalar with FADD interleave (fma-heavy + lite?)
        asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(a[i]) : "f"(c0), "f"(b[i]));
        asm volatile("add.rn.f32 %0, %0, %1;" : "+f"(b[i]) : "f"(c1));
      } else if constexpr (V == 11) {   // FMUL2 (mul.rn.f32x2)
        asm volatile("mul.rn.f32x2 %0, %0, %1;" : "+l"(p[i]) : "l"(cc));
      }
    }
  }
  long long t1 = clock64();
  float s = 0;
  for (int i = 0; i < NCH; ++i) {
    float2 u = *reinterpret_cast<float2*>(&p[i]);
    s += a[i] + b[i] + u.x + u.y;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int V>
void run(const char* name, int instr_per_inner, int warps) {
  float* out;
  long long* cyc;
  const int blocks = 148;
  cudaMalloc(&out, blocks * warps * 32 * 4);
  cudaMalloc(&cyc, blocks * 8);
  kern<V><<<blocks, warps * 32>>>(out, 1.0001f, 0.5f, -0.0f, cyc);
  cudaDeviceSynchronize();
  kern<V><<<blocks, warps * 32>>>(out, 1.0001f, 0.5f, -0.0f, cyc);
  cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < blocks; ++i) avg += h[i];
  avg /= blocks;
  // warp-instructions per SMSP per cycle
  const double winstr = (double)ITERS * NCH * instr_per_inner * warps;   // per SM
  printf("%-28s warps/SM %2d: %.3f warp-instr/clk/SMSP  (cycles %.0f)\n", name, warps, winstr / avg / 4, avg);
  cudaFree(out);
  cudaFree(cyc);
}

int main() {
  for (int w : {8, 16, 32}) {
    run<0>("FFMA rrr", 1, w);
    run<1>("FFMA imm", 1, w);
    run<2>("FFMA2", 1, w);
    run<3>("FADD2", 1, w);
    run<11>("FMUL2", 1, w);
    run<4>("FMUL+FADD scalar", 2, w);
    run<5>("FFMA2(-0)+FADD2", 2, w);
    run<6>("FMULimm+FADD", 2, w);
    run<7>("FADD", 1, w);
    run<8>("FMUL", 1, w);
    run<9>("FFMA2+IMAD", 2, w);
    run<10>("FFMA+FADD", 2, w);
  }
  return 0;
}
