// st_dispatch.cu -- kernel table, launch helpers, layout conversion kernels.
#include <cuda_runtime.h>

#include "st_kernels.cuh"

namespace st {

void* star_lookup_d3_r1(int, int, int);
void* star_lookup_d3_r2(int, int, int);
void* star_lookup_d3_r4(int, int, int);
void* star_lookup_d3_r8(int, int, int);
void* star_lookup_d2_r1(int, int, int);
void* star_lookup_d2_r2(int, int, int);
void* star_lookup_d2_r4(int, int, int);
void* star_lookup_d3_r2_v1(int, int, int);
void* star_lookup_d3_r2_v2(int, int, int);
void* star_lookup_d3_r2_v3(int, int, int);
void* star_lookup_d3_r4_v1(int, int, int);
void* star_lookup_d3_r4_v2(int, int, int);
void* star_lookup_d3_r4_v3(int, int, int);
void* star_lookup_d3_r4_v6(int, int, int);
void* star_lookup_d3_r4_v8(int, int, int);
void* star_lookup_d3_r4_v11(int, int, int);
void* star_lookup_d3_r8_v7(int, int, int);
void* star_lookup_d3_r2_v4(int, int, int);
void* star_lookup_d3_r2_v5(int, int, int);
void* star_lookup_d3_r2_v8(int, int, int);

static void* star_fn(int R, int dims, int model, int fast, int wf, int V = 0) {
  if (dims == 3 && V > 0) {
    if (R == 2) {
      switch (V) {
        case 1: return star_lookup_d3_r2_v1(model, fast, wf);
        case 2: return star_lookup_d3_r2_v2(model, fast, wf);
        case 3: return star_lookup_d3_r2_v3(model, fast, wf);
        case 4: return star_lookup_d3_r2_v4(model, fast, wf);
        case 5: return star_lookup_d3_r2_v5(model, fast, wf);
        case 8: return star_lookup_d3_r2_v8(model, fast, wf);
      }
      return nullptr;
    }
    if (R == 4) {
      switch (V) {
        case 1: return star_lookup_d3_r4_v1(model, fast, wf);
        case 2: return star_lookup_d3_r4_v2(model, fast, wf);
        case 3: return star_lookup_d3_r4_v3(model, fast, wf);
        case 6: return star_lookup_d3_r4_v6(model, fast, wf);
        case 8: return star_lookup_d3_r4_v8(model, fast, wf);
        case 11: return star_lookup_d3_r4_v11(model, fast, wf);
      }
    }
    if (R == 8 && V == 7) return star_lookup_d3_r8_v7(model, fast, wf);
    return nullptr;
  }
  if (dims == 3) {
    switch (R) {
      case 1: return star_lookup_d3_r1(model, fast, wf);
      case 2: return star_lookup_d3_r2(model, fast, wf);
      case 4: return star_lookup_d3_r4(model, fast, wf);
      case 8: return star_lookup_d3_r8(model, fast, wf);
    }
  } else if (dims == 2) {
    switch (R) {
      case 1: return star_lookup_d2_r1(model, fast, wf);
      case 2: return star_lookup_d2_r2(model, fast, wf);
      case 4: return star_lookup_d2_r4(model, fast, wf);
    }
  }
  return nullptr;
}

bool star_supported(int R, int dims) { return star_fn(R, dims, kTerms, 0, 0) != nullptr; }


static void* gen_fn(int model, int wf) {
  if (model == kWave) return wf ? (void*)&gen_kernel<kWave, true> : (void*)&gen_kernel<kWave, false>;
  return wf ? (void*)&gen_kernel<kTerms, true> : (void*)&gen_kernel<kTerms, false>;
}

static void* kernel_of(const LaunchCfg& lc) {
  return lc.star ? star_fn(lc.R, lc.dims, lc.model, lc.fast, lc.wf, lc.variant) : gen_fn(lc.model, lc.wf);
}

static int prep(void* fn, int smem) {
  if (!fn) return (int)cudaErrorInvalidDeviceFunction;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) {
      cudaGetLastError();   // not sticky: clear it, or the next launch check reports it
      return (int)e;
    }
  }
  return 0;
}

static dim3 block_of(const LaunchCfg& lc) {
  if (lc.star) return dim3(32 * (1 + lc.bx * lc.byt / 32 + (lc.wf ? 1 : 0)));  // producer (+ publisher)
  return dim3(lc.bx, lc.byt);
}

int launch_sweep(const LaunchCfg& lc, const KParams& p, int rel_level, void* stream) {
  void* fn = kernel_of(lc);
  int rc = prep(fn, lc.smem);
  if (rc) return rc;
  void* args[] = {(void*)&p, (void*)&rel_level};
  const int grid = lc.grid;
  cudaError_t e = cudaLaunchKernel(fn, dim3(grid), block_of(lc), args, (size_t)lc.smem, (cudaStream_t)stream);
  return (int)e;
}

int wavefront_grid(const LaunchCfg& lc, int sm_count) {
  void* fn = kernel_of(lc);
  int rc = prep(fn, lc.smem);
  if (rc) return -rc;
  int per_sm = 0;
  const dim3 b = block_of(lc);
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, b.x * b.y, lc.smem);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return -(int)e;
  }
  if (per_sm < 1) return -(int)cudaErrorInvalidConfiguration;
  return per_sm * sm_count;
}

int launch_wavefront(const LaunchCfg& lc, const KParams& p, void* stream) {
  void* fn = kernel_of(lc);
  int rc = prep(fn, lc.smem);
  if (rc) return rc;
  int zero = 0;
  void* args[] = {(void*)&p, (void*)&zero};
  cudaError_t e = cudaLaunchKernel(fn, dim3(lc.grid), block_of(lc), args, (size_t)lc.smem, (cudaStream_t)stream);
  return (int)e;
}

int launch_pipe(const LaunchCfg& lc, const KParams& p, void* stream) {
  void* fn = kernel_of(lc);
  int rc = prep(fn, lc.smem);
  if (rc) return rc;
  int zero = 0;
  void* args[] = {(void*)&p, (void*)&zero};
  cudaError_t e = cudaLaunchCooperativeKernel(fn, dim3(lc.grid), block_of(lc), args, (size_t)lc.smem,
                                              (cudaStream_t)stream);
  return (int)e;
}

FusedFn fused_lookup_d3_r1(int F, int ty, int fast, int model);
FusedFn fused_lookup_d3_r2(int F, int ty, int fast, int model);
FusedFn fused_lookup_d3_r4(int F, int ty, int fast, int model);

FusedFn fused_lookup(int R, int F, int ty, int fast, int model) {
  if (R == 1) return fused_lookup_d3_r1(F, ty, fast, model);
  if (R == 2) return fused_lookup_d3_r2(F, ty, fast, model);
  if (R == 4) return fused_lookup_d3_r4(F, ty, fast, model);
  return FusedFn{};
}

int fused_grid(const FusedFn& f, int sm_count) {
  int rc = prep(f.fn, f.smem);
  if (rc) return -rc;
  int per_sm = 0;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, f.fn, f.threads, f.smem);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return -(int)e;
  }
  if (per_sm < 1) return -(int)cudaErrorInvalidConfiguration;
  return per_sm * sm_count;
}

int launch_fused(const FusedFn& f, const KParams& p, int grid, void* stream) {
  int rc = prep(f.fn, f.smem);
  if (rc) return rc;
  void* args[] = {(void*)&p};
  return (int)cudaLaunchKernel(f.fn, dim3(grid), dim3(f.threads), args, (size_t)f.smem, (cudaStream_t)stream);
}

// ---- layout conversion ----------------------------------------------------
// Reference GridLayout (n dims, halo-padded, row-major, last contiguous) <->
// device pitched layout.  One thread per padded reference element.
struct RefMap {
  long long P[3];   // reference padded extents, 3D-embedded (leading 1s)
  int axis[3];      // device axis (0=z,1=y,2=x) of each embedded ref axis
  int R[3];         // halo of each embedded ref axis
};

static RefMap make_map(const DevGeom& g, int n, const long long* ref_padded) {
  RefMap m;
  for (int a = 0; a < 3; ++a) { m.P[a] = 1; m.axis[a] = a; m.R[a] = 0; }
  int dev_axes[3];
  if (n == 3) { dev_axes[0] = 0; dev_axes[1] = 1; dev_axes[2] = 2; }
  else if (n == 2) { dev_axes[0] = 0; dev_axes[1] = 2; }
  else { dev_axes[0] = 2; }
  const int rr[3] = {g.rz, g.ry, g.rx};
  int used[3] = {0, 0, 0};
  for (int i = 0; i < n; ++i) {
    const int a = 3 - n + i;
    m.P[a] = ref_padded[i];
    m.axis[a] = dev_axes[i];
    m.R[a] = rr[dev_axes[i]];
    used[dev_axes[i]] = 1;
  }
  // dummy embedded axes map onto the unused device axes (extent 1, halo 0)
  for (int a = 0; a < 3 - n; ++a)
    for (int d = 0; d < 3; ++d)
      if (!used[d]) { m.axis[a] = d; used[d] = 1; break; }
  return m;
}

template <bool TO_DEV>
__global__ void conv_kernel(const float* __restrict__ in, float* __restrict__ out,
                            DevGeom g, RefMap m, long long total) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    long long r = i;
    const long long p2 = r % m.P[2]; r /= m.P[2];
    const long long p1 = r % m.P[1];
    const long long p0 = r / m.P[1];
    long long dc[3] = {0, 0, 0};
    dc[m.axis[0]] = p0 - m.R[0];
    dc[m.axis[1]] = p1 - m.R[1];
    dc[m.axis[2]] = p2 - m.R[2];
    const long long d = dev_index(g, dc[0], dc[1], dc[2]);
    if (TO_DEV) out[d] = in[i];
    else out[i] = in[d];
  }
}

int launch_ref_to_dev(const float* ref, float* dev, const DevGeom& g, int n,
                      const long long* ref_padded, void* stream) {
  RefMap m = make_map(g, n, ref_padded);
  const long long total = m.P[0] * m.P[1] * m.P[2];
  conv_kernel<true><<<1184, 256, 0, (cudaStream_t)stream>>>(ref, dev, g, m, total);
  return (int)cudaGetLastError();
}

int launch_dev_to_ref(const float* dev, float* ref, const DevGeom& g, int n,
                      const long long* ref_padded, void* stream) {
  RefMap m = make_map(g, n, ref_padded);
  const long long total = m.P[0] * m.P[1] * m.P[2];
  conv_kernel<false><<<1184, 256, 0, (cudaStream_t)stream>>>(dev, ref, g, m, total);
  return (int)cudaGetLastError();
}

// Whole padded rows [r0, r1) (row = padded plane * Py + padded row) between
// the reference layout (rows of Px floats, contiguous) and the device layout
// (pitched rows, column xo - rx): one warp per row, coalesced both ways.
// Small grids: these run beside the persistent wavefront on the SMs it
// leaves free (overlapped host execute).
template <bool TO_DEV, bool HALO>
__global__ void __launch_bounds__(256) rows_kernel(const float* __restrict__ in, float* __restrict__ out, DevGeom g,
                                                   long long r0, long long r1) {
  constexpr int U = 8;   // loads in flight per lane (a 1-KB row is one round for Px <= 256)
  const long long Py = g.ny + 2 * g.ry;
  const int Px = g.nx + 2 * g.rx;
  const int lane = threadIdx.x & 31;
  const long long warps = (long long)gridDim.x * (blockDim.x >> 5);
  for (long long r = r0 + blockIdx.x * (long long)(blockDim.x >> 5) + (threadIdx.x >> 5); r < r1; r += warps) {
    const long long pz = r / Py, py = r - pz * Py;
    const float* __restrict__ src = TO_DEV ? in + r * Px : in + pz * g.pstride + py * g.pitch + (g.xo - g.rx);
    float* __restrict__ dst = TO_DEV ? out + pz * g.pstride + py * g.pitch + (g.xo - g.rx) : out + r * Px;
    if (HALO && pz >= g.rz && pz < g.rz + g.nz && py >= g.ry && py < g.ry + g.ny) {
      // interior row: only its x halo cells
      for (int i = lane; i < 2 * g.rx; i += 32) {
        const int x = i < g.rx ? i : g.nx + i;
        dst[x] = src[x];
      }
      continue;
    }
    for (int x0 = 0; x0 < Px; x0 += 32 * U) {
      float v[U];
#pragma unroll
      for (int k = 0; k < U; ++k) {
        const int x = x0 + lane + 32 * k;
        v[k] = x < Px ? src[x] : 0.f;
      }
#pragma unroll
      for (int k = 0; k < U; ++k) {
        const int x = x0 + lane + 32 * k;
        if (x < Px) dst[x] = v[k];
      }
    }
  }
}

int launch_rows(bool to_dev, const float* in, float* out, const DevGeom& g, long long z0, long long z1, int ctas,
                void* stream, bool halo_only) {
  const long long Py = g.ny + 2 * g.ry;
  cudaStream_t s = (cudaStream_t)stream;
  if (to_dev && halo_only)
    rows_kernel<true, true><<<ctas, 256, 0, s>>>(in, out, g, z0 * Py, z1 * Py);
  else if (to_dev)
    rows_kernel<true, false><<<ctas, 256, 0, s>>>(in, out, g, z0 * Py, z1 * Py);
  else
    rows_kernel<false, false><<<ctas, 256, 0, s>>>(in, out, g, z0 * Py, z1 * Py);
  return (int)cudaGetLastError();
}

__global__ void interior_kernel(const float* __restrict__ in, float* __restrict__ out,
                                DevGeom g, long long total) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const long long x = i % g.nx;
    const long long y = (i / g.nx) % g.ny;
    const long long z = i / ((long long)g.nx * g.ny);
    out[dev_index(g, z, y, x)] = in[i];
  }
}

// ---- palettized coefficient field ----------------------------------------
// A field with <= 256 distinct values (the layered velocity of configs 3 and
// 5 has 2) is also stored as 1-byte codes into a palette: the wave kernels
// then read 1 B instead of 4 B of m per point-update (m is a quarter of the
// wave's HBM traffic) and look the exact float up in shared memory.
// Discovery runs on the GPU: an open-addressing table of kPalSlots keys
// (float bits), warp-deduplicated inserts, an overflow flag past 256.
constexpr int kPalSlots = 1024;
constexpr unsigned kPalEmpty = 0xffffffffu;   // a NaN pattern; a field holding it is not palettized

__global__ void pal_build_kernel(const float* __restrict__ m, long long n, unsigned* slots, unsigned* count,
                                 unsigned* overflow) {
  unsigned last = kPalEmpty;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    if (*(volatile unsigned*)overflow) return;
    const unsigned key = __float_as_uint(m[i]);
    const unsigned same = __match_any_sync(__activemask(), key);
    if (key == last || (__ffs(same) - 1) != (int)(threadIdx.x & 31)) continue;   // one inserter per value per warp
    last = key;
    if (key == kPalEmpty) { atomicExch(overflow, 1u); return; }
    unsigned h = (key * 2654435761u) >> 22;   // 10 bits
    for (int probe = 0; probe < kPalSlots; ++probe, h = (h + 1) & (kPalSlots - 1)) {
      const unsigned prev = atomicCAS(slots + h, kPalEmpty, key);
      if (prev == key) break;
      if (prev == kPalEmpty) {
        if (atomicAdd(count, 1u) >= 256u) atomicExch(overflow, 1u);
        break;
      }
    }
  }
}

__global__ void pal_map_kernel(const float* __restrict__ m, DevGeom g, const float* __restrict__ pal, int npal,
                               unsigned char* __restrict__ codes) {
  __shared__ unsigned keys[256];
  for (int i = threadIdx.x; i < npal; i += blockDim.x) keys[i] = __float_as_uint(pal[i]);
  __syncthreads();
  const long long n = (long long)g.nz * g.ny * g.nx;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const unsigned key = __float_as_uint(m[i]);
    int lo = 0, hi = npal - 1;   // keys sorted ascending (as unsigned bits)
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (keys[mid] < key) lo = mid + 1; else hi = mid;
    }
    const long long x = i % g.nx, y = (i / g.nx) % g.ny, z = i / ((long long)g.nx * g.ny);
    codes[dev_index(g, z, y, x)] = (unsigned char)lo;
  }
}

int build_palette(const float* m_interior, const DevGeom& g, unsigned char* codes, float* pal_dev, float* pal_host,
                  int* npal, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  const long long n = (long long)g.nz * g.ny * g.nx;
  unsigned* work = nullptr;   // slots, count, overflow
  cudaError_t e = cudaMallocAsync(&work, sizeof(unsigned) * (kPalSlots + 2), st);
  if (e) return (int)e;
  e = cudaMemsetAsync(work, 0xff, sizeof(unsigned) * kPalSlots, st);
  if (!e) e = cudaMemsetAsync(work + kPalSlots, 0, 2 * sizeof(unsigned), st);
  if (!e) {
    pal_build_kernel<<<1184, 256, 0, st>>>(m_interior, n, work, work + kPalSlots, work + kPalSlots + 1);
    e = cudaGetLastError();
  }
  unsigned host[kPalSlots + 2];
  if (!e) e = cudaMemcpyAsync(host, work, sizeof(host), cudaMemcpyDeviceToHost, st);
  if (!e) e = cudaStreamSynchronize(st);
  cudaFreeAsync(work, st);
  if (e) return (int)e;
  *npal = 0;
  if (host[kPalSlots + 1] || host[kPalSlots] > 256u) return 0;   // not palettizable
  unsigned keys[256];
  int k = 0;
  for (int i = 0; i < kPalSlots; ++i)
    if (host[i] != kPalEmpty) keys[k++] = host[i];
  for (int i = 1; i < k; ++i)   // insertion sort (<= 256 keys)
    for (int j = i; j > 0 && keys[j - 1] > keys[j]; --j) { const unsigned t = keys[j]; keys[j] = keys[j - 1]; keys[j - 1] = t; }
  for (int i = 0; i < k; ++i) memcpy(pal_host + i, keys + i, 4);
  e = cudaMemcpyAsync(pal_dev, pal_host, sizeof(float) * k, cudaMemcpyHostToDevice, st);
  if (!e) {
    pal_map_kernel<<<1184, 256, 0, st>>>(m_interior, g, pal_dev, k, codes);
    e = cudaGetLastError();
  }
  if (!e) e = cudaStreamSynchronize(st);
  if (e) return (int)e;
  *npal = k;
  return 0;
}

int launch_interior_to_dev(const float* interior, float* dev, const DevGeom& g, void* stream) {
  const long long total = (long long)g.nz * g.ny * g.nx;
  interior_kernel<<<1184, 256, 0, (cudaStream_t)stream>>>(interior, dev, g, total);
  return (int)cudaGetLastError();
}

}  // namespace st
