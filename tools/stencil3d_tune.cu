// stencil3d_tune.cu — standalone timing of fp32 3-D 7-point designs on 1024^3
// (configs[4] 3-D half); not part of the library.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                  \
  do {                                                                         \
    cudaError_t e = (x);                                                       \
    if (e != cudaSuccess) {                                                    \
      printf("CUDA %s at line %d\n", cudaGetErrorString(e), __LINE__);         \
      exit(1);                                                                 \
    }                                                                          \
  } while (0)

// register z-march; y neighbours: plain loads (L1) ; UNZ planes per iteration
template <int BY, int ZCH, int MINB>
__global__ void __launch_bounds__(32 * BY, MINB) k_march(const float* __restrict__ in, float* __restrict__ out, long n1,
                                                         long n2, long z0, long z1, long y0, long y1, long x0, long x1) {
  const int lane = threadIdx.x;
  const long x = ((long)blockIdx.x * 32 + lane) * 4;
  const long y = y0 + (long)blockIdx.y * BY + threadIdx.y;
  if (y >= y1) return;
  const bool live = x < n2;
  const long zs = z0 + (long)blockIdx.z * ZCH, ze = min(zs + (long)ZCH, z1);
  const long pl = n1 * n2;
  auto ld = [&](float4& r, long z, long yy) {
    r = live ? __ldg(reinterpret_cast<const float4*>(in + z * pl + yy * n2 + x)) : make_float4(0, 0, 0, 0);
  };
  float4 zm, zc, zp, ym, yp;
  ld(zm, zs - 1, y);
  ld(zc, zs, y);
  for (long z = zs; z < ze; z++) {
    ld(zp, z + 1, y);
    ld(ym, z, y - 1);
    ld(yp, z, y + 1);
    float L = __shfl_up_sync(0xffffffffu, zc.w, 1);
    float R = __shfl_down_sync(0xffffffffu, zc.x, 1);
    const float* row = in + z * pl + y * n2 + x;
    if (lane == 0 && live && x > 0) L = __ldg(row - 1);
    if (lane == 31 && live && x + 4 < n2) R = __ldg(row + 4);
    float o[4];
    const float c[4] = {zc.x, zc.y, zc.z, zc.w}, m[4] = {ym.x, ym.y, ym.z, ym.w}, p[4] = {yp.x, yp.y, yp.z, yp.w},
                a[4] = {zm.x, zm.y, zm.z, zm.w}, b[4] = {zp.x, zp.y, zp.z, zp.w};
#pragma unroll
    for (int v = 0; v < 4; v++) {
      float s = (v == 0 ? L : c[v - 1]) + (v == 3 ? R : c[v + 1]);
      s = s + m[v];
      s = s + p[v];
      s = s + a[v];
      s = s + b[v];
      o[v] = s / 6.0f;
    }
    if (live) {
      float* d = out + z * pl + y * n2 + x;
      if (x >= x0 && x + 4 <= x1)
        *reinterpret_cast<float4*>(d) = make_float4(o[0], o[1], o[2], o[3]);
      else
        for (int v = 0; v < 4; v++)
          if (x + v >= x0 && x + v < x1) d[v] = o[v];
    }
    zm = zc;
    zc = zp;
  }
}

// z-window: G planes loaded together (G loads in flight per thread, like the 2-D kernel)
template <int BY, int ZCH, int G, int MINB>
__global__ void __launch_bounds__(32 * BY, MINB) k_win(const float* __restrict__ in, float* __restrict__ out, long n1,
                                                       long n2, long z0, long z1, long y0, long y1, long x0, long x1) {
  const int lane = threadIdx.x;
  const long x = ((long)blockIdx.x * 32 + lane) * 4;
  const long y = y0 + (long)blockIdx.y * BY + threadIdx.y;
  if (y >= y1) return;
  const bool live = x < n2;
  const long zs = z0 + (long)blockIdx.z * ZCH, ze = min(zs + (long)ZCH, z1);
  const long pl = n1 * n2;
  auto ld = [&](float4& r, long z, long yy) {
    r = live ? __ldg(reinterpret_cast<const float4*>(in + z * pl + yy * n2 + x)) : make_float4(0, 0, 0, 0);
  };
  float4 w[G + 2];
  ld(w[0], zs - 1, y);
  ld(w[1], zs, y);
  for (long base = zs; base < ze; base += G) {
#pragma unroll
    for (int k = 0; k < G; k++)
      if (base + 1 + k <= ze) ld(w[k + 2], base + 1 + k, y);
#pragma unroll
    for (int k = 0; k < G; k++) {
      const long z = base + k;
      if (z >= ze) break;
      float4 ym, yp;
      ld(ym, z, y - 1);
      ld(yp, z, y + 1);
      const float4 zc = w[k + 1], zm = w[k], zp = w[k + 2];
      float L = __shfl_up_sync(0xffffffffu, zc.w, 1);
      float R = __shfl_down_sync(0xffffffffu, zc.x, 1);
      const float* row = in + z * pl + y * n2 + x;
      if (lane == 0 && live && x > 0) L = __ldg(row - 1);
      if (lane == 31 && live && x + 4 < n2) R = __ldg(row + 4);
      const float c[4] = {zc.x, zc.y, zc.z, zc.w}, m[4] = {ym.x, ym.y, ym.z, ym.w}, p[4] = {yp.x, yp.y, yp.z, yp.w},
                  a[4] = {zm.x, zm.y, zm.z, zm.w}, b[4] = {zp.x, zp.y, zp.z, zp.w};
      float o[4];
#pragma unroll
      for (int v = 0; v < 4; v++) {
        float s = (v == 0 ? L : c[v - 1]) + (v == 3 ? R : c[v + 1]);
        s = s + m[v];
        s = s + p[v];
        s = s + a[v];
        s = s + b[v];
        o[v] = s / 6.0f;
      }
      if (live) {
        float* d = out + z * pl + y * n2 + x;
        if (x >= x0 && x + 4 <= x1)
          *reinterpret_cast<float4*>(d) = make_float4(o[0], o[1], o[2], o[3]);
        else
          for (int v = 0; v < 4; v++)
            if (x + v >= x0 && x + v < x1) d[v] = o[v];
      }
    }
    w[0] = w[G];
    w[1] = w[G + 1];
  }
}

// "rows": 8 warps span 1024 contiguous floats of a row (4 KB DRAM bursts); each thread
// owns R consecutive y rows (y neighbours inside come from registers, only y-1 and
// y+R are extra loads), marching z.
template <int R, int ZCH, int MINB>
__global__ void __launch_bounds__(256, MINB) k_rows(const float* __restrict__ in, float* __restrict__ out, long n1,
                                                    long n2, long z0, long z1, long y0, long y1, long x0, long x1) {
  const int lane = threadIdx.x & 31;
  const long x = ((long)blockIdx.x * 256 + threadIdx.x) * 4;
  const long ya = y0 + (long)blockIdx.y * R;  // first row of this thread
  const bool live = x < n2;
  const long zs = z0 + (long)blockIdx.z * ZCH, ze = min(zs + (long)ZCH, z1);
  const long pl = n1 * n2;
  auto ld = [&](long z, long yy) -> float4 {
    return (live && yy < n1) ? __ldg(reinterpret_cast<const float4*>(in + z * pl + yy * n2 + x))
                             : make_float4(0, 0, 0, 0);
  };
  float4 zm[R], zc[R], zp[R];
#pragma unroll
  for (int r = 0; r < R; r++) {
    zm[r] = ld(zs - 1, ya + r);
    zc[r] = ld(zs, ya + r);
  }
  for (long z = zs; z < ze; z++) {
    float4 top = ld(z, ya - 1), bot = ld(z, ya + R);
#pragma unroll
    for (int r = 0; r < R; r++) zp[r] = ld(z + 1, ya + r);
#pragma unroll
    for (int r = 0; r < R; r++) {
      const long y = ya + r;
      const float4 c = zc[r];
      const float4 ym = r == 0 ? top : zc[r - 1];
      const float4 yp = r == R - 1 ? bot : zc[r + 1];
      float L = __shfl_up_sync(0xffffffffu, c.w, 1);
      float Rr = __shfl_down_sync(0xffffffffu, c.x, 1);
      const float* row = in + z * pl + y * n2 + x;
      if (lane == 0 && live && x > 0 && y < y1) L = __ldg(row - 1);
      if (lane == 31 && live && x + 4 < n2 && y < y1) Rr = __ldg(row + 4);
      const float cc[4] = {c.x, c.y, c.z, c.w}, m[4] = {ym.x, ym.y, ym.z, ym.w}, p[4] = {yp.x, yp.y, yp.z, yp.w},
                  a[4] = {zm[r].x, zm[r].y, zm[r].z, zm[r].w}, b[4] = {zp[r].x, zp[r].y, zp[r].z, zp[r].w};
      float o[4];
#pragma unroll
      for (int v = 0; v < 4; v++) {
        float s = (v == 0 ? L : cc[v - 1]) + (v == 3 ? Rr : cc[v + 1]);
        s = s + m[v];
        s = s + p[v];
        s = s + a[v];
        s = s + b[v];
        o[v] = s / 6.0f;
      }
      if (live && y < y1) {
        float* d = out + z * pl + y * n2 + x;
        if (x >= x0 && x + 4 <= x1)
          *reinterpret_cast<float4*>(d) = make_float4(o[0], o[1], o[2], o[3]);
        else
          for (int v = 0; v < 4; v++)
            if (x + v >= x0 && x + v < x1) d[v] = o[v];
      }
    }
#pragma unroll
    for (int r = 0; r < R; r++) {
      zm[r] = zc[r];
      zc[r] = zp[r];
    }
  }
}

// "rows" + software pipelining: the loads of plane z+1's y halos and of plane z+2 are
// issued one iteration ahead, so each iteration's arithmetic overlaps the next loads.
template <int R, int ZCH, int MINB>
__global__ void __launch_bounds__(256, MINB) k_rowsp(const float* __restrict__ in, float* __restrict__ out, long n1,
                                                     long n2, long z0, long z1, long y0, long y1, long x0, long x1) {
  const int lane = threadIdx.x & 31;
  const long x = ((long)blockIdx.x * 256 + threadIdx.x) * 4;
  const long ya = y0 + (long)blockIdx.y * R;
  const bool live = x < n2;
  const long zs = z0 + (long)blockIdx.z * ZCH, ze = min(zs + (long)ZCH, z1);
  const long pl = n1 * n2;
  auto ld = [&](long z, long yy) -> float4 {
    return (live && yy < n1) ? __ldg(reinterpret_cast<const float4*>(in + z * pl + yy * n2 + x))
                             : make_float4(0, 0, 0, 0);
  };
  float4 zm[R], zc[R], zp[R];
#pragma unroll
  for (int r = 0; r < R; r++) {
    zm[r] = ld(zs - 1, ya + r);
    zc[r] = ld(zs, ya + r);
    zp[r] = ld(zs + 1, ya + r);
  }
  float4 top = ld(zs, ya - 1), bot = ld(zs, ya + R);
  for (long z = zs; z < ze; z++) {
    // next iteration's loads first
    float4 zn[R], topn, botn;
    const bool more = z + 1 < ze;
    if (more) {
#pragma unroll
      for (int r = 0; r < R; r++) zn[r] = ld(z + 2, ya + r);
      topn = ld(z + 1, ya - 1);
      botn = ld(z + 1, ya + R);
    }
#pragma unroll
    for (int r = 0; r < R; r++) {
      const long y = ya + r;
      const float4 c = zc[r];
      const float4 ym = r == 0 ? top : zc[r - 1];
      const float4 yp = r == R - 1 ? bot : zc[r + 1];
      float L = __shfl_up_sync(0xffffffffu, c.w, 1);
      float Rr = __shfl_down_sync(0xffffffffu, c.x, 1);
      const float* row = in + z * pl + y * n2 + x;
      if (lane == 0 && live && x > 0 && y < y1) L = __ldg(row - 1);
      if (lane == 31 && live && x + 4 < n2 && y < y1) Rr = __ldg(row + 4);
      const float cc[4] = {c.x, c.y, c.z, c.w}, m[4] = {ym.x, ym.y, ym.z, ym.w}, p[4] = {yp.x, yp.y, yp.z, yp.w},
                  a[4] = {zm[r].x, zm[r].y, zm[r].z, zm[r].w}, b[4] = {zp[r].x, zp[r].y, zp[r].z, zp[r].w};
      float o[4];
#pragma unroll
      for (int v = 0; v < 4; v++) {
        float s = (v == 0 ? L : cc[v - 1]) + (v == 3 ? Rr : cc[v + 1]);
        s = s + m[v];
        s = s + p[v];
        s = s + a[v];
        s = s + b[v];
        o[v] = s / 6.0f;
      }
      if (live && y < y1) {
        float* d = out + z * pl + y * n2 + x;
        if (x >= x0 && x + 4 <= x1)
          *reinterpret_cast<float4*>(d) = make_float4(o[0], o[1], o[2], o[3]);
        else
          for (int v = 0; v < 4; v++)
            if (x + v >= x0 && x + v < x1) d[v] = o[v];
      }
    }
    if (more) {
#pragma unroll
      for (int r = 0; r < R; r++) {
        zm[r] = zc[r];
        zc[r] = zp[r];
        zp[r] = zn[r];
      }
      top = topn;
      bot = botn;
    }
  }
}

// shared-memory plane tiles: the block's (BY+2) rows of plane z are staged in smem
// (double-buffered, one barrier per plane); y neighbours come from smem
template <int BY, int ZCH>
__global__ void __launch_bounds__(32 * BY) k_smem(const float* __restrict__ in, float* __restrict__ out, long n1,
                                                  long n2, long z0, long z1, long y0, long y1, long x0, long x1) {
  __shared__ float4 tile[2][BY + 2][32];
  const int lane = threadIdx.x, ty = threadIdx.y;
  const long x = ((long)blockIdx.x * 32 + lane) * 4;
  const long ybase = y0 + (long)blockIdx.y * BY;
  const long y = ybase + ty;
  const bool live = x < n2;
  const long zs = z0 + (long)blockIdx.z * ZCH, ze = min(zs + (long)ZCH, z1);
  const long pl = n1 * n2;
  auto g = [&](long z, long yy) -> float4 {
    return (live && yy < n1) ? __ldg(reinterpret_cast<const float4*>(in + z * pl + yy * n2 + x))
                             : make_float4(0, 0, 0, 0);
  };
  auto stage = [&](int buf, long z) {
    tile[buf][ty + 1][lane] = g(z, y);
    if (ty == 0) tile[buf][0][lane] = g(z, ybase - 1);
    if (ty == BY - 1) tile[buf][BY + 1][lane] = g(z, ybase + BY);
  };
  float4 zm = g(zs - 1, y);
  stage(0, zs);
  float4 nxt = g(zs + 1, y);
  __syncthreads();
  for (long z = zs; z < ze; z++) {
    const int b = (int)((z - zs) & 1);
    // prefetch plane z+1 into the other buffer (its own row is nxt)
    tile[b ^ 1][ty + 1][lane] = nxt;
    if (ty == 0) tile[b ^ 1][0][lane] = g(z + 1, ybase - 1);
    if (ty == BY - 1) tile[b ^ 1][BY + 1][lane] = g(z + 1, ybase + BY);
    float4 zp = nxt;
    if (z + 2 <= ze) nxt = g(z + 2, y);
    const float4 zc = tile[b][ty + 1][lane], ym = tile[b][ty][lane], yp = tile[b][ty + 2][lane];
    float L = __shfl_up_sync(0xffffffffu, zc.w, 1);
    float R = __shfl_down_sync(0xffffffffu, zc.x, 1);
    const float* row = in + z * pl + y * n2 + x;
    if (lane == 0 && live && x > 0 && y < y1) L = __ldg(row - 1);
    if (lane == 31 && live && x + 4 < n2 && y < y1) R = __ldg(row + 4);
    const float c[4] = {zc.x, zc.y, zc.z, zc.w}, m[4] = {ym.x, ym.y, ym.z, ym.w}, p[4] = {yp.x, yp.y, yp.z, yp.w},
                a[4] = {zm.x, zm.y, zm.z, zm.w}, bb[4] = {zp.x, zp.y, zp.z, zp.w};
    float o[4];
#pragma unroll
    for (int v = 0; v < 4; v++) {
      float s = (v == 0 ? L : c[v - 1]) + (v == 3 ? R : c[v + 1]);
      s = s + m[v];
      s = s + p[v];
      s = s + a[v];
      s = s + bb[v];
      o[v] = s / 6.0f;
    }
    if (live && y < y1) {
      float* d = out + z * pl + y * n2 + x;
      if (x >= x0 && x + 4 <= x1)
        *reinterpret_cast<float4*>(d) = make_float4(o[0], o[1], o[2], o[3]);
      else
        for (int v = 0; v < 4; v++)
          if (x + v >= x0 && x + v < x1) d[v] = o[v];
    }
    zm = zc;
    __syncthreads();
  }
}

int main() {
  const long n = 1024;
  const size_t bytes = n * n * n * 4;
  float *X, *Y, *R;
  CK(cudaMalloc(&X, bytes));
  CK(cudaMalloc(&Y, bytes));
  CK(cudaMalloc(&R, bytes));
  std::vector<float> h(n * n * n);
  for (long i = 0; i < n * n * n; i++) h[i] = (float)((i * 2654435761u) % 1000) / 1000.0f;
  CK(cudaMemcpy(X, h.data(), bytes, cudaMemcpyHostToDevice));
  const long lo = 1, hi = n - 1;
  const double alg = (double)(hi - lo) * (hi - lo) * (hi - lo) * 8;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  std::vector<float> o(n * n * n), ref(n * n * n);
  auto time_it = [&](const char* name, auto launch, bool is_ref) {
    CK(cudaMemset(Y, 0, bytes));
    for (int i = 0; i < 3; i++) launch();
    CK(cudaDeviceSynchronize());
    const int it = 20;
    cudaEventRecord(a);
    for (int i = 0; i < it; i++) launch();
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double us = ms * 1e3 / it;
    long bad = 0;
    if (is_ref) {
      CK(cudaMemcpy(R, Y, bytes, cudaMemcpyDeviceToDevice));
    } else {
      CK(cudaMemcpy(o.data(), Y, bytes, cudaMemcpyDeviceToHost));
      CK(cudaMemcpy(ref.data(), R, bytes, cudaMemcpyDeviceToHost));
      for (long i = 0; i < n * n * n; i++) bad += o[i] != ref[i];
    }
    printf("%-30s %9.1f us  %7.1f GB/s  mismatches=%ld\n", name, us, alg / us / 1e3, bad);
  };
#define MARCH(BY, ZCH, MINB)                                                                              \
  time_it("march BY" #BY " Z" #ZCH " minB" #MINB, [&] {                                                   \
    dim3 g((unsigned)((n + 127) / 128), (unsigned)((hi - lo + BY - 1) / BY), (unsigned)((hi - lo + ZCH - 1) / ZCH)); \
    k_march<BY, ZCH, MINB><<<g, dim3(32, BY)>>>(X, Y, n, n, lo, hi, lo, hi, lo, hi);                      \
  }, false)
  time_it("ref march BY8 Z16", [&] {
    dim3 g((unsigned)((n + 127) / 128), (unsigned)((hi - lo + 7) / 8), (unsigned)((hi - lo + 15) / 16));
    k_march<8, 16, 1><<<g, dim3(32, 8)>>>(X, Y, n, n, lo, hi, lo, hi, lo, hi);
  }, true);
  MARCH(8, 64, 1);
#define WIN(BY, ZCH, G, MINB)                                                                             \
  time_it("win BY" #BY " Z" #ZCH " G" #G " minB" #MINB, [&] {                                             \
    dim3 g((unsigned)((n + 127) / 128), (unsigned)((hi - lo + BY - 1) / BY), (unsigned)((hi - lo + ZCH - 1) / ZCH)); \
    k_win<BY, ZCH, G, MINB><<<g, dim3(32, BY)>>>(X, Y, n, n, lo, hi, lo, hi, lo, hi);                     \
  }, false)
  WIN(8, 32, 4, 4);
#define ROWSV(R, ZCH, MINB)                                                                              \
  time_it("rows R" #R " Z" #ZCH " minB" #MINB, [&] {                                                    \
    dim3 g((unsigned)((n + 1023) / 1024), (unsigned)((hi - lo + R - 1) / R), (unsigned)((hi - lo + ZCH - 1) / ZCH)); \
    k_rows<R, ZCH, MINB><<<g, 256>>>(X, Y, n, n, lo, hi, lo, hi, lo, hi);                                 \
  }, false)
  ROWSV(1, 32, 4);
  ROWSV(2, 32, 4);
  ROWSV(4, 32, 3);
  ROWSV(4, 64, 3);
  ROWSV(8, 64, 2);
  ROWSV(2, 64, 4);
#define ROWSP(R, ZCH, MINB)                                                                              \
  time_it("rowsp R" #R " Z" #ZCH " minB" #MINB, [&] {                                                   \
    dim3 g((unsigned)((n + 1023) / 1024), (unsigned)((hi - lo + R - 1) / R), (unsigned)((hi - lo + ZCH - 1) / ZCH)); \
    k_rowsp<R, ZCH, MINB><<<g, 256>>>(X, Y, n, n, lo, hi, lo, hi, lo, hi);                                \
  }, false)
  ROWSP(1, 32, 4);
  ROWSP(2, 32, 4);
  ROWSP(2, 32, 3);
  ROWSP(1, 64, 5);
  ROWSP(2, 16, 4);
#define SMEM(BY, ZCH)                                                                                     \
  time_it("smem BY" #BY " Z" #ZCH, [&] {                                                                 \
    dim3 g((unsigned)((n + 127) / 128), (unsigned)((hi - lo + BY - 1) / BY), (unsigned)((hi - lo + ZCH - 1) / ZCH)); \
    k_smem<BY, ZCH><<<g, dim3(32, BY)>>>(X, Y, n, n, lo, hi, lo, hi, lo, hi);                             \
  }, false)
  SMEM(8, 32);
  {
    cudaEventRecord(a);
    for (int i = 0; i < 10; i++) cudaMemcpyAsync(Y, X, bytes, cudaMemcpyDeviceToDevice);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("%-30s %9.1f us  %7.1f GB/s\n", "cudaMemcpy D2D", ms * 1e3 / 10, 2.0 * bytes / (ms * 1e-3 / 10) / 1e9);
  }
  return 0;
}
