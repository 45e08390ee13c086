// p2p_tune.cu — NVLink transfer mechanisms between two B200s (standalone; not part of
// the library).  Each GPU moves `bytes` to/from the other, both directions at once
// (the repartition pattern), as (1) SM pull: peer LDG.128 -> local STG, U loads in
// flight per lane; (2) SM push: local LDG -> peer STG.128; (3) copy engine
// cudaMemcpyPeerAsync.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17
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

template <int U>
__global__ void __launch_bounds__(256) copy_kernel(const uint4* __restrict__ src, uint4* __restrict__ dst, size_t n) {
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (; i + (U - 1) * stride < n; i += U * stride) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; u++) v[u] = src[i + u * stride];
#pragma unroll
    for (int u = 0; u < U; u++) dst[i + u * stride] = v[u];
  }
  for (; i < n; i += stride) dst[i] = src[i];
}

// all-to-all over G GPUs: every GPU pulls `bytes` from each peer (the ROW<->COL
// repartition); (a) copy engine, one stream; (b) copy engine, one stream per peer;
// (c) SM pull kernel per peer on one stream.  Time = max over GPUs.
static void all_to_all(int G, size_t bytes) {
  std::vector<void*> src(G), dst(G);
  std::vector<std::vector<cudaStream_t>> st(G, std::vector<cudaStream_t>(G));
  std::vector<cudaEvent_t> e0(G), e1(G);
  for (int g = 0; g < G; g++) {
    CK(cudaSetDevice(g));
    for (int h = 0; h < G; h++)
      if (h != g) cudaDeviceEnablePeerAccess(h, 0);
    cudaGetLastError();
    CK(cudaMalloc(&src[g], bytes));
    CK(cudaMalloc(&dst[g], bytes * G));
    for (int h = 0; h < G; h++) CK(cudaStreamCreateWithFlags(&st[g][h], cudaStreamNonBlocking));
    cudaEventCreate(&e0[g]);
    cudaEventCreate(&e1[g]);
  }
  const size_t n = bytes / 16;
  for (int mode = 0; mode < 5; mode++) {
    float best = 1e30f;
    for (int rep = 0; rep < 4; rep++) {
      for (int g = 0; g < G; g++) {
        CK(cudaSetDevice(g));
        CK(cudaDeviceSynchronize());
      }
      for (int g = 0; g < G; g++) {
        CK(cudaSetDevice(g));
        cudaEventRecord(e0[g], st[g][0]);
        for (int h = 0; h < G; h++) {
          if (h == g) continue;
          cudaStream_t s = mode == 1 ? st[g][h] : st[g][0];
          if (mode == 1) {
            cudaStreamWaitEvent(s, e0[g], 0);
          }
          if (mode == 2)
            copy_kernel<4><<<148 * 8, 256, 0, s>>>((const uint4*)src[h], (uint4*)((char*)dst[g] + h * bytes), n);
          else if (mode == 3)  // CE push: g writes its block into peer h
            CK(cudaMemcpyPeerAsync((char*)dst[h] + g * bytes, h, src[g], g, bytes, s));
          else if (mode == 4)  // SM push
            copy_kernel<4><<<148 * 8, 256, 0, s>>>((const uint4*)src[g], (uint4*)((char*)dst[h] + g * bytes), n);
          else
            CK(cudaMemcpyPeerAsync((char*)dst[g] + h * bytes, g, src[h], h, bytes, s));
        }
        if (mode == 1)
          for (int h = 0; h < G; h++)
            if (h != g && h != 0) {
              cudaEvent_t ev;
              cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
              cudaEventRecord(ev, st[g][h]);
              cudaStreamWaitEvent(st[g][0], ev, 0);
              cudaEventDestroy(ev);
            }
        cudaEventRecord(e1[g], st[g][0]);
      }
      float worst = 0;
      for (int g = 0; g < G; g++) {
        CK(cudaSetDevice(g));
        CK(cudaEventSynchronize(e1[g]));
        float ms;
        cudaEventElapsedTime(&ms, e0[g], e1[g]);
        worst = ms > worst ? ms : worst;
      }
      best = worst < best ? worst : best;
    }
    const char* nm[5] = {"CE pull one stream", "CE pull stream/peer", "SM pull x4", "CE push one stream",
                         "SM push x4"};
    printf("all-to-all G=%d %-22s %8.3f ms  per-GPU in %7.1f GB/s\n", G, nm[mode], best,
           (G - 1) * bytes / (best * 1e-3) / 1e9);
  }
}

int main(int argc, char** argv) {
  int ndev = 0;
  cudaGetDeviceCount(&ndev);
  if (argc > 2 && atoi(argv[2]) > 0) {
    all_to_all(ndev, (size_t)atol(argv[1]) << 20);
    return 0;
  }
  const size_t bytes = (argc > 1 ? atol(argv[1]) : 1024L) << 20;  // MiB per direction
  const size_t n = bytes / 16;
  void *a[2], *b[2];
  for (int g = 0; g < 2; g++) {
    CK(cudaSetDevice(g));
    CK(cudaDeviceEnablePeerAccess(1 - g, 0));
    CK(cudaMalloc(&a[g], bytes));
    CK(cudaMalloc(&b[g], bytes));
    CK(cudaMemset(a[g], g + 1, bytes));
  }
  cudaStream_t s[2];
  cudaEvent_t e0[2], e1[2];
  for (int g = 0; g < 2; g++) {
    CK(cudaSetDevice(g));
    CK(cudaStreamCreateWithFlags(&s[g], cudaStreamNonBlocking));
    cudaEventCreate(&e0[g]);
    cudaEventCreate(&e1[g]);
  }
  auto run = [&](const char* name, int mode, int grid, bool both) {
    float best = 1e30f;
    for (int rep = 0; rep < 5; rep++) {
      for (int g = 0; g < 2; g++) {
        CK(cudaSetDevice(g));
        CK(cudaDeviceSynchronize());
      }
      for (int g = 0; g < (both ? 2 : 1); g++) {
        CK(cudaSetDevice(g));
        cudaEventRecord(e0[g], s[g]);
        const uint4* peer_src = (const uint4*)a[1 - g];
        uint4* local_dst = (uint4*)b[g];
        const uint4* local_src = (const uint4*)a[g];
        uint4* peer_dst = (uint4*)b[1 - g];
        switch (mode) {
          case 1: copy_kernel<1><<<grid, 256, 0, s[g]>>>(peer_src, local_dst, n); break;
          case 4: copy_kernel<4><<<grid, 256, 0, s[g]>>>(peer_src, local_dst, n); break;
          case 8: copy_kernel<8><<<grid, 256, 0, s[g]>>>(peer_src, local_dst, n); break;
          case 14: copy_kernel<4><<<grid, 256, 0, s[g]>>>(local_src, peer_dst, n); break;
          case 18: copy_kernel<8><<<grid, 256, 0, s[g]>>>(local_src, peer_dst, n); break;
          case 20: CK(cudaMemcpyPeerAsync(b[g], g, a[1 - g], 1 - g, bytes, s[g])); break;
        }
        cudaEventRecord(e1[g], s[g]);
      }
      float worst = 0;
      for (int g = 0; g < (both ? 2 : 1); g++) {
        CK(cudaSetDevice(g));
        CK(cudaEventSynchronize(e1[g]));
        float ms;
        cudaEventElapsedTime(&ms, e0[g], e1[g]);
        if (ms > worst) worst = ms;
      }
      if (worst < best) best = worst;
    }
    printf("%-44s %s grid=%5d  %8.3f ms  %7.1f GB/s per direction\n", name, both ? "bidir" : "unidir", grid, best,
           bytes / (best * 1e-3) / 1e9);
  };
  for (bool both : {false, true}) {
    run("pull LDG.128 x1", 1, 148 * 8, both);
    run("pull LDG.128 x4", 4, 148 * 8, both);
    run("pull LDG.128 x4 (grid 148*16)", 4, 148 * 16, both);
    run("pull LDG.128 x8", 8, 148 * 8, both);
    run("pull LDG.128 x8 (grid 148*2)", 8, 148 * 2, both);
    run("push STG.128 x4", 14, 148 * 8, both);
    run("push STG.128 x8", 18, 148 * 8, both);
    run("push STG.128 x4 (grid 148*2)", 14, 148 * 2, both);
    run("copy engine cudaMemcpyPeerAsync", 20, 0, both);
  }
  return 0;
}
