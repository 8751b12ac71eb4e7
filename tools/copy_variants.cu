// copy_variants.cu -- development probe: plain contiguous copy kernels of different shapes against the
// driver's device-to-device memcpy (the kernel MEASURED_PEAKS.json's copy_ figure comes from), at the
// bench's size and larger.  Each row: a CUDA graph of NL dependent launches over rotating buffer pairs
// (>= 2 GiB footprint, L2 defeated), timed with CUDA events around one replay, best of 5.
//
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o /tmp/cv tools/copy_variants.cu
//   /tmp/cv [MiB per side ...]
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                         \
  do {                                                                                \
    cudaError_t e_ = (x);                                                             \
    if (e_ != cudaSuccess) {                                                          \
      fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
      exit(1);                                                                        \
    }                                                                                 \
  } while (0)

__device__ __forceinline__ uint4 ld_nc(const uint4 *p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}
__device__ __forceinline__ void st_plain(uint4 *p, uint4 v) {
  asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}
__device__ __forceinline__ void st_cs(uint4 *p, uint4 v) {
  asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}

// grid-stride: each thread moves U vectors a block apart per trip
template <int U, bool CS>
__global__ void __launch_bounds__(256) k_stride(const uint4 *__restrict__ s, uint4 *__restrict__ d, size_t n) {
  const size_t step = (size_t)gridDim.x * 256 * U;
  for (size_t b = (size_t)blockIdx.x * 256 * U + threadIdx.x; b < n; b += step) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; u++)
      if (b + (size_t)u * 256 < n) v[u] = ld_nc(s + b + (size_t)u * 256);
#pragma unroll
    for (int u = 0; u < U; u++)
      if (b + (size_t)u * 256 < n) CS ? st_cs(d + b + (size_t)u * 256, v[u]) : st_plain(d + b + (size_t)u * 256, v[u]);
  }
}

// contiguous chunk per CTA: CTA c moves vectors [c * n / G, (c + 1) * n / G)
template <int U>
__global__ void __launch_bounds__(256) k_chunk(const uint4 *__restrict__ s, uint4 *__restrict__ d, size_t n) {
  const size_t per = (n + gridDim.x - 1) / gridDim.x;
  const size_t lo = (size_t)blockIdx.x * per, hi = lo + per < n ? lo + per : n;
  for (size_t b = lo + threadIdx.x; b < hi; b += 256 * U) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; u++)
      if (b + (size_t)u * 256 < hi) v[u] = ld_nc(s + b + (size_t)u * 256);
#pragma unroll
    for (int u = 0; u < U; u++)
      if (b + (size_t)u * 256 < hi) st_plain(d + b + (size_t)u * 256, v[u]);
  }
}

// persistent grid, tiles of 256 * U vectors claimed in order from a global counter (zeroed before each
// launch): the active tiles stay a tight window however the CTAs drift
template <int U>
__global__ void __launch_bounds__(256) k_dyn(const uint4 *__restrict__ s, uint4 *__restrict__ d, size_t n,
                                             unsigned *ctr) {
  __shared__ unsigned t_s;
  const size_t ntiles = (n + 256 * U - 1) / (256 * U);
  for (;;) {
    if (threadIdx.x == 0) t_s = atomicAdd(ctr, 1u);
    __syncthreads();
    const size_t t = t_s;
    __syncthreads();
    if (t >= ntiles) return;
    const size_t b = t * 256 * U + threadIdx.x;
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; u++)
      if (b + (size_t)u * 256 < n) v[u] = ld_nc(s + b + (size_t)u * 256);
#pragma unroll
    for (int u = 0; u < U; u++)
      if (b + (size_t)u * 256 < n) st_plain(d + b + (size_t)u * 256, v[u]);
  }
}

struct Bufs {
  std::vector<void *> s, d;
};

template <class F>
static float timed(F launch, int pairs, int nl, cudaStream_t st) {
  for (int i = 0; i < 3; i++) launch(i % pairs, st);
  CK(cudaStreamSynchronize(st));
  cudaGraph_t g;
  cudaGraphExec_t ge;
  CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
  for (int i = 0; i < nl; i++) launch(i % pairs, st);
  CK(cudaStreamEndCapture(st, &g));
  CK(cudaGraphInstantiate(&ge, g, 0));
  CK(cudaGraphLaunch(ge, st));
  CK(cudaStreamSynchronize(st));
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  float best = 1e30f;
  for (int r = 0; r < 5; r++) {
    CK(cudaEventRecord(a, st));
    CK(cudaGraphLaunch(ge, st));
    CK(cudaEventRecord(b, st));
    CK(cudaEventSynchronize(b));
    float ms;
    CK(cudaEventElapsedTime(&ms, a, b));
    if (ms < best) best = ms;
  }
  CK(cudaGraphExecDestroy(ge));
  CK(cudaGraphDestroy(g));
  return best * 1e3f / nl;  // us per copy
}

int main(int argc, char **argv) {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  std::vector<int> sizes;
  for (int i = 1; i < argc; i++) sizes.push_back(atoi(argv[i]));
  if (sizes.empty()) sizes = {32, 256};
  cudaStream_t st;
  CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  for (int mib : sizes) {
    const size_t nb = (size_t)mib << 20, n = nb / 16;
    const int pairs = (int)std::max<size_t>(2, ((size_t)2 << 30) / (2 * nb));
    Bufs B;
    for (int i = 0; i < pairs; i++) {
      void *p, *q;
      CK(cudaMalloc(&p, nb));
      CK(cudaMalloc(&q, nb));
      CK(cudaMemset(p, i + 1, nb));
      B.s.push_back(p);
      B.d.push_back(q);
    }
    auto row = [&](const char *name, float us) {
      printf("{\"MiB\":%d,\"variant\":\"%s\",\"us\":%.2f,\"GBps\":%.0f}\n", mib, name, us, 2.0 * nb / (us * 1e-6) / 1e9);
      fflush(stdout);
    };
    const int NL = 16;
    row("memcpy", timed([&](int i, cudaStream_t s) { CK(cudaMemcpyAsync(B.d[i], B.s[i], nb, cudaMemcpyDeviceToDevice, s)); },
                        pairs, NL, st));
#define STRIDE(U, CS, K)                                                                                   \
  {                                                                                                        \
    char nm[64];                                                                                           \
    snprintf(nm, sizeof nm, "stride_u%d%s_g%dx", U, CS ? "_cs" : "", K);                                    \
    row(nm, timed([&](int i, cudaStream_t s) {                                                             \
          k_stride<U, CS><<<sms * K, 256, 0, s>>>((const uint4 *)B.s[i], (uint4 *)B.d[i], n);              \
        }, pairs, NL, st));                                                                                \
  }
    STRIDE(1, false, 8) STRIDE(2, false, 8) STRIDE(4, false, 8) STRIDE(8, false, 4) STRIDE(4, false, 4)
    STRIDE(4, true, 8) STRIDE(4, false, 16) STRIDE(2, false, 16)
    {
      const unsigned g = (unsigned)((n + 256 * 4 - 1) / (256 * 4));
      row("oneshot_u4", timed([&](int i, cudaStream_t s) {
            k_stride<4, false><<<g, 256, 0, s>>>((const uint4 *)B.s[i], (uint4 *)B.d[i], n);
          }, pairs, NL, st));
      const unsigned g2 = (unsigned)((n + 256 * 8 - 1) / (256 * 8));
      row("oneshot_u8", timed([&](int i, cudaStream_t s) {
            k_stride<8, false><<<g2, 256, 0, s>>>((const uint4 *)B.s[i], (uint4 *)B.d[i], n);
          }, pairs, NL, st));
    }
#define CHUNK(U, K)                                                                                        \
  {                                                                                                        \
    char nm[64];                                                                                           \
    snprintf(nm, sizeof nm, "chunk_u%d_g%dx", U, K);                                                       \
    row(nm, timed([&](int i, cudaStream_t s) {                                                             \
          k_chunk<U><<<sms * K, 256, 0, s>>>((const uint4 *)B.s[i], (uint4 *)B.d[i], n);                   \
        }, pairs, NL, st));                                                                                \
  }
    CHUNK(4, 8) CHUNK(4, 4) CHUNK(8, 4)
    {
      unsigned *ctr;
      CK(cudaMalloc(&ctr, 4 * 64));
      for (int K : {4, 8}) {
        char nm[64];
        snprintf(nm, sizeof nm, "dyn_u4_g%dx", K);
        row(nm, timed([&](int i, cudaStream_t s) {
              CK(cudaMemsetAsync(ctr + i, 0, 4, s));
              k_dyn<4><<<sms * K, 256, 0, s>>>((const uint4 *)B.s[i], (uint4 *)B.d[i], n, ctr + i);
            }, pairs, NL, st));
      }
      CK(cudaFree(ctr));
    }
    for (int i = 0; i < pairs; i++) {
      CK(cudaFree(B.s[i]));
      CK(cudaFree(B.d[i]));
    }
  }
  return 0;
}
