/* host_path_bench.c -- host cost of one axe_copy_plan_execute call through the C ABI (no Python): the
 * config-2 plan (the lowered TMA schedule) over 32 rotating buffer pairs, N enqueues timed with
 * CLOCK_MONOTONIC, then the device time of the same N launches with CUDA events.  Shows the library's
 * own per-call work (tensor-map cache lookup, parameter block, cudaLaunchKernelEx) apart from the
 * ctypes overhead the bench's host_us_per_call includes.  Measured (round 2, profiles/r02_host_path_c.json):
 * 4.0 us per call, of which the library's own work is 0.1 us (a build whose launcher returns before
 * cudaLaunchKernelEx: 0.10 us per call) -- the rest is the launch; past ~1000 queued launches the host
 * waits for the GPU to drain the launch queue (5.1 us per call over 2000).
 *
 *   gcc -O2 -I include tools/host_path_bench.c -o /tmp/hpb -L paper_2601_19092_b200 -laxe \
 *       -Wl,-rpath,$PWD/paper_2601_19092_b200 -L /usr/local/cuda/lib64 -lcudart && /tmp/hpb */
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>
#include <time.h>

#include "axe.h"

#define CK(x)                                                              \
  do {                                                                     \
    axe_status s_ = (x);                                                   \
    if (s_ != AXE_OK) {                                                    \
      fprintf(stderr, "%s failed: %d %s\n", #x, s_, axe_last_error());     \
      return 1;                                                            \
    }                                                                      \
  } while (0)

static double now_us(void) {
  struct timespec t;
  clock_gettime(CLOCK_MONOTONIC, &t);
  return t.tv_sec * 1e6 + t.tv_nsec * 1e-3;
}

int main(void) {
  const int64_t n = 4096;
  axe_iter rm[2] = {{n, n, NULL}, {n, 1, NULL}};
  axe_iter tl[4] = {{64, 64 * n, NULL}, {64, 64, NULL}, {64, 64 * 64, NULL}, {64, 1, NULL}};
  axe_layout *src = NULL, *dst = NULL;
  CK(axe_layout_create(rm, 2, NULL, 0, NULL, 0, &src));
  CK(axe_layout_create(tl, 4, NULL, 0, NULL, 0, &dst));
  axe_storage_digit dg = {"m", n * n, 1};
  axe_storage st_rm = {1, &dg, 0, 0, 0}, st_tl = {1, &dg, 3, 4, 3};
  axe_copy_plan *plan = NULL;
  CK(axe_copy_plan_create(src, &st_rm, dst, &st_tl, 2, AXE_KERNEL_AUTO, &plan));
  char desc[4096];
  CK(axe_copy_plan_describe(plan, desc, sizeof desc));
  enum { PAIRS = 32, N = 2000 };
  void *s[PAIRS], *d[PAIRS];
  for (int i = 0; i < PAIRS; i++) {
    if (cudaMalloc(&s[i], n * n * 2) != cudaSuccess || cudaMalloc(&d[i], n * n * 2) != cudaSuccess) return 2;
    cudaMemset(s[i], i, n * n * 2);
  }
  cudaStream_t st;
  cudaStreamCreate(&st);
  for (int i = 0; i < 64; i++) CK(axe_copy_plan_execute(plan, s[i % PAIRS], d[i % PAIRS], st));
  cudaStreamSynchronize(st);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  // host cost: the first H calls after an idle stream (fewer than the launch queue holds, so no call
  // waits for the GPU to drain it); device time: N back-to-back launches
  enum { H = 200 };
  const double h0 = now_us();
  for (int i = 0; i < H; i++) CK(axe_copy_plan_execute(plan, s[i % PAIRS], d[i % PAIRS], st));
  const double h1 = now_us();
  cudaStreamSynchronize(st);
  cudaEventRecord(e0, st);
  const double t0 = now_us();
  for (int i = 0; i < N; i++) CK(axe_copy_plan_execute(plan, s[i % PAIRS], d[i % PAIRS], st));
  const double t1 = now_us();
  cudaEventRecord(e1, st);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  printf("{\"host_us_per_call\": %.3f, \"host_us_per_call_queue_full\": %.3f, "
         "\"device_us_per_step_direct_launches\": %.3f, \"calls\": %d, \"GBps\": %.1f, \"plan\": %s}\n",
         (h1 - h0) / H, (t1 - t0) / N, ms * 1e3 / N, N, 2.0 * n * n * 2 / (ms * 1e-3 / N) / 1e9, desc);
  return 0;
}
