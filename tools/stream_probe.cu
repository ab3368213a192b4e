// Streaming probe: how fast do warps pull 8 KB tiles through one-lane TMA bulk copies, as a
// function of the stream length, warps per CTA, stages per warp and tile assignment?
// nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a tools/stream_probe.cu -o tools/stream_probe
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kTB = 8192;

__device__ __forceinline__ unsigned sa(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

template <int KW, int KS>
__global__ void __launch_bounds__(KW * 32, 1) k_stream(const double* T, long long nt, int rr, double* out) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ __align__(8) unsigned long long bars[KW][KS];
  const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
  unsigned char* wb = sm + (size_t)wl * KS * kTB;
  const long long Wn = (long long)gridDim.x * KW, w = (long long)blockIdx.x * KW + wl;
  long long t0, t1, step;
  if (rr) { t0 = w; t1 = nt; step = Wn; } else { t0 = w * nt / Wn; t1 = (w + 1) * nt / Wn; step = 1; }
  unsigned long long pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  if (lane == 0)
    for (int s = 0; s < KS; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bars[wl][s])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  auto issue = [&](int s, long long t) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bars[wl][s])), "r"(kTB) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
                 ::"r"(sa(wb + s * kTB)), "l"(T + t * 1024), "r"(kTB), "r"(sa(&bars[wl][s])), "l"(pol) : "memory");
  };
  if (lane == 0)
    for (int s = 0; s < KS; ++s)
      if (t0 + s * step < t1) issue(s, t0 + s * step);
  double acc = 0.0;
  int k = 0;
  for (long long t = t0; t < t1; t += step, ++k) {
    const int s = k % KS;
    const unsigned par = (unsigned)((k / KS) & 1);
    unsigned done = 0;
    while (!done)
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                   : "=r"(done) : "r"(sa(&bars[wl][s])), "r"(par) : "memory");
    const double2* v = reinterpret_cast<const double2*>(wb + s * kTB);
#pragma unroll
    for (int p = 0; p < 16; ++p) { const double2 a = v[p * 32 + lane]; acc += a.x + a.y; }
    __syncwarp();
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (lane == 0 && t + KS * step < t1) issue(s, t + KS * step);
  }
  if (acc == 12345.0) out[0] = acc;
}

template <int KW, int KS>
void run(const double* T, long long nt, int rr, double* out) {
  const size_t smem = (size_t)KW * KS * kTB;
  cudaFuncSetAttribute(k_stream<KW, KS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int i = 0; i < 3; ++i) k_stream<KW, KS><<<148, KW * 32, smem>>>(T, nt, rr, out);
  const int reps = 20;
  cudaEventRecord(a);
  for (int i = 0; i < reps; ++i) k_stream<KW, KS><<<148, KW * 32, smem>>>(T, nt, rr, out);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  const double us = ms * 1000.0 / reps;
  printf("KW=%2d KS=%d rr=%d tiles=%7lld  %8.2f us  %7.1f GB/s\n", KW, KS, rr, nt, us,
         nt * (double)kTB / us * 1e-3);
}

int main() {
  const long long maxt = 60000;
  double* T;
  double* out;
  cudaMalloc(&T, maxt * kTB);
  cudaMalloc(&out, 8);
  cudaMemset(T, 0, maxt * kTB);
  for (long long nt : {8320LL, 16640LL, 58653LL})
    for (int rr = 0; rr < 2; ++rr) {
      run<12, 2>(T, nt, rr, out);
      run<16, 1>(T, nt, rr, out);
      run<8, 3>(T, nt, rr, out);
      run<4, 6>(T, nt, rr, out);
      run<2, 12>(T, nt, rr, out);
    }
  return 0;
}
