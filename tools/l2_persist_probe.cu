// L2 persistence probe: does a 70 MB buffer stay L2-resident across a 700 MB stream when it
// is covered by a persisting access-policy window (or loaded with an evict_last policy)?
#include <cstdio>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(256) k_read(const double2* __restrict__ p, long long n2,
                                              double* out, int mode) {
  unsigned long long pol;
  if (mode == 1)
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  else
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  double acc = 0.0;
  const long long stride = (long long)gridDim.x * blockDim.x;
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  for (; i + 7 * stride < n2; i += 8 * stride) {
    double2 v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if (mode == 0) {
        v[k] = __ldcg(p + i + k * stride);
      } else {
        asm volatile("ld.global.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;"
                     : "=d"(v[k].x), "=d"(v[k].y) : "l"(p + i + k * stride), "l"(pol));
      }
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) acc += v[k].x + v[k].y;
  }
  for (; i < n2; i += stride) {
    const double2 v = __ldcg(p + i);
    acc += v.x + v.y;
  }
  if (acc == 12345.678) out[0] = acc;
}

int main() {
  cudaDeviceProp pr;
  cudaGetDeviceProperties(&pr, 0);
  printf("l2 %d MB, persistingL2CacheMaxSize %d MB, accessPolicyMaxWindowSize %d MB\n",
         pr.l2CacheSize >> 20, pr.persistingL2CacheMaxSize >> 20,
         pr.accessPolicyMaxWindowSize >> 20);
  const long long wb = 70ll << 20, sb = 700ll << 20, wcap = 96ll << 20;
  double2 *W, *S;
  double* out;
  cudaMalloc(&W, wcap);
  cudaMalloc(&S, sb);
  cudaMalloc(&out, 8);
  cudaMemset(W, 0, wcap);
  cudaMemset(S, 0, sb);
  cudaStream_t s;
  cudaStreamCreate(&s);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int grid = pr.multiProcessorCount * 4;
  for (int variant = 0; variant < 4; ++variant) {
    // 0: plain; 1: evict_last loads of W (others evict_first); 2: persisting window;
    // 3: persisting window with carve-out = max
    cudaStreamAttrValue av = {};
    if (variant >= 2) {
      size_t carve = variant == 3 ? pr.persistingL2CacheMaxSize : (size_t)wb;
      if (carve > (size_t)pr.persistingL2CacheMaxSize) carve = pr.persistingL2CacheMaxSize;
      cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, carve);
      av.accessPolicyWindow.base_ptr = W;
      av.accessPolicyWindow.num_bytes = wb;
      av.accessPolicyWindow.hitRatio = (float)((double)carve / wb > 1.0 ? 1.0 : (double)carve / wb);
      av.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
      av.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    } else {
      cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, 0);
      av.accessPolicyWindow.num_bytes = 0;
    }
    cudaStreamSetAttribute(s, cudaStreamAttributeAccessPolicyWindow, &av);
    cudaCtxResetPersistingL2Cache();
    float tw = 0, ts = 0;
    const int reps = 20;
    for (int r = 0; r < reps + 2; ++r) {
      cudaEventRecord(e0, s);
      k_read<<<grid, 256, 0, s>>>(W, wb / 16, out, variant == 1 ? 1 : 0);
      cudaEventRecord(e1, s);
      cudaEventSynchronize(e1);
      float a;
      cudaEventElapsedTime(&a, e0, e1);
      cudaEventRecord(e0, s);
      k_read<<<grid, 256, 0, s>>>(S, sb / 16, out, variant == 1 ? 2 : 0);
      cudaEventRecord(e1, s);
      cudaEventSynchronize(e1);
      float b;
      cudaEventElapsedTime(&b, e0, e1);
      if (r >= 2) {
        tw += a;
        ts += b;
      }
    }
    printf("variant %d: W read %.1f us (%.0f GB/s), stream %.1f us (%.0f GB/s) err=%s\n", variant,
           1e3 * tw / reps, wb / (1e6 * tw / reps), 1e3 * ts / reps, sb / (1e6 * ts / reps),
           cudaGetErrorString(cudaGetLastError()));
  }
  // effective L2 capacity for an immediate re-read: read W twice back to back (no stream in
  // between), time the second read; W sizes 16..96 MB; policy: 0 normal, 1 evict_last
  cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, 0);
  cudaStreamAttrValue av0 = {};
  cudaStreamSetAttribute(s, cudaStreamAttributeAccessPolicyWindow, &av0);
  for (int pol = 0; pol < 2; ++pol)
    for (int mb = 16; mb <= 96; mb += 8) {
      const long long b = (long long)mb << 20;
      float t2 = 0;
      for (int r = 0; r < 6; ++r) {
        k_read<<<grid, 256, 0, s>>>(S, sb / 16, out, 0);  // flush
        k_read<<<grid, 256, 0, s>>>(W, b / 16, out, pol);
        cudaEventRecord(e0, s);
        k_read<<<grid, 256, 0, s>>>(W, b / 16, out, pol);
        cudaEventRecord(e1, s);
        cudaEventSynchronize(e1);
        float a;
        cudaEventElapsedTime(&a, e0, e1);
        if (r >= 1) t2 += a;
      }
      t2 /= 5;
      printf("reread pol=%d %3d MB: %.1f us (%.0f GB/s)\n", pol, mb, 1e3 * t2, b / (1e6 * t2));
    }
  return 0;
}
