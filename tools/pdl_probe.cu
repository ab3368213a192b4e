// Probe: programmatic dependent launch inside stream capture (diagnostic).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k1(int* p) { asm volatile("griddepcontrol.wait;" ::: "memory"); p[threadIdx.x] += 1; asm volatile("griddepcontrol.launch_dependents;"); }
__global__ void k2(int* p) { asm volatile("griddepcontrol.wait;" ::: "memory"); p[threadIdx.x] *= 2; }
template <typename K, typename... A> cudaError_t L(K k, cudaStream_t s, int attr, A... a) {
  cudaLaunchConfig_t c = {}; c.gridDim = dim3(4); c.blockDim = dim3(32); c.stream = s;
  cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1; c.attrs = at; c.numAttrs = attr;
  return cudaLaunchKernelEx(&c, k, a...);
}
int main() {
  int* p; cudaMalloc(&p, 128 * 4); cudaMemset(p, 0, 128 * 4);
  cudaStream_t s; cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  for (int mode = 0; mode < 4; ++mode) {
    cudaGraph_t g; cudaGetLastError();
    cudaError_t e0 = cudaStreamBeginCapture(s, mode < 2 ? cudaStreamCaptureModeThreadLocal : cudaStreamCaptureModeGlobal);
    cudaError_t e1 = L(k1, s, mode & 1, p);
    cudaError_t e2 = L(k2, s, 1, p);
    cudaError_t e3 = L(k1, s, 1, p);
    cudaError_t e4 = cudaStreamEndCapture(s, &g);
    printf("mode %d: begin %s k1 %s k2 %s k1b %s end %s\n", mode, cudaGetErrorString(e0), cudaGetErrorString(e1), cudaGetErrorString(e2), cudaGetErrorString(e3), cudaGetErrorString(e4));
    if (e4 == cudaSuccess) { cudaGraphExec_t x; cudaError_t e5 = cudaGraphInstantiate(&x, g, 0); printf("  inst %s\n", cudaGetErrorString(e5)); if (!e5) { printf("  launch %s\n", cudaGetErrorString(cudaGraphLaunch(x, s))); printf("  sync %s\n", cudaGetErrorString(cudaStreamSynchronize(s))); } }
  }
  // eager (no capture)
  printf("eager: %s %s %s\n", cudaGetErrorString(L(k1, s, 1, p)), cudaGetErrorString(L(k2, s, 1, p)), cudaGetErrorString(cudaStreamSynchronize(s)));
  return 0;
}
