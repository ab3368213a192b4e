// Stand-alone timing of the fp64 tensor-core GEMM (dk_dense.cu) on set-up shapes.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include \
//        -o tools/gemm_bench tools/gemm_bench.cu
#include "../paper_1510_02148_b200/csrc/dk_dense.cu"

#include <cstdio>

int main() {
  const int d = 10917, ld = 10918;
  double *A, *C;
  cudaMalloc(&A, (size_t)d * ld * 8);
  cudaMalloc(&C, (size_t)d * ld * 8);
  cudaMemset(A, 0, (size_t)d * ld * 8);
  cudaMemset(C, 0, (size_t)d * ld * 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  struct Case { const char* name; bool ta, tb; int M, N, K, tri; double beta; int kshift; };
  Case cases[] = {
      {"square 8192 NN", false, false, 8192, 8192, 8192, 0, 1.0, INT_MIN},
      {"square 8192 NT", false, true, 8192, 8192, 8192, 0, 1.0, INT_MIN},
      {"syrk K=128 lower", false, true, 10789, 10789, 128, 1, 1.0, INT_MIN},
      {"syrk K=128 full", false, true, 10789, 10789, 128, 0, 1.0, INT_MIN},
      {"syrk K=128 full b0", false, true, 10789, 10789, 128, 0, 0.0, INT_MIN},
      {"syrk K=256 lower", false, true, 10661, 10661, 256, 1, 1.0, INT_MIN},
      {"syrk K=512 full", false, true, 10661, 10661, 512, 0, 1.0, INT_MIN},
      {"lauum TA upper", true, false, 10917, 10917, 10917, 2, 0.0, 0},
      {"trsm N=128", false, true, 10789, 128, 128, 0, 0.0, INT_MIN},
  };
  for (int nt : {4, 2}) {
  dk::g_gemm_nt = nt;
  printf("-- n8 tiles per warp: %d\n", nt);
  for (auto& c : cases) {
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(e0);
      dk::gemm_mma(c.ta, c.tb, A, ld, A, ld, C, ld, c.M, c.N, c.K, -1.0, c.beta, c.tri, c.kshift,
                   0);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      double fl = 2.0 * c.M * (double)c.N * c.K;
      if (c.tri) fl *= 0.5;
      if (c.kshift != INT_MIN) fl *= 0.5;
      if (rep == 2)
        printf("%-22s %9.3f ms  %6.1f TF/s (useful)  err=%s\n", c.name, ms, fl / ms / 1e9,
               cudaGetErrorString(cudaGetLastError()));
    }
  }
  }
  return 0;
}
