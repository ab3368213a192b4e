// Standalone check of nd_tree_inverse: E = graph Laplacian of a label graph + I (SPD), in
// nested-dissection order; W = L^-1 must satisfy W E W^T = I.
// nvcc -O3 -std=c++17 -I paper_1510_02148_b200/csrc -I include -gencode arch=compute_100a,code=sm_100a \
//   tools/nd_tree_check.cu paper_1510_02148_b200/csrc/{dk_profile,dk_dense,dk_coarse,dk_kernels}.cu -o tools/nd_tree_check
#include <cmath>
#include <cstdio>
#include <vector>
#include "dk_launch.h"
int main(int argc, char** argv) {
  const char* pp = argc > 1 ? argv[1] : "/tmp/ptr.bin";
  const char* cp = argc > 2 ? argv[2] : "/tmp/col.bin";
  FILE* f = fopen(pp, "rb");
  std::vector<int> ptr;
  int v;
  while (fread(&v, 4, 1, f) == 1) ptr.push_back(v);
  fclose(f);
  const int d = (int)ptr.size() - 1;
  std::vector<int> col(ptr.back());
  f = fopen(cp, "rb");
  if (fread(col.data(), 4, col.size(), f) != col.size()) return 1;
  fclose(f);
  std::vector<int> perm;
  std::vector<dk::NDTreeNode> tree;
  dk::nd_order(d, ptr, col, perm, &tree);
  std::vector<int> inv(d);
  for (int i = 0; i < d; ++i) inv[perm[i]] = i;
  const int ld = d + (d & 1);
  std::vector<double> E((size_t)d * ld, 0.0);
  for (int r = 0; r < d; ++r) {
    double s = 1.0;
    for (int k = ptr[r]; k < ptr[r + 1]; ++k) {
      const double w = 1.0 + 0.001 * ((r * 7 + col[k] * 13) % 17) + 0.001 * ((col[k] * 7 + r * 13) % 17);
      E[(size_t)inv[r] * ld + inv[col[k]]] = -w;
      s += w;
    }
    E[(size_t)inv[r] * ld + inv[r]] = s;
  }
  printf("d %d nodes %zu\n", d, tree.size());
  double *dE, *dW;
  cudaMalloc(&dE, E.size() * 8);
  cudaMalloc(&dW, E.size() * 8);
  cudaMemcpy(dE, E.data(), E.size() * 8, cudaMemcpyHostToDevice);
  cudaMemset(dW, 0, E.size() * 8);
  cudaStream_t s;
  cudaStreamCreate(&s);
  double mn = 0;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a, s);
  int err = dk::nd_tree_inverse(dE, d, ld, tree, dW, &mn, s);
  cudaEventRecord(b, s);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  printf("err %d min_diag_sq %g  %.2f ms\n", err, mn, ms);
  std::vector<double> W(E.size());
  cudaMemcpy(W.data(), dW, W.size() * 8, cudaMemcpyDeviceToHost);
  // check rows of W E W^T = I on a sample of rows
  double worst = 0;
  for (int t = 0; t < 40; ++t) {
    const int i = (int)((long long)t * 2654435761LL % d), j = (int)((long long)(t + 7) * 40503LL % d);
    double acc = 0;  // (W E W^T)_{ij} = sum_{k,l} W_ik E_kl W_jl with E from the host copy
    std::vector<double> ew(d, 0.0);  // E W_j^T
    for (int k = 0; k < d; ++k) {
      double sum = 0;
      for (int l = 0; l <= j; ++l) sum += E[(size_t)k * ld + l] * W[(size_t)j * ld + l];
      ew[k] = sum;
    }
    for (int k = 0; k <= i; ++k) acc += W[(size_t)i * ld + k] * ew[k];
    worst = fmax(worst, fabs(acc - (i == j ? 1.0 : 0.0)));
  }
  printf("max |W E W^T - I| over samples %.3e\n", worst);
  return 0;
}
