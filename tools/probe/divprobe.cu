#include <cstdio>
__global__ void k(const double* a, const double* b, double* o, int n) { int i = threadIdx.x; if (i < n) o[i] = a[i] / b[i]; }
__global__ void kf(const float* a, const float* b, float* o, int n) { int i = threadIdx.x; if (i < n) o[i] = a[i] / b[i]; }
int main() {
  const int n = 6;
  double ha[n] = {-9.14e-322, 5e-324, 1e-310, 1.0, 1e-310, 3.0}, hb[n] = {0.0, 0.0, 0.0, 0.0, 1e300, 1e-310}, ho[n];
  float fa[3] = {-1.036e-42f, 1e-45f, 1.0f}, fb[3] = {0.f, 0.f, 0.f}, fo[3];
  double *da, *db, *dout; float *fa_d, *fb_d, *fo_d;
  cudaMalloc(&da, sizeof ha); cudaMalloc(&db, sizeof hb); cudaMalloc(&dout, sizeof ho);
  cudaMalloc(&fa_d, sizeof fa); cudaMalloc(&fb_d, sizeof fb); cudaMalloc(&fo_d, sizeof fo);
  cudaMemcpy(da, ha, sizeof ha, cudaMemcpyHostToDevice); cudaMemcpy(db, hb, sizeof hb, cudaMemcpyHostToDevice);
  cudaMemcpy(fa_d, fa, sizeof fa, cudaMemcpyHostToDevice); cudaMemcpy(fb_d, fb, sizeof fb, cudaMemcpyHostToDevice);
  k<<<1, 32>>>(da, db, dout, n); kf<<<1, 32>>>(fa_d, fb_d, fo_d, 3);
  cudaMemcpy(ho, dout, sizeof ho, cudaMemcpyDeviceToHost); cudaMemcpy(fo, fo_d, sizeof fo, cudaMemcpyDeviceToHost);
  for (int i = 0; i < n; ++i) printf("%g/%g = %g (host %g)\n", ha[i], hb[i], ho[i], ha[i] / hb[i]);
  for (int i = 0; i < 3; ++i) printf("%g/%g = %g (host %g)\n", fa[i], fb[i], fo[i], fa[i] / fb[i]);
}
