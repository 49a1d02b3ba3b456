// Device check of the router epilogue's running top-K insertion (bo_gemm.cu topk_insert):
// tie-heavy random rows, one thread per row, compared with a stable host sort.
#include <cstdio>
#include <cmath>
#include <vector>
#include <random>
#include <algorithm>
template <int KMAX>
__host__ __device__ __forceinline__ void topk_insert(float (&tv)[KMAX], int (&ti)[KMAX], float v, int e) {
  bool beats[KMAX];
#pragma unroll
  for (int j = 0; j < KMAX; ++j) beats[j] = v > tv[j];
#pragma unroll
  for (int j = KMAX - 1; j > 0; --j) {
    tv[j] = beats[j] ? (beats[j - 1] ? tv[j - 1] : v) : tv[j];
    ti[j] = beats[j] ? (beats[j - 1] ? ti[j - 1] : e) : ti[j];
  }
  tv[0] = beats[0] ? v : tv[0];
  ti[0] = beats[0] ? e : ti[0];
}
__global__ void k(const float* L, int n, int m, int* out) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  float tv[8]; int ti[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) { tv[j] = -INFINITY; ti[j] = j; }
  for (int c = 0; c < m; c += 32) {
    float a[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) a[i] = c + i < m ? L[(size_t)t * m + c + i] : 0.f;
#pragma unroll
    for (int i = 0; i < 32; ++i) if (c + i < m) topk_insert<8>(tv, ti, a[i], c + i);
  }
  for (int j = 0; j < 8; ++j) out[t * 8 + j] = ti[j];
}
int main() {
  const int n = 4096;
  int bad = 0;
  for (int m : {32, 64, 128}) {
    std::mt19937 rng(m);
    std::vector<float> L((size_t)n * m);
    for (auto& x : L) x = (float)((int)(rng() % 9) - 4) * 0.5f;
    float* dL; int* dO;
    cudaMalloc(&dL, L.size() * 4); cudaMalloc(&dO, n * 8 * 4);
    cudaMemcpy(dL, L.data(), L.size() * 4, cudaMemcpyHostToDevice);
    k<<<(n + 127) / 128, 128>>>(dL, n, m, dO);
    std::vector<int> O(n * 8);
    cudaMemcpy(O.data(), dO, O.size() * 4, cudaMemcpyDeviceToHost);
    int badm = 0;
    for (int t = 0; t < n; ++t) {
      std::vector<int> idx(m); for (int i = 0; i < m; ++i) idx[i] = i;
      std::stable_sort(idx.begin(), idx.end(), [&](int a, int b) { return L[(size_t)t * m + a] > L[(size_t)t * m + b]; });
      for (int j = 0; j < 8; ++j) if (idx[j] != O[t * 8 + j]) { if (badm < 3) { printf("m=%d t=%d j=%d dev", m, t, j); for (int q = 0; q < 8; ++q) printf(" %d", O[t*8+q]); printf(" | ref"); for (int q = 0; q < 8; ++q) printf(" %d", idx[q]); printf("\n"); } badm++; break; }
    }
    printf("m=%d bad rows %d of %d (%s)\n", m, badm, n, cudaGetErrorString(cudaGetLastError()));
    bad += badm;
  }
  return bad ? 1 : 0;
}
