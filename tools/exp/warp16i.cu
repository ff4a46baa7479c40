#include <cstdio>
#include <cuda_runtime.h>
constexpr int kLD = 65;
// 1/sqrt(x) from a float seed and two Newton steps in FP64 (the FP64 sqrt and divide
// sequences cost several hundred cycles each on the pivot's critical path); exact
// fallback outside the float range
__device__ __forceinline__ double rsqrt_fast(double x) {
  if (x > 1e-30 && x < 1e30) {
    double y = (double)rsqrtf((float)x);
    const double hx = 0.5 * x;
    y = y * fma(-hx * y, y, 1.5);
    y = y * fma(-hx * y, y, 1.5);
    return y;
  }
  return 1.0 / sqrt(x);
}

constexpr unsigned kFull = 0xffffffffu;

// One warp factors the 16 x 16 lower block of a at (o, o) in registers (lane & 15 = row;
// lanes 16..31 mirror 0..15 so every shuffle is warp-uniform) and writes L and L^{-1}
// (into w) back to shared memory. Returns the first failing local pivot or -1.
// The step loops are deliberately not unrolled (the register row is rotated instead of
// indexed): a fully unrolled body is ~30 KB of straight-line SASS whose instruction fetch,
// not the arithmetic, set the pace (27k cycles measured vs ~4k for this form).
__device__ int warp_potf2_inv16(double* a, double* w, int o, int bvalid, double* bc) {
  // bc: 2 x 32 doubles of shared scratch, double-buffered by step parity:
  // [0,16) column j of L, [16,32) row j of W
  const int lane = threadIdx.x & 31, row = lane & 15;
  double r[16], wr[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    r[k] = (k <= row) ? a[(o + row) + (o + k) * kLD] : 0.0;
    wr[k] = (k == row) ? 1.0 : 0.0;
  }
  int fail = -1;
  // step j: factor column j of L and, interleaved, step j of the substitution L W = I
  // (row j of W is final once scaled by 1/l_jj; rows below subtract l_ij W_j). The column
  // and the row are broadcast through shared memory: a 64-bit shuffle costs ~10 issue
  // cycles per lane-pair on one warp, a broadcast LDS far less.
  long long T0 = clock64(), TA = 0, TB = 0, TC = 0, TD = 0;
#pragma unroll 1
  for (int j = 0; j < 16; ++j) {
    long long s0 = clock64();
    double* cb = bc + 32 * (j & 1);
    // r[0] holds column j of this row (rotated)
    const double pj = __shfl_sync(kFull, r[0], j);
    if (fail < 0 && j < bvalid && (!(pj > 0.0) || !isfinite(pj))) fail = j;
    const double y = rsqrt_fast(pj);
    long long s1 = clock64(); TA += s1 - s0;
    double lij = r[0];
    if (row == j) {
      lij = pj * y;
#pragma unroll
      for (int k = 0; k < 16; ++k) wr[k] *= y;
      if (lane == j) {
#pragma unroll
        for (int k = 0; k < 16; ++k) cb[16 + k] = wr[k];
      }
    } else if (row > j) {
      lij = r[0] * y;
    }
    if (lane < 16) {
      cb[row] = lij;
      if (row >= j) a[(o + row) + (o + j) * kLD] = lij;
    }
    __syncwarp();
    long long s2 = clock64(); TB += s2 - s1;
    if (row > j) {
#pragma unroll
      for (int k = 1; k < 16; ++k) {
        if (row >= j + k) r[k] = fma(-lij, cb[(j + k) & 15], r[k]);
      }
#pragma unroll
      for (int k = 0; k < 16; ++k) wr[k] = fma(-lij, cb[16 + k], wr[k]);
    }
    long long s3 = clock64(); TC += s3 - s2;
#pragma unroll
    for (int k = 0; k < 15; ++k) r[k] = r[k + 1];
    r[15] = 0.0;
    TD += clock64() - s3;
  }
  if (threadIdx.x == 0) printf("loop %lld: pivot+rsqrt %lld, publish %lld, update %lld, rotate %lld\n", clock64() - T0, TA, TB, TC, TD);
  if (fail >= 0) return fail;
  if (lane < 16) {
#pragma unroll
    for (int k = 0; k < 16; ++k) w[(o + row) + (o + k) * kLD] = (k <= row) ? wr[k] : 0.0;
  }
  return -1;
}

__global__ void bench(double* out, long long* clk, int reps) {
  __shared__ double a[20 * 65], w[20 * 65], bc[64];
  const int lane = threadIdx.x;
  for (int e = lane; e < 20 * 65; e += 32) { a[e] = 0.0; w[e] = 0.0; }
  __syncwarp();
  long long tot = 0;
  for (int rep = 0; rep < reps; ++rep) {
    for (int e = lane; e < 16 * 16; e += 32) { int i = e & 15, k = e >> 4; a[i + k * kLD] = (i == k) ? 20.0 : 1.0 / (1 + i + k); }
    __syncwarp();
    long long t0 = clock64();
    int f = warp_potf2_inv16(a, w, 0, 16, bc);
    __syncwarp();
    long long t1 = clock64();
    tot += t1 - t0;
    if (f >= 0) out[1] = f;
  }
  if (lane == 0) { clk[0] = tot / reps; out[0] = w[5 + 3 * kLD]; }
}
int main() {
  double* d; long long* c; cudaMalloc(&d, 16); cudaMalloc(&c, 8);
  bench<<<1, 32>>>(d, c, 1); cudaDeviceSynchronize();
  bench<<<1, 32>>>(d, c, 2); cudaDeviceSynchronize();
  long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("warp_potf2_inv16: %lld cycles/call (%s)\n", h, cudaGetErrorString(cudaGetLastError()));
}
