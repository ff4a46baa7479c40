// Latency of a 32 x 32 Cholesky factor + triangular inverse inside one CTA (tools only):
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo f32_bench.cu -o f32_bench
// V1: warp 0 factors (lane i = row i in registers, pivot diagonal replicated in every lane,
//     column broadcast by shfl) and forms W = L^-1 by Gauss-Jordan on the identity rows.
// V2: warp 0 factors and publishes each column to shared memory; warp 1 forms W columns
//     (lane c = column c) trailing the factor.
// V3: factor only.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                              \
  do {                                                                     \
    cudaError_t e = (x);                                                   \
    if (e != cudaSuccess) {                                                \
      printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e));     \
      exit(1);                                                             \
    }                                                                      \
  } while (0)

constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ double rsqrt_mufu(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double hx = 0.5 * x;
  y = y * fma(-hx * y, y, 1.5);
  y = y * fma(-hx * y, y, 1.5);
  return y;
}

// lane i holds row i of A (a[c], c <= i meaningful). On return a = row i of L, w = row i of W.
template <bool INV>
__device__ __forceinline__ int factor32(double (&a)[32], double (&w)[32], double (&rs)[32]) {
  const int lane = threadIdx.x & 31;
  double dg[32];
#pragma unroll
  for (int c = 0; c < 32; ++c) dg[c] = __shfl_sync(kFull, a[c], c);
  if (INV) {
#pragma unroll
    for (int c = 0; c < 32; ++c) w[c] = (c == lane) ? 1.0 : 0.0;
  }
  int fail = -1;
#pragma unroll
  for (int p = 0; p < 32; ++p) {
    const double d = dg[p];
    if (fail < 0 && (!(d > 0.0) || !isfinite(d))) fail = p;
    const double r = rsqrt_mufu(d);
    rs[p] = r;
    const double l = (lane >= p) ? a[p] * r : 0.0;
    a[p] = l;
#pragma unroll
    for (int c = p + 1; c < 32; ++c) {
      const double lc = __shfl_sync(kFull, l, c);
      a[c] = fma(-l, lc, a[c]);
      dg[c] = fma(-lc, lc, dg[c]);
    }
    if (INV) {
#pragma unroll
      for (int c = 0; c <= p; ++c) {
        const double wp = __shfl_sync(kFull, w[c], p) * r;  // row p of W, scaled
        w[c] = (lane == p) ? wp : ((lane > p) ? fma(-l, wp, w[c]) : w[c]);
      }
    }
  }
  return fail;
}

struct Out {
  long long t0, t1;
  int fail;
};

// V1 / V3
template <bool INV>
__global__ void k_v1(const double* A, double* L, double* W, Out* out, int reps) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __shared__ double sw[32 * 33];
  if (warp == 0) {
    double a[32], w[32], rs[32];
    long long t0 = 0, t1 = 0;
    int f = 0;
    for (int it = 0; it < reps; ++it) {
#pragma unroll
      for (int c = 0; c < 32; ++c) a[c] = (c <= lane) ? A[lane + 32 * c] : 0.0;
      __syncwarp();
      t0 = clock64();
      f = factor32<INV>(a, w, rs);
      __syncwarp();
      // consume every result so nothing is dead code
      double s = 0.0;
#pragma unroll
      for (int c = 0; c < 32; ++c) s += a[c] + (INV ? w[c] : 0.0);
      sw[lane] = s;
      __syncwarp();
      t1 = clock64();
    }
#pragma unroll
    for (int c = 0; c < 32; ++c) {
      L[lane + 32 * c] = a[c];
      if (INV) W[lane + 32 * c] = w[c];
    }
    if (lane == 0) {
      out->t0 = t0;
      out->t1 = t1;
      out->fail = f + (int)(sw[0] * 0.0);
    }
  }
}

// V2: warp 0 factors, publishes column p (l values) + r_p to shared memory and a counter;
// warp 1 lane c builds column c of W: w(p) = s(p) r_p; s(i) -= l_ip w(p), i > p.
__global__ void k_v2(const double* A, double* L, double* W, Out* out, int reps) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __shared__ double col[32][33];  // col[p][i] = l_ip
  __shared__ double rr[32];
  __shared__ volatile int cnt;
  long long t0 = 0, t1 = 0;
  int f = 0;
  for (int it = 0; it < reps; ++it) {
    if (threadIdx.x == 0) cnt = 0;
    __syncthreads();
    if (warp == 0) {
      double a[32], w[32], rs[32];
#pragma unroll
      for (int c = 0; c < 32; ++c) a[c] = (c <= lane) ? A[lane + 32 * c] : 0.0;
      __syncwarp();
      t0 = clock64();
      // factor, publishing each column as it is finished
      double dg[32];
#pragma unroll
      for (int c = 0; c < 32; ++c) dg[c] = __shfl_sync(kFull, a[c], c);
      f = -1;
#pragma unroll
      for (int p = 0; p < 32; ++p) {
        const double d = dg[p];
        if (f < 0 && (!(d > 0.0) || !isfinite(d))) f = p;
        const double r = rsqrt_mufu(d);
        const double l = (lane >= p) ? a[p] * r : 0.0;
        a[p] = l;
        col[p][lane] = l;
        if (lane == 0) rr[p] = r;
        __syncwarp();
        if (lane == 0) {
          __threadfence_block();
          cnt = p + 1;
        }
#pragma unroll
        for (int c = p + 1; c < 32; ++c) {
          const double lc = __shfl_sync(kFull, l, c);
          a[c] = fma(-l, lc, a[c]);
          dg[c] = fma(-lc, lc, dg[c]);
        }
      }
      (void)w;
      (void)rs;
#pragma unroll
      for (int c = 0; c < 32; ++c) L[lane + 32 * c] = a[c];
    } else if (warp == 1) {
      double s[32];
#pragma unroll
      for (int i = 0; i < 32; ++i) s[i] = (i == lane) ? 1.0 : 0.0;
#pragma unroll
      for (int p = 0; p < 32; ++p) {
        while (cnt <= p) {
        }
        __syncwarp();
        const double wp = s[p] * rr[p];
        s[p] = wp;
#pragma unroll
        for (int i = p + 1; i < 32; ++i) s[i] = fma(-col[p][i], wp, s[i]);
      }
      t1 = clock64();
      // s[i] = W(i, lane)
#pragma unroll
      for (int i = 0; i < 32; ++i) W[i + 32 * lane] = (i >= lane) ? s[i] : 0.0;
    }
    __syncthreads();
  }
  __shared__ long long st0;
  if (threadIdx.x == 0) st0 = t0;
  __syncthreads();
  if (threadIdx.x == 32) {
    out->t0 = st0;
    out->t1 = t1;
    out->fail = 0;
  }
  (void)f;
}


__device__ __forceinline__ double rcp_mufu(double x) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  double e = fma(-x, y, 1.0);
  y = fma(y, e, y);
  e = fma(-x, y, 1.0);
  y = fma(y, e, y);
  return y;
}
__device__ __forceinline__ double2 ld2(const double* p) { return *reinterpret_cast<const double2*>(p); }

// V4: warp 0 factors (next pivot by one shfl, columns broadcast through shared memory),
// warp 1 forms W columns trailing it (same shared columns)
template <bool WARP1, bool RANGE, bool SLEEP, bool RCP = false>
__global__ void k_v4(const double* A, double* L, double* W, Out* out, int reps) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __shared__ __align__(16) double col[32 * 32];
  __shared__ double rr[32];
  __shared__ volatile int cnt;
  long long t0 = 0, t1 = 0, t2 = 0;
  int f = -1;
  for (int it = 0; it < reps; ++it) {
    if (threadIdx.x == 0) cnt = 0;
    __syncthreads();
    if (warp == 0) {
      double a[32];
#pragma unroll
      for (int c = 0; c < 32; ++c) a[c] = (c <= lane) ? A[lane + 32 * c] : 0.0;
      __syncwarp();
      t0 = clock64();
      double dcur = __shfl_sync(kFull, a[0], 0);
      f = -1;
#pragma unroll
      for (int p = 0; p < 32; ++p) {
        if (f < 0 && (!(dcur > 0.0) || !isfinite(dcur))) f = p;
        double r;
        if (!RANGE || (dcur >= 1e-300 && dcur <= 1e300)) r = rsqrt_mufu(dcur);
        else r = 1.0 / sqrt(dcur);
        if (RCP && p < 31) {
          const double q = a[p] * a[p];
          const double dn = fma(-q, rcp_mufu(dcur), a[p + 1]);
          dcur = __shfl_sync(kFull, dn, p + 1);
        }
        const double l = (lane >= p) ? a[p] * r : 0.0;
        a[p] = l;
        if (!RCP && p < 31) {
          const double dn = fma(-l, l, a[p + 1]);
          dcur = __shfl_sync(kFull, dn, p + 1);
        }
        col[p * 32 + lane] = l;
        if (lane == 0) rr[p] = r;
        __syncwarp();
        if (lane == 0) {
          __threadfence_block();
          cnt = p + 1;
        }
#pragma unroll
        for (int c = (p + 1) & ~1; c < 32; c += 2) {
          const double2 lc = ld2(col + p * 32 + c);
          if (c > p) a[c] = fma(-l, lc.x, a[c]);
          if (c + 1 > p) a[c + 1] = fma(-l, lc.y, a[c + 1]);
        }
      }
      t1 = clock64();
#pragma unroll
      for (int c = 0; c < 32; ++c) L[lane + 32 * c] = a[c];
    } else if (warp == 1 && WARP1) {
      double s[32];
#pragma unroll
      for (int i = 0; i < 32; ++i) s[i] = (i == lane) ? 1.0 : 0.0;
#pragma unroll
      for (int p = 0; p < 32; ++p) {
        while (cnt <= p) {
          if (SLEEP) __nanosleep(32);
        }
        __threadfence_block();
        const double wp = s[p] * rr[p];
        s[p] = wp;
#pragma unroll
        for (int i = (p + 1) & ~1; i < 32; i += 2) {
          const double2 lc = ld2(col + p * 32 + i);
          if (i > p) s[i] = fma(-lc.x, wp, s[i]);
          if (i + 1 > p) s[i + 1] = fma(-lc.y, wp, s[i + 1]);
        }
      }
      t2 = clock64();
#pragma unroll
      for (int i = 0; i < 32; ++i) W[i + 32 * lane] = (i >= lane) ? s[i] : 0.0;
    }
    __syncthreads();
  }
  __shared__ long long st[2];
  if (threadIdx.x == 0) { st[0] = t0; st[1] = t1; }
  __syncthreads();
  if (threadIdx.x == 32) {
    out->t0 = st[0];
    out->t1 = t2;
    out->fail = (int)(st[1] - st[0]);
  }
}


// V5: two pivots per round (2x2 blocked pivot chain): column pair (p, p+1) formed with two
// rsqrt, one shared-memory broadcast round and one mbarrier-free counter signal per pair
template <bool WARP1>
__global__ void k_v5(const double* A, double* L, double* W, Out* out, int reps) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __shared__ __align__(16) double col[32 * 32];
  __shared__ double rr[32];
  __shared__ volatile int cnt;
  long long t0 = 0, t1 = 0, t2 = 0;
  for (int it = 0; it < reps; ++it) {
    if (threadIdx.x == 0) cnt = 0;
    __syncthreads();
    if (warp == 0) {
      double a[32];
#pragma unroll
      for (int c = 0; c < 32; ++c) a[c] = (c <= lane) ? A[lane + 32 * c] : 0.0;
      __syncwarp();
      t0 = clock64();
      double d1 = __shfl_sync(kFull, a[0], 0);
#pragma unroll
      for (int p = 0; p < 32; p += 2) {
        const double r1 = rsqrt_mufu(d1);
        const double l1 = (lane >= p) ? a[p] * r1 : 0.0;
        const double l21 = __shfl_sync(kFull, l1, p + 1);
        const double d2 = __shfl_sync(kFull, fma(-l1, l1, a[p + 1]), p + 1);
        const double r2 = rsqrt_mufu(d2);
        const double l2 = (lane >= p + 1) ? fma(-l1, l21, a[p + 1]) * r2 : 0.0;
        if (p + 2 < 32) d1 = __shfl_sync(kFull, fma(-l2, l2, fma(-l1, l1, a[p + 2])), p + 2);
        a[p] = l1;
        a[p + 1] = l2;
        col[p * 32 + lane] = l1;
        col[(p + 1) * 32 + lane] = l2;
        if (lane == 0) {
          rr[p] = r1;
          rr[p + 1] = r2;
        }
        __syncwarp();
#pragma unroll
        for (int c = (p + 2); c < 32; c += 2) {
          const double2 c1 = ld2(col + p * 32 + c);
          const double2 c2 = ld2(col + (p + 1) * 32 + c);
          a[c] = fma(-l2, c2.x, fma(-l1, c1.x, a[c]));
          a[c + 1] = fma(-l2, c2.y, fma(-l1, c1.y, a[c + 1]));
        }
        if (WARP1 && lane == 0) {
          __threadfence_block();
          cnt = p + 2;
        }
      }
      t1 = clock64();
#pragma unroll
      for (int c = 0; c < 32; ++c) L[lane + 32 * c] = a[c];
    } else if (warp == 1 && WARP1) {
      double s[32];
#pragma unroll
      for (int i = 0; i < 32; ++i) s[i] = (i == lane) ? 1.0 : 0.0;
#pragma unroll
      for (int p = 0; p < 32; ++p) {
        if ((p & 1) == 0)
          while (cnt <= p) __nanosleep(20);
        __threadfence_block();
        const double wp = s[p] * rr[p];
        s[p] = wp;
#pragma unroll
        for (int i = (p + 1) & ~1; i < 32; i += 2) {
          const double2 lc = ld2(col + p * 32 + i);
          if (i > p) s[i] = fma(-lc.x, wp, s[i]);
          if (i + 1 > p) s[i + 1] = fma(-lc.y, wp, s[i + 1]);
        }
      }
      t2 = clock64();
#pragma unroll
      for (int i = 0; i < 32; ++i) W[i + 32 * lane] = (i >= lane) ? s[i] : 0.0;
    }
    __syncthreads();
  }
  __shared__ long long st[2];
  if (threadIdx.x == 0) { st[0] = t0; st[1] = t1; }
  __syncthreads();
  if (threadIdx.x == (WARP1 ? 32 : 0)) {
    out->t0 = st[0];
    out->t1 = WARP1 ? t2 : st[1];
    out->fail = (int)(st[1] - st[0]);
  }
}

int main(int argc, char** argv) {
  const int reps = argc > 1 ? atoi(argv[1]) : 3;
  const int n = 32;
  std::vector<double> G(n * n), A(n * n, 0.0);
  srand(3);
  for (auto& g : G) g = rand() / double(RAND_MAX) - 0.5;
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      double s = (i == j) ? 4.0 : 0.0;
      for (int k = 0; k < n; ++k) s += G[i * n + k] * G[j * n + k];
      A[i + j * n] = s;
    }
  // host reference
  std::vector<double> Lr(n * n, 0.0), Wr(n * n, 0.0);
  for (int j = 0; j < n; ++j) {
    double d = A[j + j * n];
    for (int k = 0; k < j; ++k) d -= Lr[j + k * n] * Lr[j + k * n];
    Lr[j + j * n] = std::sqrt(d);
    for (int i = j + 1; i < n; ++i) {
      double s = A[i + j * n];
      for (int k = 0; k < j; ++k) s -= Lr[i + k * n] * Lr[j + k * n];
      Lr[i + j * n] = s / Lr[j + j * n];
    }
  }
  for (int c = 0; c < n; ++c)
    for (int i = c; i < n; ++i) {
      double s = (i == c) ? 1.0 : 0.0;
      for (int k = c; k < i; ++k) s -= Lr[i + k * n] * Wr[k + c * n];
      Wr[i + c * n] = s / Lr[i + i * n];
    }
  double *dA, *dL, *dW;
  Out* dO;
  CK(cudaMalloc(&dA, 8 * n * n));
  CK(cudaMalloc(&dL, 8 * n * n));
  CK(cudaMalloc(&dW, 8 * n * n));
  CK(cudaMalloc(&dO, sizeof(Out)));
  CK(cudaMemcpy(dA, A.data(), 8 * n * n, cudaMemcpyHostToDevice));
  auto check = [&](const char* name, bool inv) {
    std::vector<double> L(n * n), W(n * n);
    Out o;
    CK(cudaMemcpy(L.data(), dL, 8 * n * n, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(W.data(), dW, 8 * n * n, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(&o, dO, sizeof(Out), cudaMemcpyDeviceToHost));
    double eL = 0, eW = 0;
    for (int i = 0; i < n; ++i)
      for (int j = 0; j <= i; ++j) {
        eL = fmax(eL, fabs(L[i + j * n] - Lr[i + j * n]));
        if (inv) eW = fmax(eW, fabs(W[i + j * n] - Wr[i + j * n]));
      }
    printf("%s: %lld cycles (%.2f us at 1.965 GHz), max|dL| %.2e max|dW| %.2e fail %d\n", name,
           o.t1 - o.t0, (o.t1 - o.t0) / 1965.0, eL, eW, o.fail);
  };
  CK(cudaMemset(dW, 0, 8 * n * n));
  k_v1<false><<<1, 128>>>(dA, dL, dW, dO, reps);
  CK(cudaDeviceSynchronize());
  check("V3 factor only       ", false);
  k_v1<true><<<1, 128>>>(dA, dL, dW, dO, reps);
  CK(cudaDeviceSynchronize());
  check("V1 factor + GJ inv   ", true);
  k_v2<<<1, 128>>>(dA, dL, dW, dO, reps);
  CK(cudaDeviceSynchronize());
  check("V2 factor | W warp   ", true);
  k_v4<true, true, false><<<1, 128>>>(dA, dL, dW, dO, reps);
  CK(cudaDeviceSynchronize());
  check("V4 smem bcast + W warp (fail = factor-only cycles)", true);
  k_v4<false, true, false><<<1, 128>>>(dA, dL, dW, dO, reps);
  CK(cudaDeviceSynchronize());
  check("V4b no W warp", false);
  k_v4<false, false, false><<<1, 128>>>(dA, dL, dW, dO, reps);
  CK(cudaDeviceSynchronize());
  check("V4c no W warp, no range branch", false);
  k_v4<true, false, true><<<1, 128>>>(dA, dL, dW, dO, reps);
  CK(cudaDeviceSynchronize());
  check("V4d W warp nanosleep spin, no range branch", true);
  k_v4<true, false, true, true><<<1, 128>>>(dA, dL, dW, dO, reps);
  CK(cudaDeviceSynchronize());
  check("V4e = V4d with the rcp pivot chain", true);
  k_v5<false><<<1, 128>>>(dA, dL, dW, dO, reps);
  CK(cudaDeviceSynchronize());
  check("V5 two pivots per round, factor only", false);
  k_v5<true><<<1, 128>>>(dA, dL, dW, dO, reps);
  CK(cudaDeviceSynchronize());
  check("V5 two pivots per round + W warp (fail = factor cycles)", true);
  return 0;
}
