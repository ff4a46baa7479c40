// Row access to J for the structure analysis (structure.cu): the stored dense J of a host QP,
// or the device-built QP's J generated on the fly from its row descriptors and
// Gall = [G_0 .. G_{T-1}] (G_k = A_K^k B), so the built QP's J is never materialised
// (1 GB at config 3, 6.5 GB at config 4). Both give the same values, bit
// for bit, so the analysis (hashes, verification, the gathered prototypes P) is identical.
#pragma once
#include <cstdint>

namespace cmpc {

// one row of J: kind 0 mixed (E + F K), 1 state, 2 input; upper bound or lower; stage t; index i
struct RowDesc {
  int kind, upper, t, i;
};

// J as the reference stores it: m x n column-major, ld = m
struct DenseJ {
  const double* J;
  int64_t ld;
  struct Row {
    const double* p;
    int64_t ld;
    __device__ __forceinline__ double operator()(int64_t j) const { return p[j * ld]; }
  };
  __device__ __forceinline__ Row row(int64_t r) const { return Row{J + r, ld}; }
};

// J of the device-built QP (reduction.cpp:191-251): state row (t, i) = +-[G_{t-1} | .. | G_0]
// row i, input row +-(K Gall) row i plus the unit at its own input, mixed row +-((E + F K)
// Gall) row i plus F at its own stage
struct BuiltJ {
  const RowDesc* rows;
  const double *G, *KG, *EG, *F;
  int nx, nu, nc;
  struct Row {
    RowDesc q;
    const double *G, *KG, *EG, *F;
    int nx, nu, nc;
    __device__ __forceinline__ double operator()(int64_t col) const {
      const int j = (int)(col / nu), cc = (int)(col - (int64_t)j * nu);
      const double sg = q.upper ? 1.0 : -1.0;
      double v = 0.0;
      if (j < q.t) {
        const int64_t gc = (int64_t)(q.t - 1 - j) * nu + cc;  // column of G_{t-1-j}
        if (q.kind == 1) v = G[q.i + gc * nx];
        else if (q.kind == 2) v = KG ? KG[q.i + gc * nu] : 0.0;
        else v = EG[q.i + gc * nc];
        v *= sg;
      }
      if (q.kind == 2 && col == (int64_t)q.t * nu + q.i) v += sg;
      if (q.kind == 0 && j == q.t) v += sg * F[q.i + (int64_t)cc * nc];
      return v;
    }
  };
  __device__ __forceinline__ Row row(int64_t r) const { return Row{rows[r], G, KG, EG, F, nx, nu, nc}; }
};

}  // namespace cmpc
