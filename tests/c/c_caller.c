/* A plain C caller of the drop-in boundary (include/condmpc_cuda.h): what a binding written
 * against the header does. Compiled with gcc -std=c11 -Wall -Werror against
 * the header and linked against libcondmpc_cuda.so by tests/test_c_caller.py, so a drift
 * between the header and the library's exports fails the build; run on a GPU it solves the
 * reference's bound_toy (proj/tests/test_ipm.cpp:28-31: H = 4, h = 2, -v <= 0) with the
 * reference's expectations (:378-385: v ~ 0, z ~ 2, s > 0) and a second 1-D case whose upper
 * bound is active (v = 0.5, objective -1.5). */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include "condmpc_cuda.h"

static int n_log = 0;
static void on_log(void* user, const double* rec) {
  (void)user;
  (void)rec;
  ++n_log;
}

static int solve_toy(double H, double h, double J, double d, double* v_out, double* obj, double* z_out,
                     double* s_out) {
  cmpc_ctx* ctx = NULL;
  if (cmpc_ctx_create(&ctx, 0) != CMPC_OK) {
    fprintf(stderr, "ctx_create: %s\n", cmpc_last_error());
    return 1;
  }
  if (cmpc_load_qp(ctx, 1, 1, &H, &h, 0.0, &J, &d, 0) != CMPC_OK) {
    fprintf(stderr, "load_qp: %s\n", cmpc_last_error());
    cmpc_ctx_destroy(ctx);
    return 1;
  }
  const double opts[5] = {1e-8, 0.1, 0.2, 0.995, 1e-4}; /* tol, mu_init, kappa_mu, tau, armijo_eta */
  double v = 0.0, s = 0.0, lam = 0.0, z = 0.0, out[14];
  const int rc = cmpc_solve(ctx, opts, 200, &v, &s, &lam, &z, out, on_log, NULL, NULL);
  cmpc_ctx_destroy(ctx);
  if (rc != CMPC_OK) {
    fprintf(stderr, "solve: %s\n", cmpc_last_error());
    return 1;
  }
  if (out[0] != 0.0) {
    fprintf(stderr, "status %g\n", out[0]);
    return 1;
  }
  *v_out = v;
  *obj = out[3];
  *z_out = z;
  *s_out = s;
  return 0;
}

int main(void) {
  if (cmpc_abi_version() != 1) {
    fprintf(stderr, "abi version %d\n", cmpc_abi_version());
    return 2;
  }
  double v = 0.0, obj = 0.0, z = 0.0, s = 0.0;
  /* bound_toy: min 2 v^2 + 2 v  s.t.  -v <= 0: the bound is active, v = 0, z = 2 */
  if (solve_toy(4.0, 2.0, -1.0, 0.0, &v, &obj, &z, &s)) return 1;
  if (fabs(v) > 1e-7 || fabs(z - 2.0) > 2e-5 || !(s > 0.0) || !(z > 0.0)) {
    fprintf(stderr, "bound_toy: v %.17g z %.17g s %.17g\n", v, z, s);
    return 1;
  }
  /* min 2 v^2 - 4 v  s.t.  v <= 0.5: the bound is active, v = 0.5, objective -1.5 */
  if (solve_toy(4.0, -4.0, 1.0, 0.5, &v, &obj, &z, &s)) return 1;
  if (fabs(v - 0.5) > 1e-6 || fabs(obj + 1.5) > 1e-6) {
    fprintf(stderr, "bound: v %.17g obj %.17g\n", v, obj);
    return 1;
  }
  /* errors surface as codes, not crashes */
  if (cmpc_load_qp(NULL, 1, 1, NULL, NULL, 0.0, NULL, NULL, 0) >= 0) return 3;
  printf("c caller ok: %d log records\n", n_log);
  return 0;
}
