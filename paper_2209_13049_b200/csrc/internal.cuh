// Device-resident condensed-space IPM context and the launcher interface between
// the kernel files (structure.cu, syrk.cu, chol.cu, vec.cu) and the C ABI (capi.cu)
// plus the host loop (ipm_host.cpp).
//
// Data layout in HBM (all FP64, column-major like Eigen::MatrixXd):
//   H   n x n (ld n)          J   m x n (ld m, the caller's dense constraint Jacobian)
//   P   ldp x n               the distinct rows of J ("prototypes"), K-major: J = Pi P
//                             with Pi an m x p signed selection (each row of J is +-1 x one
//                             prototype). SYRK prototypes (>=2 nonzeros) come first, sorted
//                             by their nonzero prefix width hi ascending; singleton rows
//                             (one nonzero, e.g. input bounds) are diagonal terms.
//   M   n x n lower           H + J' diag(z/s) J (+ shift); L n x n lower Cholesky factor
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "common.cuh"
#include "../../include/condmpc_cuda.h"

namespace cmpc {

constexpr int kTile = 64;      // SYRK / Cholesky output tile
constexpr int kBK = 32;        // SYRK k rows per pipeline stage
constexpr int kPartBlocks = 2048;  // max grid of the m-length row passes: one row per thread up to 524k rows

// small scalar packet read back at the two sync points of an iteration
struct Packet {
  // residual pass (packet A)
  double kkt, max_r1, max_r3, max_comp, max_lam, max_s, max_z, max_h;
  double obj_vHv, obj_hv, sum_log_s, sum_abs_r3, objective;
  // step (packet B)
  double alpha_s_min, alpha_z_min;  // tau-ratio minima (1.0 when no blocking entry)
  double d_gpv, d_ps_s;             // (Hv+h).pv, sum ps/s
  long long info;                   // Cholesky failing pivot + 1 (0 = ok)
  long long any_nonpos;             // trial slack positivity violated
  // trial merit pieces
  double t_vHv, t_hv, t_sum_log, t_sum_abs;
  double pad[8];
};

// the allreduced groups of the sharded solve are contiguous
static_assert(offsetof(Packet, sum_abs_r3) == offsetof(Packet, sum_log_s) + 8, "packet layout");
static_assert(offsetof(Packet, max_z) == offsetof(Packet, max_r3) + 32, "packet layout");
static_assert(offsetof(Packet, alpha_z_min) == offsetof(Packet, alpha_s_min) + 8, "packet layout");
static_assert(offsetof(Packet, t_sum_abs) == offsetof(Packet, t_sum_log) + 8, "packet layout");

// NVTX range for profilers (nsys / ncu --nvtx); header-only NVTX 3, free without a tool attached
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

struct Workspace;
struct ProblemDev;

struct Ctx {
  int device = 0;
  // row-sharded solve (comm.cpp): this context holds rows of J; partial sums are allreduced
  void* comm = nullptr;  // ncclComm_t, or the LoopGroup when comm_loop
  bool comm_loop = false;  // in-process loopback communicator (tests: N ranks on one GPU)
  int nranks = 1, rank = 0;
  int64_t m_all = -1;    // rows of the whole QP (kkt scaling); -1 = m
  cudaStream_t stream = nullptr;
  bool owns_stream = true;
  void* prob = nullptr;  // ProblemDev (builder.cu): the structured problem behind a device-built QP
  bool pk_autoreset = false;  // inside the host loop: k_publish resets the packet's accumulators

  int64_t n = 0, m = 0;
  double h0 = 0.0;
  // problem (device)
  double *H = nullptr, *h = nullptr, *J = nullptr, *d = nullptr;
  bool owns_J = true;

  // structure of J
  int64_t ps = 0;   // SYRK prototypes
  int64_t pz = 0;   // singleton prototypes (incl. all-zero rows)
  int64_t p = 0;    // ps + pz
  int64_t ldp = 0;  // padded leading dimension of P (multiple of kBK, >= ps)
  double* P = nullptr;           // ldp x n
  int32_t* hi = nullptr;         // ps: nonzero prefix width
  int32_t* start_col = nullptr;  // n+1: first SYRK prototype with hi > c
  int32_t* row_map = nullptr;    // m: proto << 1 | (sign < 0)
  int32_t* mem_ptr = nullptr;    // p+1
  int32_t* mem_rows = nullptr;   // m: row << 1 | (sign < 0)
  int64_t zero_k = -1;           // prototype index of the all-zero row group (-1: none)
  int32_t* sing_col = nullptr;   // pz (ascending)
  double* sing_val = nullptr;    // pz
  int32_t* sing_ptr = nullptr;   // n+1: singleton prototypes of column j are [sing_ptr[j], sing_ptr[j+1])
  int32_t* proto_big = nullptr;  // prototypes with more than 8 member rows (k_proto_reduce warp path)
  int nbig = 0;
  int64_t nzero = 0;  // member rows of the zero prototype (zero_k)
  bool h_symmetric = false;      // H == H' bitwise: H x as column dots
  std::vector<int32_t> h_start_col;

  // Markov-table prototypes (markov.cu): for a device-built QP whose SYRK
  // prototypes are all state rows, P is never stored. State row (t, i) of J is
  // [G_{t-1} .. G_0] row i (G_k = A_K^k B), a window of row i of the Markov table
  //   MK[q, s] = G_{T-1-s/nu}[order(q), s % nu]   (nq x T nu, column-major, ld ldmk)
  // starting at column (T - t) nu; the table's zero tail ends every row's nonzero prefix.
  // The prototype space is laid out stage-major in 32-row chunks: stage t holds Q rows
  // [0, cnt_t) (states ordered by the first stage their B-response is nonzero, so these are
  // exactly the states whose row at stage t is nonzero), padded to a chunk multiple.
  // option "markov": 0 never, 1 (default) when the QP allows it and the materialised P would
  // exceed kMarkovMinBytes (below that P is L2-sized and its plain passes are the faster
  // ones), 2 whenever the QP allows it
  int opt_markov = 1;
  bool markov = false;           // active for the loaded QP
  double* mk = nullptr;          // the Markov table
  int64_t ldmk = 0, mk_cols = 0, mk_nq = 0;
  int mk_T = 0, mk_nu = 0, mk_nchunks = 0;
  int64_t mk_ps = 0;             // prototype rows of the layout (32 x chunks)
  int mk_nx = 0;                 // sources: states [0, nx), inputs [nx, nx + nu), mixed after
  bool mk_inputs = false;        // input rows are table rows (feedback K)
  int32_t* mk_pos = nullptr;     // source (state, input, mixed row) -> table row (-1: none)
  int32_t* mk_base = nullptr;    // T + 2: first prototype row of stage t (t = 0..T; [T+1] = ps)
  int32_t* mk_cnt = nullptr;     // T + 1: padded rows of stage t
  int2* mk_chunk = nullptr;      // per chunk: {table row, column shift (T - t) nu}
  int4* mk_clist = nullptr;      // SYRK plan: chunk lists per column block (full, thin), per
                                 // position {table row, column shift, prototype row}
  int32_t* mk_rbend = nullptr;   // per 32-row table block: end of its nonzero columns
  std::vector<int2> h_mk_chunk;
  std::vector<int32_t> h_mk_width;  // per chunk: its widest row's nonzero prefix (= first row's)

  // SYRK work decomposition (syrk.cu): segments (a k range of one tile) grouped in pieces
  int nunits = 0, ntiles = 0, nctas = 0, npieces = 0;
  int4* units = nullptr;          // segments {tile_i | tile_j << 10 | shape << 20, k0, k1, tile}
  int32_t* cta_ptr = nullptr;     // npieces+1 into units
  unsigned* syrk_ctl = nullptr;   // piece counter, retired CTAs, reduction item counter, per-tile done counts
  int2* tiles = nullptr;          // ntiles {ti, tj}
  int32_t* tile_ptr = nullptr;    // ntiles+1 into tile_units
  int32_t* tile_units = nullptr;  // segment ids per tile in k order (bits 30-31: valid rows 16 x code, 0 = 64)
  double* partial = nullptr;      // nunits x 64 x 64
  double* rhs_part = nullptr;     // nunits x 128: fused P' q half-sums of the diagonal segments
  long long* syrk_prof = nullptr; // debug timeline: {start ns, end ns, smid} per piece (null: off)
  std::vector<double> syrk_cta_cost;  // per piece: segments, k steps per shape (debug timeline)
  void* tmap_P = nullptr;         // CUtensorMap (128 B), host copy passed by value: box {16, 64}
  void* tmap_P32 = nullptr;       // the same over box {16, 32} (thin units' A operand)

  // iterate and per-iteration buffers (device)
  double *v = nullptr, *s = nullptr, *lam = nullptr, *z = nullptr, *r1 = nullptr, *r2 = nullptr,
         *r3 = nullptr;
  double *Hv = nullptr, *Jtl = nullptr, *y = nullptr, *sigma = nullptr, *omega = nullptr,
         *q = nullptr, *rhs = nullptr, *M = nullptr, *L = nullptr;
  double* tq = nullptr;  // J'(r2 - sigma r3) of the step (the SYRK's fused right-hand side part)
  double* Mpack = nullptr;  // sharded: the lower triangle of M packed for the allreduce
  // J'lambda carried along: the recovery forms J' p_lambda = (M - H) pv - tq,
  // the accepted step adds alpha J' p_lambda to Jtl, and the residual pass skips its J pass
  double* JtPl = nullptr;
  bool jtl_recur = false;  // unsharded with rows: the residual after a step reuses Jtl
  // per-context options (cmpc_ctx_set_option; defaults = the measured best forms)
  bool opt_jtl_recur = true;  // "jtl_recurrence": carry J'lambda (else the direct pass)
  int opt_rhs_pass = 0;       // "rhs_pass": 0/1 = fused into the SYRK, 2 = its own pass over P
  bool opt_graphs = true;     // "graphs": capture the per-iteration segments as CUDA graphs
  bool opt_small = true;      // "small_path": whole solve in one CTA when the QP fits (small.cu)
  bool opt_spec = true;       // "speculate": enqueue update + residuals behind the step segment
  // small.cu: the dense J kept for the one-CTA solver (null when the QP does not fit)
  double* Jsmall = nullptr;
  double* small_log = nullptr;
  int64_t small_log_cap = 0;
  double* small_res = nullptr;
  double *pv = nullptr, *ps_ = nullptr, *pl = nullptr, *pzd = nullptr, *Jpv = nullptr,
         *vt = nullptr, *yt = nullptr, *Hvt = nullptr;
  double* yv = nullptr;  // P v of the current point (prototype-indexed, like y = P pv)
  double* part = nullptr;     // kPartBlocks x 16 partial sums
  double* colpart = nullptr;  // Pt q partial: nchunks x n
  int colchunks = 0;
  double* hmax = nullptr;
  double* d_mu = nullptr;    // barrier value on the device (kernels read it: graph-safe)
  // accepted step {alpha, alpha_z, go} on the device, then the residual pass's merit snapshot
  // {max_lam, v'Hv, h'v, sum log s, sum |r3|} (trial0_decide)
  double* d_alpha = nullptr;
  double* stage = nullptr;   // pinned ring for the host -> device scalars (mu, alpha): a copy from
  int stage_i = 0;           // pageable memory is staged and synchronous, from pinned a plain DMA
  // CUDA graphs of the two per-iteration segments (captured on the second iteration)
  cudaStream_t stream2 = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
  cudaGraphExec_t g_step = nullptr, g_next = nullptr;
  long long g_step_nodes = 0, g_next_nodes = 0;
  double g_tau = 0.0;
  double g_eta = 0.0;  // eta baked into the captured seg_step (trial0_decide)
  double* Winv = nullptr;    // inverses of the 32 x 32 diagonal blocks of L
  double* Lt = nullptr;      // packed 32 x 32 off-diagonal tiles of L (dataflow Cholesky)
  unsigned* df_flags = nullptr;  // per-tile done flags (generation stamped)
  unsigned* df_ctl = nullptr;    // generation, exit count, failure, pivot, task counter
  double* df_y = nullptr;        // fused forward-solve blocks (nt x 32)
  double* df_part = nullptr;     // per diagonal block: the pre-accumulated A_{d,d-1}, A_dd and b_d - sum L y
  unsigned* df_pflags = nullptr; // their done flags
  double* df_x = nullptr;        // distributed backward solve (large n): solved blocks (nt x 32)
  unsigned* df_xflags = nullptr; // their done flags
  int df_grid = 148;
  Packet* pk = nullptr;      // device packet
  Packet* pk_host = nullptr; // pinned, device-mapped mirror
  Packet* pk_map = nullptr;  // device address of pk_host (k_publish writes it directly)
  Packet* pk_host_b = nullptr;  // second mirror: seg_step's publish (packet B)
  Packet* pk_map_b = nullptr;
  volatile unsigned long long* pub_host = nullptr;  // mapped publish sequence number
  unsigned long long* pub_map = nullptr;            // its device address
  unsigned long long* pub_dev = nullptr;            // device-side publish counter
  unsigned long long pub_expect = 0;                // publishes enqueued so far
  double mu = 0.0;

  // events for per-phase timing
  cudaEvent_t ev0 = nullptr, ev1 = nullptr, ev2 = nullptr, ev3 = nullptr, ev4 = nullptr;  // ev4: after k_syrk
  double syrk_flops = 0.0;   // algorithmic: sum over prototypes of hi (hi + 1)
  double syrk_bytes = 0.0;   // algorithmic: 8 x nonzeros of P (one read)
};

// ---- structure.cu
void analyze_structure(Ctx& c);
struct BuiltJ;  // jrows.cuh
// the analysis over the device-built QP's J, generated row by row (never stored)
void analyze_structure_built(Ctx& c, const BuiltJ& J);
// the built problem's J (null: the QP was loaded, not built)
const BuiltJ* prob_rows(Ctx& c);
void free_structure(Ctx& c);

// ---- markov.cu
// the Markov table and chunk layout of a built QP (false: not applicable, P is materialised)
bool markov_prepare(Ctx& c);
void markov_free(Ctx& c);
// structure.cu: prototype order -> Markov layout (false: a SYRK prototype is not a state row)
struct MarkovRemap {
  const void* rows;  // RowDesc*
  const int32_t* pos;
  const int32_t* base;
  int64_t ps;  // prototype rows of the Markov layout
  bool force;  // option markov = 2: no size threshold
  int nx, nu;  // source offsets (states, inputs, mixed rows)
  bool inputs;
};
constexpr double kMarkovMinBytes = 64e6;
void launch_markov_gemv(Ctx& c, const double* x, double* y);
void launch_markov_ptq(Ctx& c, const double* q, double* out);

// ---- syrk.cu
void syrk_plan(Ctx& c);
// M(lower) = H + P' diag(omega) P + (singleton diagonal); writes full symmetric M when mirror
void launch_condense(Ctx& c, bool mirror, bool with_rhs = false, cudaEvent_t after_syrk = nullptr);
void syrk_free(Ctx& c);
// ---- small.cu: the whole IPM loop in one CTA for QPs that fit in shared memory
bool small_fits(int64_t n, int64_t m);
int small_solve(Ctx& c, const double* opts, int64_t max_iter, double* v_out, double* s_out, double* lam_out,
                double* z_out, double* out, cmpc_log_fn log, void* user);

// ---- bsyrk.cu: lockstep-batch condensation (batch.cu): B instances sharing H and P, one CTA
// per instance; per-instance omega/q in prototype space at stride s_proto, M (n x n lower),
// tq, rhs and r1 (n) at their natural strides; inactive instances (act = 0) are skipped
struct BatchSyrk {
  int2* chunks = nullptr;            // 32-row chunks of P in processing order: {first row, width}
  int nchunks = 0;
  unsigned char reg[15][4] = {};     // each consumer warp's 16 x 16 output regions
  double flops_per_instance = 0.0;   // algorithmic: sum over SYRK rows of hi (hi + 1)
  int64_t B = 0;
};
void syrk_plan_batch(Ctx& c, int64_t B, BatchSyrk& out, cudaStream_t st);
void syrk_free_batch(BatchSyrk& b, cudaStream_t st);
void launch_condense_batch(Ctx& c, BatchSyrk& bs, cudaStream_t st, const double* omega, const double* q,
                           int64_t s_proto, double* M, double* tq, double* rhs, const double* r1,
                           const int* act);

// ---- chol.cu
// L = chol(M + delta I) (lower, upper zeroed); failing pivot+1 in c.pk->info; with rhs,
// the same kernel also solves L L' x = rhs (x written only when the factorization succeeds)
void launch_cholesky(Ctx& c, const double* M, double* L, double delta, const double* rhs = nullptr,
                     double* x = nullptr);
void chol_alloc(Ctx& c);
void chol_free(Ctx& c);
// diagonal-block inverses of an externally provided factor (set_factor)
void launch_factor_inverses(Ctx& c, const double* L);
// x = L^{-T} L^{-1} b (in place on x allowed); uses the diagonal-block inverses
void launch_chol_solve(Ctx& c, const double* L, const double* b, double* x);

// ---- batch.cu (lockstep batch of instances sharing H and J)
struct BatchCtx;
BatchCtx* batch_create(Ctx& base, int64_t B);
void batch_destroy(BatchCtx* b);
void batch_set_affine(BatchCtx& b, const double* h, const double* h0, const double* d);
void batch_condense(BatchCtx& b, const double* sigma, const double* w, double* M_out, double* tq_out);
void batch_solve(BatchCtx& b, const double* opts, int64_t max_iter, double* v_out, double* scal, double* stats);

// ---- comm.cpp (NCCL, opened at run time)
enum class CommType { f64, i64 };
enum class CommOp { sum, max, min };
void comm_unique_id(void* out128);
void comm_attach(Ctx& c, const void* id128, int nranks, int rank);
void comm_detach(Ctx& c);
// in-place allreduce on c.stream (no-op without a communicator)
void comm_allreduce(Ctx& c, void* buf, size_t count, CommType type, CommOp op);
void comm_group(Ctx& c, bool start);
// loopback communicator: N contexts on one device, one host thread each (comm.cpp)
void* comm_loop_create(int nranks, int device);
void comm_loop_destroy(void* group);
void comm_loop_attach(Ctx& c, void* group, int rank);
void comm_loop_allreduce(Ctx& c, void* buf, size_t count, CommType type, CommOp op);
// the sharded solve's packed-M buffer (allocated when a communicator attaches)
void comm_buffers(Ctx& c);
inline int64_t rows_all(const Ctx& c) { return c.m_all >= 0 ? c.m_all : c.m; }

// ---- vec.cu
void launch_zero_packet(Ctx& c);
// copy the packet into the mapped host mirror and bump the publish sequence (the host spins
// on it instead of a stream synchronize + D2H copy); returns the sequence value to wait for
unsigned long long launch_publish(Ctx& c, bool slot_b = false);
// max |h| (after h changed)
void launch_hmax(Ctx& c);
// set the barrier value (host copy and the device scalar the kernels read)
void set_mu(Ctx& c, double mu);
// residuals at the current state (r1, r2, r3, kkt, objective pieces) -> packet A;
// reuse_trial: the state was just moved to the last evaluated line-search trial point
// gated: nothing runs unless the step was taken (d_alpha[2] != 0; the speculative seg_next)
// publish >= 0: the last kernel also publishes the packet into slot A (0) or B (1)
void launch_residuals(Ctx& c, bool reuse_trial = false, bool gated = false, int publish = -1);
// r2 and complementarity only (after a barrier change) -> packet kkt at the new mu, from the
// residual maxima of `a` (the current point's residual packet) and the recomputed max_comp
void launch_residuals_mu(Ctx& c, const Packet& a);
// sigma = z/s, omega, q = Pi'(r2 - sigma r3) (one launch; the singleton diagonal is added by k_syrk_reduce)
void launch_prepare_step(Ctx& c, const double* sigma_override);
// rhs = -r1 + (P' q + singletons): the partial product (this context's rows) and the final
// combination; launch_rhs does both (unsharded)
void launch_rhs_partial(Ctx& c);
void launch_rhs_final(Ctx& c);
void launch_rhs(Ctx& c);
// Jpv, ps, plambda, pz, fraction-to-boundary minima, line-search derivative pieces
void launch_recover(Ctx& c, double tau);
// merit pieces of trial (alpha): v_t = v + alpha pv, s_t = s + alpha ps; with
// alpha_from_device the step is alpha_max = min(1, packet tau-ratio minimum)
// linear: J v_t from the current point's and the direction's prototype values (yv + alpha y,
// valid inside the host loop after launch_residuals and launch_recover) instead of a P pass
// builder.cu
void prob_build(Ctx& c, const cmpc_lq_problem& in, double** H, double** h, double* h0, double** J,
                double** d, int64_t* m);
void prob_refresh(Ctx& c, const double* x_bar);
void prob_recover(Ctx& c, const double* v_dev, double* x, double* u, double* obj);
void prob_free(Ctx& c);

void launch_reset_packet_all(Ctx& c);
void launch_debug_sum(Ctx& c, const double* x, int64_t n, int slot);
// decide: also the speculative trial-0 acceptance into d_alpha (trial0_decide, vec.cu)
void launch_trial(Ctx& c, double alpha, bool alpha_from_device, bool linear = false,
                  bool decide = false, double eta = 0.0, int publish = -1);
// line-search derivative pieces for externally set directions: (Hv+h).pv, sum ps/s
void launch_ls_pieces(Ctx& c);
// v = 0, s = max(1, d), z = mu / s, lambda = z (ipm.cpp:170-177)
void launch_init_state(Ctx& c, double mu);
// iterate update v,s,lambda += alpha p; z += alpha_z pz
void launch_update(Ctx& c, double alpha, double alpha_z);
// the same with the step lengths already on the device (set_alpha)
void set_alpha(Ctx& c, double alpha, double alpha_z);
void launch_update_dev(Ctx& c);
// y = P x (+ singletons), Jx_r = sign y[proto]; optional
void launch_Jx(Ctx& c, const double* x, double* y, double* Jx);
// out = P' q + singleton scatter
void launch_Jtq(Ctx& c, const double* q, double* out);
// Hx
void launch_Hx(Ctx& c, const double* x, double* out);
// stand-alone fraction_to_boundary minima into out[2] (device)
void launch_fraction_to_boundary(cudaStream_t st, int64_t m, const double* s, const double* ps,
                                 const double* z, const double* pz, double tau, double* out);
// pack (to_packed) / unpack the lower triangle of the n x n column-major M
void launch_pack_lower(Ctx& c, double* M, double* packed, bool to_packed);
void vec_alloc(Ctx& c);
void vec_free(Ctx& c);

}  // namespace cmpc
