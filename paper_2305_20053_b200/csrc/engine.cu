// engine.cu -- sdn_handle and the C ABI declared in include/saadino.h.
//
// One handle owns one device's shard of the SAA sample set, the replicated
// surrogate (weights, projections), the tracking form / decoder, and all
// work buffers.  Per evaluation (reference saa_objective, riskopt.py:227-243,
// over SurrogateEvaluator, riskopt.py:178-194) the device runs:
//   zbias (W1_z V_z^T z + b1, once)  ->  forward GEMM chain with fused
//   bias/activation/residual epilogues (derivatives kept for the sweep)  ->
//   QoI + fp64 block moments  ->  [collective on the moments]  ->
//   [exact CVaR: radix top-k selection]  ->  weighted seeds on the active
//   rows  ->  reverse GEMM chain  ->  fp64 column sums of dL/dS_1  ->
//   projection through V_z W1_z^T to the d_z gradient  ->  [collective].
// The reverse sweep replaces the reference's forward-mode z-Jacobian
// (surrogate.py:195-233, >=95% of its CPU time): sum_i w_i dQ_i/dz is
// linear in the seeds, so one weighted sweep gives the risk gradient.
#include "../../include/saadino.h"
#include "common.cuh"
#include "gemm_simt.cuh"
#include "kernels.cuh"
#include "gemm_tc.cuh"
#include "refine.cuh"
#include "train.cuh"
#include "small.cuh"

// SMs left to side-stream work (the exact-CVaR selection + fp64 band
// refinement, a cooperative kernel on this many blocks) while the main stream's
// persistent sweep GEMMs run (sdn_eval_multi).  Balances the two paths of the
// c2 step; re-measured after each change to either path (latest, with the
// depth-3 reverse ring: 0.370 ms at 24-28, 0.358-0.367 at 32-44).
constexpr int SDN_SIDE_SMS_DEFAULT = 16;   // the exact-CVaR selections are off the critical path (deferred sums)

#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>
#include <cstdio>
#include <cstdlib>
#include <functional>
#include <vector>

using namespace sdn;

static thread_local std::string g_err;
static int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}
#define CU(call)                                                                          \
  do {                                                                                    \
    cudaError_t e_ = (call);                                                              \
    if (e_ != cudaSuccess)                                                                \
      return fail(SDN_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_));     \
  } while (0)
#define CHECK_LAUNCH(h)                                                                   \
  do {                                                                                    \
    cudaError_t e_ = cudaGetLastError();                                                  \
    if (e_ != cudaSuccess)                                                                \
      return fail(SDN_ERR_CUDA, std::string("kernel launch: ") + cudaGetErrorString(e_)); \
  } while (0)
#define TRY(x)                 \
  do {                         \
    int rc_ = (x);             \
    if (rc_ != SDN_OK) return rc_; \
  } while (0)

static inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }
static inline int pad4(int x) { return (x + 3) & ~3; }

// reverse-sweep work buffers (one set per handle)
struct SweepBufs {
  float* E = nullptr;           // seeds (rows x r_u)
  float* G = nullptr;           // residual gradient stream (rows x maxw)
  float* Ub[2] = {nullptr, nullptr};
  double* tsum = nullptr;       // fused column-sum partials (TC chains)
  double* cpart = nullptr;      // SIMT column-sum partials (crb x maxw)
  double* csum = nullptr;
  TcOperand act[2];             // bf16x3 split of the sweep operand (ping-pong)
  TcOperand seed;
  int64_t rows = 0;
  double* W = nullptr;          // per-row risk weights (rows x planes)
  int planes = 0;               // risks the partial buffers hold
};

struct sdn_handle {
  // ---- configuration
  int L = 0;                    // weight matrices (hidden + output)
  std::vector<int> w;           // widths, L + 1
  int r_m = 0, r_z = 0, d_z = 0, d_zp = 0, r_u = 0, h1 = 0, maxw = 0;
  int act = ACT_ELU, residual = 1, gemm = SDN_GEMM_AUTO, device = 0;
  int ldx = 0;                  // padded [r_m | d_z] input width for per-row z
  int64_t cap = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  std::vector<void*> allocs;
  int64_t launches = 0;
  int num_sms = 148;

  // ---- model (device)
  bool have_model = false;
  std::vector<float*> W;        // W[0] = W1[:, :r_m] * in_scale (h1 x r_m); W[l] as given
  std::vector<float*> b;
  std::vector<char> res;        // residual flag per layer
  float* Wx = nullptr;          // h1 x ldx : [W0m' | Pz32 | 0]
  double* Pz = nullptr;         // h1 x d_z  = W0z V_z^T (fp64)
  double* PzT = nullptr;        // d_z x h1  (transposed, for the gradient projection)
  float* Pz32 = nullptr;        // h1 x d_zp
  float* Pz32t = nullptr;       // d_z x h1
  float* omean = nullptr;
  float* ostd = nullptr;
  TcWeights tcw;                // bf16x3 operand copies for the tensor-core path

  // ---- QoI
  bool have_form = false;
  float* c = nullptr;
  double q0 = 0.0;
  bool have_dec = false;
  int64_t d_u = 0;
  float* U = nullptr;           // d_u x r_u
  float* ub = nullptr;          // d_u
  float* Kg = nullptr;          // r_u x r_u Gram U^T M U
  float* cdec = nullptr;        // r_u
  double q0dec = 0.0;

  // ---- samples
  float* MR = nullptr;
  int64_t n = 0, goff = 0;

  // ---- work buffers
  float* H[2] = {nullptr, nullptr};
  std::vector<float*> D;        // per hidden layer, cap x w[l+1]
  float* Y = nullptr;           // cap x r_u (phi)
  float* KPhi = nullptr;        // cap x r_u
  double* Q = nullptr;          // cap
  float* E = nullptr;           // cap x r_u (seeds, compacted)
  float* G = nullptr;           // cap x maxw (residual gradient stream)
  float* Ub[2] = {nullptr, nullptr};
  float* Gz = nullptr;          // cap x d_zp (per-sample G)
  int* rowidx = nullptr;
  int* counts = nullptr;
  int* offs = nullptr;
  int* n_act_dev = nullptr;
  uint8_t* sel = nullptr;
  double* qpart = nullptr;      // qgrid x STATS_LEN
  int qgrid = 0;
  double* partial_multi = nullptr;   // per-risk partials of sdn_eval_multi (device)
  double* hpart_multi = nullptr;     // pinned host copy
  int* hidx = nullptr;               // pinned CVaR indices
  int multi_cap = 0;
  int64_t hidx_cap = 0;
  int crb = 0;
  double* stats_loc = nullptr;  // STATS_LEN
  double* partial_loc = nullptr;
  double* zdev = nullptr;       // d_z
  float* zb = nullptr;          // h1
  double* cand_vals = nullptr;  // candidate scratch (exact CVaR, multi-rank)
  double* cand_gidx = nullptr;
  uint8_t* cand_mask = nullptr;
  int64_t n_cand = 0;           // candidates of the last sdn_eval_select
  // sdn_eval_multi_launch -> sdn_eval_multi_wait
  bool pending = false;
  std::vector<sdn_risk> pend_risks;
  int64_t pend_ktot = 0;
  bool pend_idx = false;
  int64_t cand_cap = 0;
  // pinned staging
  double* hz = nullptr;         // d_z + SDN_RMAX (z, then each risk's t)
  double* hstats = nullptr;     // STATS_LEN
  double* hpart = nullptr;      // partial len

  // ---- profiling (per kernel class CUDA-event timing, sdn_profile)
  bool prof = false;
  int pcls = 9;                 // class of the next GEMM launch (PC_OTHER)
  int64_t prows = 0;            // its true row count (-1: device-side n_act)
  struct ProfRec { int cls; cudaEvent_t a, b; double flops; double bytes; int64_t rows; double per_row; };
  std::vector<ProfRec> recs;
  std::vector<cudaEvent_t> pool;
  size_t pool_used = 0;

  // ---- evaluation state
  sdn_risk risk{};
  sdn_risk fwd_risk{};          // the risk the last forward ran with (its t / eps fed the moments)
  double shift = 0.0;
  bool have_mean = false;
  double last_mean = 0.0;
  bool fwd_done = false;
  // Q refinement (fp64 re-evaluation of decision-boundary rows)
  float* W0raw = nullptr;       // h1 x r_m : W1[:, :r_m] as given (fp32)
  float* iscale = nullptr;      // r_m input scale
  double* zb64 = nullptr;       // h1 : b1 + Pz z in fp64
  double* ref64[2] = {nullptr, nullptr};   // ref_rows x maxw ping-pong
  int ref_rows = 0;
  double* thr_dev = nullptr;    // exact-CVaR threshold value (top-k output)
  int* ref_blockcnt = nullptr;  // k_refine grid scratch
  int* ref_rowidx = nullptr;    // k_refine band rows
  unsigned* ref_ghist = nullptr;           // k_refine selection histograms (2 x grid x 256)
  unsigned long long* ref_gmm = nullptr;   // k_refine selection min / max keys (2 x grid)
  double* Qr = nullptr;         // exact-CVaR selection copy of Q (threshold band refined in fp64)
  float* seed_a2 = nullptr;     // r_u: 2 sigma        (fused output-layer seeds)
  float* seed_b2 = nullptr;     // r_u: 2 sigma c
  bool seed_fused = false;      // the last forward wrote the sweep's unit seeds
  bool qr_valid = false;
  double* wpart = nullptr;      // k_weights block partials (qgrid x 2 SDN_RMAX)
  double* vsum = nullptr;       // 2 SDN_RMAX: per-risk sum_{w != 0} Q, count
  int* red_counter = nullptr;   // last-block reduction counters (k_qoi, k_weights), self re-arming
  int* fwdflags = nullptr;      // forward chain row-block readiness (L x fwd_mtiles)
  int* bwdflags = nullptr;      // reverse chain row-block readiness (L x fwd_mtiles)
  int fwd_mtiles = 0;
  unsigned* ref_bar = nullptr;  // k_refine grid barrier
  int ref_grid = 0;
  bool ref_ok = false;          // the fp64 refinement can run (L <= REF_MAX_LAYERS)
  const double* ref_tp = nullptr;  // device-side t of the refinement window (set by refine_window)
  // side stream (overlapped exact-CVaR selection in sdn_eval_multi)
  cudaStream_t side = nullptr;
  cudaEvent_t ev_fwd = nullptr, ev_side = nullptr, ev_qoi = nullptr, ev_idx = nullptr;
  int* x_counts = nullptr;
  int* x_offs = nullptr;
  std::vector<int*> x_rowidx, x_nact;
  std::vector<uint8_t*> x_mask;
  std::vector<int64_t> x_k;     // k of each kept selection (multi-rank phases)
  std::vector<int64_t*> x_gidx; // global indices of each kept selection (ascending)
  std::vector<int64_t> x_gcap;
  // short tail (k_sel_colsum_sl + k_finalize_export): sliced selected-row sums, finalise + export in one launch
  // QoI partials written by the output layer's epilogue (cap x r_u/16 chunk planes), summed by k_qoi_part
  double* qp = nullptr;
  bool qoi_fuse = true;         // env SDN_NO_QOI_FUSE=1: k_qoi reads Y back instead
  bool q_fused = false;         // the last forward wrote qp
  bool z_by_kernel = false;     // upload_z used the fetch kernel (k_zbias may launch programmatically behind it)
  bool tail_fuse = true;        // env SDN_NO_TAIL_FUSE=1 disables (c2: 0.3117 -> 0.3086 ms with the direct host writes)
  bool tail_export = false;     // env SDN_TAIL_EXPORT=1: the finalise kernel writes the host results itself (no export launch)
  bool exp_want = false, exp_done = false;   // enqueue_multi asks the tail to export; the tail says it did
  double *exp_s = nullptr, *exp_p = nullptr; // host-mapped destinations (stats, partials)
  int* exp_b = nullptr;                      // ... band log
  int exp_np = 0, exp_nb = 0;
  int sm_avail = 0;             // SMs the persistent GEMMs may use
  int side_sms = SDN_SIDE_SMS_DEFAULT;   // env SDN_SIDE_SMS (default clamped to a quarter of the SMs)
  bool no_overlap = false;               // env SDN_NO_OVERLAP=1
  SweepBufs sw0;                // sweep buffers
  SweepBufs* sw = &sw0;
  int* band_log = nullptr;      // band row counts: [0] forward window, [1 + i] exact risk i
  int* hband = nullptr;         // pinned mirror
  int band_cap = 0;
  double* K64 = nullptr;        // decoded-frame Gram / c in fp64
  double* c64dec = nullptr;
  // batched control Jacobian (c5): scratch kept across calls (no per-call
  // allocation); tensor-core chains hold the tangents as bf16x3 splits
  int64_t jac_rows = 0;         // tangent-row capacity of the scratch below
  TcOperand jtan[2];            // tangent split ping-pong (rows x maxw)
  TcOperand jjr;                // std . dy/dz split (rows x r_u), the decoder GEMM's A
  TcOperand usplit;             // decoder basis split (d_u16 x r_u)
  int64_t d_u16 = 0;
  float* jT[2] = {nullptr, nullptr};   // SIMT tangents (rows x maxw)
  float* jJt = nullptr;         // SIMT std . dy/dz (rows x r_u)
  int64_t jin_cap = 0;          // host-input scratch (sdn_jacobian_batch): samples
  // grow-only device scratch for the host-facing entry points (no per-call
  // cudaMalloc/cudaFree; freed at destroy)
  void* scr[8] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
  size_t scr_bytes[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  TcOperand lift_in;            // lift: phi split (rows x r_u)
  float *jmr = nullptr, *jz = nullptr, *jX = nullptr, *jJ = nullptr;
  bool no_refine = false;       // env SDN_NO_REFINE=1 (precision studies)
  // small sample sets: the whole evaluation in one launch (small.cuh)
  bool no_small = false;        // env SDN_NO_SMALL=1
  std::vector<float*> WT;       // transposed fp32 weights (w[l] x w[l+1]) of the one-launch path
  double* small_part = nullptr; // per-CTA partials
  int64_t small_gen = -1;       // handle generation the transposes were taken at
  bool ref_trace = false;       // env SDN_REFINE_TRACE=1
  // H1 training state (sdn_train_*), allocated on first use
  struct Train {
    bool ready = false;
    int64_t n = 0;
    int bcap = 0;
    float *dm = nullptr, *dz = nullptr, *du = nullptr, *dj = nullptr;
    std::vector<int64_t> woff, boff;   // parameter offsets (W_l, b_l), reference layout
    int64_t count = 0;
    double *P = nullptr, *G = nullptr, *M = nullptr, *V = nullptr;
    double* mask = nullptr;            // optional (padded networks)
    float* P32 = nullptr;
    float *scale = nullptr, *mu = nullptr, *sig = nullptr;
    int* idx = nullptr;
    float *Y = nullptr, *Jt = nullptr, *GA = nullptr, *GT = nullptr, *GS = nullptr, *GU = nullptr;
    float *GA2 = nullptr, *GT2 = nullptr;
    float *GSt = nullptr, *GUt = nullptr, *zpart = nullptr;   // split-K weight-gradient scratch
    int zmax = 8;
    std::vector<float*> A, S, T, U;  // per layer (A[0] = X, T[0] = tangent seed)
    double* part = nullptr;
    double* hloss = nullptr;           // pinned
    std::vector<void*> allocs;
  } tr;
  // CUDA graph of the last evaluation configuration (sdn_eval_multi)
  bool use_graphs = true;       // env SDN_NO_GRAPH=1 disables
  cudaGraphExec_t gexec = nullptr;
  cudaEvent_t dev_ev[2] = {nullptr, nullptr};   // device span of the last sdn_eval_multi
  // stage timeline inside the evaluation graph (env SDN_TIMELINE=1: event
  // record nodes at stage boundaries, printed after each sdn_eval_multi)
  bool tl_on = false;
  cudaEvent_t tl[12] = {};
  bool tl_hit[12] = {};
  double last_dev_ms = 0.0;
  std::vector<double> gkey;
  int64_t glaunches = 0;
  int64_t gen = 0;              // bumped by every set_* call (invalidates the graph)
  unsigned long long* ref_trace_dev = nullptr;
  bool selected = false;        // exact CVaR selection done
  int64_t kk = 0;               // exact CVaR k (global)
  bool compacted = false;
  double hzz = 0.0;             // z.z of the current evaluation
  std::vector<double> zhost;

  int plen() const { return d_z + 2; }
};

template <class T>
static int dalloc(sdn_handle* h, T** p, size_t count) {
  void* q = nullptr;
  size_t bytes = std::max<size_t>(count * sizeof(T), 16);
  cudaError_t e = cudaMalloc(&q, bytes);
  if (e != cudaSuccess) return fail(SDN_ERR_NOMEM, std::string("cudaMalloc: ") + cudaGetErrorString(e));
  h->allocs.push_back(q);
  *p = reinterpret_cast<T*>(q);
  return SDN_OK;
}

// grow-only scratch slot (stream-ordered reuse: callers are serialised on the
// handle's stream; a grown buffer is freed after a stream sync)
enum ScratchSlot { SCR_A = 0, SCR_B, SCR_C, SCR_D, SCR_E, SCR_F, SCR_G, SCR_H };
template <class T>
static int scratch(sdn_handle* h, int slot, size_t count, T** p) {
  const size_t bytes = std::max<size_t>(count * sizeof(T), 16);
  if (bytes > h->scr_bytes[slot]) {
    if (h->scr[slot]) {
      cudaStreamSynchronize(h->stream);
      cudaFree(h->scr[slot]);
      h->scr[slot] = nullptr;
      h->scr_bytes[slot] = 0;
    }
    if (cudaMalloc(&h->scr[slot], bytes) != cudaSuccess) return fail(SDN_ERR_NOMEM, "scratch allocation failed");
    h->scr_bytes[slot] = bytes;
  }
  *p = reinterpret_cast<T*>(h->scr[slot]);
  return SDN_OK;
}

// ---------------------------------------------------------------------------
// profiling: events bracket each launch on the handle's stream

enum ProfClass { PC_FWD_GEMM = 0, PC_BWD_GEMM, PC_QOI, PC_SELECT, PC_COMPACT, PC_SEED, PC_COLSUM, PC_FINAL,
                 PC_ZBIAS, PC_OTHER, PC_REFINE, PC_TANGENT, PC_DECODE, PC_N };

static cudaEvent_t prof_event(sdn_handle* h) {
  if (h->pool_used == h->pool.size()) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    h->pool.push_back(e);
  }
  return h->pool[h->pool_used++];
}

struct ProfScope {
  sdn_handle* h; int cls; double flops, bytes; int64_t rows; double per_row; cudaEvent_t a = nullptr;
  // flops/bytes are totals when rows >= 0; when rows < 0 the count is the
  // device-side n_act and per_row scales it at read time
  ProfScope(sdn_handle* h_, int cls_, double flops_, double bytes_, int64_t rows_ = 0, double per_row_ = 0.0)
      : h(h_), cls(cls_), flops(flops_), bytes(bytes_), rows(rows_), per_row(per_row_) {
    if (h->prof) { a = prof_event(h); cudaEventRecord(a, h->stream); }
  }
  ~ProfScope() {
    if (!h->prof) return;
    cudaEvent_t b = prof_event(h);
    cudaEventRecord(b, h->stream);
    h->recs.push_back({cls, a, b, flops, bytes, rows, per_row});
  }
};

// ---------------------------------------------------------------------------
// GEMM dispatch

static inline bool al16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

// stage boundary mark (SDN_TIMELINE=1): an event record node on `st`
static inline void tl_mark(sdn_handle* h, int i, cudaStream_t st = nullptr) {
  if (!h->tl_on) return;
  if (!h->tl[i]) cudaEventCreate(&h->tl[i]);
  cudaEventRecordWithFlags(h->tl[i], st ? st : h->stream, cudaEventRecordExternal);
  h->tl_hit[i] = true;
}
static const char* const TL_NAMES[12] = {"start", "z-bias", "forward GEMMs", "QoI+moments", "side: start",
                                          "side: selection+refine+compaction", "reverse chain (pre-join)",
                                          "join wait", "sweep weights", "last reverse GEMM + sums",
                                          "column sums + finalize", "end"};

template <int BM, int BN, int TM, int TN, bool AT, bool BT, class Epi>
static void launch_simt(sdn_handle* h, int64_t M, const int* Mdev, int N, int K, const float* A,
                        int64_t lda, const float* B, int64_t ldb, Epi epi, bool vec) {
  dim3 grid((unsigned)cdiv(M, BM), (unsigned)cdiv(N, BN));
  dim3 block((BM / TM) * (BN / TN));
  if (vec)
    gemm_simt_kernel<BM, BN, 16, TM, TN, AT, BT, true, Epi>
        <<<grid, block, 0, h->stream>>>(M, Mdev, N, K, A, lda, B, ldb, epi);
  else
    gemm_simt_kernel<BM, BN, 16, TM, TN, AT, BT, false, Epi>
        <<<grid, block, 0, h->stream>>>(M, Mdev, N, K, A, lda, B, ldb, epi);
  h->launches++;
}

// C = opA(A) opB(B) with a fused epilogue; M rows (Mdev: device row count
// upper-bounded by M, for compacted sweeps).  Routes to tcgen05 when the
// handle allows it and the shape qualifies.
// route: -1 per-GEMM policy, 0 SIMT, 1 tcgen05 (a chain decided up front)
template <bool AT, bool BT, class Epi>
static int gemm(sdn_handle* h, int64_t M, const int* Mdev, int N, int K, const float* A, int64_t lda,
                const float* B, int64_t ldb, Epi epi, const TcOperand* tcB = nullptr,
                const TcOperand* tcA = nullptr, int route = -1, TcFlags fl = TcFlags{}) {
  if (M <= 0 || N <= 0) return SDN_OK;
  const int64_t rows = h->prows ? h->prows : M;
  h->prows = 0;
  ProfScope ps(h, h->pcls, rows >= 0 ? 2.0 * rows * N * K : 0.0, 0.0, rows, 2.0 * N * K);
  h->pcls = PC_OTHER;
  bool use_tc = route != 0 && h->gemm != SDN_GEMM_SIMT && !AT && tcB && tcA && h->tcw.enabled &&
                tc_gemm_supported(M, N, K) && tcA->ld % 8 == 0 && tcB->ld % 8 == 0;
  if (route == 1 && !use_tc) return fail(SDN_ERR_STATE, "tensor-core chain without a tensor-core GEMM");
  if (use_tc && route < 0 && h->gemm == SDN_GEMM_AUTO) {
    // small GEMMs (c1, CVaR tails) fill more SMs with 64x64 SIMT tiles
    const int64_t mrows = rows >= 0 ? rows : M;
    const int64_t tiles = cdiv(mrows, 128) * cdiv(N, N <= 128 ? 128 : 256);
    if (tiles < h->num_sms / 2) use_tc = false;
  }
  if (use_tc) {
    g_tc_pdl_now = h->sm_avail == h->num_sms;   // no PDL while SMs are reserved for the side stream
    int rc = tc_gemm(h->tcw, h->stream, h->sm_avail, M, Mdev, N, K, *tcA, *tcB, epi, rows, fl);
    h->launches++;
    if (rc != 0) return fail(SDN_ERR_CUDA, "tcgen05 GEMM launch failed (" + std::to_string(rc) + ")");
    CHECK_LAUNCH(h);
    return SDN_OK;
  }
  bool vec = !AT && (K % 4 == 0) && (lda % 4 == 0) && (ldb % 4 == 0) && al16(A) && al16(B) &&
             (BT || N % 4 == 0);
  // tile size from the rows that will actually run (compacted sweeps pass
  // the device count in Mdev and the known count as the row hint)
  int64_t tiles128 = cdiv(rows >= 0 ? rows : M, 128) * cdiv(N, 128);
  if (tiles128 >= 2 * h->num_sms)
    launch_simt<128, 128, 8, 8, AT, BT>(h, M, Mdev, N, K, A, lda, B, ldb, epi, vec);
  else
    launch_simt<64, 64, 4, 4, AT, BT>(h, M, Mdev, N, K, A, lda, B, ldb, epi, vec);
  CHECK_LAUNCH(h);
  return SDN_OK;
}

// ---------------------------------------------------------------------------
// forward / backward building blocks

// Whether a whole layer chain over `rows` rows runs on the tensor cores.  A
// chain is routed as one unit so that intermediates only the SIMT path reads
// (fp32 H for residuals, fp32 U) are skipped when every GEMM is tcgen05.
static bool chain_tc(sdn_handle* h, int64_t rows) {
  // softmax layers run SIMT chains (row kernels between the GEMMs)
  if (!h->tcw.enabled || h->gemm == SDN_GEMM_SIMT || rows < 1 || h->act == ACT_SOFTMAX) return false;
  for (int l = 0; l < h->L; ++l) {
    const int n_out = h->w[l + 1], n_in = (l == 0) ? h->r_m : h->w[l];
    if (!tc_gemm_supported(rows, n_out, n_in) || n_in % 8 || n_out % 8) return false;
    if (l >= 1 && !tc_gemm_supported(rows, n_in, n_out)) return false;
  }
  if (h->gemm == SDN_GEMM_TC) return true;
  // auto: the tcgen05 chain (narrow N tiles for short chains) beats the SIMT
  // tiles down to a single 128-row tile (c1: 113 vs 176 us per evaluation);
  // only a handful of rows stays on the exact-fp32 SIMT path
  return rows >= 64;
}

// layer chain on `nrows` rows.  Layer 0 input: X (ld0, K0) with weight W0 and
// bias0 (either MR + zb, or [m_r | z] + b0).  store_D keeps act' for the sweep.
// Hs (optional) replaces the hidden ping-pong buffers; simt forces the exact
// fp32 SIMT chain (Q refinement).
static int run_forward(sdn_handle* h, int64_t nrows, const float* X, int64_t ld0, int K0,
                       const float* W0, int64_t ldW0, const float* bias0, bool store_D,
                       float* phi_out, const TcOperand* tcX0, float* const* Hs = nullptr,
                       bool simt = false, bool fuse_seed = false) {
  const int L = h->L;
  const bool tcc = !simt && chain_tc(h, nrows);
  float* const* Hb = Hs ? Hs : h->H;
  // row-block readiness flags between the chain's GEMMs (PDL early start)
  static const bool no_rflags = getenv("SDN_NO_RFLAGS") != nullptr;
  const bool rflags = tcc && !Hs && nrows <= h->cap && !no_rflags;
  if (rflags) {
    CU(cudaMemsetAsync(h->fwdflags, 0, sizeof(int) * (size_t)L * h->fwd_mtiles, h->stream));
  }
  auto flags_of = [&](int l) -> TcFlags {
    TcFlags f;
    if (!rflags) return f;
    if (l >= 1 && (l > 1 || tcX0)) f.in = h->fwdflags + (size_t)(l - 1) * h->fwd_mtiles;
    if (l < L - 1) f.out = h->fwdflags + (size_t)l * h->fwd_mtiles;
    return f;
  };
  int cur = 0;
  const float* in = X;
  int64_t ldin = ld0;
  int l_start = 0;
  // persistent chain: the hidden layers (equal widths, tensor-core operands
  // from layer 0 on) in one launch; the output layer follows as its own GEMM
  {
    const int NH = L - 1, Nw = h->w[1];
    // (only when a layer's 128 x 256 tiles fill at least half the GPU, as
    // tc_gemm's 256-column rule: small batches (c1) keep the per-layer GEMMs'
    // narrower tiles, which spread over more SMs)
    bool ok = tcc && rflags && tcX0 && g_tc_chain && NH >= 2 && NH <= SDN_CHAIN_MAX && h->act != ACT_SOFTMAX &&
              h->tcw.enabled && Nw % 16 == 0 && Nw > 128 && tcX0->ld % 8 == 0 && K0 % 8 == 0 &&
              cdiv(nrows, 128) * cdiv(Nw, 256) >= h->num_sms / 2;
    for (int l = 1; l < NH && ok; ++l) ok = h->w[l + 1] == Nw && h->res[l];
    if (ok) {
      std::vector<FwdChainLayerHost> ls;
      int c = 0;
      for (int l = 0; l < NH; ++l) {
        FwdChainLayerHost x{};
        const TcFlags f = flags_of(l);
        x.A = l == 0 ? tcX0 : &h->tcw.act[c];
        x.B = &h->tcw.fwd[l];
        x.S = &h->tcw.act[l == 0 ? 0 : 1 - c];
        x.P = l == 0 ? nullptr : &h->tcw.act[c];
        x.D = store_D ? h->D[l] : nullptr;
        x.bias = l == 0 ? bias0 : h->b[l];
        x.K = l == 0 ? K0 : h->w[l];
        x.fl = f;
        ls.push_back(x);
        c = l == 0 ? 0 : 1 - c;
      }
      // optionally the output layer too (phi = mu + sigma (acc + b), and the
      // reverse sweep's unit seeds when fused) as the chain's last layer:
      // measured slower at c2 (device span 0.330 -> 0.342 ms: its 128-column
      // layer on 256-column tiles at the end of every CTA's list), so off by
      // default; SDN_CHAIN_OUT=1 enables it
      static const bool chain_out = getenv("SDN_CHAIN_OUT") && getenv("SDN_CHAIN_OUT")[0] == '1';
      const bool out_in_chain = chain_out && h->r_u % 16 == 0 && h->r_u >= 16;
      if (out_in_chain) {
        FwdChainLayerHost x{};
        x.A = &h->tcw.act[c];
        x.B = &h->tcw.fwd[L - 1];
        const bool seeds = fuse_seed && L > 1;
        x.S = seeds ? &h->sw->seed : nullptr;
        x.D = phi_out;
        x.bias = h->b[L - 1];
        x.K = h->w[L - 1];
        x.fl = flags_of(L - 1);
        x.N = h->r_u;
        x.kind = 1;
        x.scale = h->ostd;
        x.shift = h->omean;
        x.a2 = h->seed_a2;
        x.b2 = h->seed_b2;
        ls.push_back(x);
        if (seeds) h->seed_fused = true;
      }
      double fl_sum = 0.0;
      for (int l = 0; l < NH; ++l) fl_sum += 2.0 * nrows * Nw * (l == 0 ? K0 : h->w[l]);
      if (out_in_chain) fl_sum += 2.0 * nrows * h->r_u * h->w[L - 1];
      ProfScope ps(h, PC_FWD_GEMM, fl_sum, 0.0);
      g_tc_pdl_now = h->sm_avail == h->num_sms;
      const int64_t tiles = cdiv(nrows, 128) * cdiv(Nw, 256) * NH;
      const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(tiles, h->sm_avail));
      const int rc = tc_fwd_chain(h->tcw, h->stream, grid, nrows, Nw, h->act, ls);
      h->launches++;
      if (rc != 0) return fail(SDN_ERR_CUDA, "tcgen05 forward chain launch failed (" + std::to_string(rc) + ")");
      CHECK_LAUNCH(h);
      cur = c;
      l_start = out_in_chain ? L : NH;
      in = nullptr;
      ldin = Nw;
    }
  }
  for (int l = l_start; l < L; ++l) {
    const int n_in = h->w[l], n_out = h->w[l + 1];
    const float* Wl = (l == 0) ? W0 : h->W[l];
    const int64_t ldW = (l == 0) ? ldW0 : n_in;
    const int K = (l == 0) ? K0 : n_in;
    const float* bl = (l == 0) ? bias0 : h->b[l];
    const bool tc = tcc && (l > 0 || tcX0);      // layer 0 of per-row-z inputs stays SIMT
    const TcOperand* tA = !tc ? nullptr : (l == 0) ? tcX0 : &h->tcw.act[cur];
    const TcOperand* tB = !tc ? nullptr : &h->tcw.fwd[l];
    h->pcls = PC_FWD_GEMM;
    h->prows = nrows;
    if (l == L - 1) {
      EpiAffine e{bl, h->ostd, h->omean, phi_out, (int64_t)n_out};
      if (fuse_seed && tc && L > 1) {      // + the reverse sweep's unit seeds (bf16x3 split)
        EpiAffineSeed es{e, h->seed_a2, h->seed_b2, TcEpiSplit{&h->sw->seed}};
        if (h->qoi_fuse && n_out == h->r_u && n_out % 16 == 0 && nrows <= h->cap && phi_out == h->Y) {
          es.cq = h->c; es.qp = h->qp; es.qld = h->cap;     // + the QoI's chunk partials (launch_qoi: k_qoi_part)
          h->q_fused = true;
        }
        TRY((gemm<false, true>(h, nrows, nullptr, n_out, K, in, ldin, Wl, ldW, es, tB, tA, 1, flags_of(l))));
        h->seed_fused = true;
      } else {
        TRY((gemm<false, true>(h, nrows, nullptr, n_out, K, in, ldin, Wl, ldW, e, tB, tA, tc ? 1 : 0,
                               tc ? flags_of(l) : TcFlags{})));
      }
    } else {
      float* out = Hb[(l == 0) ? 0 : 1 - cur];
      if (h->act == ACT_SOFTMAX) {                // S + b, then the row softmax (SIMT chain)
        EpiFwdHidden e{bl, nullptr, out, nullptr, (int64_t)n_out, ACT_IDENTITY};
        TRY((gemm<false, true>(h, nrows, nullptr, n_out, K, in, ldin, Wl, ldW, e, nullptr, nullptr, 0)));
        k_softmax_rows<<<(unsigned)cdiv(nrows, 8), 256, 0, h->stream>>>(nrows, n_out, out,
                                                                      store_D ? h->D[l] : nullptr,
                                                                      h->res[l] ? in : nullptr);
        h->launches++;
        CHECK_LAUNCH(h);
        cur = (l == 0) ? 0 : 1 - cur;
        in = out;
        ldin = n_out;
        continue;
      }
      // in a tensor-core chain the residual is read from the bf16 split of the
      // layer input (the A operand), and the fp32 H is never needed
      const bool split_prev = tc && h->res[l];
      EpiFwdHidden e{bl, (h->res[l] && !split_prev ? in : nullptr), tcc ? nullptr : out,
                     store_D ? h->D[l] : nullptr, (int64_t)n_out, h->act};
      TcEpiSplit split = tcc ? TcEpiSplit{&h->tcw.act[(l == 0) ? 0 : 1 - cur]} : TcEpiSplit{nullptr};
      TcEpiSplit prev = split_prev ? TcEpiSplit{&h->tcw.act[cur]} : TcEpiSplit{nullptr};
      TRY((gemm<false, true>(h, nrows, nullptr, n_out, K, in, ldin, Wl, ldW,
                             TcChain<EpiFwdHidden>{e, split, prev}, tB, tA, tc ? 1 : 0,
                             tc ? flags_of(l) : TcFlags{})));
      cur = (l == 0) ? 0 : 1 - cur;
      in = out;
      ldin = n_out;
    }
  }
  return SDN_OK;
}

// weighted column sums of the unified sweep (backward_multi): per-row risk
// weights W (sweep rows x R), partial plane stride, and a hook run right
// before the last GEMM (where the weights are first needed)
struct SweepSum {
  const double* W = nullptr;
  int R = 1;
  int64_t plane = 0;
  std::function<int()> before_last;
  float* U0 = nullptr;          // store u = dL/dS_0 too (deferred exact-CVaR sums)
  // weights computed in the last GEMM's epilogue (wfun) from Q and the moments
  int wfun = 0;
  RiskSet rs{};
  const double* Q = nullptr;
  const double* st = nullptr;
  double shift = 0.0;
};

// reverse sweep over `nmax` (device count n_act_dev) compacted rows from the
// seeds E.  SIMT chains (or want_u0) leave dL/dS_0 (rows x w[1]) in *u0_out;
// tensor-core chains fuse the (weighted) sample sum into the last GEMM and
// leave fp64 column-sum partials in h->sw->tsum (*u0_out = nullptr, *nrb =
// partial rows, device-bounded by n_act_dev).
static int run_backward(sdn_handle* h, int64_t nmax, const int* n_act_dev, const int* rowidx,
                        float** u0_out, int64_t rows_hint, bool want_u0 = false, int64_t* nrb = nullptr,
                        const SweepSum* ss = nullptr) {
  const int L = h->L;
  if (L == 1) {
    if (ss && ss->before_last) TRY(ss->before_last());
    *u0_out = h->sw->E;
    return SDN_OK;
  }
  const bool tcc = chain_tc(h, rows_hint >= 0 ? rows_hint : nmax);
  const int route = tcc ? 1 : 0;
  int cur = 0;
  int l_top = L - 1;
  // persistent reverse chain: the dense sweep's steps l = L-1 .. 2 (equal
  // widths) in one launch; the summing step (l = 1) follows as its own GEMM
  {
    const int NW = h->w[1];
    bool ok = tcc && g_bwd_chain && ss && !want_u0 && !rowidx && !n_act_dev && L >= 4 && L - 2 <= SDN_CHAIN_MAX &&
              h->act != ACT_SOFTMAX && NW % 16 == 0 && NW > 128 && nmax <= h->cap &&
              cdiv(nmax, 128) * cdiv(NW, 256) >= h->num_sms / 2;
    for (int l = 1; l < L && ok; ++l) ok = h->w[l] == NW;
    if (ok) {
      std::vector<BwdChainLayerHost> ls;
      CU(cudaMemsetAsync(h->bwdflags, 0, sizeof(int) * (size_t)L * h->fwd_mtiles, h->stream));
      double fl_sum = 0.0;
      int c = 0, step = 0;
      for (int l = L - 1; l >= 2; --l, ++step) {
        BwdChainLayerHost x{};
        x.A = (l == L - 1) ? &h->sw->seed : &h->sw->act[c];
        x.B = &h->tcw.bwd[l];
        x.S = &h->sw->act[1 - c];
        x.R = (l < L - 1 && h->res[l]) ? h->sw->G : nullptr;
        x.G = h->res[l - 1] ? h->sw->G : nullptr;
        x.D = h->D[l - 1];
        x.ldD = NW;
        x.K = h->w[l + 1];
        x.fl.in = step > 0 ? h->bwdflags + (size_t)(step - 1) * h->fwd_mtiles : nullptr;
        x.fl.out = h->bwdflags + (size_t)step * h->fwd_mtiles;
        fl_sum += 2.0 * nmax * NW * x.K;
        ls.push_back(x);
        c = 1 - c;
      }
      ProfScope ps(h, PC_BWD_GEMM, fl_sum, 0.0);
      g_tc_pdl_now = h->sm_avail == h->num_sms;
      const int64_t tiles = cdiv(nmax, 128) * cdiv(NW, 256) * (int64_t)ls.size();
      const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(tiles, h->sm_avail));
      const int rc = tc_bwd_chain(h->tcw, h->stream, grid, nmax, NW, ls);
      h->launches++;
      if (rc != 0) return fail(SDN_ERR_CUDA, "tcgen05 reverse chain launch failed (" + std::to_string(rc) + ")");
      CHECK_LAUNCH(h);
      cur = c;
      l_top = 1;
    }
  }
  for (int l = l_top; l >= 1; --l) {
    // GEMM l: g_{l-1} = (res[l] ? g_l : 0) + u_l W_l, u_{l-1} = D_{l-1} g_{l-1}
    const int K = h->w[l + 1], N = h->w[l];
    const float* A = (l == L - 1) ? h->sw->E : h->sw->Ub[cur];
    const TcOperand* tA = !tcc ? nullptr : (l == L - 1) ? &h->sw->seed : &h->sw->act[cur];
    const TcOperand* tB = tcc ? &h->tcw.bwd[l] : nullptr;
    const float* resid = (l < L - 1 && h->res[l]) ? h->sw->G : nullptr;
    if (l == 1 && ss && ss->before_last) TRY(ss->before_last());
    h->pcls = PC_BWD_GEMM;
    h->prows = rows_hint;
    if (l == 1 && tcc && !want_u0) {
      EpiBwdSum e{resid, h->D[0], (int64_t)N, rowidx, (int64_t)N, h->sw->tsum, (int64_t)N};
      if (ss) {
        e.W = ss->W; e.R = ss->R; e.plane = ss->plane; e.U0 = ss->U0;
        if (ss->wfun) { e.W = nullptr; e.wfun = 1; e.rs = ss->rs; e.Q = ss->Q; e.st = ss->st; e.shift = ss->shift; }
      }
      TRY((gemm<false, false>(h, nmax, n_act_dev, N, K, A, K, h->W[l], N, e, tB, tA, route)));
      *u0_out = nullptr;
      if (nrb) *nrb = cdiv(nmax, 128) * 4;
      return SDN_OK;
    }
    const bool last = (l == 1);
    const bool smax = h->act == ACT_SOFTMAX;     // derivative applied by a row kernel below
    EpiBwd e{resid, h->res[l - 1] ? h->sw->G : nullptr, smax ? nullptr : h->D[l - 1], (int64_t)N, rowidx,
             (!tcc || last) ? h->sw->Ub[1 - cur] : nullptr, (int64_t)N};
    TcEpiSplit split = (tcc && !last) ? TcEpiSplit{&h->sw->act[1 - cur]} : TcEpiSplit{nullptr};
    TRY((gemm<false, false>(h, nmax, n_act_dev, N, K, A, K, h->W[l], N, TcChain<EpiBwd>{e, split}, tB, tA,
                            route)));
    if (smax) {
      k_softmax_bwd<<<(unsigned)cdiv(nmax, 8), 256, 0, h->stream>>>(nmax, n_act_dev, rowidx, N, h->D[l - 1],
                                                                    h->sw->Ub[1 - cur]);
      h->launches++;
      CHECK_LAUNCH(h);
    }
    cur = 1 - cur;
  }
  *u0_out = h->sw->Ub[cur];
  return SDN_OK;
}

// ---------------------------------------------------------------------------
// C ABI

extern "C" {

const char* sdn_last_error(void) { return g_err.c_str(); }
int sdn_version(void) { return 1; }

int sdn_create(const sdn_config* cfg, sdn_handle** out) {
  if (!cfg || !out) return fail(SDN_ERR_ARG, "null argument");
  if (cfg->n_layers < 1 || !cfg->widths) return fail(SDN_ERR_ARG, "need at least one layer");
  for (int i = 0; i <= cfg->n_layers; ++i)
    if (cfg->widths[i] < 1) return fail(SDN_ERR_ARG, "all widths must be positive");
  if (cfg->r_m < 1 || cfg->d_z < 1 || cfg->r_m >= cfg->widths[0])
    return fail(SDN_ERR_ARG, "need 1 <= r_m < widths[0] and d_z >= 1");
  if (cfg->activation < 0 || cfg->activation > 5) return fail(SDN_ERR_ARG, "unknown activation");
  if (cfg->max_samples < 1) return fail(SDN_ERR_ARG, "max_samples must be >= 1");
  for (int i = 1; i <= cfg->n_layers; ++i)
    if (cfg->widths[i] % 4 != 0) return fail(SDN_ERR_ARG, "layer output widths must be multiples of 4");
  if (cfg->r_m % 4 != 0) return fail(SDN_ERR_ARG, "r_m must be a multiple of 4");

  sdn_handle* h = new sdn_handle();
  h->L = cfg->n_layers;
  h->w.assign(cfg->widths, cfg->widths + cfg->n_layers + 1);
  h->r_m = cfg->r_m;
  h->r_z = h->w[0] - h->r_m;
  h->d_z = cfg->d_z;
  h->d_zp = pad4(cfg->d_z);
  h->r_u = h->w[h->L];
  h->h1 = h->w[1];
  h->maxw = *std::max_element(h->w.begin() + 1, h->w.end());
  h->act = cfg->activation;
  h->residual = cfg->residual;
  h->gemm = cfg->gemm;
  h->device = cfg->device;
  h->ldx = pad4(h->r_m + h->d_z);
  h->cap = cfg->max_samples;
  h->res.assign(h->L, 0);
  for (int l = 1; l < h->L - 1; ++l) h->res[l] = (h->residual && h->w[l] == h->w[l + 1]) ? 1 : 0;

  auto bail = [&](int rc) { sdn_destroy(h); return rc; };
  cudaError_t e = cudaSetDevice(h->device);
  if (e != cudaSuccess) { delete h; return fail(SDN_ERR_CUDA, std::string("cudaSetDevice: ") + cudaGetErrorString(e)); }
  cudaDeviceGetAttribute(&h->num_sms, cudaDevAttrMultiProcessorCount, h->device);
  h->sm_avail = h->num_sms;
  e = cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking);
  if (e != cudaSuccess) { delete h; return fail(SDN_ERR_CUDA, "cudaStreamCreate failed"); }
  h->own_stream = true;

  const int64_t cap = h->cap;
  int rc;
  h->W.assign(h->L, nullptr);
  h->b.assign(h->L, nullptr);
  for (int l = 0; l < h->L; ++l) {
    int n_in = (l == 0) ? h->r_m : h->w[l];
    if ((rc = dalloc(h, &h->W[l], (size_t)h->w[l + 1] * n_in))) return bail(rc);
    if ((rc = dalloc(h, &h->b[l], h->w[l + 1]))) return bail(rc);
  }
  if ((rc = dalloc(h, &h->Wx, (size_t)h->h1 * h->ldx))) return bail(rc);
  if ((rc = dalloc(h, &h->Pz, (size_t)h->h1 * h->d_z))) return bail(rc);
  if ((rc = dalloc(h, &h->PzT, (size_t)h->h1 * h->d_z))) return bail(rc);
  if ((rc = dalloc(h, &h->Pz32, (size_t)h->h1 * h->d_zp))) return bail(rc);
  if ((rc = dalloc(h, &h->Pz32t, (size_t)h->h1 * h->d_z))) return bail(rc);
  if ((rc = dalloc(h, &h->omean, h->r_u))) return bail(rc);
  if ((rc = dalloc(h, &h->ostd, h->r_u))) return bail(rc);
  if ((rc = dalloc(h, &h->c, h->r_u))) return bail(rc);
  if ((rc = dalloc(h, &h->MR, (size_t)cap * h->r_m))) return bail(rc);
  for (int i = 0; i < 2; ++i) {
    if ((rc = dalloc(h, &h->H[i], (size_t)cap * h->maxw))) return bail(rc);
    if ((rc = dalloc(h, &h->Ub[i], (size_t)cap * h->maxw))) return bail(rc);
  }
  h->D.assign(std::max(h->L - 1, 0), nullptr);
  for (int l = 0; l < h->L - 1; ++l)
    if ((rc = dalloc(h, &h->D[l], (size_t)cap * h->w[l + 1]))) return bail(rc);
  if ((rc = dalloc(h, &h->Y, (size_t)cap * h->r_u))) return bail(rc);
  if ((rc = dalloc(h, &h->E, (size_t)cap * h->r_u))) return bail(rc);
  if ((rc = dalloc(h, &h->G, (size_t)cap * h->maxw))) return bail(rc);
  if ((rc = dalloc(h, &h->Q, cap))) return bail(rc);
  if ((rc = dalloc(h, &h->rowidx, cap))) return bail(rc);
  if ((rc = dalloc(h, &h->sel, cap))) return bail(rc);
  const int nb1024 = (int)cdiv(cap, 1024);
  if ((rc = dalloc(h, &h->counts, nb1024))) return bail(rc);
  if ((rc = dalloc(h, &h->offs, nb1024))) return bail(rc);
  if ((rc = dalloc(h, &h->n_act_dev, 1))) return bail(rc);
  h->qgrid = (int)std::min<int64_t>(cdiv(cap, 8), 2 * h->num_sms);
  if ((rc = dalloc(h, &h->qpart, (size_t)h->qgrid * STATS_LEN))) return bail(rc);
  if ((rc = dalloc(h, &h->qp, (size_t)cap * (size_t)cdiv(h->r_u, 16)))) return bail(rc);
  h->crb = (int)std::min<int64_t>(cdiv(cap, 8), 16);
  if ((rc = dalloc(h, &h->stats_loc, STATS_LEN))) return bail(rc);
  if ((rc = dalloc(h, &h->partial_loc, h->plen()))) return bail(rc);
  if ((rc = dalloc(h, &h->zdev, h->d_z + SDN_RMAX))) return bail(rc);   // [z | per-risk t]
  if ((rc = dalloc(h, &h->zb, h->h1))) return bail(rc);
  if ((rc = dalloc(h, &h->zb64, h->h1))) return bail(rc);
  if ((rc = dalloc(h, &h->W0raw, (size_t)h->h1 * h->r_m))) return bail(rc);
  if ((rc = dalloc(h, &h->iscale, h->r_m))) return bail(rc);
  if ((rc = dalloc(h, &h->thr_dev, 1))) return bail(rc);
  h->ref_rows = (int)std::min<int64_t>(cap, REFINE_ROWS);
  {
    cudaFuncSetAttribute(k_refine, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)sizeof(double) * REF_RB * REF_KC);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_refine, REF_THREADS, sizeof(double) * REF_RB * REF_KC);
    h->ref_grid = h->num_sms;                     // one block per SM, all co-resident
    h->ref_ok = per_sm >= 1 && h->L <= REF_MAX_LAYERS;   // any width (K chunks), any band size (row chunks)
  }
  if ((rc = dalloc(h, &h->ref_blockcnt, h->num_sms))) return bail(rc);
  if ((rc = dalloc(h, &h->ref_rowidx, cap))) return bail(rc);
  if ((rc = dalloc(h, &h->ref_ghist, (size_t)2 * h->num_sms * 256))) return bail(rc);
  if ((rc = dalloc(h, &h->ref_gmm, (size_t)2 * h->num_sms))) return bail(rc);
  if ((rc = dalloc(h, &h->Qr, cap))) return bail(rc);
  if ((rc = dalloc(h, &h->seed_a2, h->r_u))) return bail(rc);
  if ((rc = dalloc(h, &h->seed_b2, h->r_u))) return bail(rc);
  if ((rc = dalloc(h, &h->wpart, (size_t)h->qgrid * 2 * SDN_RMAX))) return bail(rc);
  if ((rc = dalloc(h, &h->vsum, 2 * SDN_RMAX))) return bail(rc);
  if ((rc = dalloc(h, &h->red_counter, 4))) return bail(rc);

  h->fwd_mtiles = 2 * (int)cdiv(cap, 256);        // 128-row blocks, whole 256-row pair tiles
  if ((rc = dalloc(h, &h->fwdflags, (size_t)h->L * h->fwd_mtiles))) return bail(rc);
  if ((rc = dalloc(h, &h->bwdflags, (size_t)h->L * h->fwd_mtiles))) return bail(rc);
  if (cudaMemset(h->red_counter, 0, 4 * sizeof(int)) != cudaSuccess) return bail(fail(SDN_ERR_CUDA, "memset"));
  if ((rc = dalloc(h, &h->ref_bar, 2))) return bail(rc);
  if (cudaMemset(h->ref_bar, 0, 2 * sizeof(unsigned)) != cudaSuccess) return bail(fail(SDN_ERR_CUDA, "memset"));
  for (int i = 0; i < 2; ++i)
    if ((rc = dalloc(h, &h->ref64[i], (size_t)h->ref_rows * h->maxw))) return bail(rc);
  h->band_cap = 8;
  if ((rc = dalloc(h, &h->band_log, h->band_cap))) return bail(rc);
  if (cudaHostAlloc((void**)&h->hband, sizeof(int) * h->band_cap, cudaHostAllocMapped) != cudaSuccess)
    return bail(fail(SDN_ERR_NOMEM, "cudaHostAlloc failed"));
  if (cudaHostAlloc((void**)&h->hz, sizeof(double) * (h->d_z + SDN_RMAX), cudaHostAllocMapped) != cudaSuccess ||
      cudaHostAlloc((void**)&h->hstats, sizeof(double) * STATS_LEN, cudaHostAllocMapped) != cudaSuccess ||
      cudaHostAlloc((void**)&h->hpart, sizeof(double) * h->plen(), cudaHostAllocMapped) != cudaSuccess)
    return bail(fail(SDN_ERR_NOMEM, "cudaHostAlloc failed"));
  { const char* e = getenv("SDN_NO_REFINE"); h->no_refine = e && e[0] == '1'; }
  { const char* e = getenv("SDN_NO_SMALL"); h->no_small = e && e[0] == '1'; }
  { const char* e = getenv("SDN_NO_OVERLAP"); h->no_overlap = e && e[0] == '1'; }
  { const char* e = getenv("SDN_REFINE_TRACE"); h->ref_trace = e && e[0] == '1'; }
  { const char* e = getenv("SDN_NO_GRAPH"); h->use_graphs = !(e && e[0] == '1'); }
  { const char* e = getenv("SDN_TIMELINE"); h->tl_on = e && e[0] == '1'; }
  h->tail_fuse = !(getenv("SDN_NO_TAIL_FUSE") && getenv("SDN_NO_TAIL_FUSE")[0] == '1');
  h->qoi_fuse = !(getenv("SDN_NO_QOI_FUSE") && getenv("SDN_NO_QOI_FUSE")[0] == '1');
  h->tail_export = getenv("SDN_TAIL_EXPORT") && getenv("SDN_TAIL_EXPORT")[0] == '1';
  h->side_sms = std::max(1, std::min(SDN_SIDE_SMS_DEFAULT, h->num_sms / 4));
  { const char* e = getenv("SDN_SIDE_SMS");
    if (e) h->side_sms = std::max(1, std::min(atoi(e), h->num_sms / 2)); }
  h->tcw.enabled = false;
  if (h->gemm != SDN_GEMM_SIMT) {
    if ((rc = tc_alloc(h, h->tcw))) return bail(rc);
  }
  h->sw0.E = h->E;
  h->sw0.G = h->G;
  h->sw0.Ub[0] = h->Ub[0];
  h->sw0.Ub[1] = h->Ub[1];
  h->sw0.act[0] = h->tcw.act[0];
  h->sw0.act[1] = h->tcw.act[1];
  h->sw0.seed = h->tcw.seed;
  h->sw0.rows = cap;
  h->sw = &h->sw0;
  *out = h;
  return SDN_OK;
}

int sdn_destroy(sdn_handle* h) {
  if (!h) return SDN_OK;
  cudaSetDevice(h->device);
  if (h->stream) cudaStreamSynchronize(h->stream);
  for (cudaEvent_t e : h->dev_ev)
    if (e) cudaEventDestroy(e);
  for (cudaEvent_t e : h->tl)
    if (e) cudaEventDestroy(e);
  for (void* p : h->allocs) cudaFree(p);
  for (void* p : h->scr)
    if (p) cudaFree(p);
  if (h->U) cudaFree(h->U);
  if (h->ub) cudaFree(h->ub);
  if (h->Kg) cudaFree(h->Kg);
  if (h->cdec) cudaFree(h->cdec);
  if (h->KPhi) cudaFree(h->KPhi);
  if (h->Gz) cudaFree(h->Gz);
  if (h->cand_vals) cudaFree(h->cand_vals);
  if (h->cand_gidx) cudaFree(h->cand_gidx);
  if (h->cand_mask) cudaFree(h->cand_mask);
  if (h->hz) cudaFreeHost(h->hz);
  if (h->hstats) cudaFreeHost(h->hstats);
  if (h->hpart) cudaFreeHost(h->hpart);
  if (h->hband) cudaFreeHost(h->hband);
  if (h->ref_trace_dev) cudaFree(h->ref_trace_dev);
  if (h->K64) cudaFree(h->K64);
  if (h->c64dec) cudaFree(h->c64dec);
  if (h->partial_multi) cudaFree(h->partial_multi);
  if (h->hpart_multi) cudaFreeHost(h->hpart_multi);
  if (h->hidx) cudaFreeHost(h->hidx);
  tc_free(h->tcw);
  if (h->gexec) cudaGraphExecDestroy(h->gexec);
  for (void* p : h->tr.allocs) cudaFree(p);
  if (h->tr.hloss) cudaFreeHost(h->tr.hloss);
  if (h->side) { cudaStreamSynchronize(h->side); cudaStreamDestroy(h->side); }
  if (h->ev_fwd) cudaEventDestroy(h->ev_fwd);
  if (h->ev_side) cudaEventDestroy(h->ev_side);
  if (h->ev_qoi) cudaEventDestroy(h->ev_qoi);
  if (h->ev_idx) cudaEventDestroy(h->ev_idx);
  if (h->own_stream && h->stream) cudaStreamDestroy(h->stream);
  delete h;
  return SDN_OK;
}

int sdn_set_stream(sdn_handle* h, void* stream) {
  if (!h) return fail(SDN_ERR_ARG, "null handle");
  CU(cudaSetDevice(h->device));
  if (stream) {
    CU(cudaStreamSynchronize(h->stream));
    if (h->own_stream) cudaStreamDestroy(h->stream);
    h->stream = reinterpret_cast<cudaStream_t>(stream);
    h->own_stream = false;
  }
  return SDN_OK;
}

int sdn_synchronize(sdn_handle* h) {
  if (!h) return fail(SDN_ERR_ARG, "null handle");
  CU(cudaStreamSynchronize(h->stream));
  return SDN_OK;
}

int64_t sdn_kernel_launches(sdn_handle* h) { return h ? h->launches : -1; }

int sdn_set_model(sdn_handle* h, const float* const* W, const float* const* b, const float* in_scale,
                  const float* out_mean, const float* out_std, const float* Vz) {
  if (!h || !W || !b || !in_scale || !out_mean || !out_std) return fail(SDN_ERR_ARG, "null argument");
  CU(cudaSetDevice(h->device));
  const int n0 = h->w[0], h1 = h->h1, r_m = h->r_m, r_z = h->r_z, d_z = h->d_z;
  if (!Vz && r_z != d_z) return fail(SDN_ERR_ARG, "V_z = identity needs r_z == d_z");
  // layer 0 split: W0m' = W0[:, :r_m] * in_scale ; Pz = W0[:, r_m:] V_z^T (fp64)
  std::vector<float> w0m((size_t)h1 * r_m);
  std::vector<double> pz((size_t)h1 * d_z, 0.0);
  std::vector<float> pz32((size_t)h1 * h->d_zp, 0.0f), pz32t((size_t)d_z * h1), wx((size_t)h1 * h->ldx, 0.0f);
  for (int c = 0; c < h1; ++c) {
    const float* row = W[0] + (size_t)c * n0;
    for (int j = 0; j < r_m; ++j) {
      w0m[(size_t)c * r_m + j] = (float)((double)row[j] * (double)in_scale[j]);
      wx[(size_t)c * h->ldx + j] = w0m[(size_t)c * r_m + j];
    }
    for (int k = 0; k < d_z; ++k) {
      double s = 0.0;
      if (Vz)
        for (int j = 0; j < r_z; ++j) s += (double)row[r_m + j] * (double)Vz[(size_t)k * r_z + j];
      else
        s = row[r_m + k];
      pz[(size_t)c * d_z + k] = s;
      pz32[(size_t)c * h->d_zp + k] = (float)s;
      pz32t[(size_t)k * h1 + c] = (float)s;
      wx[(size_t)c * h->ldx + r_m + k] = (float)s;
    }
  }
  CU(cudaMemcpy(h->W[0], w0m.data(), w0m.size() * 4, cudaMemcpyHostToDevice));
  {
    std::vector<float> raw((size_t)h1 * r_m);
    for (int c = 0; c < h1; ++c)
      for (int j = 0; j < r_m; ++j) raw[(size_t)c * r_m + j] = W[0][(size_t)c * n0 + j];
    CU(cudaMemcpy(h->W0raw, raw.data(), raw.size() * 4, cudaMemcpyHostToDevice));
    CU(cudaMemcpy(h->iscale, in_scale, (size_t)r_m * 4, cudaMemcpyHostToDevice));
  }
  for (int l = 1; l < h->L; ++l)
    CU(cudaMemcpy(h->W[l], W[l], (size_t)h->w[l + 1] * h->w[l] * 4, cudaMemcpyHostToDevice));
  for (int l = 0; l < h->L; ++l) CU(cudaMemcpy(h->b[l], b[l], (size_t)h->w[l + 1] * 4, cudaMemcpyHostToDevice));
  CU(cudaMemcpy(h->Pz, pz.data(), pz.size() * 8, cudaMemcpyHostToDevice));
  {
    std::vector<double> pzt((size_t)d_z * h1);
    for (int c = 0; c < h1; ++c)
      for (int k = 0; k < d_z; ++k) pzt[(size_t)k * h1 + c] = pz[(size_t)c * d_z + k];
    CU(cudaMemcpy(h->PzT, pzt.data(), pzt.size() * 8, cudaMemcpyHostToDevice));
  }
  CU(cudaMemcpy(h->Pz32, pz32.data(), pz32.size() * 4, cudaMemcpyHostToDevice));
  CU(cudaMemcpy(h->Pz32t, pz32t.data(), pz32t.size() * 4, cudaMemcpyHostToDevice));
  CU(cudaMemcpy(h->Wx, wx.data(), wx.size() * 4, cudaMemcpyHostToDevice));
  CU(cudaMemcpy(h->omean, out_mean, (size_t)h->r_u * 4, cudaMemcpyHostToDevice));
  CU(cudaMemcpy(h->ostd, out_std, (size_t)h->r_u * 4, cudaMemcpyHostToDevice));
  if (h->tcw.enabled) TRY(tc_set_weights(h, h->tcw));
  if (h->have_form) {
    k_seedcoef<<<1, 256>>>(h->r_u, h->ostd, h->c, h->seed_a2, h->seed_b2);
    CU(cudaDeviceSynchronize());
  }
  h->have_model = true;
  h->have_mean = false;
  h->gen++;
  return SDN_OK;
}

int sdn_set_tracking(sdn_handle* h, const float* c, double q0) {
  if (!h || !c) return fail(SDN_ERR_ARG, "null argument");
  CU(cudaSetDevice(h->device));
  CU(cudaMemcpy(h->c, c, (size_t)h->r_u * 4, cudaMemcpyHostToDevice));
  h->q0 = q0;
  h->have_form = true;
  k_seedcoef<<<1, 256>>>(h->r_u, h->ostd, h->c, h->seed_a2, h->seed_b2);
  CU(cudaDeviceSynchronize());
  h->have_mean = false;
  h->gen++;
  return SDN_OK;
}

int sdn_set_samples(sdn_handle* h, const float* m_r, int64_t n, int64_t global_offset, int32_t on_device) {
  if (!h || (!m_r && n > 0)) return fail(SDN_ERR_ARG, "null argument");
  if (n < 0 || n > h->cap) return fail(SDN_ERR_ARG, "sample count exceeds the handle capacity");
  CU(cudaSetDevice(h->device));
  if (n > 0)
    CU(cudaMemcpyAsync(h->MR, m_r, (size_t)n * h->r_m * 4,
                       on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, h->stream));
  CU(cudaStreamSynchronize(h->stream));
  h->n = n;
  h->goff = global_offset;
  h->fwd_done = false;
  h->gen++;
  if (h->tcw.enabled) TRY(tc_set_samples(h, h->tcw, h->MR, n));
  return SDN_OK;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// evaluation phases

static int check_risk(const sdn_risk* r) {
  if (!r) return fail(SDN_ERR_ARG, "null risk");
  if (r->kind < 0 || r->kind > 3) return fail(SDN_ERR_ARG, "unknown risk kind");
  if ((r->kind == SDN_RISK_CVAR_SMOOTH || r->kind == SDN_RISK_CVAR_EXACT) && !(r->beta >= 0.0 && r->beta < 1.0))
    return fail(SDN_ERR_ARG, "beta must be in [0, 1)");
  if (r->kind == SDN_RISK_MEANVAR && !(r->beta >= 0.0)) return fail(SDN_ERR_ARG, "variance weight must be >= 0");
  if (r->kind == SDN_RISK_CVAR_SMOOTH && !(r->eps > 0.0)) return fail(SDN_ERR_ARG, "eps must be positive");
  if (r->qoi != SDN_QOI_REDUCED && r->qoi != SDN_QOI_DECODED) return fail(SDN_ERR_ARG, "unknown QoI frame");
  return SDN_OK;
}

static int ceil_count(double x) { return (int)std::ceil(x - 1e-9); }   // riskopt.py:56-58

// z and the risks' t values -> pinned staging -> device (one copy; a captured
// graph replays it, so z and t are per-call parameters of the graph)
static void stage_z(sdn_handle* h, const double* z, const sdn_risk* risks, int n_risks) {
  double zz = 0.0;
  h->zhost.assign(z, z + h->d_z);
  for (int k = 0; k < h->d_z; ++k) { h->hz[k] = z[k]; zz += z[k] * z[k]; }
  for (int r = 0; r < SDN_RMAX; ++r) h->hz[h->d_z + r] = r < n_risks ? risks[r].t : 0.0;
  h->hzz = zz;
}
// (z reaches the device once -- by a one-block fetch kernel or a copy node -- rather than every
// k_zbias block reading it from host-mapped memory, which measured slower)
__global__ void k_fetch_small(int n, const double* __restrict__ src_host, double* __restrict__ dst) {
  asm volatile("griddepcontrol.launch_dependents;");       // k_zbias loads its Pz rows meanwhile
  for (int i = threadIdx.x; i < n; i += blockDim.x) dst[i] = src_host[i];
}
static int upload_z(sdn_handle* h, const double* z, const sdn_risk* risks, int n_risks) {
  stage_z(h, z, risks, n_risks);
  h->z_by_kernel = false;
  // one small block reads the pinned (host-mapped) staging buffer over PCIe instead of a copy node: the same
  // device span, a cheaper graph launch on the host (c2 e2e 50.2 -> 50.6 M samples/s); SDN_Z_KERNEL=0: the copy node
  static const bool zk = !(getenv("SDN_Z_KERNEL") && getenv("SDN_Z_KERNEL")[0] == '0');
  if (zk) {
    double* src = nullptr;
    CU(cudaHostGetDevicePointer((void**)&src, h->hz, 0));
    k_fetch_small<<<1, 128, 0, h->stream>>>(h->d_z + SDN_RMAX, src, h->zdev);
    h->z_by_kernel = true;
    h->launches++;
    CHECK_LAUNCH(h);
    return SDN_OK;
  }
  CU(cudaMemcpyAsync(h->zdev, h->hz, sizeof(double) * (h->d_z + SDN_RMAX), cudaMemcpyHostToDevice, h->stream));
  return SDN_OK;
}

static int compact_rows(sdn_handle* h, int kind, double t, double eps, const double* tdev = nullptr,
                        int* count_out = nullptr, const uint8_t* sel = nullptr, int* rowidx_out = nullptr);

// Q refinement.  Rows whose chain Q (bf16x3 or fp32, ~1e-5
// relative) lies within REFINE_REL |Q| of a decision boundary -- the
// smoothed-CVaR window [t, t + eps] (kind RISK_BAND) or the exact-CVaR
// threshold (RISK_BAND_EXACT, value in thr_dev) -- are compacted and
// re-evaluated by an fp64 chain on the same fp32 weights (the oracle's
// arithmetic), and their Q replaced in place.  No host round trip: the band
// count stays on the device (*count); bands of more than ref_rows rows run in
// row chunks, and a large exact-CVaR band is reselected cooperatively.
static int refine_band(sdn_handle* h, int kind, double t, double eps, bool dec, int* count,
                       uint8_t* mask = nullptr, double* Qt = nullptr, int64_t k = 0, bool do_refine = true) {
  do_refine = do_refine && h->ref_ok;
  if (!do_refine && k == 0) return SDN_OK;
  RefineArgs a{};
  a.n = h->n; a.kind = kind; a.t = t; a.eps = eps; a.tdev = h->thr_dev; a.tp = h->ref_tp;
  a.rowidx = h->ref_rowidx; a.count = count; a.blockcnt = h->ref_blockcnt; a.bar = h->ref_bar;
  a.L = h->L;
  for (int l = 0; l < h->L && l < REF_MAX_LAYERS; ++l) {
    const bool first = l == 0;
    a.layer[l] = RefineLayer{first ? h->W0raw : h->W[l], h->b[l], first ? h->r_m : h->w[l], h->w[l + 1],
                             (l > 0 && l < h->L - 1 && h->res[l]) ? 1 : 0};
  }
  a.MR = h->MR; a.iscale = h->iscale; a.zb64 = h->zb64; a.act = h->act; a.omean = h->omean; a.ostd = h->ostd;
  a.buf[0] = h->ref64[0]; a.buf[1] = h->ref64[1]; a.cap_rows = h->ref_rows;
  a.r_u = h->r_u; a.c32 = h->c; a.K64 = dec ? h->K64 : nullptr; a.c64 = dec ? h->c64dec : nullptr;
  a.q0 = dec ? h->q0dec : h->q0; a.Q = Qt ? Qt : h->Q; a.mask = mask;
  a.k = k; a.ghist = h->ref_ghist; a.gmm = h->ref_gmm; a.refine = do_refine ? 1 : 0;
  a.softmax = h->act == ACT_SOFTMAX ? 1 : 0;
  void* args[] = {&a};
  ProfScope ps(h, k > 0 ? PC_SELECT : PC_REFINE, 0.0, k > 0 ? 8.0 * 8.0 * h->n : 0.0);
  if (h->ref_trace) {
    if (!h->ref_trace_dev) CU(cudaMalloc(&h->ref_trace_dev, 64 * sizeof(unsigned long long)));
    CU(cudaMemsetAsync(h->ref_trace_dev, 0, 64 * sizeof(unsigned long long), h->stream));
    a.trace = h->ref_trace_dev;
  }
  CU(cudaLaunchCooperativeKernel((const void*)k_refine, dim3(h->ref_grid), dim3(REF_THREADS), args,
                                 sizeof(double) * REF_RB * REF_KC, h->stream));
  h->launches++;
  if (h->ref_trace) {                 // debug: phase timestamps of block 0 (env SDN_REFINE_TRACE=1)
    unsigned long long tr[64];
    CU(cudaStreamSynchronize(h->stream));
    CU(cudaMemcpy(tr, h->ref_trace_dev, sizeof(tr), cudaMemcpyDeviceToHost));
    fprintf(stderr, "k_refine grid %d k %lld:", h->ref_grid, (long long)k);
    for (int i = 1; i < 64; ++i)
      if (tr[i]) fprintf(stderr, " [%d]%.1f", i, (tr[i] - tr[0]) * 1e-3);
    fprintf(stderr, " us\n");
  }
  return SDN_OK;
}

// smoothed CVaR: refine the window rows, then retake the moments from Q
static int refine_window(sdn_handle* h, const sdn_risk* risk, bool dec, int qg, double* stats_dev,
                         const double* tp) {
  if (risk->kind != SDN_RISK_CVAR_SMOOTH || h->n == 0 || h->no_refine || !h->ref_ok) return SDN_OK;
  h->ref_tp = tp;
  int rc = refine_band(h, RISK_BAND, risk->t, risk->eps, dec, h->band_log);
  h->ref_tp = nullptr;
  TRY(rc);
  { ProfScope ps(h, PC_QOI, 0.0, 8.0 * h->n);
  k_moments<<<qg, 256, 0, h->stream>>>(h->n, h->Q, h->shift, risk->t, risk->eps, h->qpart, tp);
  k_sum_rows<<<(unsigned)cdiv(STATS_LEN, 8), 256, 0, h->stream>>>(qg, STATS_LEN, h->qpart, stats_dev); }
  h->launches += 2;
  CHECK_LAUNCH(h);
  return SDN_OK;
}

// phase 1: forward over the shard; local moments -> stats_dev (device)
// (all, n_all): the evaluation's risks, whose t values travel with z (graph
// parameters); slot: this forward's risk among them
static int launch_qoi(sdn_handle* h, const sdn_risk* risk, double* stats_dev, const double* tp);

// (defer_qoi: the caller launches the QoI itself, launch_qoi -- sdn_eval_multi
// puts it on the side stream so the reverse sweep starts right after the forward)
static int eval_forward(sdn_handle* h, const double* z, const sdn_risk* risk, double* stats_dev,
                        bool store_D, const sdn_risk* all = nullptr, int n_all = 0, int slot = 0,
                        bool fuse_seed = false, bool defer_qoi = false) {
  if (!all) { all = risk; n_all = 1; slot = 0; }
  h->seed_fused = false;
  h->q_fused = false;
  if (!h->have_model) return fail(SDN_ERR_STATE, "set_model first");
  if (risk->qoi == SDN_QOI_REDUCED && !h->have_form) return fail(SDN_ERR_STATE, "set_tracking first");
  if (risk->qoi == SDN_QOI_DECODED && !h->have_dec) return fail(SDN_ERR_STATE, "set_decoder first");
  TRY(check_risk(risk));
  // CVaR decisions need the fp64 boundary refinement: never
  // return a possibly wrong selection silently
  for (int i = 0; i < n_all; ++i)
    if ((all[i].kind == SDN_RISK_CVAR_SMOOTH || all[i].kind == SDN_RISK_CVAR_EXACT) && !h->ref_ok && !h->no_refine)
      return fail(SDN_ERR_STATE, "CVaR risks need the fp64 boundary refinement, which supports at most 16 layers");
  CU(cudaSetDevice(h->device));
  h->risk = *risk;
  h->fwd_risk = *risk;
  h->selected = false;
  h->compacted = false;
  h->qr_valid = false;
  const bool dec = risk->qoi == SDN_QOI_DECODED;
  const double q0 = dec ? h->q0dec : h->q0;
  // moments accumulate (Q - shift) in fp64; shift = q0 keeps every evaluation
  // stateless and deterministic (cancellation ~1e-16 (Qbar - q0)^2 / var)
  h->shift = q0;
  TRY(upload_z(h, z, all, n_all));
  const double* tp = h->zdev + h->d_z + slot;
  { ProfScope ps(h, PC_ZBIAS, 2.0 * h->h1 * h->d_z, 8.0 * h->h1 * h->d_z);
  // (behind the z fetch kernel: a programmatic dependent launch -- its blocks load their Pz rows while z arrives)
  static const bool zpdl = !(getenv("SDN_NO_PDL") || (getenv("SDN_Z_PDL") && getenv("SDN_Z_PDL")[0] == '0'));
  cudaLaunchConfig_t zc{};
  zc.gridDim = dim3((unsigned)cdiv(h->h1, 8)); zc.blockDim = dim3(256); zc.dynamicSmemBytes = 0; zc.stream = h->stream;
  cudaLaunchAttribute za[1];
  za[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  za[0].val.programmaticStreamSerializationAllowed = (zpdl && h->z_by_kernel && !h->tl_on && !h->prof) ? 1 : 0;
  zc.attrs = za; zc.numAttrs = 1;
  CU(cudaLaunchKernelEx(&zc, k_zbias, h->h1, h->d_z, (const double*)h->Pz, (const double*)h->zdev,
                        (const float*)h->b[0], h->zb, h->zb64)); }
  tl_mark(h, 1);
  h->launches++;
  CHECK_LAUNCH(h);
  if (h->n > 0) {
    TRY(run_forward(h, h->n, h->MR, h->r_m, h->r_m, h->W[0], h->r_m, h->zb, store_D, h->Y,
                    h->tcw.enabled ? &h->tcw.mr : nullptr, nullptr, false, fuse_seed && !dec && store_D));
    tl_mark(h, 2);
    if (dec) {
      TRY((gemm<false, true>(h, h->n, nullptr, h->r_u, h->r_u, h->Y, h->r_u, h->Kg, h->r_u,
                             EpiStore{h->KPhi, (int64_t)h->r_u})));
    }
  }
  h->fwd_done = true;
  if (!defer_qoi) TRY(launch_qoi(h, risk, stats_dev, tp));
  return SDN_OK;
}

// per-sample QoI + moments (and the smoothed-CVaR window refinement) on h->stream
static int launch_qoi(sdn_handle* h, const sdn_risk* risk, double* stats_dev, const double* tp) {
  const bool dec = risk->qoi == SDN_QOI_DECODED;
  const double q0 = dec ? h->q0dec : h->q0;
  const int qg = (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(std::max<int64_t>(h->n, 1), 8), h->qgrid));
  // Q also goes to the exact-CVaR selection's copy (sel_q: no copy node ahead of the selection), unless a
  // smoothed-CVaR window refinement is about to change Q in place
  // (study switch SDN_Q2_WRITE=1, off: measured 1-2 us slower per c2 evaluation than the copy node)
  static const bool q2w = getenv("SDN_Q2_WRITE") && getenv("SDN_Q2_WRITE")[0] == '1';
  double* q2 = (q2w && risk->kind != SDN_RISK_CVAR_SMOOTH && h->Qr && h->n > 0) ? h->Qr : nullptr;
  if (h->q_fused && !dec && h->n > 0) {             // the output layer left the row's chunk partials
    const int nch = h->r_u / 16;
    const int g = (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(h->n, 128), h->qgrid));
    ProfScope ps(h, PC_QOI, 2.0 * h->n * nch, 8.0 * h->n * (nch + 1));
    k_qoi_part<<<g, 128, 0, h->stream>>>(h->n, nch, h->qp, h->cap, q0, h->shift, risk->t,
                                         risk->kind == SDN_RISK_CVAR_SMOOTH ? risk->eps : 1.0, h->Q, h->qpart, tp,
                                         h->red_counter, stats_dev, q2);
  } else
  { ProfScope ps(h, PC_QOI, 4.0 * h->n * h->r_u, 4.0 * h->n * h->r_u * (dec ? 2 : 1) + 8.0 * h->n);
  k_qoi<<<qg, 256, 0, h->stream>>>(h->n, h->r_u, h->Y, dec ? h->KPhi : nullptr, dec ? h->cdec : h->c, q0,
                                   h->shift, risk->t, risk->kind == SDN_RISK_CVAR_SMOOTH ? risk->eps : 1.0,
                                   h->Q, h->qpart, tp, h->red_counter, stats_dev, q2); }
  if (q2) h->qr_valid = true;
  tl_mark(h, 3, h->stream);
  h->launches += 1;
  CHECK_LAUNCH(h);
  TRY(refine_window(h, risk, dec, qg, stats_dev, tp));
  return SDN_OK;
}

// ensure candidate scratch for `count` entries
static int ensure_cand(sdn_handle* h, int64_t count) {
  if (count <= h->cand_cap) return SDN_OK;
  if (h->cand_vals) cudaFree(h->cand_vals);
  if (h->cand_gidx) cudaFree(h->cand_gidx);
  if (h->cand_mask) cudaFree(h->cand_mask);
  CU(cudaMalloc(&h->cand_vals, sizeof(double) * count));
  CU(cudaMalloc(&h->cand_gidx, sizeof(double) * count));
  CU(cudaMalloc(&h->cand_mask, count));
  h->cand_cap = count;
  return SDN_OK;
}

// ordered compaction of flagged rows -> rowidx / n_act_dev
static int compact_rows(sdn_handle* h, int kind, double t, double eps, const double* tdev, int* count_out,
                        const uint8_t* sel, int* rowidx_out) {
  const int nb = (int)cdiv(std::max<int64_t>(h->n, 1), 1024);
  if (!sel) sel = h->sel;
  ProfScope ps(h, PC_COMPACT, 0.0, 2.0 * (8.0 + 1.0) * h->n);
  if (kind == RISK_CVAR_EXACT && h->n <= COMPACT1_MAX) {     // a mask, few rows: one block, one launch
    k_compact_mask1<<<1, 1024, 0, h->stream>>>(h->n, sel, rowidx_out ? rowidx_out : h->rowidx,
                                               count_out ? count_out : h->n_act_dev);
    h->launches += 1;
    CHECK_LAUNCH(h);
    if (!rowidx_out) h->compacted = true;
    return SDN_OK;
  }
  k_flag_count<<<nb, 1024, 0, h->stream>>>(h->n, kind, h->Q, sel, t, eps, tdev, h->counts);
  k_scan_counts<<<1, 32, 0, h->stream>>>(nb, h->counts, h->offs, count_out ? count_out : h->n_act_dev);
  k_compact<<<nb, 1024, 0, h->stream>>>(h->n, kind, h->Q, sel, t, eps, tdev, h->offs,
                                        rowidx_out ? rowidx_out : h->rowidx);
  h->launches += 3;
  CHECK_LAUNCH(h);
  if (!rowidx_out) h->compacted = true;
  return SDN_OK;
}

// exact top-k selection mask (value desc, global index asc); SMEM-resident
// keys when they fit, else the global-memory radix select
static int launch_topk(sdn_handle* h, int64_t n, int64_t k, const double* vals, const double* gidx, uint8_t* mask,
                       double* thr = nullptr) {
  if (n <= TOPK_SMEM_MAX) {
    static unsigned attr = 0;                      // per device
    int dev = 0;
    cudaGetDevice(&dev);
    if (!(attr & (1u << (dev & 31)))) {
      cudaFuncSetAttribute(k_topk_select_smem, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)TOPK_SMEM_BYTES);
      attr |= 1u << (dev & 31);
    }
    k_topk_select_smem<<<1, 1024, TOPK_SMEM_BYTES, h->stream>>>((int)n, k, vals, gidx, mask, thr);
  } else {
    k_topk_select<<<1, 1024, 0, h->stream>>>(n, k, vals, gidx, mask, thr);
  }
  h->launches++;
  CHECK_LAUNCH(h);
  return SDN_OK;
}

// local exact top-k (single rank): selection mask over the shard's Q.  With
// band_count, the rows within refinement error of the threshold are
// re-evaluated in fp64 and reselected among themselves.
// The exact-CVaR selection works on its own copy of Q, so that the fp64
// refinement of the threshold band decides the selection only: every weight
// and value (and the other risks of the evaluation) use the chain's Q.
static double* sel_q(sdn_handle* h) {
  if (!h->qr_valid) {
    cudaMemcpyAsync(h->Qr, h->Q, sizeof(double) * std::max<int64_t>(h->n, 1), cudaMemcpyDeviceToDevice, h->stream);
    h->qr_valid = true;
  }
  return h->Qr;
}

static int select_local(sdn_handle* h, int64_t k, int* band_count = nullptr, uint8_t* mask = nullptr,
                        int* rowidx_out = nullptr, int* count_out = nullptr) {
  const bool refine = band_count && !h->no_refine;
  if (!mask) mask = h->sel;
  double* Qs = sel_q(h);
  // study switch SDN_TOPK_SMEM=1: the top-k by the single-CTA shared-memory radix select (no grid
  // barriers), then the cooperative kernel only for the band refinement and the reselection
  static const bool topk_smem = getenv("SDN_TOPK_SMEM") && getenv("SDN_TOPK_SMEM")[0] == '1';
  if (topk_smem && h->n <= TOPK_SMEM_MAX && refine && h->ref_ok) {
    TRY(launch_topk(h, h->n, k, Qs, nullptr, mask, h->thr_dev));
    TRY(refine_band(h, RISK_BAND_EXACT, 0.0, 0.0, h->risk.qoi == SDN_QOI_DECODED, band_count, mask, Qs, 0, true));
  } else {
  // one cooperative launch: top-k, then (refine) the fp64 threshold band and
  // the reselection among it
  TRY(refine_band(h, RISK_BAND_EXACT, 0.0, 0.0, h->risk.qoi == SDN_QOI_DECODED, band_count, mask, Qs, k,
                  refine));
  }
  TRY(compact_rows(h, RISK_CVAR_EXACT, 0.0, 1.0, nullptr, count_out, mask, rowidx_out));
  h->selected = true;
  return SDN_OK;
}

// per-handle buffers of the unified sweep for R risks: weights, weight
// partials, and R partial planes of the column sums (grown on demand)
static int ensure_sweep(sdn_handle* h, SweepBufs& b, int R) {
  if (R <= b.planes) return SDN_OK;
  const int64_t rows = b.rows;
  int rc;
  if ((rc = dalloc(h, &b.tsum, (size_t)R * cdiv(rows, 128) * 4 * h->maxw))) return rc;
  if ((rc = dalloc(h, &b.cpart, (size_t)R * h->crb * h->maxw))) return rc;
  if ((rc = dalloc(h, &b.csum, (size_t)R * h->maxw))) return rc;
  if ((rc = dalloc(h, &b.W, (size_t)R * std::max<int64_t>(rows, 1)))) return rc;
  b.planes = R;
  return SDN_OK;
}

// One reverse sweep for R risks.  Unit seeds over the union of
// the risks' active rows (all rows when a mean / mean+variance risk is
// present, else the ordered union of the CVaR rows), per-row weights
// w_i^(r), weighted fp64 column sums per risk, projection through PzT ->
// partials[r * plen] = [grad (d_z) | sum_{w != 0} Q | #{w != 0}].
// `join` runs before the first use of the exact-CVaR masks (side-stream
// selections, sdn_eval_multi): before the union compaction, or -- dense --
// right before the last GEMM, so the selections overlap the sweep.
static int backward_multi(sdn_handle* h, const sdn_risk* risks, int R, const uint8_t* const* masks,
                          const int64_t* ks, const double* stats_dev, double* partials,
                          const std::function<int()>& join = {}, const double* tdev = nullptr,
                          const int* const* sel_rows = nullptr, const std::function<int()>& qjoin = {}) {
  if (!h->fwd_done) return fail(SDN_ERR_STATE, "eval_forward first");
  if (R < 1 || R > SDN_RMAX) return fail(SDN_ERR_ARG, "1..8 risks per sweep");
  RiskSet rs{};
  rs.R = R;
  rs.tdev = tdev;                     // per-risk t on the device, in list order (sdn_eval_multi)
  bool dense = false, all_exact = true, any_grad = false;
  int64_t ksum = 0;
  for (int r = 0; r < R; ++r) {
    const sdn_risk& k = risks[r];
    const bool exact = k.kind == SDN_RISK_CVAR_EXACT;
    if (exact && (!masks || !masks[r])) return fail(SDN_ERR_STATE, "exact CVaR needs the selection phase");
    rs.kind[r] = k.kind;
    rs.beta[r] = k.beta;
    rs.eps[r] = k.kind == SDN_RISK_CVAR_SMOOTH ? k.eps : 1.0;
    rs.t[r] = k.t;
    rs.kinv[r] = exact ? 1.0 / (double)ks[r] : 0.0;
    rs.mask[r] = exact ? masks[r] : nullptr;
    dense |= k.kind == SDN_RISK_MEAN || k.kind == SDN_RISK_MEANVAR;
    all_exact &= exact;
    ksum += exact ? ks[r] : 0;
    any_grad |= k.need_grad != 0;
  }
  const bool dec = risks[0].qoi == SDN_QOI_DECODED;
  SweepBufs& sw = *h->sw;
  TRY(ensure_sweep(h, sw, R));
  // sweep rows
  const int* rowidx = nullptr;
  const int* nact = nullptr;
  int64_t nmax = h->n, rows_hint = h->n;
  if (!dense && h->n > 0) {
    if (join) TRY(join());
    const int nb = (int)cdiv(h->n, 1024);
    { ProfScope ps(h, PC_COMPACT, 0.0, 9.0 * h->n);
    k_union_count<<<nb, 1024, 0, h->stream>>>(h->n, rs, h->Q, h->counts);
    k_scan_counts<<<1, 32, 0, h->stream>>>(nb, h->counts, h->offs, h->n_act_dev);
    k_union_compact<<<nb, 1024, 0, h->stream>>>(h->n, rs, h->Q, h->offs, h->rowidx); }
    h->launches += 3;
    CHECK_LAUNCH(h);
    rowidx = h->rowidx;
    nact = h->n_act_dev;
    h->compacted = true;
    nmax = all_exact ? std::min<int64_t>(h->n, ksum) : h->n;
    rows_hint = all_exact ? nmax : -1;
  }
  if (nmax > sw.rows) return fail(SDN_ERR_STATE, "sweep buffers too small");
  // weights + value partials (the first read of the masks and of Q)
  const int wg = (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(std::max<int64_t>(nmax, 1), 256), h->qgrid));
  // deferred exact CVaR (dense sweep overlapped with the selections): the
  // last reverse GEMM runs without waiting for them -- dense risks' weights
  // are known after the forward moments -- and also stores u = dL/dS_0; once
  // the selections join, each exact risk's sums are taken over its k selected
  // rows of u (k_sel_colsum).  The masks are then never on the sweep's path.
  const bool defer = join && dense && sel_rows && !rowidx && h->n > 0 &&
                     chain_tc(h, nmax) && h->sw == &h->sw0 && h->L >= 2;
  RiskSet rs_w = rs;
  if (defer)
    for (int r = 0; r < R; ++r)
      if (rs.kind[r] == SDN_RISK_CVAR_EXACT) rs_w.mask[r] = nullptr;
  auto weights = [&]() -> int {
    ProfScope ps(h, PC_SEED, 0.0, 0.0, rows_hint, 8.0 * (1 + R));
    k_weights<<<wg, 256, 0, h->stream>>>(nmax, nact, rowidx, rs_w, h->Q, stats_dev, h->shift, sw.W, h->wpart,
                                         h->red_counter + 1, h->vsum);
    h->launches += 1;
    CHECK_LAUNCH(h);
    return SDN_OK;
  };
  const size_t fsm = sizeof(double) * h->h1;
  if (!any_grad || h->n == 0) {
    if (dense && join) TRY(join());
    TRY(weights());
    k_finalize_multi<<<dim3(1, R), 256, fsm, h->stream>>>(0, 0, h->h1, h->d_z, nullptr, h->PzT, h->vsum, h->plen(),
                                                          partials);
    h->launches++;
    CHECK_LAUNCH(h);
    return SDN_OK;
  }
  const bool tcs = chain_tc(h, rows_hint >= 0 ? rows_hint : nmax);
  if (!(dense && h->seed_fused && tcs && h->sw == &h->sw0)) {   // else: written by the output layer
  ProfScope ps(h, PC_SEED, 0.0, 0.0, rows_hint, 8.0 * h->r_u);
  const int sg = (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(nmax, 8), 4 * h->num_sms));
  k_seed<<<sg, 256, 0, h->stream>>>(nmax, nact, rowidx, h->r_u, h->Y, dec ? h->KPhi : nullptr,
                                    dec ? h->cdec : h->c, h->ostd, nullptr, nullptr, RISK_UNIT, 0.0, 0.0, 1.0,
                                    0.0, 0.0, sw.E, tcs ? sw.seed.hi : nullptr, tcs ? sw.seed.lo : nullptr);
  h->launches++;
  CHECK_LAUNCH(h);
  }
  const int64_t tplane = cdiv(sw.rows, 128) * 4 * h->maxw;
  SweepSum ssum;
  ssum.W = sw.W;
  ssum.R = R;
  ssum.plane = tplane;
  ssum.before_last = [&]() -> int {
    tl_mark(h, 6);
    if (qjoin) TRY(qjoin());                      // Q and the moments (QoI on the side stream)
    if (dense && join && !defer) TRY(join());
    tl_mark(h, 7);
    const int rc = defer ? SDN_OK : weights();   // deferred: the last GEMM weighs its rows itself
    tl_mark(h, 8);
    return rc;
  };
  if (defer) {
    ssum.U0 = sw.Ub[0];
    ssum.wfun = 1;
    ssum.rs = rs_w;
    ssum.Q = h->Q;
    ssum.st = stats_dev;
    ssum.shift = h->shift;
  }
  float* u0 = nullptr;
  int64_t nrb = 0;
  TRY(run_backward(h, nmax, nact, rowidx, &u0, rows_hint, false, &nrb, &ssum));
  tl_mark(h, 9);
  const double* part;
  int nrb_fin;
  int64_t plane;
  if (u0) {
    ProfScope ps(h, PC_COLSUM, 0.0, 0.0, rows_hint, 4.0 * h->h1);
    dim3 cg((unsigned)cdiv(h->h1, 32), (unsigned)h->crb);
    k_colsum_w<<<cg, dim3(32, 8), 0, h->stream>>>(nmax, nact, h->h1, u0, sw.W, R, sw.cpart);
    part = sw.cpart;
    nrb_fin = h->crb;
    plane = (int64_t)h->crb * h->h1;
  } else {
    ProfScope ps(h, PC_COLSUM, 0.0, 8.0 * nrb * h->h1 * R);
    k_colsum64<<<dim3((unsigned)cdiv(h->h1, 32), R), dim3(32, 32), 0, h->stream>>>((int)nrb, nact, h->h1, sw.tsum,
                                                                                sw.csum, tplane);
    part = sw.csum;
    nrb_fin = 1;
    plane = h->h1;
  }
  h->launches++;
  CHECK_LAUNCH(h);
  // short tail: sliced sums over the selected rows, one finalise + export launch
  const int S = std::max(1, std::min(8, h->crb));
  const bool short_tail = h->tail_fuse && !h->prof && !u0;      // sliced selected-row sums
  const bool fin_export = (h->tail_export || short_tail) && !h->prof && !u0;   // finalise writes the host results itself
  FinArgs fa{};
  for (int r = 0; r < R; ++r) fa.risk[r] = FinRisk{part + (int64_t)r * plane, nrb_fin, 1.0};
  if (defer) {
    TRY(join());
    for (int r = 0; r < R; ++r) {
      if (rs.kind[r] != SDN_RISK_CVAR_EXACT) continue;
      ProfScope ps(h, PC_COLSUM, 0.0, 4.0 * ks[r] * h->h1);
      if (short_tail) {
        // (cpart: the SIMT sweep's partial planes, idle here: R x crb x maxw >= R x S x h1)
        double* sl = sw.cpart + (int64_t)r * h->crb * h->maxw;
        k_sel_colsum_sl<<<dim3((unsigned)cdiv(h->h1, 32), S), dim3(32, 32), 0, h->stream>>>(
            ks[r], sel_rows[r], h->h1, sw.Ub[0], h->h1, h->Q, sl, h->vsum + 2 * r);
        fa.risk[r] = FinRisk{sl, S, rs.kinv[r]};
      } else {
        k_sel_colsum<<<(unsigned)cdiv(h->h1, 32), dim3(32, 32), 0, h->stream>>>(
            ks[r], sel_rows[r], h->h1, sw.Ub[0], h->h1, rs.kinv[r], h->Q, sw.csum + (int64_t)r * h->h1,
            h->vsum + 2 * r);
      }
      h->launches++;
      CHECK_LAUNCH(h);
    }
  }
  { ProfScope ps(h, PC_FINAL, 0.0, 8.0 * nrb_fin * h->h1 * R);
  if (fin_export) {
    fa.h1 = h->h1; fa.d_z = h->d_z; fa.plen = h->plen();
    fa.PzT = h->PzT; fa.vsum = h->vsum; fa.out = partials;
    if (h->exp_want && partials == h->partial_multi) {
      fa.stats = stats_dev; fa.hstats = h->exp_s; fa.nstats = STATS_LEN;
      fa.hpart = h->exp_p; fa.npart = h->exp_np;
      fa.band = h->band_log; fa.hband = h->exp_b; fa.nband = h->exp_nb;
      h->exp_done = true;
    }
    // (programmatic dependent launch behind the last sum kernel: its blocks prefetch their PzT rows meanwhile)
    static const bool fpdl = !(getenv("SDN_NO_PDL") || (getenv("SDN_FIN_PDL") && getenv("SDN_FIN_PDL")[0] == '0'));
    cudaLaunchConfig_t fc{};
    fc.gridDim = dim3((unsigned)cdiv(h->d_z, 8), R); fc.blockDim = dim3(256); fc.dynamicSmemBytes = fsm;
    fc.stream = h->stream;
    cudaLaunchAttribute fat[1];
    fat[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    fat[0].val.programmaticStreamSerializationAllowed = (fpdl && !h->tl_on) ? 1 : 0;
    fc.attrs = fat; fc.numAttrs = 1;
    CU(cudaLaunchKernelEx(&fc, k_finalize_export, fa));
  } else {
    k_finalize_multi<<<dim3((unsigned)cdiv(h->d_z, 8), R), 256, fsm, h->stream>>>(
        nrb_fin, plane, h->h1, h->d_z, part, h->PzT, h->vsum, h->plen(), partials);
  } }
  h->launches++;
  CHECK_LAUNCH(h);
  return SDN_OK;
}

// phase 3 for the current risk (sdn_eval, multi-rank phases)
static int eval_backward(sdn_handle* h, const double* stats_dev, double* partial_dev) {
  const uint8_t* m = h->sel;
  const int64_t k = h->kk;
  if (h->risk.kind == SDN_RISK_CVAR_EXACT && !h->selected)
    return fail(SDN_ERR_STATE, "exact CVaR needs the selection phase");
  return backward_multi(h, &h->risk, 1, &m, &k, stats_dev, partial_dev);
}

// host combination of the (global) moments and partials of one risk
static int finish_host(sdn_handle* h, const sdn_risk& r, const double* st, const double* pt, sdn_result* res,
                       double* grad_z) {
  const double n = st[0];
  if (!(n > 0)) return fail(SDN_ERR_ARG, "empty sample set");
  const double m1 = st[1] / n;
  const double qmean = h->shift + m1;
  const double qvar = std::max(st[2] / n - m1 * m1, 0.0);
  double value = 0.0, grad_t = 0.0;
  switch (r.kind) {
    case SDN_RISK_MEAN: value = qmean; break;
    case SDN_RISK_MEANVAR: value = qmean + r.beta * qvar; break;
    case SDN_RISK_CVAR_SMOOTH: {
      const double s = 1.0 / (n * (1.0 - r.beta));
      value = r.t + s * st[3];
      grad_t = 1.0 - s * st[4];
      break;
    }
    default: value = pt[h->d_z] / pt[h->d_z + 1]; break;
  }
  value += r.alpha * h->hzz;
  if (grad_z)
    for (int k = 0; k < h->d_z; ++k) grad_z[k] = (r.need_grad ? pt[k] : 0.0) + 2.0 * r.alpha * h->zhost[k];
  if (std::isfinite(qmean)) { h->last_mean = qmean; h->have_mean = true; }
  if (res) {
    res->value = value;
    res->grad_t = grad_t;
    res->n_samples = (int64_t)n;
    res->n_selected = r.kind == SDN_RISK_CVAR_EXACT ? (int64_t)pt[h->d_z + 1]
                      : r.kind == SDN_RISK_CVAR_SMOOTH ? (int64_t)st[5] : (int64_t)n;
    res->q_mean = qmean;
    res->q_var = qvar;
    res->n_refined = 0;
  }
  return SDN_OK;
}

// per-exact-risk selection buffers (sdn_eval_multi)
static int ensure_xsel(sdn_handle* h, int n_exact) {
  int rc;
  while ((int)h->x_rowidx.size() < n_exact) {
    int* r = nullptr;
    int* c = nullptr;
    uint8_t* m = nullptr;
    if ((rc = dalloc(h, &r, h->cap))) return rc;
    if ((rc = dalloc(h, &c, 1))) return rc;
    if ((rc = dalloc(h, &m, h->cap))) return rc;
    h->x_rowidx.push_back(r);
    h->x_nact.push_back(c);
    h->x_mask.push_back(m);
  }
  return SDN_OK;
}

// side stream for overlapped selections (sdn_eval_multi)
static int ensure_side(sdn_handle* h) {
  if (h->side) return SDN_OK;
  CU(cudaStreamCreateWithFlags(&h->side, cudaStreamNonBlocking));
  CU(cudaEventCreateWithFlags(&h->ev_fwd, cudaEventDisableTiming));
  CU(cudaEventCreateWithFlags(&h->ev_side, cudaEventDisableTiming));
  CU(cudaEventCreateWithFlags(&h->ev_qoi, cudaEventDisableTiming));
  CU(cudaEventCreateWithFlags(&h->ev_idx, cudaEventDisableTiming));
  const int nb1024 = (int)cdiv(h->cap, 1024);
  int rc;
  if ((rc = dalloc(h, &h->x_counts, nb1024))) return rc;
  if ((rc = dalloc(h, &h->x_offs, nb1024))) return rc;
  return SDN_OK;
}

// enqueue on the side stream with its own compaction scratch (the helpers
// read these handle fields); the refinement grid fits the reserved SMs
struct SideScope {
  sdn_handle* h;
  cudaStream_t s0;
  int *c0, *o0;
  int g0;
  explicit SideScope(sdn_handle* h_) : h(h_), s0(h_->stream), c0(h_->counts), o0(h_->offs), g0(h_->ref_grid) {
    h->stream = h->side;
    h->counts = h->x_counts;
    h->offs = h->x_offs;
    h->ref_grid = h->side_sms;
  }
  ~SideScope() {
    h->stream = s0;
    h->counts = c0;
    h->offs = o0;
    h->ref_grid = g0;
  }
};

// refined-row count of a risk from the band log (read back with the
// results): smoothed CVaR -> the forward window (slot 0), exact CVaR -> its
// threshold band (exact_slot, -1 = none)
static int64_t refined_count(sdn_handle* h, const sdn_risk& r, int exact_slot) {
  if (h->no_refine || !h->ref_ok) return 0;
  int64_t v = 0;
  if (r.kind == SDN_RISK_CVAR_SMOOTH) v = h->hband[0];
  else if (r.kind == SDN_RISK_CVAR_EXACT && exact_slot > 0) v = h->hband[exact_slot];
  return v;
}

static int eval_finish(sdn_handle* h, const double* stats_dev, const double* partial_dev, sdn_result* res,
                       double* grad_z, int exact_slot = -1) {
  {                                   // results -> host-mapped memory (one kernel, no copy nodes)
    double *dst_s = nullptr, *dst_p = nullptr;
    int* dst_b = nullptr;
    CU(cudaHostGetDevicePointer((void**)&dst_s, h->hstats, 0));
    CU(cudaHostGetDevicePointer((void**)&dst_p, h->hpart, 0));
    CU(cudaHostGetDevicePointer((void**)&dst_b, h->hband, 0));
    k_export<<<1, 256, 0, h->stream>>>(stats_dev, dst_s, STATS_LEN, partial_dev, dst_p, h->plen(), h->band_log,
                                       dst_b, 2);
    h->launches++;
    CHECK_LAUNCH(h);
  }
  CU(cudaStreamSynchronize(h->stream));
  TRY(finish_host(h, h->risk, h->hstats, h->hpart, res, grad_z));
  res->n_refined = refined_count(h, h->risk, exact_slot);
  return SDN_OK;
}

extern "C" {

int sdn_partial_len(sdn_handle* h) { return h ? h->plen() : -1; }

int sdn_eval(sdn_handle* h, const double* z, const sdn_risk* risk, sdn_result* res, double* grad_z,
             int64_t* cvar_idx) {
  if (!h || !z || !risk) return fail(SDN_ERR_ARG, "null argument");
  if (h->n < 1) return fail(SDN_ERR_ARG, "empty sample set");
  return sdn_eval_multi(h, z, risk, 1, res, grad_z, risk->kind == SDN_RISK_CVAR_EXACT ? cvar_idx : nullptr);
}

// ---- small sample sets (BASELINE config 1): one launch per evaluation (small.cuh)
constexpr int64_t SMALL_MAX_ROWS = 1024;
__global__ void k_transpose32(int rows, int cols, const float* __restrict__ A, float* __restrict__ AT) {
  __shared__ float tile[32][33];
  const int x = blockIdx.x * 32 + threadIdx.x, y0 = blockIdx.y * 32;
  for (int j = threadIdx.y; j < 32; j += 8)
    if (x < cols && y0 + j < rows) tile[j][threadIdx.x] = A[(int64_t)(y0 + j) * cols + x];
  __syncthreads();
  const int tx = blockIdx.y * 32 + threadIdx.x, ty0 = blockIdx.x * 32;
  for (int j = threadIdx.y; j < 32; j += 8)
    if (tx < rows && ty0 + j < cols) AT[(int64_t)(ty0 + j) * rows + tx] = tile[threadIdx.x][j];
}
// rows per CTA: 4 (more CTAs, shorter FFMA chains: measured faster) or 8 (SDN_SMALL_RB=8)
static int small_rb() {
  static const int rb = getenv("SDN_SMALL_RB") && atoi(getenv("SDN_SMALL_RB")) == 8 ? 8 : 4;
  return rb;
}
static bool small_eligible(const sdn_handle* h, const sdn_risk* risks, int n_risks) {
  if (h->no_small || h->prof || h->gemm != SDN_GEMM_AUTO || h->n < 1 || h->n > SMALL_MAX_ROWS) return false;
  if (h->L < 1 || h->L > SM_MAXL || h->act == ACT_SOFTMAX || h->r_m > SM_MAXW) return false;
  for (int l = 0; l < h->L; ++l)
    if (h->w[l + 1] > SM_MAXW) return false;
  if (small_smem_bytes(small_rb(), h->L - 1) > TC_SMEM_MAX - 2048) return false;
  for (int i = 0; i < n_risks; ++i) {
    if (risks[i].kind != SDN_RISK_MEAN && risks[i].kind != SDN_RISK_MEANVAR) return false;
    if (risks[i].qoi != SDN_QOI_REDUCED) return false;
  }
  return h->have_form;
}
// buffers and weight transposes (outside any graph capture)
static int ensure_small(sdn_handle* h) {
  int rc;
  if (!h->small_part) {
    if ((rc = dalloc(h, &h->small_part, (size_t)cdiv(std::max<int64_t>(h->cap, 1), 4) * (2 * h->h1 + 4)))) return rc;
  }
  if ((int)h->WT.size() < h->L) {
    h->WT.resize(h->L, nullptr);
    for (int l = 0; l < h->L; ++l) {
      const int K = l == 0 ? h->r_m : h->w[l];
      if ((rc = dalloc(h, &h->WT[l], (size_t)K * h->w[l + 1]))) return rc;
    }
    h->small_gen = -1;
  }
  if (h->small_gen != h->gen) {
    for (int l = 0; l < h->L; ++l) {
      const int K = l == 0 ? h->r_m : h->w[l], N = h->w[l + 1];
      k_transpose32<<<dim3((unsigned)cdiv(K, 32), (unsigned)cdiv(N, 32)), dim3(32, 8), 0, h->stream>>>(N, K, h->W[l],
                                                                                                h->WT[l]);
    }
    h->launches += h->L;
    CHECK_LAUNCH(h);
    h->small_gen = h->gen;
    static unsigned attr = 0;                      // per device
    if (!(attr & (1u << (h->device & 31)))) {
      CU(cudaFuncSetAttribute(k_small_eval<4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)std::min<size_t>(small_smem_bytes(4, SM_MAXL - 1), TC_SMEM_MAX - 2048)));
      CU(cudaFuncSetAttribute(k_small_eval<8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)std::min<size_t>(small_smem_bytes(8, SM_MAXL - 1), TC_SMEM_MAX - 2048)));
      attr |= 1u << (h->device & 31);
    }
  }
  return SDN_OK;
}
static int enqueue_small(sdn_handle* h, const double* z, const sdn_risk* risks, int n_risks) {
  CU(cudaSetDevice(h->device));
  h->risk = risks[0];
  h->fwd_risk = risks[0];
  h->seed_fused = false;
  h->q_fused = false;
  h->selected = false;
  h->compacted = false;
  h->qr_valid = false;
  h->fwd_done = false;                             // the layer buffers are not written on this path
  h->shift = h->q0;
  TRY(upload_z(h, z, risks, n_risks));
  SmallArgs a{};
  a.L = h->L; a.n = (int)h->n; a.r_m = h->r_m; a.d_z = h->d_z; a.r_u = h->r_u; a.h1 = h->h1; a.act = h->act;
  a.R = n_risks; a.plen = h->plen();
  a.w[0] = h->r_m;
  for (int l = 0; l < h->L; ++l) {
    a.w[l + 1] = h->w[l + 1];
    a.res[l] = (l > 0 && l < h->L - 1 && h->res[l]) ? 1 : 0;
    a.W[l] = h->W[l]; a.WT[l] = h->WT[l]; a.b[l] = h->b[l];
  }
  a.MR = h->MR; a.Pz = h->Pz; a.z = h->zdev; a.omean = h->omean; a.ostd = h->ostd; a.c = h->c;
  a.q0 = h->q0; a.shift = h->shift;
  for (int i = 0; i < n_risks; ++i) { a.kind[i] = risks[i].kind; a.beta[i] = risks[i].beta; }
  a.Q = h->Q; a.part = h->small_part; a.PzT = h->PzT; a.stats = h->stats_loc; a.out = h->partial_multi;
  a.counter = h->red_counter + 3;
  CU(cudaHostGetDevicePointer((void**)&a.hstats, h->hstats, 0));
  CU(cudaHostGetDevicePointer((void**)&a.hpart, h->hpart_multi, 0));
  CU(cudaHostGetDevicePointer((void**)&a.hband, h->hband, 0));
  a.nband = n_risks + 1;
  static const bool trace = getenv("SDN_SMALL_TRACE") != nullptr;     // study switch: phase stamps, printed per call
  static unsigned long long* tbuf = nullptr;
  if (trace) {
    if (!tbuf) CU(cudaMalloc(&tbuf, 16 * sizeof(unsigned long long)));
    a.trace = tbuf;
  }
  const int rb = small_rb();
  tl_mark(h, 1);
  if (rb == 8)
    k_small_eval<8><<<(unsigned)cdiv(h->n, 8), SM_THREADS, small_smem_bytes(8, h->L - 1), h->stream>>>(a);
  else
    k_small_eval<4><<<(unsigned)cdiv(h->n, 4), SM_THREADS, small_smem_bytes(4, h->L - 1), h->stream>>>(a);
  h->launches++;
  CHECK_LAUNCH(h);
  if (trace && !h->use_graphs) {
    unsigned long long hb[9];
    CU(cudaMemcpyAsync(hb, tbuf, sizeof(hb), cudaMemcpyDeviceToHost, h->stream));
    CU(cudaStreamSynchronize(h->stream));
    fprintf(stderr, "k_small_eval: CTA 0 [start 0 | inputs %.1f | forward %.1f | Q+seeds %.1f | sweep %.1f | partials %.1f] "
            "last CTA [ticket %.1f | combined %.1f | end %.1f] us\n", (hb[1] - hb[0]) / 1e3, (hb[2] - hb[0]) / 1e3,
            (hb[3] - hb[0]) / 1e3, (hb[4] - hb[0]) / 1e3, (hb[5] - hb[0]) / 1e3, (hb[6] - hb[0]) / 1e3,
            (hb[7] - hb[0]) / 1e3, (hb[8] - hb[0]) / 1e3);
  }
  return SDN_OK;
}

// several risk functionals from ONE forward pass and ONE reverse sweep (e.g.
// c2: mean+variance and exact CVaR).  At most one smoothed-CVaR entry (its
// t/eps feed the forward-time moments and window refinement).
//
// The device work is enqueued by enqueue_multi (no host sync inside); for a
// repeated risk configuration it is captured once into a CUDA graph and
// replayed: one launch per evaluation instead of ~30, which is what bounds
// small problems (c1) and the optimizer loop.  z and each risk's t (the
// smoothed-CVaR variable changes every optimizer step) are staged in pinned
// memory on every call and read by the graph's first copy node.
static int enqueue_multi(sdn_handle* h, const double* z, const sdn_risk* risks, int n_risks, bool want_idx,
                         const std::vector<int64_t>& kks, const std::vector<int64_t>& koff, int smooth,
                         bool any_grad) {
  if (small_eligible(h, risks, n_risks)) return enqueue_small(h, z, risks, n_risks);
  const int plen = h->plen();
  int n_exact = 0;
  bool dense = false;
  for (int i = 0; i < n_risks; ++i) {
    n_exact += risks[i].kind == SDN_RISK_CVAR_EXACT;
    dense |= risks[i].kind == SDN_RISK_MEAN || risks[i].kind == SDN_RISK_MEANVAR;
  }
  // a dense sweep over all rows: the output layer writes its unit seeds
  // Overlap (a dense risk present, see below): the QoI runs first on the side
  // stream -- the sweep's unit seeds never read Q, so the reverse chain starts
  // right behind the forward; Q and the moments join before the last GEMM
  const bool overlap = dense && n_exact > 0 && !h->prof && !h->no_overlap;
  static const bool qoi_main = getenv("SDN_QOI_MAIN") && getenv("SDN_QOI_MAIN")[0] == '1';   // study switch
  const bool qoi_side = overlap && smooth < 0 && any_grad && h->tcw.enabled && !qoi_main;
  TRY(eval_forward(h, z, &risks[smooth >= 0 ? smooth : 0], h->stats_loc, any_grad, risks, n_risks,
                   smooth >= 0 ? smooth : 0, dense && any_grad, qoi_side));
  std::vector<const uint8_t*> masks(n_risks, nullptr);
  std::vector<const int*> sel_rows(n_risks, nullptr);
  auto select_all = [&]() -> int {
    for (int i = 0, e = 0; i < n_risks; ++i) {
      if (risks[i].kind != SDN_RISK_CVAR_EXACT) continue;
      h->risk = risks[i];
      TRY(select_local(h, kks[i], h->band_log + 1 + i, h->x_mask[e], h->x_rowidx[e], h->x_nact[e]));
      masks[i] = h->x_mask[e];
      sel_rows[i] = h->x_rowidx[e];
      ++e;
    }
    return SDN_OK;
  };
  // the selections' indices -> host (on the stream that made them)
  auto copy_idx = [&]() -> int {
    if (!want_idx) return SDN_OK;
    for (int i = 0, e = 0; i < n_risks; ++i) {
      if (risks[i].kind != SDN_RISK_CVAR_EXACT) continue;
      CU(cudaMemcpyAsync(h->hidx + koff[i], h->x_rowidx[e], sizeof(int) * kks[i], cudaMemcpyDeviceToHost,
                         h->stream));
      ++e;
    }
    return SDN_OK;
  };
  // Overlap (a dense risk present): the selections (top-k, fp64 refinement
  // of the threshold band, index compaction) only read Q, and the one sweep
  // first needs the masks at its last GEMM -- so they run on the side stream
  // (side_sms SMs kept free of the persistent GEMMs meanwhile) while the main
  // stream seeds and runs the first L-2 sweep GEMMs.  The sweep's seeds are
  // unit weights (no Q read), so the in-place refinement of Q cannot race.
  // (Profiling runs serialise: its class timers are stream-ordered.)
  std::function<int()> join, qjoin;
  if (overlap) {
    CU(cudaEventRecord(h->ev_fwd, h->stream));
    CU(cudaStreamWaitEvent(h->side, h->ev_fwd, 0));
    tl_mark(h, 4, h->side);
    {
      SideScope ss(h);
      if (qoi_side) {
        TRY(launch_qoi(h, &risks[0], h->stats_loc, h->zdev + h->d_z));
        CU(cudaEventRecord(h->ev_qoi, h->side));
        qjoin = [h]() -> int {
          CU(cudaStreamWaitEvent(h->stream, h->ev_qoi, 0));
          return SDN_OK;
        };
      }
      TRY(select_all());
    }
    tl_mark(h, 5, h->side);
    CU(cudaEventRecord(h->ev_side, h->side));
    {                                 // the index copies stay off the path the tail waits for
      SideScope ss(h);
      TRY(copy_idx());
    }
    CU(cudaEventRecord(h->ev_idx, h->side));
    h->sm_avail = h->num_sms - h->side_sms;
    join = [h]() -> int {
      h->sm_avail = h->num_sms;
      CU(cudaStreamWaitEvent(h->stream, h->ev_side, 0));
      return SDN_OK;
    };
  } else {
    TRY(select_all());
    TRY(copy_idx());
  }
  h->risk = risks[0];
  // results -> host-mapped memory: by the sweep's fused tail when it runs,
  // else by one export kernel (no copy nodes either way)
  double *dst_s = nullptr, *dst_p = nullptr;
  int* dst_b = nullptr;
  CU(cudaHostGetDevicePointer((void**)&dst_s, h->hstats, 0));
  CU(cudaHostGetDevicePointer((void**)&dst_p, h->hpart_multi, 0));
  CU(cudaHostGetDevicePointer((void**)&dst_b, h->hband, 0));
  h->exp_want = true;
  h->exp_done = false;
  h->exp_s = dst_s; h->exp_p = dst_p; h->exp_b = dst_b;
  h->exp_np = n_risks * plen; h->exp_nb = n_risks + 1;
  int rc = backward_multi(h, risks, n_risks, masks.data(), kks.data(), h->stats_loc, h->partial_multi, join,
                          h->zdev + h->d_z, sel_rows.data(), qjoin);
  h->sm_avail = h->num_sms;
  h->exp_want = false;
  if (rc) return rc;
  if (overlap) CU(cudaStreamWaitEvent(h->stream, h->ev_idx, 0));   // the side stream rejoins (index copies done)
  if (!h->exp_done) {
    k_export<<<1, 256, 0, h->stream>>>(h->stats_loc, dst_s, STATS_LEN, h->partial_multi, dst_p, n_risks * plen,
                                       h->band_log, dst_b, n_risks + 1);
    h->launches++;
    CHECK_LAUNCH(h);
  }
  return SDN_OK;
}

// graph cache key of an evaluation configuration
static std::vector<double> graph_key(sdn_handle* h, const sdn_risk* risks, int n_risks, bool want_idx) {
  std::vector<double> k{(double)h->gen, (double)h->n, (double)n_risks, want_idx ? 1.0 : 0.0};
  for (int i = 0; i < n_risks; ++i) {
    k.push_back(risks[i].kind);
    k.push_back(risks[i].qoi);
    k.push_back(risks[i].beta);
    k.push_back(risks[i].eps);
    k.push_back(risks[i].need_grad);
  }
  return k;
}

static void drop_graph(sdn_handle* h) {
  if (h->gexec) cudaGraphExecDestroy(h->gexec);
  h->gexec = nullptr;
  h->gkey.clear();
}

int sdn_eval_multi_launch(sdn_handle* h, const double* z, const sdn_risk* risks, int32_t n_risks, int32_t want_idx_i) {
  if (!h || !z || !risks || n_risks < 1) return fail(SDN_ERR_ARG, "null argument");
  h->pending = false;
  if (h->n < 1) return fail(SDN_ERR_ARG, "empty sample set");
  if (n_risks > SDN_RMAX) return fail(SDN_ERR_ARG, "at most 8 risks per evaluation");
  int smooth = -1, any_grad = 0;
  for (int i = 0; i < n_risks; ++i) {
    TRY(check_risk(&risks[i]));
    if (risks[i].qoi != risks[0].qoi) return fail(SDN_ERR_ARG, "all risks must share the QoI frame");
    if (risks[i].kind == SDN_RISK_CVAR_SMOOTH) {
      if (smooth >= 0) return fail(SDN_ERR_ARG, "at most one smoothed CVaR per multi-evaluation");
      smooth = i;
    }
    any_grad |= risks[i].need_grad;
  }
  if (!h->have_model) return fail(SDN_ERR_STATE, "set_model first");
  if (risks[0].qoi == SDN_QOI_REDUCED && !h->have_form) return fail(SDN_ERR_STATE, "set_tracking first");
  if (risks[0].qoi == SDN_QOI_DECODED && !h->have_dec) return fail(SDN_ERR_STATE, "set_decoder first");
  CU(cudaSetDevice(h->device));
  // host-side buffers (never allocated while a graph is being captured)
  const int plen = h->plen();
  std::vector<int64_t> koff(n_risks, -1), kks(n_risks, 0);
  int64_t ktot = 0;
  int n_exact = 0;
  bool dense = false;
  for (int i = 0; i < n_risks; ++i) {
    dense |= risks[i].kind == SDN_RISK_MEAN || risks[i].kind == SDN_RISK_MEANVAR;
    if (risks[i].kind == SDN_RISK_CVAR_EXACT) {
      kks[i] = std::max(ceil_count((1.0 - risks[i].beta) * (double)h->n), 1);   // riskopt.py:80
      koff[i] = ktot;
      ktot += kks[i];
      ++n_exact;
    }
  }
  if (n_risks > h->multi_cap || ktot > h->hidx_cap) {
    drop_graph(h);
    if (h->partial_multi) cudaFree(h->partial_multi);
    if (h->hpart_multi) cudaFreeHost(h->hpart_multi);
    if (h->hidx) cudaFreeHost(h->hidx);
    h->multi_cap = std::max(n_risks, 4);
    h->hidx_cap = std::max<int64_t>(ktot, 1);
    CU(cudaMalloc(&h->partial_multi, sizeof(double) * h->multi_cap * plen));
    CU(cudaHostAlloc((void**)&h->hpart_multi, sizeof(double) * h->multi_cap * plen, cudaHostAllocMapped));
    CU(cudaHostAlloc((void**)&h->hidx, sizeof(int) * h->hidx_cap, 0));
  }
  if (n_risks + 1 > h->band_cap) {
    drop_graph(h);
    int* bl = nullptr;
    int* hb = nullptr;
    CU(cudaMalloc(&bl, sizeof(int) * (n_risks + 1)));
    CU(cudaHostAlloc((void**)&hb, sizeof(int) * (n_risks + 1), cudaHostAllocMapped));
    h->allocs.push_back(bl);
    if (h->hband) cudaFreeHost(h->hband);
    h->band_log = bl;                // (the old block stays in allocs until destroy)
    h->hband = hb;
    h->band_cap = n_risks + 1;
  }
  TRY(ensure_xsel(h, n_exact));
  if (!h->dev_ev[0]) {
    CU(cudaEventCreate(&h->dev_ev[0]));
    CU(cudaEventCreate(&h->dev_ev[1]));
  }
  if (dense && n_exact > 0) TRY(ensure_side(h));
  TRY(ensure_sweep(h, *h->sw, n_risks));
  if (small_eligible(h, risks, n_risks)) TRY(ensure_small(h));
  // graph path (z and every risk's t are per-call graph parameters, staged
  // in pinned memory); not when profiling / tracing (host timers and syncs)
  const bool use_graph = h->use_graphs && !h->prof && !h->ref_trace;
  const bool want_idx = want_idx_i != 0;
  if (use_graph) {
    const std::vector<double> key = graph_key(h, risks, n_risks, want_idx);
    if (!h->gexec || key != h->gkey) {
      drop_graph(h);
      const int64_t l0 = h->launches;
      CU(cudaStreamBeginCapture(h->stream, cudaStreamCaptureModeRelaxed));
      // the device span events are nodes of the graph itself (first and last):
      // the span excludes any host delay in submitting the replay
      cudaError_t ee = cudaEventRecordWithFlags(h->dev_ev[0], h->stream, cudaEventRecordExternal);
      tl_mark(h, 0);
      int rc = ee == cudaSuccess ? enqueue_multi(h, z, risks, n_risks, want_idx, kks, koff, smooth, any_grad != 0)
                                 : fail(SDN_ERR_CUDA, "event record node");
      tl_mark(h, 11);
      if (rc == SDN_OK && cudaEventRecordWithFlags(h->dev_ev[1], h->stream, cudaEventRecordExternal) != cudaSuccess)
        rc = fail(SDN_ERR_CUDA, "event record node");
      cudaGraph_t g = nullptr;
      cudaError_t ce = cudaStreamEndCapture(h->stream, &g);
      if (rc != SDN_OK) { if (g) cudaGraphDestroy(g); return rc; }
      if (ce != cudaSuccess) return fail(SDN_ERR_CUDA, std::string("graph capture: ") + cudaGetErrorString(ce));
      ce = cudaGraphInstantiate(&h->gexec, g, 0);
      cudaGraphDestroy(g);
      if (ce != cudaSuccess) { h->gexec = nullptr; return fail(SDN_ERR_CUDA, "graph instantiate failed"); }
      h->gkey = key;
      h->glaunches = h->launches - l0;
      h->launches = l0;
    } else {
      // per-call host state of eval_forward / upload_z
      h->risk = risks[0];
      h->fwd_risk = risks[smooth >= 0 ? smooth : 0];
      h->selected = h->compacted = h->qr_valid = false;
      h->shift = risks[0].qoi == SDN_QOI_DECODED ? h->q0dec : h->q0;
      stage_z(h, z, risks, n_risks);
      h->fwd_done = true;
      h->qr_valid = n_exact > 0;
    }
    CU(cudaGraphLaunch(h->gexec, h->stream));
    h->launches += h->glaunches;
  } else {
    CU(cudaEventRecord(h->dev_ev[0], h->stream));
    TRY(enqueue_multi(h, z, risks, n_risks, want_idx, kks, koff, smooth, any_grad != 0));
    CU(cudaEventRecord(h->dev_ev[1], h->stream));
  }
  h->pend_risks.assign(risks, risks + n_risks);
  h->pend_ktot = ktot;
  h->pend_idx = want_idx;
  h->pending = true;
  return SDN_OK;
}

// wait for the evaluation sdn_eval_multi_launch enqueued and read its results
int sdn_eval_multi_wait(sdn_handle* h, sdn_result* res, double* grads, int64_t* cvar_idx) {
  if (!h || !res) return fail(SDN_ERR_ARG, "null argument");
  if (!h->pending) return fail(SDN_ERR_STATE, "sdn_eval_multi_launch first");
  if (cvar_idx && !h->pend_idx) return fail(SDN_ERR_ARG, "indices were not requested at launch");
  h->pending = false;
  CU(cudaSetDevice(h->device));
  const int n_risks = (int)h->pend_risks.size();
  const sdn_risk* risks = h->pend_risks.data();
  const int64_t ktot = h->pend_ktot;
  const int plen = h->plen();
  CU(cudaStreamSynchronize(h->stream));
  {
    float t = 0.f;
    h->last_dev_ms = cudaEventElapsedTime(&t, h->dev_ev[0], h->dev_ev[1]) == cudaSuccess ? (double)t : -1.0;
  }
  if (h->tl_on && h->tl_hit[0] && h->tl_hit[11]) {      // stage timeline (us from the graph's first node)
    fprintf(stderr, "timeline:");
    for (int i = 1; i < 12; ++i) {
      float t = 0.f;
      if (h->tl_hit[i] && cudaEventElapsedTime(&t, h->tl[0], h->tl[i]) == cudaSuccess)
        fprintf(stderr, " | %s %.1f", TL_NAMES[i], 1e3 * t);
    }
    fprintf(stderr, "\n");
  }
  for (int i = 0; i < n_risks; ++i) {
    TRY(finish_host(h, risks[i], h->hstats, h->hpart_multi + (size_t)i * plen, &res[i],
                    grads ? grads + (size_t)i * h->d_z : nullptr));
    res[i].n_refined = refined_count(h, risks[i], 1 + i);
  }
  if (cvar_idx)
    for (int64_t j = 0; j < ktot; ++j) cvar_idx[j] = h->goff + h->hidx[j];
  return SDN_OK;
}

int sdn_eval_multi(sdn_handle* h, const double* z, const sdn_risk* risks, int32_t n_risks, sdn_result* res,
                   double* grads, int64_t* cvar_idx) {
  if (!h || !z || !risks || n_risks < 1 || !res) return fail(SDN_ERR_ARG, "null argument");
  TRY(sdn_eval_multi_launch(h, z, risks, n_risks, cvar_idx != nullptr));
  return sdn_eval_multi_wait(h, res, grads, cvar_idx);
}

int sdn_last_device_ms(sdn_handle* h, double* ms) {
  if (!h || !ms) return fail(SDN_ERR_ARG, "null argument");
  *ms = h->last_dev_ms;
  return SDN_OK;
}

int sdn_profile(sdn_handle* h, int32_t enable) {
  if (!h) return fail(SDN_ERR_ARG, "null handle");
  CU(cudaStreamSynchronize(h->stream));
  h->prof = enable != 0;
  h->recs.clear();
  h->pool_used = 0;
  return SDN_OK;
}

// per-class totals since sdn_profile(h, 1): ms, algorithmic flops, bytes,
// launches.  Arrays of length n_cls (<= SDN_PROF_CLASSES).
int sdn_profile_read(sdn_handle* h, int32_t n_cls, double* ms, double* flops, double* bytes, int64_t* count) {
  if (!h || !ms || !flops || !bytes || !count) return fail(SDN_ERR_ARG, "null argument");
  CU(cudaStreamSynchronize(h->stream));
  for (int c = 0; c < n_cls; ++c) { ms[c] = 0; flops[c] = 0; bytes[c] = 0; count[c] = 0; }
  int nact = 0;
  CU(cudaMemcpy(&nact, h->n_act_dev, sizeof(int), cudaMemcpyDeviceToHost));
  for (auto& r : h->recs) {
    if (r.cls < 0 || r.cls >= n_cls) continue;
    float t = 0.0f;
    CU(cudaEventElapsedTime(&t, r.a, r.b));
    ms[r.cls] += t;
    double f = r.flops, b = r.bytes;
    if (r.rows < 0) f += (double)nact * r.per_row;
    else if (r.per_row > 0.0 && r.flops == 0.0 && r.bytes == 0.0) b += (double)r.rows * r.per_row;
    flops[r.cls] += f;
    bytes[r.cls] += b;
    count[r.cls] += 1;
  }
  return SDN_OK;
}

int sdn_eval_forward(sdn_handle* h, const double* z, const sdn_risk* risk, double* stats_dev) {
  if (!h || !z || !risk || !stats_dev) return fail(SDN_ERR_ARG, "null argument");
  return eval_forward(h, z, risk, stats_dev, risk->need_grad != 0);
}

int sdn_eval_candidates(sdn_handle* h, int64_t k, double* cand_dev) {
  if (!h || !cand_dev || k < 1) return fail(SDN_ERR_ARG, "bad argument");
  if (!h->fwd_done) return fail(SDN_ERR_STATE, "eval_forward first");
  CU(cudaSetDevice(h->device));
  const int64_t kl = std::min<int64_t>(k, h->n);
  if (kl > 0) {
    TRY(launch_topk(h, h->n, kl, sel_q(h), nullptr, h->sel));
    TRY(compact_rows(h, RISK_CVAR_EXACT, 0.0, 1.0));
  } else {
    CU(cudaMemsetAsync(h->n_act_dev, 0, sizeof(int), h->stream));
  }
  k_export_candidates<<<(unsigned)cdiv(k, 256), 256, 0, h->stream>>>(k, h->n_act_dev, h->rowidx, sel_q(h), h->goff,
                                                                      cand_dev);
  h->launches++;
  CHECK_LAUNCH(h);
  return SDN_OK;
}

int sdn_eval_select(sdn_handle* h, const double* all_cand_dev, int32_t n_ranks, int64_t k) {
  if (!h || !all_cand_dev || n_ranks < 1 || k < 1) return fail(SDN_ERR_ARG, "bad argument");
  CU(cudaSetDevice(h->device));
  const int64_t nc = (int64_t)n_ranks * k;
  TRY(ensure_cand(h, nc));
  k_unpack_candidates<<<(unsigned)cdiv(nc, 256), 256, 0, h->stream>>>(n_ranks, k, all_cand_dev, h->cand_vals,
                                                                      h->cand_gidx);
  TRY(launch_topk(h, nc, k, h->cand_vals, h->cand_gidx, h->cand_mask, h->thr_dev));
  h->n_cand = nc;
  CU(cudaMemsetAsync(h->sel, 0, std::max<int64_t>(h->n, 1), h->stream));
  k_scatter_selection<<<(unsigned)cdiv(nc, 256), 256, 0, h->stream>>>(nc, h->cand_mask, h->cand_gidx, h->goff,
                                                                      h->n, h->sel);
  h->launches += 3;
  CHECK_LAUNCH(h);
  TRY(compact_rows(h, RISK_CVAR_EXACT, 0.0, 1.0));
  h->kk = k;
  h->selected = true;
  return SDN_OK;
}

// multi-rank exact CVaR: after a global selection (sdn_eval_select, which
// leaves the global threshold on the device), re-evaluate this shard's rows
// within refinement error of it in fp64 (Q updated in place).  The caller
// then repeats candidates -> all-gather -> select on the refined Q.
int sdn_eval_refine_band(sdn_handle* h) {
  if (!h) return fail(SDN_ERR_ARG, "null handle");
  if (!h->fwd_done || !h->selected) return fail(SDN_ERR_STATE, "eval_select first");
  CU(cudaSetDevice(h->device));
  if (h->no_refine || h->n == 0) return SDN_OK;
  TRY(refine_band(h, RISK_BAND_EXACT, 0.0, 0.0, h->risk.qoi == SDN_QOI_DECODED, h->band_log + 1, nullptr,
                  sel_q(h)));
  h->selected = false;
  return SDN_OK;
}

// multi-rank, several risks: keep the current exact-CVaR selection (after
// its final sdn_eval_select) in slot `slot` for sdn_eval_backward_multi
int sdn_eval_keep_selection(sdn_handle* h, int32_t slot) {
  if (!h || slot < 0 || slot >= SDN_RMAX) return fail(SDN_ERR_ARG, "bad argument");
  if (!h->fwd_done || !h->selected) return fail(SDN_ERR_STATE, "eval_select first");
  CU(cudaSetDevice(h->device));
  TRY(ensure_xsel(h, slot + 1));
  if ((int)h->x_k.size() < slot + 1) h->x_k.resize(slot + 1, 0);
  CU(cudaMemcpyAsync(h->x_mask[slot], h->sel, std::max<int64_t>(h->n, 1), cudaMemcpyDeviceToDevice, h->stream));
  h->x_k[slot] = h->kk;
  // the global selection (identical on every rank) as ascending global indices
  if ((int)h->x_gidx.size() < slot + 1) { h->x_gidx.resize(slot + 1, nullptr); h->x_gcap.resize(slot + 1, 0); }
  if (h->x_gcap[slot] < h->kk) {
    int rc;
    if ((rc = dalloc(h, &h->x_gidx[slot], h->kk))) return rc;
    h->x_gcap[slot] = h->kk;
  }
  k_selection_gidx<<<1, 1024, 0, h->stream>>>(h->n_cand, h->cand_mask, h->cand_gidx, h->kk, h->x_gidx[slot]);
  h->launches++;
  CHECK_LAUNCH(h);
  return SDN_OK;
}

// multi-rank: the kept exact-CVaR selection of `slot` as k ascending GLOBAL
// sample indices (host buffer; every rank returns the same set)
int sdn_eval_selection(sdn_handle* h, int32_t slot, int64_t k, int64_t* idx_out) {
  if (!h || !idx_out || slot < 0) return fail(SDN_ERR_ARG, "bad argument");
  if (slot >= (int)h->x_gidx.size() || !h->x_gidx[slot]) return fail(SDN_ERR_STATE, "eval_keep_selection first");
  if (k != h->x_k[slot]) return fail(SDN_ERR_ARG, "k does not match the kept selection");
  CU(cudaSetDevice(h->device));
  CU(cudaMemcpyAsync(idx_out, h->x_gidx[slot], sizeof(int64_t) * k, cudaMemcpyDeviceToHost, h->stream));
  CU(cudaStreamSynchronize(h->stream));
  return SDN_OK;
}

// multi-rank, several risks: ONE reverse sweep for all of them (the i-th
// exact-CVaR risk in the list uses kept selection slot i); partials_dev holds
// n_risks x sdn_partial_len(h) doubles (one all-reduce for all risks)
int sdn_eval_backward_multi(sdn_handle* h, const sdn_risk* risks, int32_t n_risks, const double* stats_dev,
                            double* partials_dev) {
  if (!h || !risks || !stats_dev || !partials_dev || n_risks < 1 || n_risks > SDN_RMAX)
    return fail(SDN_ERR_ARG, "bad argument");
  if (!h->fwd_done) return fail(SDN_ERR_STATE, "eval_forward first");
  CU(cudaSetDevice(h->device));
  std::vector<const uint8_t*> masks(n_risks, nullptr);
  std::vector<int64_t> ks(n_risks, 0);
  for (int i = 0, e = 0; i < n_risks; ++i) {
    TRY(check_risk(&risks[i]));
    if (risks[i].qoi != h->risk.qoi) return fail(SDN_ERR_ARG, "risks must keep the forward's QoI frame");
    if (risks[i].kind != SDN_RISK_CVAR_EXACT) continue;
    if (e >= (int)h->x_k.size() || h->x_k[e] < 1) return fail(SDN_ERR_STATE, "exact CVaR needs a kept selection");
    masks[i] = h->x_mask[e];
    ks[i] = h->x_k[e];
    ++e;
  }
  TRY(ensure_sweep(h, *h->sw, n_risks));
  return backward_multi(h, risks, n_risks, masks.data(), ks.data(), stats_dev, partials_dev);
}

// next reverse sweep after one forward (multi-risk): same QoI frame; a
// smoothed CVaR must be the forward's own risk (its t/eps fed the moments)
int sdn_eval_set_risk(sdn_handle* h, const sdn_risk* risk) {
  if (!h || !risk) return fail(SDN_ERR_ARG, "null argument");
  TRY(check_risk(risk));
  if (!h->fwd_done) return fail(SDN_ERR_STATE, "eval_forward first");
  if (risk->qoi != h->risk.qoi) return fail(SDN_ERR_ARG, "risk must keep the forward's QoI frame");
  if (risk->kind == SDN_RISK_CVAR_SMOOTH &&
      (h->fwd_risk.kind != SDN_RISK_CVAR_SMOOTH || risk->t != h->fwd_risk.t || risk->eps != h->fwd_risk.eps))
    return fail(SDN_ERR_ARG, "smoothed CVaR must be the forward's risk");
  h->risk = *risk;
  h->compacted = false;
  h->selected = false;
  return SDN_OK;
}

int sdn_eval_backward(sdn_handle* h, const double* stats_dev, double* partial_dev) {
  if (!h || !stats_dev || !partial_dev) return fail(SDN_ERR_ARG, "null argument");
  CU(cudaSetDevice(h->device));
  return eval_backward(h, stats_dev, partial_dev);
}

int sdn_eval_finish(sdn_handle* h, const double* stats_dev, const double* partial_dev, sdn_result* res,
                    double* grad_z) {
  if (!h || !stats_dev || !partial_dev) return fail(SDN_ERR_ARG, "null argument");
  CU(cudaSetDevice(h->device));
  return eval_finish(h, stats_dev, partial_dev, res, grad_z);
}

int sdn_last_q(sdn_handle* h, const double** q_dev, int64_t* n) {
  if (!h || !q_dev || !n) return fail(SDN_ERR_ARG, "null argument");
  *q_dev = h->Q;
  *n = h->n;
  return SDN_OK;
}

int sdn_last_qsel(sdn_handle* h, const double** q_dev, int64_t* n) {
  if (!h || !q_dev || !n) return fail(SDN_ERR_ARG, "null argument");
  *q_dev = h->qr_valid ? h->Qr : h->Q;
  *n = h->n;
  return SDN_OK;
}

// per-sample (Q, G): unit weights through the same sweep, then G = dL/dS_0 Pz
int sdn_eval_samples(sdn_handle* h, const double* z, int32_t qoi, double* Qout, double* Gout) {
  if (!h || !z || !Qout) return fail(SDN_ERR_ARG, "null argument");
  if (h->n < 1) return fail(SDN_ERR_ARG, "empty sample set");
  sdn_risk r{};
  r.kind = SDN_RISK_MEAN;
  r.qoi = qoi;
  r.beta = 0.0;
  r.eps = 1.0;
  r.need_grad = Gout != nullptr;
  TRY(eval_forward(h, z, &r, h->stats_loc, Gout != nullptr));
  if (Gout) {
    if (!h->Gz) CU(cudaMalloc(&h->Gz, sizeof(float) * h->cap * h->d_zp));
    const bool dec = qoi == SDN_QOI_DECODED;
    const int sg = (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(h->n, 8), 4 * h->num_sms));
    k_seed<<<sg, 256, 0, h->stream>>>(h->n, nullptr, nullptr, h->r_u, h->Y, dec ? h->KPhi : nullptr,
                                      dec ? h->cdec : h->c, h->ostd, h->Q, h->stats_loc, RISK_UNIT, 0.0, 0.0,
                                      1.0, 0.0, 0.0, h->E);
    h->launches++;
    CHECK_LAUNCH(h);
    if (h->tcw.enabled) TRY(tc_split_seed(h, h->tcw, h->E, h->n, nullptr));
    float* u0 = nullptr;
    TRY(run_backward(h, h->n, nullptr, nullptr, &u0, h->n, /*want_u0=*/true));
    TRY((gemm<false, false>(h, h->n, nullptr, h->d_zp, h->h1, u0, h->h1, h->Pz32, h->d_zp,
                            EpiStore{h->Gz, (int64_t)h->d_zp})));
    double* gd = nullptr;
    CU(cudaMalloc(&gd, sizeof(double) * h->n * h->d_z));
    k_copy_g<<<(unsigned)std::min<int64_t>(cdiv(h->n * h->d_z, 256), 65535), 256, 0, h->stream>>>(
        h->n, h->d_z, h->d_zp, h->Gz, gd);
    h->launches++;
    cudaError_t e = cudaMemcpyAsync(Gout, gd, sizeof(double) * h->n * h->d_z, cudaMemcpyDeviceToHost, h->stream);
    cudaError_t e2 = cudaStreamSynchronize(h->stream);
    cudaFree(gd);
    if (e != cudaSuccess || e2 != cudaSuccess) return fail(SDN_ERR_CUDA, "G download failed");
  }
  CU(cudaMemcpyAsync(Qout, h->Q, sizeof(double) * h->n, cudaMemcpyDeviceToHost, h->stream));
  CU(cudaStreamSynchronize(h->stream));
  return SDN_OK;
}

// rows with their own z: X = [m_r | z] through Wx = [W0m' | Pz]
static int forward_rows(sdn_handle* h, const float* mr_dev, const float* z_dev, int64_t n, float* X, bool store_D,
                        float* phi_dev) {
  k_build_x<<<(unsigned)n, 128, 0, h->stream>>>(n, h->r_m, h->d_z, h->ldx, mr_dev, z_dev, X);
  h->launches++;
  CHECK_LAUNCH(h);
  return run_forward(h, n, X, h->ldx, h->ldx, h->Wx, h->ldx, h->b[0], store_D, phi_dev, nullptr);
}

int sdn_forward_batch(sdn_handle* h, const float* m_r, const float* z, int64_t n, float* phi) {
  if (!h || !m_r || !z || !phi) return fail(SDN_ERR_ARG, "null argument");
  if (!h->have_model) return fail(SDN_ERR_STATE, "set_model first");
  if (n < 0) return fail(SDN_ERR_ARG, "negative row count");
  CU(cudaSetDevice(h->device));
  const int64_t chunk = h->cap;
  float *mr = nullptr, *zz = nullptr, *X = nullptr;
  TRY(scratch(h, SCR_A, (size_t)chunk * h->r_m, &mr));
  TRY(scratch(h, SCR_B, (size_t)chunk * h->d_z, &zz));
  TRY(scratch(h, SCR_C, (size_t)chunk * h->ldx, &X));
  int rc = SDN_OK;
  for (int64_t s = 0; s < n && rc == SDN_OK; s += chunk) {
    const int64_t m = std::min(chunk, n - s);
    if (cudaMemcpyAsync(mr, m_r + s * h->r_m, sizeof(float) * m * h->r_m, cudaMemcpyHostToDevice, h->stream) ||
        cudaMemcpyAsync(zz, z + s * h->d_z, sizeof(float) * m * h->d_z, cudaMemcpyHostToDevice, h->stream)) {
      rc = fail(SDN_ERR_CUDA, "upload failed");
      break;
    }
    rc = forward_rows(h, mr, zz, m, X, false, h->Y);
    if (rc == SDN_OK &&
        (cudaMemcpyAsync(phi + s * h->r_u, h->Y, sizeof(float) * m * h->r_u, cudaMemcpyDeviceToHost, h->stream) ||
         cudaStreamSynchronize(h->stream)))
      rc = fail(SDN_ERR_CUDA, "download failed");
  }
  cudaStreamSynchronize(h->stream);
  return rc;
}

// forward-mode control Jacobian (surrogate.py:195-233) on the device:
// tangent rows (i*d_z + k) through the chain; decoded: U (std . J)
// (test_acceptance.py:326).  The tangent GEMMs run on the tensor cores
// (bf16x3, act' gathered per sample in the epilogue, tangents kept only as
// the next GEMM's split) whenever the forward chain does; the output is
// scattered straight into J[i, u, k] by the last GEMM's epilogue (a warp's
// 32 rows are consecutive k of one or two samples: coalesced).

static bool jac_tc(sdn_handle* h) {
  return h->tcw.enabled && h->gemm != SDN_GEMM_SIMT && h->L >= 2 && h->act != ACT_SOFTMAX;
}

// scratch for `rows` tangent rows (grown, never shrunk; freed at destroy)
static int jac_scratch(sdn_handle* h, int64_t rows, bool decoded) {
  if (rows <= h->jac_rows && (!decoded || h->jjr.hi || !jac_tc(h))) return SDN_OK;
  const int64_t cap = std::max(rows, h->jac_rows);
  const int wmax = std::max(h->maxw, h->r_u);
  int rc;
  if (jac_tc(h)) {
    for (int i = 0; i < 2; ++i)
      if (tc_buf(h, h->tcw, h->jtan[i], cap, wmax)) return fail(SDN_ERR_NOMEM, "jacobian scratch");
    if (decoded && tc_buf(h, h->tcw, h->jjr, cap, h->r_u)) return fail(SDN_ERR_NOMEM, "jacobian scratch");
  } else {
    for (int i = 0; i < 2; ++i)
      if ((rc = dalloc(h, &h->jT[i], (size_t)cap * wmax))) return rc;
    if ((rc = dalloc(h, &h->jJt, (size_t)cap * h->r_u))) return rc;
  }
  h->jac_rows = cap;
  return SDN_OK;
}

// tangent-row budget of one chunk (~1.5 GB of scratch)
static int64_t jac_chunk_samples(sdn_handle* h, bool decoded) {
  const int64_t per_row = 4ll * (2 * std::max(h->maxw, h->r_u) + (decoded ? h->r_u : 0));
  const int64_t rows = std::max<int64_t>(h->d_z, (1536ll << 20) / per_row);
  return std::max<int64_t>(1, std::min<int64_t>(h->cap, rows / h->d_z));
}

// Jacobians of m samples whose forward (act' in D[l] rows dro .. dro + m)
// is done, into J (device, m x outw x d_z)
static int jac_rows(sdn_handle* h, int64_t dro, int64_t m, bool decoded, float* J) {
  const int d_z = h->d_z, L = h->L;
  const int64_t rows = m * d_z;
  TRY(jac_scratch(h, rows, decoded));
  const float* D0 = h->act == ACT_SOFTMAX ? nullptr : h->D[0] + dro * h->w[1];
  if (jac_tc(h)) {
    // seed (the tangent of x_z = V_z^T z through W1_z is the constant Pz), as a split
    TcOperand* Tc = &h->jtan[0];
    TcOperand* Tn = &h->jtan[1];
    { ProfScope ps(h, PC_SEED, 0.0, 4.0 * rows * Tc->ld);
      k_tangent_seed_split<<<(unsigned)std::min<int64_t>(cdiv(rows, 8), 32ll * h->num_sms), 256, 0, h->stream>>>(
          rows, d_z, h->h1, Tc->ld, D0, h->Pz32t, Tc->hi, Tc->lo); }
    h->launches++;
    CHECK_LAUNCH(h);
    for (int l = 1; l < L - 1; ++l) {
      TcChain<EpiTanTc> e{EpiTanTc{h->D[l] + dro * h->w[l + 1], (int64_t)h->w[l + 1], d_z}, TcEpiSplit{Tn},
                          TcEpiSplit{h->res[l] ? Tc : nullptr}};
      ProfScope ps(h, PC_TANGENT, 2.0 * rows * h->w[l + 1] * h->w[l], 0.0);
      const int rc = tc_gemm(h->tcw, h->stream, h->sm_avail, rows, nullptr, h->w[l + 1], h->w[l], *Tc,
                             h->tcw.fwd[l], e, rows);
      h->launches++;
      if (rc) return fail(SDN_ERR_CUDA, "tangent GEMM launch failed (" + std::to_string(rc) + ")");
      CHECK_LAUNCH(h);
      std::swap(Tc, Tn);
    }
    const int Kl = h->w[L - 1];
    int rc;
    if (!decoded) {
      ProfScope ps(h, PC_TANGENT, 2.0 * rows * h->r_u * Kl, 4.0 * rows * h->r_u);
      rc = tc_gemm(h->tcw, h->stream, h->sm_avail, rows, nullptr, h->r_u, Kl, *Tc, h->tcw.fwd[L - 1],
                   EpiJacScatter{h->ostd, J, d_z, (int64_t)h->r_u}, rows);
    } else {
      { ProfScope ps(h, PC_TANGENT, 2.0 * rows * h->r_u * Kl, 0.0);
        rc = tc_gemm(h->tcw, h->stream, h->sm_avail, rows, nullptr, h->r_u, Kl, *Tc, h->tcw.fwd[L - 1],
                     EpiScaleSplit{h->ostd, TcEpiSplit{&h->jjr}}, rows); }
      h->launches++;
      // decoder GEMM: HBM-write bound (4 d_u bytes per tangent row)
      ProfScope ps(h, PC_DECODE, 0.0, 4.0 * rows * h->d_u);
      if (rc == 0)
        rc = tc_gemm(h->tcw, h->stream, h->sm_avail, rows, nullptr, (int)h->d_u16, h->r_u, h->jjr, h->usplit,
                     EpiJacScatter{nullptr, J, d_z, h->d_u, h->d_u}, rows);
    }
    h->launches++;
    if (rc) return fail(SDN_ERR_CUDA, "jacobian GEMM launch failed (" + std::to_string(rc) + ")");
    CHECK_LAUNCH(h);
    return SDN_OK;
  }
  // SIMT chains (small widths / softmax / SDN_GEMM_SIMT)
  float* Tc = h->jT[0];
  float* Tn = h->jT[1];
  k_tangent_seed<<<(unsigned)rows, 128, 0, h->stream>>>(rows, d_z, h->h1, L == 1 ? nullptr : D0, h->Pz32t, Tc);
  h->launches++;
  if (L > 1 && h->act == ACT_SOFTMAX) {          // T = a (U - a.U), U = (W1_z V_z^T)_k
    k_softmax_tangent<<<(unsigned)cdiv(rows, 8), 256, 0, h->stream>>>(rows, d_z, h->h1, h->D[0] + dro * h->w[1],
                                                                      Tc, nullptr);
    h->launches++;
  }
  for (int l = 1; l < L - 1; ++l) {
    const bool smax = h->act == ACT_SOFTMAX;
    EpiTangent e{smax ? nullptr : h->D[l] + dro * h->w[l + 1], (int64_t)h->w[l + 1], d_z,
                 (h->res[l] && !smax) ? Tc : nullptr, Tn, (int64_t)h->w[l + 1]};
    TRY((gemm<false, true>(h, rows, nullptr, h->w[l + 1], h->w[l], Tc, h->w[l], h->W[l], h->w[l], e, nullptr,
                           nullptr, 0)));
    if (smax) {
      k_softmax_tangent<<<(unsigned)cdiv(rows, 8), 256, 0, h->stream>>>(rows, d_z, h->w[l + 1],
                                                                        h->D[l] + dro * h->w[l + 1], Tn,
                                                                        h->res[l] ? Tc : nullptr);
      h->launches++;
    }
    std::swap(Tc, Tn);
  }
  if (L >= 2) {
    if (!decoded) {
      EpiJacScatter e{h->ostd, J, d_z, (int64_t)h->r_u};
      TRY((gemm<false, true>(h, rows, nullptr, h->r_u, h->w[L - 1], Tc, h->w[L - 1], h->W[L - 1], h->w[L - 1], e,
                             nullptr, nullptr, 0)));
      return SDN_OK;
    }
    EpiAffine e{nullptr, h->ostd, nullptr, h->jJt, (int64_t)h->r_u};
    TRY((gemm<false, true>(h, rows, nullptr, h->r_u, h->w[L - 1], Tc, h->w[L - 1], h->W[L - 1], h->w[L - 1], e,
                           nullptr, nullptr, 0)));
  } else {                                       // linear model: dy/dz rows are the seed (w[1] = r_u)
    k_scale_cols<<<(unsigned)cdiv(rows * h->r_u, 256), 256, 0, h->stream>>>(rows, h->r_u, h->ostd, Tc,
                                                                            decoded ? h->jJt : nullptr, J, d_z);
    h->launches++;
    if (!decoded) return SDN_OK;
  }
  EpiJacScatter e{nullptr, J, d_z, h->d_u};
  TRY((gemm<false, true>(h, rows, nullptr, (int)h->d_u, h->r_u, h->jJt, h->r_u, h->U, h->r_u, e, nullptr, nullptr,
                         0)));
  return SDN_OK;
}

int sdn_jacobian_batch(sdn_handle* h, const float* m_r, const float* z, int64_t n, int32_t decoded, float* J) {
  if (!h || !m_r || !z || !J) return fail(SDN_ERR_ARG, "null argument");
  if (!h->have_model) return fail(SDN_ERR_STATE, "set_model first");
  if (decoded && !h->have_dec) return fail(SDN_ERR_STATE, "set_decoder first");
  if (n < 0) return fail(SDN_ERR_ARG, "negative row count");
  CU(cudaSetDevice(h->device));
  const int d_z = h->d_z;
  const int64_t outw = decoded ? h->d_u : h->r_u;
  const int64_t chunk = jac_chunk_samples(h, decoded != 0);
  if (chunk > h->jin_cap) {
    int rc;
    if ((rc = dalloc(h, &h->jmr, (size_t)chunk * h->r_m)) || (rc = dalloc(h, &h->jz, (size_t)chunk * d_z)) ||
        (rc = dalloc(h, &h->jX, (size_t)chunk * h->ldx)) ||
        (rc = dalloc(h, &h->jJ, (size_t)chunk * std::max<int64_t>(h->d_u, h->r_u) * d_z)))
      return rc;
    h->jin_cap = chunk;
  }
  for (int64_t s = 0; s < n; s += chunk) {
    const int64_t m = std::min(chunk, n - s);
    CU(cudaMemcpyAsync(h->jmr, m_r + s * h->r_m, sizeof(float) * m * h->r_m, cudaMemcpyHostToDevice, h->stream));
    CU(cudaMemcpyAsync(h->jz, z + s * d_z, sizeof(float) * m * d_z, cudaMemcpyHostToDevice, h->stream));
    TRY(forward_rows(h, h->jmr, h->jz, m, h->jX, true, h->Y));
    TRY(jac_rows(h, 0, m, decoded != 0, h->jJ));
    CU(cudaMemcpyAsync(J + s * outw * d_z, h->jJ, sizeof(float) * m * outw * d_z, cudaMemcpyDeviceToHost, h->stream));
  }
  CU(cudaStreamSynchronize(h->stream));
  return SDN_OK;
}

// the resident samples (sdn_set_samples) at one control z: J_dev (device,
// n x outw x d_z) -- the benchmarked c5 path: no host transfer but z
int sdn_jacobian_samples(sdn_handle* h, const double* z, int32_t decoded, float* J_dev) {
  if (!h || !z || !J_dev) return fail(SDN_ERR_ARG, "null argument");
  if (!h->have_model) return fail(SDN_ERR_STATE, "set_model first");
  if (decoded && !h->have_dec) return fail(SDN_ERR_STATE, "set_decoder first");
  if (h->n < 1) return fail(SDN_ERR_ARG, "empty sample set");
  CU(cudaSetDevice(h->device));
  const int64_t outw = decoded ? h->d_u : h->r_u;
  sdn_risk r{};
  r.kind = SDN_RISK_MEAN;
  TRY(upload_z(h, z, &r, 1));
  k_zbias<<<(unsigned)cdiv(h->h1, 8), 256, 0, h->stream>>>(h->h1, h->d_z, h->Pz, h->zdev, h->b[0], h->zb, h->zb64);
  h->launches++;
  CHECK_LAUNCH(h);
  TRY(run_forward(h, h->n, h->MR, h->r_m, h->r_m, h->W[0], h->r_m, h->zb, true, h->Y,
                  h->tcw.enabled ? &h->tcw.mr : nullptr));
  const int64_t chunk = jac_chunk_samples(h, decoded != 0);
  for (int64_t s = 0; s < h->n; s += chunk) {
    const int64_t m = std::min(chunk, h->n - s);
    TRY(jac_rows(h, s, m, decoded != 0, J_dev + s * outw * h->d_z));
  }
  return SDN_OK;
}

// decoder: Gram K = U^T M U (split-K fp64), c = U^T M (b - u_t), q0 (host fp64)
static int set_decoder_impl(sdn_handle* h, int64_t d_u, const float* U, const float* ubias, const float* Mdiag,
                            const int64_t* indptr, const int32_t* indices, const float* data, const float* u_target);

int sdn_set_decoder(sdn_handle* h, int64_t d_u, const float* U, const float* ubias, const float* Mdiag,
                    const float* u_target) {
  if (!h || !U || !ubias || !Mdiag || !u_target || d_u < 1) return fail(SDN_ERR_ARG, "bad argument");
  return set_decoder_impl(h, d_u, U, ubias, Mdiag, nullptr, nullptr, nullptr, u_target);
}

// general sparse (CSR) state mass, e.g. the consistent P1 mass: the reduced
// tracking form only needs M U, M (b - u_t): one SpMM and one SpMV at set-up
int sdn_set_decoder_csr(sdn_handle* h, int64_t d_u, const float* U, const float* ubias, const int64_t* indptr,
                        const int32_t* indices, const float* data, const float* u_target) {
  if (!h || !U || !ubias || !indptr || !indices || !data || !u_target || d_u < 1)
    return fail(SDN_ERR_ARG, "bad argument");
  if (indptr[0] != 0) return fail(SDN_ERR_ARG, "CSR indptr must start at 0");
  for (int64_t d = 0; d < d_u; ++d)
    if (indptr[d + 1] < indptr[d]) return fail(SDN_ERR_ARG, "CSR indptr must be non-decreasing");
  const int64_t nnz = indptr[d_u];
  for (int64_t e = 0; e < nnz; ++e)
    if (indices[e] < 0 || indices[e] >= d_u) return fail(SDN_ERR_ARG, "CSR column index out of range");
  return set_decoder_impl(h, d_u, U, ubias, nullptr, indptr, indices, data, u_target);
}

static int set_decoder_impl(sdn_handle* h, int64_t d_u, const float* U, const float* ubias, const float* Mdiag,
                            const int64_t* indptr, const int32_t* indices, const float* data, const float* u_target) {
  CU(cudaSetDevice(h->device));
  const int r_u = h->r_u;
  // everything on the device: Um = diag(M) U, c and q0 (fixed-order fp64
  // block sums), the Gram K = Um^T U (split-K fp64 GEMM); one read-back of q0
  if (h->U) { cudaFree(h->U); h->U = nullptr; }
  if (h->ub) { cudaFree(h->ub); h->ub = nullptr; }
  if (!h->Kg) CU(cudaMalloc(&h->Kg, sizeof(float) * r_u * r_u));
  if (!h->cdec) CU(cudaMalloc(&h->cdec, sizeof(float) * r_u));
  if (!h->KPhi) CU(cudaMalloc(&h->KPhi, sizeof(float) * h->cap * r_u));
  if (!h->c64dec) CU(cudaMalloc(&h->c64dec, sizeof(double) * r_u));
  const int64_t d16 = (d_u + 15) / 16 * 16;
  CU(cudaMalloc(&h->U, sizeof(float) * d_u * r_u));
  CU(cudaMalloc(&h->ub, sizeof(float) * d16));      // zero-padded to the tensor-core operand's rows
  CU(cudaMemsetAsync(h->ub, 0, sizeof(float) * d16, h->stream));
  float *Um = nullptr, *Md = nullptr, *ut = nullptr, *cdat = nullptr;
  double *K64 = nullptr, *q0d = nullptr, *msv = nullptr;
  int64_t* cptr = nullptr;
  int32_t* cidx = nullptr;
  const int64_t nnz = indptr ? indptr[d_u] : 0;
  auto cleanup = [&]() {
    cudaFree(Um); cudaFree(Md); cudaFree(ut); cudaFree(q0d); cudaFree(msv); cudaFree(cptr); cudaFree(cidx);
    cudaFree(cdat);
  };
  if (cudaMalloc(&Um, sizeof(float) * d_u * r_u) || cudaMalloc(&ut, sizeof(float) * d_u) ||
      cudaMalloc(&q0d, sizeof(double)) || cudaMalloc(&msv, sizeof(double) * d_u) ||
      cudaMalloc(&K64, sizeof(double) * r_u * r_u) ||
      (Mdiag ? cudaMalloc(&Md, sizeof(float) * d_u)
             : (cudaMalloc(&cptr, sizeof(int64_t) * (d_u + 1)) ||
                cudaMalloc(&cidx, sizeof(int32_t) * std::max<int64_t>(nnz, 1)) ||
                cudaMalloc(&cdat, sizeof(float) * std::max<int64_t>(nnz, 1))))) {
    cleanup();
    return fail(SDN_ERR_NOMEM, "decoder scratch allocation failed");
  }
  int rc = SDN_OK;
  if (cudaMemcpyAsync(h->U, U, sizeof(float) * d_u * r_u, cudaMemcpyHostToDevice, h->stream) ||
      cudaMemcpyAsync(h->ub, ubias, sizeof(float) * d_u, cudaMemcpyHostToDevice, h->stream) ||
      cudaMemcpyAsync(ut, u_target, sizeof(float) * d_u, cudaMemcpyHostToDevice, h->stream) ||
      cudaMemsetAsync(K64, 0, sizeof(double) * r_u * r_u, h->stream) ||
      (Mdiag ? cudaMemcpyAsync(Md, Mdiag, sizeof(float) * d_u, cudaMemcpyHostToDevice, h->stream)
             : (cudaMemcpyAsync(cptr, indptr, sizeof(int64_t) * (d_u + 1), cudaMemcpyHostToDevice, h->stream) ||
                cudaMemcpyAsync(cidx, indices, sizeof(int32_t) * nnz, cudaMemcpyHostToDevice, h->stream) ||
                cudaMemcpyAsync(cdat, data, sizeof(float) * nnz, cudaMemcpyHostToDevice, h->stream))))
    rc = fail(SDN_ERR_CUDA, "decoder upload failed");
  if (rc == SDN_OK) {
    const unsigned rg = (unsigned)std::min<int64_t>(cdiv(d_u, 8), 4096);
    if (Mdiag)
      k_dec_scale<<<(unsigned)std::min<int64_t>(cdiv(d_u * r_u, 256), 4096), 256, 0, h->stream>>>(d_u, r_u, h->U, Md, Um);
    else
      k_dec_spmm<<<rg, 256, 0, h->stream>>>(d_u, r_u, h->U, cptr, cidx, cdat, Um);
    k_dec_ms<<<rg, 256, 0, h->stream>>>(d_u, h->ub, ut, Md, cptr, cidx, cdat, msv);
    h->launches++;
    k_dec_c<<<(unsigned)(r_u + 1), 256, 0, h->stream>>>(d_u, r_u, h->U, h->ub, msv, ut, h->c64dec, q0d);
    k_f64_to_f32<<<1, 256, 0, h->stream>>>(r_u, h->c64dec, h->cdec);
    h->launches += 3;
    const int64_t kc = 2048;
    for (int64_t k0 = 0; k0 < d_u && rc == SDN_OK; k0 += kc) {
      const int kl = (int)std::min(kc, d_u - k0);
      // K += (Um[k0:k0+kl])^T U[k0:k0+kl]  (A stored K x M: AT)
      rc = gemm<true, false>(h, r_u, nullptr, r_u, kl, Um + k0 * r_u, r_u, h->U + k0 * r_u, r_u,
                             EpiAccum64{K64, (int64_t)r_u});
    }
  }
  double q0 = 0.0;
  if (rc == SDN_OK) {
    k_f64_to_f32<<<(unsigned)cdiv(r_u * r_u, 256), 256, 0, h->stream>>>((int64_t)r_u * r_u, K64, h->Kg);
    h->launches++;
    if (cudaMemcpyAsync(&q0, q0d, sizeof(double), cudaMemcpyDeviceToHost, h->stream) ||
        cudaStreamSynchronize(h->stream))
      rc = fail(SDN_ERR_CUDA, "decoder set-up failed");
  }
  // the decoder basis as a tensor-core operand (rows padded to 16) for the
  // decoded Jacobian GEMM
  if (rc == SDN_OK && h->tcw.enabled) {
    if (!h->usplit.hi || h->usplit.rows < d16) {
      if (tc_buf(h, h->tcw, h->usplit, d16, r_u)) rc = fail(SDN_ERR_NOMEM, "decoder operand allocation failed");
    }
    if (rc == SDN_OK) {
      cudaMemsetAsync(h->usplit.hi, 0, sizeof(__nv_bfloat16) * 2 * h->usplit.rows * r_u, h->stream);
      k_split<<<(unsigned)std::min<int64_t>(cdiv(d_u * r_u, 256), 4096), 256, 0, h->stream>>>(
          d_u, nullptr, r_u, r_u, h->U, r_u, h->usplit.hi, h->usplit.lo);
      h->launches++;
      h->d_u16 = d16;
    }
  }
  cleanup();
  if (h->K64) cudaFree(h->K64);
  h->K64 = K64;                 // kept (fp64) for the refinement chain's decoded QoI
  if (rc) return rc;
  CU(cudaGetLastError());
  h->d_u = d_u;
  h->q0dec = q0;
  h->have_dec = true;
  h->have_mean = false;
  h->gen++;
  return SDN_OK;
}

// u = U phi + b  (pod.py:36-40)
int sdn_lift(sdn_handle* h, const float* phi, int64_t n, float* u) {
  if (!h || !phi || !u) return fail(SDN_ERR_ARG, "null argument");
  if (!h->have_dec) return fail(SDN_ERR_STATE, "set_decoder first");
  if (n < 0) return fail(SDN_ERR_ARG, "negative row count");
  CU(cudaSetDevice(h->device));
  const int64_t chunk = std::max<int64_t>(1, std::min<int64_t>(std::max<int64_t>(n, 1), (int64_t)(512ll << 20) / (4 * h->d_u)));
  float *p = nullptr, *o = nullptr;
  const int64_t ldo = std::max<int64_t>(h->d_u16, h->d_u);   // padded rows on the tensor-core path
  TRY(scratch(h, SCR_D, (size_t)chunk * h->r_u, &p));
  TRY(scratch(h, SCR_E, (size_t)chunk * ldo, &o));
  // tensor cores when the decoder operand exists and the chunk fills the GPU
  const bool tc = h->tcw.enabled && h->usplit.hi && h->gemm != SDN_GEMM_SIMT && chunk >= 128ll * h->num_sms / 4;
  if (tc && (!h->lift_in.hi || h->lift_in.rows < chunk)) {
    if (tc_buf(h, h->tcw, h->lift_in, chunk, h->r_u)) return fail(SDN_ERR_NOMEM, "lift operand allocation failed");
  }
  for (int64_t s = 0; s < n; s += chunk) {
    const int64_t m = std::min(chunk, n - s);
    CU(cudaMemcpyAsync(p, phi + s * h->r_u, sizeof(float) * m * h->r_u, cudaMemcpyHostToDevice, h->stream));
    if (tc) {
      // u = U phi + b (pod.py:36-40): phi split, then one tcgen05 GEMM against the split U
      k_split<<<(unsigned)std::min<int64_t>(cdiv(m * h->r_u, 256), 4096), 256, 0, h->stream>>>(
          m, nullptr, h->r_u, h->r_u, p, h->r_u, h->lift_in.hi, h->lift_in.lo);
      h->launches++;
      ProfScope ps(h, PC_DECODE, 2.0 * m * h->d_u * h->r_u, 4.0 * m * h->d_u);
      // (TMA-store epilogue into rows padded to d_u16; the padding is dropped by the 2-D copy out)
      const int rc = tc_gemm(h->tcw, h->stream, h->sm_avail, m, nullptr, (int)h->d_u16, h->r_u, h->lift_in,
                             h->usplit, EpiAffine{h->ub, nullptr, nullptr, o, ldo}, m);
      h->launches++;
      if (rc) return fail(SDN_ERR_CUDA, "lift GEMM launch failed (" + std::to_string(rc) + ")");
      CHECK_LAUNCH(h);
    } else {
      TRY((gemm<false, true>(h, m, nullptr, (int)h->d_u, h->r_u, p, h->r_u, h->U, h->r_u,
                             EpiAffine{h->ub, nullptr, nullptr, o, ldo})));
    }
    CU(cudaMemcpy2DAsync(u + s * h->d_u, sizeof(float) * h->d_u, o, sizeof(float) * ldo, sizeof(float) * h->d_u, m,
                         cudaMemcpyDeviceToHost, h->stream));
  }
  CU(cudaStreamSynchronize(h->stream));
  return SDN_OK;
}

// encoder K1: m_r = (m - mean) diag(M) V_m, split-K in fp64 (randfield.py:67-72)
int sdn_encode_fields(sdn_handle* h, const float* m, int64_t n, int64_t d_m, const float* Vm, const float* Mdiag,
                      float m_mean, int64_t global_offset, int32_t on_device) {
  if (!h || !m || !Vm || !Mdiag || n < 0 || d_m < 1) return fail(SDN_ERR_ARG, "bad argument");
  if (n > h->cap) return fail(SDN_ERR_ARG, "sample count exceeds the handle capacity");
  CU(cudaSetDevice(h->device));
  const int r_m = h->r_m;
  // everything on the device: Vmm = diag(M) V_m (fp32 of the fp64 product),
  // bias_j = -m_mean sum_d Vmm[d, j] (fixed-order fp64), the split-K product
  // accumulated in fp64, then MR = float(acc + bias).  (The products stay on
  // the FMA pipe in fp32: the input whitening 1/sqrt(lambda_j) amplifies the
  // encoder's error by up to ~6500x at c4's highest mode, which a bf16x3
  // product error of ~2^-16 cannot absorb -- DESIGN.md section 3.)
  const int64_t rows_chunk = std::max<int64_t>(1, std::min<int64_t>(std::max<int64_t>(n, 1), (int64_t)(1ll << 30) / (4 * d_m)));
  float *V = nullptr, *Vraw = nullptr, *Md = nullptr, *mb = nullptr;
  double *acc = nullptr, *bd = nullptr;
  TRY(scratch(h, SCR_A, (size_t)d_m * r_m, &V));
  TRY(scratch(h, SCR_B, (size_t)d_m * r_m, &Vraw));
  TRY(scratch(h, SCR_C, (size_t)d_m, &Md));
  TRY(scratch(h, SCR_D, (size_t)std::max<int64_t>(n, 1) * r_m, &acc));
  TRY(scratch(h, SCR_E, (size_t)r_m, &bd));
  if (!on_device) TRY(scratch(h, SCR_F, (size_t)std::max<int64_t>(rows_chunk, std::min<int64_t>(n, 16384)) * d_m, &mb));
  CU(cudaMemcpyAsync(Vraw, Vm, sizeof(float) * d_m * r_m, cudaMemcpyHostToDevice, h->stream));
  CU(cudaMemcpyAsync(Md, Mdiag, sizeof(float) * d_m, cudaMemcpyHostToDevice, h->stream));
  k_dec_scale<<<(unsigned)std::min<int64_t>(cdiv(d_m * r_m, 256), 4096), 256, 0, h->stream>>>(d_m, r_m, Vraw, Md, V);
  k_enc_bias<<<(unsigned)r_m, 256, 0, h->stream>>>(d_m, r_m, V, (double)m_mean, bd);
  h->launches += 2;
  CU(cudaMemsetAsync(acc, 0, sizeof(double) * std::max<int64_t>(n, 1) * r_m, h->stream));
  const int64_t kc = 1024;
  // Tensor cores (default when the handle has them and the shard fills a few
  // tiles; SDN_ENC_TC=0: the FMA-pipe GEMM).  Both operands are split into
  // three bf16 planes (24 mantissa bits); per 1024-column K chunk two launches
  // (k_split3's layout): pass A, a bf16x3 GEMM over the chunk's segments
  // (a0;a1)x(b0;b1) and (a1;a2)x(b1;b2); pass B, hi-only products a2 b0 + a0 b2.
  // Together every term a_i b_j with i + j <= 2 -- the fp32 product to ~2^-24,
  // which the input whitening downstream needs -- with
  // fp32 accumulation in TMEM within a launch and fp64 accumulation across
  // launches, as on the FMA path.
  static const bool enc_tc_off = getenv("SDN_ENC_TC") && getenv("SDN_ENC_TC")[0] == '0';
  const bool enc_tc = !enc_tc_off && h->tcw.enabled && h->gemm != SDN_GEMM_SIMT && r_m % 16 == 0 && n >= 512 &&
                      tc_encode_fn() != nullptr;
  const int nch = (int)cdiv(d_m, kc);               // K chunks (planes zero-padded to whole chunks)
  const int64_t lda = 4 * kc, ldb2 = 2 * kc;          // row pitch inside a chunk (chunk-major planes)
  __nv_bfloat16 *PA = nullptr, *PB = nullptr, *PB2 = nullptr;
  int64_t tc_rows = 0;
  if (enc_tc) {
    tc_rows = cdiv(std::min<int64_t>(n, 16384), 128) * 128;      // up to 16384 rows per pass: 128 256-column tiles per launch
    TRY(scratch(h, SCR_G, (size_t)nch * tc_rows * lda + 2 * kc, &PA));
    TRY(scratch(h, SCR_H, (size_t)nch * r_m * (lda + ldb2) + 2 * kc, &PB));
    PB2 = PB + (int64_t)nch * r_m * lda;
    k_split3_transpose<<<dim3((unsigned)cdiv((int64_t)nch * kc, 32), (unsigned)cdiv(r_m, 32)), dim3(32, 8), 0, h->stream>>>(
        d_m, r_m, V, nch, (int)kc, PB, PB2);
    h->launches++;
    CHECK_LAUNCH(h);
  }
  for (int64_t s = 0; s < n; s += (enc_tc ? tc_rows : rows_chunk)) {
    const int64_t rows = std::min(enc_tc ? tc_rows : rows_chunk, n - s);
    const float* src = m + s * d_m;
    if (!on_device) {
      CU(cudaMemcpyAsync(mb, src, sizeof(float) * rows * d_m, cudaMemcpyHostToDevice, h->stream));
      src = mb;
    }
    ProfScope ps(h, PC_OTHER, 2.0 * rows * r_m * d_m, 4.0 * rows * d_m);
    if (enc_tc) {
      k_split3<<<(unsigned)std::min<int64_t>(cdiv(rows * nch * kc / 8, 256), 65536), 256, 0, h->stream>>>(
          rows, (int)d_m, d_m, src, nch, (int)kc, tc_rows, PA);
      h->launches++;
      CHECK_LAUNCH(h);
      for (int c = 0; c < nch; ++c) {
        TcOperand ta, tb;
        TcFlags fl;
        // pass A: hi = (a0, a1), lo = (a1, a2) -- the same rows one segment on
        ta.hi = PA + (int64_t)c * tc_rows * lda; ta.lo = ta.hi + kc; ta.ld = (int)lda; ta.rows = rows;
        tb.hi = PB + (int64_t)c * r_m * lda; tb.lo = tb.hi + kc; tb.ld = (int)lda; tb.rows = r_m;
        TRY((gemm<false, true>(h, rows, nullptr, r_m, (int)(2 * kc), src, d_m, V, r_m,
                               EpiAccum64{acc + s * r_m, (int64_t)r_m}, &tb, &ta, 1, fl)));
        // pass B: hi-only a2 b0 + a0 b2 (the lo halves are loaded and ignored)
        // (lo = the hi rows shifted by 16 bytes: the same cache lines, never multiplied; the buffers carry slack)
        ta.hi = PA + (int64_t)c * tc_rows * lda + 2 * kc; ta.lo = ta.hi + 8;
        tb.hi = PB2 + (int64_t)c * r_m * ldb2; tb.lo = tb.hi + 8; tb.ld = (int)ldb2;
        fl.hi_only = 1;
        TRY((gemm<false, true>(h, rows, nullptr, r_m, (int)(2 * kc), src, d_m, V, r_m,
                               EpiAccum64{acc + s * r_m, (int64_t)r_m}, &tb, &ta, 1, fl)));
      }
      continue;
    }
    for (int64_t k0 = 0; k0 < d_m; k0 += kc) {
      const int kl = (int)std::min(kc, d_m - k0);
      TRY((gemm<false, false>(h, rows, nullptr, r_m, kl, src + k0, d_m, V + k0 * r_m, r_m,
                              EpiAccum64{acc + s * r_m, (int64_t)r_m})));
    }
  }
  if (n > 0) {
    k_enc_finish<<<(unsigned)std::min<int64_t>(cdiv(n * r_m, 256), 4096), 256, 0, h->stream>>>(n, r_m, acc, bd, h->MR);
    h->launches++;
  }
  CU(cudaStreamSynchronize(h->stream));
  CU(cudaGetLastError());
  h->n = n;
  h->goff = global_offset;
  h->fwd_done = false;
  h->gen++;
  if (h->tcw.enabled) TRY(tc_set_samples(h, h->tcw, h->MR, n));
  return SDN_OK;
}

// order statistics: indices of the k largest values (value desc, index asc),
// returned in ascending index order
int sdn_select_topk(sdn_handle* h, const double* values, int64_t n, int64_t k, int32_t on_device, int64_t* idx) {
  if (!h || !values || !idx || n < 1 || k < 1 || k > n) return fail(SDN_ERR_ARG, "bad argument");
  CU(cudaSetDevice(h->device));
  double* v = nullptr;
  uint8_t* mask = nullptr;
  int *cnt = nullptr, *offs = nullptr, *na = nullptr, *ri = nullptr;
  const int nb = (int)cdiv(n, 1024);
  TRY(scratch(h, SCR_A, (size_t)n, &v));
  TRY(scratch(h, SCR_B, (size_t)n, &mask));
  TRY(scratch(h, SCR_C, (size_t)2 * nb + 1, &cnt));
  TRY(scratch(h, SCR_D, (size_t)k, &ri));
  offs = cnt + nb;
  na = cnt + 2 * nb;
  CU(cudaMemcpyAsync(v, values, sizeof(double) * n, on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                     h->stream));
  TRY(launch_topk(h, n, k, v, nullptr, mask));
  k_flag_count<<<nb, 1024, 0, h->stream>>>(n, RISK_CVAR_EXACT, v, mask, 0.0, 1.0, nullptr, cnt);
  k_scan_counts<<<1, 32, 0, h->stream>>>(nb, cnt, offs, na);
  k_compact<<<nb, 1024, 0, h->stream>>>(n, RISK_CVAR_EXACT, v, mask, 0.0, 1.0, nullptr, offs, ri);
  h->launches += 4;
  std::vector<int> hi(k);
  cudaError_t e = cudaMemcpyAsync(hi.data(), ri, sizeof(int) * k, cudaMemcpyDeviceToHost, h->stream);
  cudaError_t e2 = cudaStreamSynchronize(h->stream);
  if (e != cudaSuccess || e2 != cudaSuccess) return fail(SDN_ERR_CUDA, "top-k failed");
  for (int64_t i = 0; i < k; ++i) idx[i] = hi[i];
  return SDN_OK;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// kernel-tuning entry: time one layer-1 forward GEMM (A = activation operand,
// B = W_1) `reps` times.  mode 0: tcgen05 mainloop with a null epilogue;
// 1: tcgen05 with the fused hidden-layer epilogue; 2: SIMT with the same
// epilogue.  ms[0] = average device ms per launch.
extern "C" int sdn_debug_gemm(sdn_handle* h, int64_t M, int32_t mode, int32_t reps, double* ms) {
  if (!h || !ms || h->L < 3 || M < 1 || M > h->cap) return fail(SDN_ERR_ARG, "bad argument");
  if (mode != 2 && !h->tcw.enabled) return fail(SDN_ERR_STATE, "tensor-core path unavailable");
  CU(cudaSetDevice(h->device));
  const int K = h->w[1], N = h->w[2];
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  // modes 3..6 drop parts of the fused epilogue: 3 no D, 4 no split, 5 no
  // residual input, 6 only the fp32 H store
  const bool keepD = mode < 3 || (mode != 3 && mode < 6), keepS = mode < 4 || (mode != 4 && mode < 6);
  const bool keepP = mode < 5, keepH = mode != 7 && mode < 8;
  // mode 8: the production tensor-core chain epilogue (no fp32 H, residual
  // read from the input's bf16 split, D + split outputs)
  // mode 9: the chain epilogue with the identity activation (arithmetic share of ELU);
  // 10 / 11 / 12: the chain epilogue without the act' store / the split store / the residual input
  // 13 / 14: the chain epilogue with the MMAs skipped / MMAs and TMA loads
  // skipped (epilogue pace alone)
  // composite study modes: base | 256 skip MMAs | 512 skip TMA loads | 1024 no act' store |
  // 2048 no split store | 4096 no residual input
  const int flags = mode & ~255;
  mode &= 255;
  // 8192 / 16384: ring epilogue without the proxy fence / without TMEM loads;
  // SDN_EPI_TRACE: ring-epilogue phase stamps of one warp printed after the timing
  // 32768: the mainloop TMA-loads only the hi halves (timing study; results wrong)
  int skip = mode == 13 ? 1 : mode == 14 ? 3 : ((flags >> 8) & 3) | ((flags & 8192) ? 16 : 0) | ((flags & 16384) ? 32 : 0) |
             ((flags & 32768) ? 128 : 0);
  unsigned long long* eptr = nullptr;
  if (getenv("SDN_EPI_TRACE")) {
    cudaMalloc(&eptr, 96 * sizeof(unsigned long long));
    cudaMemset(eptr, 0, 96 * sizeof(unsigned long long));
    cudaMemcpyToSymbol(g_tc_eptr, &eptr, sizeof(eptr));
    skip |= 64;
  }
  cudaMemcpyToSymbol(g_tc_dbg_skip, &skip, sizeof(int));
  const bool chainm = mode == 8 || mode >= 9;
  const bool noD = mode == 10 || (flags & 1024), noS = mode == 11 || (flags & 2048), noP = mode == 12 || (flags & 4096);
  EpiFwdHidden e{h->b[1], (h->res[1] && keepP && !chainm) ? h->H[0] : nullptr, keepH ? h->H[1] : nullptr,
                 ((keepD || chainm) && !noD) ? h->D[1] : nullptr, (int64_t)N,
                 mode == 9 ? (int)ACT_IDENTITY : h->act};
  TcChain<EpiFwdHidden> ch{e, TcEpiSplit{((keepS || chainm) && !noS) ? &h->tcw.act[1] : nullptr},
                           TcEpiSplit{(chainm && h->res[1] && !noP) ? &h->tcw.act[0] : nullptr}};
  h->tcw.act[0].rows = M;
  int rc = 0;
  // 20 / 21: the dense reverse-sweep chain step (layer 2) / the summing last
  // step (layer 1) on the sweep buffers of a previous evaluation (flags as above:
  // 1024 no G store, 2048 no split store, 4096 no residual-gradient input)
  if ((mode == 20 || mode == 21) && (!h->sw || h->sw->rows < M || h->sw->planes < 1 || h->L < 4))
    return fail(SDN_ERR_STATE, "debug reverse GEMM: run a multi-risk evaluation first (L >= 4)");
  for (int it = 0; it <= reps && rc == 0; ++it) {
    if (it == 1) cudaEventRecord(a, h->stream);
    if (mode == 20) {
      SweepBufs& sw = *h->sw;
      EpiBwd e{noP ? nullptr : sw.G, noD ? nullptr : sw.G, h->D[1], (int64_t)h->w[2], nullptr, nullptr, (int64_t)h->w[2]};
      TcChain<EpiBwd> cb{e, TcEpiSplit{noS ? nullptr : &sw.act[1]}};
      rc = tc_gemm(h->tcw, h->stream, h->num_sms, M, nullptr, h->w[2], h->w[3], sw.act[0], h->tcw.bwd[2], cb);
      continue;
    }
    if (mode == 21) {
      SweepBufs& sw = *h->sw;
      EpiBwdSum e{noP ? nullptr : sw.G, h->D[0], (int64_t)h->w[1], nullptr, (int64_t)h->w[1], sw.tsum, (int64_t)h->w[1]};
      e.W = sw.W; e.R = sw.planes; e.plane = cdiv(sw.rows, 128) * 4 * h->maxw;
      rc = tc_gemm(h->tcw, h->stream, h->num_sms, M, nullptr, h->w[1], h->w[2], sw.act[0], h->tcw.bwd[1], e);
      continue;
    }
    if (mode == 0) rc = tc_gemm(h->tcw, h->stream, h->num_sms, M, nullptr, N, K, h->tcw.act[0], h->tcw.fwd[1], EpiNull{});
    else if (mode != 2) rc = tc_gemm(h->tcw, h->stream, h->num_sms, M, nullptr, N, K, h->tcw.act[0], h->tcw.fwd[1], ch);
    else { launch_simt<128, 128, 8, 8, false, true>(h, M, nullptr, N, K, h->H[0], K, h->W[1], K, ch, true); }
  }
  cudaEventRecord(b, h->stream);
  cudaError_t err = cudaEventSynchronize(b);
  if (getenv("SDN_TRACE") && mode != 2 && rc == 0) {
    // one more launch with per-phase clock64 stamps of CTA 0 (stderr)
    unsigned long long* tr = nullptr;
    cudaMalloc(&tr, 128 * sizeof(unsigned long long));
    cudaMemset(tr, 0, 128 * sizeof(unsigned long long));
    g_tc_trace = tr;
    if (mode == 0) rc = tc_gemm(h->tcw, h->stream, h->num_sms, M, nullptr, N, K, h->tcw.act[0], h->tcw.fwd[1], EpiNull{});
    else rc = tc_gemm(h->tcw, h->stream, h->num_sms, M, nullptr, N, K, h->tcw.act[0], h->tcw.fwd[1], ch);
    g_tc_trace = nullptr;
    cudaStreamSynchronize(h->stream);
    unsigned long long ht[128];
    cudaMemcpy(ht, tr, sizeof(ht), cudaMemcpyDeviceToHost);
    cudaFree(tr);
    fprintf(stderr, "trace mode %d M %lld: tma[kb0..3] %lld %lld %lld %lld | mma_done %lld | epi_start %lld |", mode,
            (long long)M, (long long)(ht[1] - ht[0]), (long long)(ht[2] - ht[0]), (long long)(ht[3] - ht[0]),
            (long long)(ht[4] - ht[0]), (long long)(ht[5] - ht[0]), (long long)(ht[8] - ht[0]));
    for (int i = 0; i < 8; ++i)
      if (ht[9 + 2 * i]) fprintf(stderr, " c%d[%lld,%lld]", i, (long long)(ht[9 + 2 * i] - ht[0]), (long long)(ht[10 + 2 * i] - ht[0]));
    fprintf(stderr, "\n");
  }
  skip = 0;
  cudaMemcpyToSymbol(g_tc_dbg_skip, &skip, sizeof(int));
  if (eptr) {
    unsigned long long et[96];
    cudaMemcpy(et, eptr, sizeof(et), cudaMemcpyDeviceToHost);
    cudaFree(eptr);
    fprintf(stderr, "ring epilogue phases (cycles from chunk start: rbar, tmem, math, reclaim, issue, staged+fenced, stored)\n");
    for (int c = 0; c < 12; ++c) {
      if (!et[c * 8]) continue;
      fprintf(stderr, "  tile %d chunk %d @%lld:", c / 6, c % 6, (long long)(et[c * 8] - et[0]));
      for (int k = 1; k < 8; ++k) fprintf(stderr, " %lld", (long long)(et[c * 8 + k] - et[c * 8]));
      fprintf(stderr, "\n");
    }
  }
  float t = 0.f;
  cudaEventElapsedTime(&t, a, b);
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  if (rc || err != cudaSuccess) return fail(SDN_ERR_CUDA, std::string("debug gemm: ") + cudaGetErrorString(cudaGetLastError()));
  ms[0] = t / std::max(reps, 1);
  return SDN_OK;
}


// ---------------------------------------------------------------------------
// H1 training (reference surrogate.py:263-405), SIMT
// chains with fp64 gradients and fp64 master parameters (train.cuh)

// G64 (n_out x n_in) += X^T Y, X: K x n_out, Y: K x n_in (row-major), K large:
// transpose X to n_out x K, split K over gridDim.z so the small output fills
// the GPU, reduce the fp32 partials in a fixed order into fp64
static int tr_wgrad(sdn_handle* h, int n_out, int n_in, int64_t K, const float* X, const float* Y, double* G64) {
  auto& t = h->tr;
  float* Xt = K <= t.bcap ? t.GSt : t.GUt;
  k_tr_transpose<<<dim3((unsigned)cdiv(n_out, 32), (unsigned)cdiv(K, 32)), dim3(32, 8), 0, h->stream>>>(K, n_out, X, Xt);
  const int64_t tiles = cdiv(n_out, 64) * cdiv(n_in, 64);
  int Z = (int)std::min<int64_t>({(int64_t)t.zmax, std::max<int64_t>(1, cdiv(2 * h->num_sms, tiles)),
                                  std::max<int64_t>(1, K / 128)});
  const bool vec = (K % 4 == 0) && (n_in % 4 == 0);
  dim3 grid((unsigned)cdiv(n_out, 64), (unsigned)cdiv(n_in, 64), (unsigned)Z);
  EpiStoreZ e{t.zpart, (int64_t)n_in, (int64_t)n_out * n_in};
  if (vec)
    gemm_simt_kernel<64, 64, 16, 4, 4, false, false, true, EpiStoreZ><<<grid, 256, 0, h->stream>>>(
        n_out, nullptr, n_in, (int)K, Xt, K, Y, n_in, e);
  else
    gemm_simt_kernel<64, 64, 16, 4, 4, false, false, false, EpiStoreZ><<<grid, 256, 0, h->stream>>>(
        n_out, nullptr, n_in, (int)K, Xt, K, Y, n_in, e);
  k_tr_sum_z<<<(unsigned)std::min<int64_t>(cdiv((int64_t)n_out * n_in, 256), 4 * h->num_sms), 256, 0, h->stream>>>(
      (int64_t)n_out * n_in, Z, t.zpart, G64);
  h->launches += 3;
  CHECK_LAUNCH(h);
  return SDN_OK;
}

static int tr_alloc(sdn_handle* h, void** p, size_t bytes) {
  CU(cudaMalloc(p, std::max<size_t>(bytes, 16)));
  h->tr.allocs.push_back(*p);
  return SDN_OK;
}

extern "C" {

int sdn_train_setup(sdn_handle* h, const float* m_r, const float* z, const float* u_r, const float* j_r, int64_t n,
                    int32_t batch_cap) {
  if (!h || !m_r || !z || !u_r || n < 1 || batch_cap < 1) return fail(SDN_ERR_ARG, "bad argument");
  if (h->act == ACT_SOFTMAX || h->residual) return fail(SDN_ERR_ARG, "device training supports elementwise activations without residual blocks");
  if (h->r_z != h->d_z) return fail(SDN_ERR_ARG, "device training needs V_z = I (the reference network)");
  CU(cudaSetDevice(h->device));
  auto& t = h->tr;
  for (void* p : t.allocs) cudaFree(p);
  t = sdn_handle::Train{};
  const int L = h->L, d_z = h->d_z, r_m = h->r_m, r_u = h->r_u, B = batch_cap;
  const int n0 = h->w[0];
  t.n = n;
  t.bcap = B;
  TRY(tr_alloc(h, (void**)&t.dm, sizeof(float) * n * r_m));
  TRY(tr_alloc(h, (void**)&t.dz, sizeof(float) * n * d_z));
  TRY(tr_alloc(h, (void**)&t.du, sizeof(float) * n * r_u));
  CU(cudaMemcpy(t.dm, m_r, sizeof(float) * n * r_m, cudaMemcpyHostToDevice));
  CU(cudaMemcpy(t.dz, z, sizeof(float) * n * d_z, cudaMemcpyHostToDevice));
  CU(cudaMemcpy(t.du, u_r, sizeof(float) * n * r_u, cudaMemcpyHostToDevice));
  if (j_r) {
    TRY(tr_alloc(h, (void**)&t.dj, sizeof(float) * n * r_u * d_z));
    CU(cudaMemcpy(t.dj, j_r, sizeof(float) * n * r_u * d_z, cudaMemcpyHostToDevice));
  }
  int64_t off = 0;
  for (int l = 0; l < L; ++l) {
    t.woff.push_back(off);
    off += (int64_t)h->w[l + 1] * h->w[l];
    t.boff.push_back(off);
    off += h->w[l + 1];
  }
  t.count = off;
  for (double** q : {&t.P, &t.G, &t.M, &t.V}) TRY(tr_alloc(h, (void**)q, sizeof(double) * off));
  TRY(tr_alloc(h, (void**)&t.P32, sizeof(float) * off));
  TRY(tr_alloc(h, (void**)&t.scale, sizeof(float) * r_m));
  TRY(tr_alloc(h, (void**)&t.mu, sizeof(float) * r_u));
  TRY(tr_alloc(h, (void**)&t.sig, sizeof(float) * r_u));
  TRY(tr_alloc(h, (void**)&t.idx, sizeof(int) * B));
  const int mw = std::max(h->maxw, n0);
  TRY(tr_alloc(h, (void**)&t.Y, sizeof(float) * B * r_u));
  TRY(tr_alloc(h, (void**)&t.Jt, sizeof(float) * B * d_z * r_u));
  for (float** q : {&t.GA, &t.GS, &t.GA2}) TRY(tr_alloc(h, (void**)q, sizeof(float) * B * mw));
  for (float** q : {&t.GT, &t.GU, &t.GT2}) TRY(tr_alloc(h, (void**)q, sizeof(float) * B * d_z * mw));
  TRY(tr_alloc(h, (void**)&t.GSt, sizeof(float) * B * mw));
  TRY(tr_alloc(h, (void**)&t.GUt, sizeof(float) * B * d_z * mw));
  TRY(tr_alloc(h, (void**)&t.zpart, sizeof(float) * t.zmax * mw * mw));
  t.A.assign(L + 1, nullptr);
  t.T.assign(L + 1, nullptr);
  t.S.assign(L, nullptr);
  t.U.assign(L, nullptr);
  for (int l = 0; l <= L; ++l) {
    TRY(tr_alloc(h, (void**)&t.A[l], sizeof(float) * B * h->w[l]));
    TRY(tr_alloc(h, (void**)&t.T[l], sizeof(float) * B * d_z * h->w[l]));
  }
  for (int l = 0; l < L; ++l) {
    TRY(tr_alloc(h, (void**)&t.S[l], sizeof(float) * B * h->w[l + 1]));
    TRY(tr_alloc(h, (void**)&t.U[l], sizeof(float) * B * d_z * h->w[l + 1]));
  }
  TRY(tr_alloc(h, (void**)&t.part, sizeof(double) * 2 * 64));
  if (!t.hloss) CU(cudaHostAlloc((void**)&t.hloss, sizeof(double) * 2, 0));
  t.ready = true;
  return SDN_OK;
}

// parameters in the reference layout (W_l: n_out x n_in incl. the full first
// layer [m | z] columns), fp64; resets the Adam state
int sdn_train_set_params(sdn_handle* h, const double* const* W, const double* const* b, const double* in_scale,
                         const double* out_mean, const double* out_std) {
  if (!h || !W || !b || !in_scale || !out_mean || !out_std) return fail(SDN_ERR_ARG, "null argument");
  auto& t = h->tr;
  if (!t.ready) return fail(SDN_ERR_STATE, "sdn_train_setup first");
  CU(cudaSetDevice(h->device));
  std::vector<double> P(t.count);
  for (int l = 0; l < h->L; ++l) {
    std::memcpy(&P[t.woff[l]], W[l], sizeof(double) * h->w[l + 1] * h->w[l]);
    std::memcpy(&P[t.boff[l]], b[l], sizeof(double) * h->w[l + 1]);
  }
  CU(cudaMemcpy(t.P, P.data(), sizeof(double) * t.count, cudaMemcpyHostToDevice));
  CU(cudaMemset(t.M, 0, sizeof(double) * t.count));
  CU(cudaMemset(t.V, 0, sizeof(double) * t.count));
  k_tr_f64_to_f32<<<256, 256, 0, h->stream>>>(t.count, t.P, t.P32);
  std::vector<float> f(std::max(h->r_m, h->r_u));
  for (int j = 0; j < h->r_m; ++j) f[j] = (float)in_scale[j];
  CU(cudaMemcpy(t.scale, f.data(), sizeof(float) * h->r_m, cudaMemcpyHostToDevice));
  for (int j = 0; j < h->r_u; ++j) f[j] = (float)out_mean[j];
  CU(cudaMemcpy(t.mu, f.data(), sizeof(float) * h->r_u, cudaMemcpyHostToDevice));
  for (int j = 0; j < h->r_u; ++j) f[j] = (float)out_std[j];
  CU(cudaMemcpy(t.sig, f.data(), sizeof(float) * h->r_u, cudaMemcpyHostToDevice));
  CU(cudaStreamSynchronize(h->stream));
  return SDN_OK;
}

// per-parameter update mask (same layout as the parameters; 0 freezes an entry)
int sdn_train_set_mask(sdn_handle* h, const double* const* mW, const double* const* mb) {
  if (!h || !mW || !mb) return fail(SDN_ERR_ARG, "null argument");
  auto& t = h->tr;
  if (!t.ready) return fail(SDN_ERR_STATE, "sdn_train_setup first");
  CU(cudaSetDevice(h->device));
  if (!t.mask) TRY(tr_alloc(h, (void**)&t.mask, sizeof(double) * t.count));
  std::vector<double> m(t.count);
  for (int l = 0; l < h->L; ++l) {
    std::memcpy(&m[t.woff[l]], mW[l], sizeof(double) * h->w[l + 1] * h->w[l]);
    std::memcpy(&m[t.boff[l]], mb[l], sizeof(double) * h->w[l + 1]);
  }
  CU(cudaMemcpy(t.mask, m.data(), sizeof(double) * t.count, cudaMemcpyHostToDevice));
  return SDN_OK;
}

int sdn_train_get_params(sdn_handle* h, double* const* W, double* const* b) {
  if (!h || !W || !b) return fail(SDN_ERR_ARG, "null argument");
  auto& t = h->tr;
  if (!t.ready) return fail(SDN_ERR_STATE, "sdn_train_setup first");
  CU(cudaSetDevice(h->device));
  CU(cudaStreamSynchronize(h->stream));
  std::vector<double> P(t.count);
  CU(cudaMemcpy(P.data(), t.P, sizeof(double) * t.count, cudaMemcpyDeviceToHost));
  for (int l = 0; l < h->L; ++l) {
    std::memcpy(W[l], &P[t.woff[l]], sizeof(double) * h->w[l + 1] * h->w[l]);
    std::memcpy(b[l], &P[t.boff[l]], sizeof(double) * h->w[l + 1]);
  }
  return SDN_OK;
}

// gradient of the last sdn_train_step (fp64, reference layout)
int sdn_train_get_grad(sdn_handle* h, double* const* gW, double* const* gb) {
  if (!h || !gW || !gb) return fail(SDN_ERR_ARG, "null argument");
  auto& t = h->tr;
  if (!t.ready) return fail(SDN_ERR_STATE, "sdn_train_setup first");
  CU(cudaSetDevice(h->device));
  CU(cudaStreamSynchronize(h->stream));
  std::vector<double> G(t.count);
  CU(cudaMemcpy(G.data(), t.G, sizeof(double) * t.count, cudaMemcpyDeviceToHost));
  for (int l = 0; l < h->L; ++l) {
    std::memcpy(gW[l], &G[t.woff[l]], sizeof(double) * h->w[l + 1] * h->w[l]);
    std::memcpy(gb[l], &G[t.boff[l]], sizeof(double) * h->w[l + 1]);
  }
  return SDN_OK;
}

// one loss_and_grad over the batch idx (B records) and, when lr > 0, one Adam
// step (step = 1-based update count for the bias corrections); *loss = the
// batch loss (surrogate.py:263-335, 382-403)
int sdn_train_step(sdn_handle* h, const int64_t* idx, int32_t B, double lam, double lr, int64_t step,
                   double* loss) {
  if (!h || !idx || !loss || B < 1) return fail(SDN_ERR_ARG, "bad argument");
  auto& t = h->tr;
  if (!t.ready) return fail(SDN_ERR_STATE, "sdn_train_setup first");
  if (B > t.bcap) return fail(SDN_ERR_ARG, "batch exceeds the setup capacity");
  if (lam > 0.0 && !t.dj) return fail(SDN_ERR_ARG, "jacobian_weight > 0 requires Jacobian data");
  CU(cudaSetDevice(h->device));
  const int L = h->L, d_z = h->d_z, r_u = h->r_u;
  const bool tan = lam > 0.0;
  const int64_t BT = (int64_t)B * d_z;
  std::vector<int> ih(B);
  for (int b = 0; b < B; ++b) {
    if (idx[b] < 0 || idx[b] >= t.n) return fail(SDN_ERR_ARG, "record index out of range");
    ih[b] = (int)idx[b];
  }
  CU(cudaMemcpyAsync(t.idx, ih.data(), sizeof(int) * B, cudaMemcpyHostToDevice, h->stream));
  k_tr_gather<<<B, 128, 0, h->stream>>>(B, t.idx, t.dm, t.dz, t.du, t.dj, h->r_m, d_z, r_u, t.scale, t.mu, t.sig,
                                        t.A[0], t.Y, tan ? t.Jt : nullptr, tan ? t.T[0] : nullptr);
  h->launches++;
  CHECK_LAUNCH(h);
  // forward with tangents
  for (int l = 0; l < L; ++l) {
    const int n_in = h->w[l], n_out = h->w[l + 1];
    const float* W = t.P32 + t.woff[l];
    const float* bb = t.P32 + t.boff[l];
    const bool last = l == L - 1;
    float* Sout = last ? t.A[L] : t.S[l];
    float* Uout = last ? t.T[L] : t.U[l];
    TRY((gemm<false, true>(h, B, nullptr, n_out, n_in, t.A[l], n_in, W, n_in,
                           EpiAffine{bb, nullptr, nullptr, Sout, (int64_t)n_out}, nullptr, nullptr, 0)));
    if (tan)
      TRY((gemm<false, true>(h, BT, nullptr, n_out, n_in, t.T[l], n_in, W, n_in, EpiStore{Uout, (int64_t)n_out},
                             nullptr, nullptr, 0)));
    if (!last) {
      k_tr_act<<<dim3(B, (unsigned)cdiv(n_out, 128)), 128, 0, h->stream>>>(B, d_z, n_out, h->act, t.S[l],
                                                                         tan ? t.U[l] : nullptr, t.A[l + 1],
                                         tan ? t.T[l + 1] : nullptr);
      h->launches++;
    }
  }
  // loss and output seeds
  const int lg = 32;
  k_tr_loss<<<lg, 256, 0, h->stream>>>(B, d_z, r_u, lam, t.A[L], t.Y, tan ? t.T[L] : nullptr, t.Jt, t.GA, t.GT,
                                       t.part);
  k_sum_rows<<<1, 256, 0, h->stream>>>(lg, 2, t.part, t.part + 2 * lg);
  h->launches += 2;
  CHECK_LAUNCH(h);
  // reverse: GA/GT hold dLoss/d(layer outputs); gradients into G (fp64)
  CU(cudaMemsetAsync(t.G, 0, sizeof(double) * t.count, h->stream));
  float *GA = t.GA, *GT = t.GT, *GAn = t.GA2, *GTn = t.GT2;
  for (int l = L - 1; l >= 0; --l) {
    const int n_in = h->w[l], n_out = h->w[l + 1];
    const float* W = t.P32 + t.woff[l];
    const float *GS, *GU;
    if (l == L - 1) {
      GS = GA;
      GU = GT;
    } else {
      k_tr_bwd<<<dim3(B, (unsigned)cdiv(n_out, 128)), 128, 0, h->stream>>>(B, d_z, n_out, h->act, t.S[l],
                                                                         tan ? t.U[l] : nullptr, GA,
                                         tan ? GT : nullptr, t.GS, t.GU);
      h->launches++;
      GS = t.GS;
      GU = t.GU;
    }
    // gW = GS^T A_l (+ GU^T T_l): K-contiguous transposes, split-K SIMT GEMMs
    // into fp32 partials, fixed-order fp64 reduction; gb = colsum(GS)
    TRY(tr_wgrad(h, n_out, n_in, B, GS, t.A[l], t.G + t.woff[l]));
    if (tan) TRY(tr_wgrad(h, n_out, n_in, BT, GU, t.T[l], t.G + t.woff[l]));
    k_tr_colsum<<<(unsigned)cdiv(n_out, 128), 128, 0, h->stream>>>(B, n_out, GS, t.G + t.boff[l]);
    h->launches++;
    if (l > 0) {                                 // GA = GS W, GT = GU W
      TRY((gemm<false, false>(h, B, nullptr, n_in, n_out, GS, n_out, W, n_in, EpiStore{GAn, (int64_t)n_in},
                              nullptr, nullptr, 0)));
      if (tan)
        TRY((gemm<false, false>(h, BT, nullptr, n_in, n_out, GU, n_out, W, n_in, EpiStore{GTn, (int64_t)n_in},
                                nullptr, nullptr, 0)));
      std::swap(GA, GAn);
      std::swap(GT, GTn);
    }
  }
  CHECK_LAUNCH(h);
  CU(cudaMemcpyAsync(t.hloss, t.part + 2 * lg, sizeof(double) * 2, cudaMemcpyDeviceToHost, h->stream));
  if (lr > 0.0) {
    const double b1 = 0.9, b2 = 0.999;
    const double c1 = 1.0 - std::pow(b1, (double)step), c2 = 1.0 - std::pow(b2, (double)step);
    k_tr_adam<<<(unsigned)std::min<int64_t>(cdiv(t.count, 256), 4 * h->num_sms), 256, 0, h->stream>>>(
        t.count, t.P, t.G, t.M, t.V, t.P32, lr, b1, b2, 1e-8, c1, c2, t.mask);
    h->launches++;
  }
  CU(cudaStreamSynchronize(h->stream));
  *loss = (t.hloss[0] + lam * t.hloss[1]) / (double)B;
  return SDN_OK;
}

}  // extern "C"
