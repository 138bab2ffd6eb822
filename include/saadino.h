/*
 * saadino.h -- C ABI of the B200 SAA risk / control-gradient engine for
 * MR-DINO surrogates (arxiv 2305.20053).  Plain C: pointers, sizes, int
 * status codes; no torch or C++ types.  Library: paper_2305_20053_b200/libsaadino.so
 *
 * One handle = one CUDA device = one shard of the SAA sample set.  Across
 * processes (one per GPU) the caller combines the handle's small exchange
 * buffers with its own collective; a single-process
 * caller uses sdn_eval(), which chains every phase locally.
 *
 * Reference interfaces each entry point replaces (paths relative to
 * /root/reference/pkg/src/ouukit):
 *   sdn_set_model      <- SurrogateModel fields / init_model           surrogate.py:149-157, 241-256
 *   sdn_set_tracking   <- build_tracking_form / ReducedTrackingForm     pod.py:46-62, 104-110
 *   sdn_set_decoder    <- PODBasis.lift + TrackingTarget (full frame)   pod.py:36-40, riskopt.py:89-109
 *   sdn_set_samples    <- SurrogateEvaluator.__init__ (m_r copy)        riskopt.py:166-172
 *   sdn_encode_fields  <- KLEBasis.encode, pipeline's per-sample loop   randfield.py:67-72, pipeline.py:357-360
 *   sdn_eval           <- saa_objective(prob, z, t) over the surrogate  riskopt.py:227-243 (+178-194)
 *   sdn_eval_samples   <- SurrogateEvaluator.__call__ -> (Q, G)         riskopt.py:178-194
 *   sdn_forward_batch  <- SurrogateModel.forward_batch                  surrogate.py:187-191
 *   sdn_jacobian_batch <- SurrogateModel.z_jacobian_batch (+ decode)    surrogate.py:229-233, tests/test_acceptance.py:326
 *   sdn_select_topk    <- mc_cvar / mc_var order statistics             riskopt.py:56-82
 *
 * Errors: every function returns SDN_OK (0) or a negative code; the message
 * of the last failure on the calling thread is sdn_last_error().  Argument
 * errors mirror the reference's ValueError cases (riskopt.py:28,64-67,
 * 211-216,236-237; surrogate.py:188-189).  Non-finite samples propagate as
 * NaN into the value and gradient, which minimize() treats as a rejected
 * step (riskopt.py:341).
 */
#ifndef SAADINO_H
#define SAADINO_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SDN_OK 0
#define SDN_ERR_ARG (-1)     /* invalid argument (reference: ValueError) */
#define SDN_ERR_CUDA (-2)    /* CUDA runtime failure */
#define SDN_ERR_STATE (-3)   /* call order (e.g. eval before set_model) */
#define SDN_ERR_NOMEM (-4)

/* activations: identity/tanh/softplus/sigmoid as surrogate.py:42-63; elu (BASELINE) */
#define SDN_ACT_IDENTITY 0
#define SDN_ACT_TANH 1
#define SDN_ACT_SOFTPLUS 2
#define SDN_ACT_SIGMOID 3
#define SDN_ACT_ELU 4
#define SDN_ACT_SOFTMAX 5   /* per-layer vector softmax (surrogate.py:65-66, 175-177); SIMT chains */

/* risk kinds: mean / smoothed CVaR as RiskSpec (riskopt.py:204-216), plus
 * mean + beta*variance and exact CVaR by device selection (BASELINE) */
#define SDN_RISK_MEAN 0
#define SDN_RISK_CVAR_SMOOTH 1
#define SDN_RISK_MEANVAR 2
#define SDN_RISK_CVAR_EXACT 3

/* QoI frame: reduced (pod.py:46-62) or decoded full frame (riskopt.py:103-108) */
#define SDN_QOI_REDUCED 0
#define SDN_QOI_DECODED 1

/* GEMM back end for the MLP chain */
#define SDN_GEMM_AUTO 0
#define SDN_GEMM_SIMT 1      /* fp32 FFMA */
#define SDN_GEMM_TC 2        /* tcgen05 bf16x3 split, fp32 accumulate in TMEM */

typedef struct sdn_handle sdn_handle;

typedef struct sdn_config {
  int32_t n_layers;          /* number of weight matrices (hidden + output) */
  const int32_t* widths;     /* n_layers + 1 widths; widths[0] = r_m + r_z */
  int32_t r_m;               /* field coefficients */
  int32_t d_z;               /* controls (V_z is d_z x r_z, r_z = widths[0] - r_m) */
  int32_t activation;        /* SDN_ACT_* */
  int32_t residual;          /* 1: equal-width hidden layers add their input */
  int32_t gemm;              /* SDN_GEMM_* */
  int32_t device;            /* CUDA ordinal */
  int64_t max_samples;       /* capacity of this shard */
} sdn_config;

typedef struct sdn_risk {
  int32_t kind;              /* SDN_RISK_* */
  int32_t qoi;               /* SDN_QOI_* */
  double beta;               /* CVaR level / variance weight */
  double eps;                /* smoothing width (smoothed CVaR) */
  double t;                  /* auxiliary variable (smoothed CVaR) */
  double alpha;              /* control cost alpha ||z||^2 */
  int32_t need_grad;         /* 0: value only (line-search trials) */
} sdn_risk;

typedef struct sdn_result {
  double value;
  double grad_t;             /* smoothed CVaR only, else 0 */
  int64_t n_samples;         /* global sample count */
  int64_t n_selected;        /* CVaR exact: k; smoothed: active samples */
  double q_mean, q_var;      /* sample moments of Q (for reporting) */
  int64_t n_refined;         /* rows of this rank re-evaluated in fp64 at the
                                risk's decision boundary (smoothed-CVaR window,
                                exact-CVaR threshold band); never skipped */
} sdn_result;

const char* sdn_last_error(void);
int sdn_version(void);

int sdn_create(const sdn_config* cfg, sdn_handle** out);
int sdn_destroy(sdn_handle* h);

/* Use an external CUDA stream (cudaStream_t) for all work; 0 = own stream. */
int sdn_set_stream(sdn_handle* h, void* stream);
int sdn_synchronize(sdn_handle* h);

/* Weights W_l (n_out x n_in row-major, torch Linear layout) and biases;
 * in_scale (r_m), out_mean/out_std (r_u), Vz (d_z x r_z row-major, NULL = I).
 * All host pointers (float32). */
int sdn_set_model(sdn_handle* h, const float* const* W, const float* const* b,
                  const float* in_scale, const float* out_mean, const float* out_std,
                  const float* Vz);

/* Reduced tracking form c (r_u), q0. */
int sdn_set_tracking(sdn_handle* h, const float* c, double q0);

/* Decoder U (d_u x r_u row-major), bias (d_u), lumped mass diag (d_u),
 * target (d_u): enables SDN_QOI_DECODED. */
int sdn_set_decoder(sdn_handle* h, int64_t d_u, const float* U, const float* ubias,
                    const float* Mdiag, const float* u_target);

/* The same with a general sparse state mass M in CSR (indptr: d_u + 1 int64,
 * indices: nnz int32 columns, data: nnz values; host pointers) -- the
 * reference's q_tracking takes any scipy sparse target.M (riskopt.py:103-108),
 * e.g. the consistent P1 mass of fem.py:119-126 with lumped=False. */
int sdn_set_decoder_csr(sdn_handle* h, int64_t d_u, const float* U, const float* ubias,
                        const int64_t* indptr, const int32_t* indices, const float* data,
                        const float* u_target);

/* Encoded samples m_r (n x r_m row-major).  on_device != 0: device pointer.
 * global_offset = index of row 0 in the global sample set (CVaR tie-break). */
int sdn_set_samples(sdn_handle* h, const float* m_r, int64_t n, int64_t global_offset,
                    int32_t on_device);

/* Encode nodal fields on the device: m_r = V_m^T diag(M) (m - m_mean).
 * m (n x d_m), Vm (d_m x r_m), Mdiag (d_m); host pointers unless on_device.
 * Stores the result as this shard's samples (like sdn_set_samples). */
int sdn_encode_fields(sdn_handle* h, const float* m, int64_t n, int64_t d_m,
                      const float* Vm, const float* Mdiag, float m_mean,
                      int64_t global_offset, int32_t on_device);

/* Full single-process evaluation: value, grad_z (d_z), CVaR indices.
 * z: host (d_z) float64.  grad_z: host (d_z) float64 or NULL.
 * cvar_idx: host int64 (k) or NULL (exact CVaR). */
int sdn_eval(sdn_handle* h, const double* z, const sdn_risk* risk, sdn_result* res,
             double* grad_z, int64_t* cvar_idx);

/* Several risk functionals sharing ONE forward pass (e.g. mean+variance and
 * exact CVaR, BASELINE config 2).  res[n_risks]; grads (n_risks x d_z) or
 * NULL; cvar_idx receives each exact-CVaR selection in order, or NULL. */
int sdn_eval_multi(sdn_handle* h, const double* z, const sdn_risk* risks, int32_t n_risks,
                   sdn_result* res, double* grads, int64_t* cvar_idx);
/* sdn_eval_multi in two halves: _launch enqueues the evaluation on the
 * handle's stream (one CUDA-graph replay) and returns at once; _wait blocks
 * until it is done and reads the results (same arguments as sdn_eval_multi;
 * cvar_idx only if want_idx was set at launch).  Lets a caller record its own
 * stream events around the device work, or overlap host work with it. */
int sdn_eval_multi_launch(sdn_handle* h, const double* z, const sdn_risk* risks, int32_t n_risks,
                          int32_t want_idx);
int sdn_eval_multi_wait(sdn_handle* h, sdn_result* res, double* grads, int64_t* cvar_idx);

/* Per-sample evaluator protocol: Q (n) and G (n x d_z) as float64 host arrays. */
int sdn_eval_samples(sdn_handle* h, const double* z, int32_t qoi, double* Q, double* G);

/* Surrogate primal / Jacobian on arbitrary rows (host pointers, float32):
 * m_r (n x r_m), z (n x d_z, one control per row as forward_batch takes it);
 * phi (n x r_u); J (n x r_u x d_z), or decoded U J (n x d_u x d_z) when
 * decoded != 0 (needs sdn_set_decoder). */
int sdn_forward_batch(sdn_handle* h, const float* m_r, const float* z, int64_t n,
                      float* phi);
int sdn_jacobian_batch(sdn_handle* h, const float* m_r, const float* z, int64_t n,
                       int32_t decoded, float* J);
/* Batched control Jacobian of the handle's resident samples (sdn_set_samples)
 * at one control z (host, d_z float64) -- BASELINE config 5: dq/dz per
 * sample, J_dev a DEVICE buffer of n x r_u x d_z floats, or decoded
 * U (std . dq/dz) of n x d_u x d_z (test_acceptance.py:326), same layout as
 * z_jacobian_batch (surrogate.py:195-233).  Enqueued on the handle's stream;
 * returns without waiting (sdn_synchronize).  Multi-GPU: each rank passes its
 * shard's buffer (no exchange). */
int sdn_jacobian_samples(sdn_handle* h, const double* z, int32_t decoded, float* J_dev);

/* Decoded states u = U phi + b for the rows' phi (n x r_u) -> (n x d_u). */
int sdn_lift(sdn_handle* h, const float* phi, int64_t n, float* u);

/* Order statistics on device: indices of the k largest of values (n, float64,
 * host or device), ordered by value desc then index asc.  idx: host int64. */
int sdn_select_topk(sdn_handle* h, const double* values, int64_t n, int64_t k,
                    int32_t on_device, int64_t* idx);

/* ---- multi-process phases (one handle per rank) -------------------------
 * The caller owns two device exchange buffers (float64) it can all-reduce /
 * all-gather with its own collective on the handle's stream:
 *   stats   : SDN_STATS_LEN doubles    (sum-reduce)
 *   partial : sdn_partial_len(h) doubles (sum-reduce)
 *   cand    : 2*k doubles per rank (exact CVaR candidates; all-gather)
 * Sequence: eval_forward -> [allreduce stats] -> [cvar_exact: eval_candidates
 * -> allgather cand -> eval_select] -> eval_backward -> [allreduce partial]
 * -> eval_finish.  Every phase is asynchronous on the handle's stream. */
#define SDN_STATS_LEN 8
int sdn_partial_len(sdn_handle* h);
int sdn_eval_forward(sdn_handle* h, const double* z, const sdn_risk* risk,
                     double* stats_dev);
int sdn_eval_candidates(sdn_handle* h, int64_t k, double* cand_dev);
int sdn_eval_select(sdn_handle* h, const double* all_cand_dev, int32_t n_ranks, int64_t k);

/* Multi-rank exact CVaR, optional: after sdn_eval_select, re-evaluate in fp64
 * the rows of this shard whose Q lies within refinement error of the global
 * threshold (Q refined in place); then repeat sdn_eval_candidates ->
 * all-gather -> sdn_eval_select.  Single-rank sdn_eval / sdn_eval_multi do
 * the equivalent internally. */
int sdn_eval_refine_band(sdn_handle* h);

/* Several risks over one forward (multi-rank): after the final sdn_eval_select
 * of each exact-CVaR risk, sdn_eval_keep_selection(h, slot) keeps it (slots in
 * the order the exact risks appear in the list); sdn_eval_backward_multi then
 * runs ONE reverse sweep for all risks (unit seeds, per-risk weighted column
 * sums) into partials_dev = n_risks x sdn_partial_len(h) doubles, all-reduced
 * together; finish each risk with sdn_eval_set_risk + sdn_eval_finish on its
 * slice.  (sdn_eval_multi does the same on one handle.) */
int sdn_eval_keep_selection(sdn_handle* h, int32_t slot);
/* The kept selection of `slot` as k ascending GLOBAL sample indices (host
 * buffer idx_out, k = the risk's ceil-count over the global N).  Every rank
 * holds the same merged selection, so every rank returns the same indices --
 * the sharded counterpart of sdn_eval's cvar_idx (riskopt.py:73-82: the
 * samples mc_cvar averages, ordered by index). */
int sdn_eval_selection(sdn_handle* h, int32_t slot, int64_t k, int64_t* idx_out);
int sdn_eval_backward_multi(sdn_handle* h, const sdn_risk* risks, int32_t n_risks, const double* stats_dev,
                            double* partials_dev);
int sdn_eval_backward(sdn_handle* h, const double* stats_dev, double* partial_dev);
/* Switch the risk for the next sweep sharing the last forward (multi-risk). */
int sdn_eval_set_risk(sdn_handle* h, const sdn_risk* risk);
int sdn_eval_finish(sdn_handle* h, const double* stats_dev, const double* partial_dev,
                    sdn_result* res, double* grad_z);

/* Local per-sample outputs of the last evaluation (device pointers, read-only;
 * valid until the next call): Q (n, float64). */
int sdn_last_q(sdn_handle* h, const double** q_dev, int64_t* n);
/* Q as used by the last exact-CVaR selection: the chain's Q with the rows
 * near the threshold re-evaluated in fp64; = sdn_last_q when
 * no exact selection ran since the last forward. */
int sdn_last_qsel(sdn_handle* h, const double** q_dev, int64_t* n);

/* H1 (derivative-informed) training on the device (reference
 * surrogate.py:263-405).  The handle's network shape and
 * activation define the model (elementwise activations, no residual blocks,
 * V_z = I, as the reference's network).  The dataset is resident on the device
 * (j_r: n x r_u x d_z, may be null for jacobian_weight = 0); parameters are fp64
 * masters in the reference layout (W_l: n_out x n_in over the full [m | z]
 * input, b_l); sdn_train_step computes loss_and_grad over the batch idx and,
 * when lr > 0, applies one Adam step (0.9, 0.999, 1e-8; step = 1-based count). */
int sdn_train_setup(sdn_handle* h, const float* m_r, const float* z, const float* u_r, const float* j_r,
                    int64_t n, int32_t batch_cap);
int sdn_train_set_params(sdn_handle* h, const double* const* W, const double* const* b, const double* in_scale,
                         const double* out_mean, const double* out_std);
int sdn_train_set_mask(sdn_handle* h, const double* const* mW, const double* const* mb);   /* 0 = frozen entry */
int sdn_train_get_params(sdn_handle* h, double* const* W, double* const* b);
int sdn_train_get_grad(sdn_handle* h, double* const* gW, double* const* gb);
int sdn_train_step(sdn_handle* h, const int64_t* idx, int32_t B, double jacobian_weight, double lr, int64_t step,
                   double* loss);

/* Instrumentation.  sdn_profile(h, 1) starts CUDA-event timing of every
 * launch by kernel class (0 fwd GEMM, 1 reverse GEMM, 2 QoI+moments,
 * 3 top-k select, 4 compaction, 5 seeds, 6 column sums, 7 finalise,
 * 8 zbias, 9 other, 10 fp64 Q refinement); sdn_profile_read returns per-class device ms,
 * algorithmic flops and bytes, and launch counts. */
#define SDN_PROF_CLASSES 13
int sdn_profile(sdn_handle* h, int32_t enable);
int sdn_profile_read(sdn_handle* h, int32_t n_cls, double* ms, double* flops, double* bytes,
                     int64_t* count);

/* Device time (CUDA events on the handle's stream, ms) of the last
 * sdn_eval_multi: from its first enqueued operation to its last (graph
 * replay included), host staging and result post-processing excluded. */
int sdn_last_device_ms(sdn_handle* h, double* ms);

/* Kernel tuning: average ms of one layer-1 forward GEMM over M rows
 * (mode 0 tcgen05 + null epilogue, 1 tcgen05 + fused epilogue, 2 SIMT). */
int sdn_debug_gemm(sdn_handle* h, int64_t M, int32_t mode, int32_t reps, double* ms);

/* Number of kernels this handle has launched (lifetime). */
int64_t sdn_kernel_launches(sdn_handle* h);

#ifdef __cplusplus
}
#endif
#endif /* SAADINO_H */
