/*
 * odpo.h -- C ABI of libodpo.so, the B200 (sm_100a) Online-DPO learner hot path.
 *
 * The method (arXiv 2410.18252, "Asynchronous RLHF"): Online DPO samples two
 * completions per prompt, ranks them with the reward model into chosen y+ and
 * rejected y- (Sec 2.1; App A.1), and maximises
 *
 *     E log sigma( beta log pi(y+|x)/pi_init(y+|x) - beta log pi(y-|x)/pi_init(y-|x) )
 *                                                             (Sec 2.1)
 *
 * Three calls follow the paper's statement of the problem:
 *   odpo_pair_select              rewards -> (chosen, rejected) pairs
 *   odpo_seq_logprobs             logits, tokens, mask -> log pi(y|x)
 *   odpo_seq_ppl                  the same -> per-completion perplexity (KL proxy)
 *   odpo_online_dpo_loss_fwd_bwd  policy logits, ref log-probs, beta ->
 *                                 -log sigma loss, statistics, dlogits
 *
 * General conventions (all calls):
 *  - Every tensor argument is a DEVICE pointer unless noted; the caller allocates and
 *    owns every buffer (outputs included).  The library never allocates, frees or
 *    synchronises, and keeps no per-call global state.
 *  - Calls are asynchronous and stream-ordered on `stream` (a cudaStream_t passed as
 *    void*; NULL = the legacy default stream).  Calls are re-entrant across streams and
 *    devices; the current device must own the pointers.
 *  - ARGUMENT errors are synchronous return codes (odpo_status).  DATA-dependent
 *    errors are OR-ed into a caller-owned device uint32 `status` word (ODPO_FLAG_*),
 *    read by the caller at its own sync point; outputs of flagged sequences/pairs are
 *    unspecified (except EMPTY_SEQ, where the sequence log-prob is 0).
 *  - Logits are [B, T, V] with element strides (stride_b, stride_t) and contiguous V;
 *    logits[b, t, :] is the (pre-shifted) distribution that produced tokens[b, t]
 *    (reading R1).  The logits base pointer and both strides in bytes must
 *    be multiples of 16 (128-bit vector path; no scalar fallback) -> ODPO_ERR_ALIGNMENT.
 *    V need not be a multiple of the vector width.
 *  - tokens are int32 [B, T]; mask is uint8 [B, T] (1 = response token that counts).
 *    Rows with mask = 0 are never read, so their logits may hold anything.
 */
#ifndef ODPO_H
#define ODPO_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  ODPO_OK = 0,
  ODPO_ERR_INVALID_ARG = 1, /* null required pointer, bad size, beta/invT <= 0 or non-finite, ... */
  ODPO_ERR_ALIGNMENT = 2,   /* logits/dlogits base or stride (bytes) not a multiple of 16 */
  ODPO_ERR_WORKSPACE = 3,   /* workspace NULL or smaller than odpo_workspace_bytes() */
  ODPO_ERR_UNSUPPORTED = 4, /* shape beyond the 32-bit work-ticket range, unknown schedule */
  ODPO_ERR_CUDA = 5         /* a launch failed (cudaGetLastError after launch) */
} odpo_status;

typedef enum { ODPO_F32 = 0, ODPO_BF16 = 1 } odpo_dtype;

/* Data-dependent status bits, OR-ed into *status on the device. */
enum {
  ODPO_FLAG_TOKEN_RANGE = 1,       /* a token outside [0, V) where mask = 1 */
  ODPO_FLAG_NONFINITE_LOGIT = 2,   /* NaN or +inf in a read row, an all -inf row, or a -inf sampled logit */
  ODPO_FLAG_EMPTY_SEQ = 4,         /* a sequence with no mask = 1 token (its log-prob := 0) */
  ODPO_FLAG_NONFINITE_REWARD = 8,  /* a shaped reward is NaN or +-inf */
  ODPO_FLAG_DUP_ROW = 16,          /* chosen == rejected, or a sequence referenced by two pairs */
  ODPO_FLAG_DEGENERATE_PAIR = 32,  /* informational: max reward == min reward in a group */
  ODPO_FLAG_PAIR_RANGE = 64        /* a pair_rows entry outside [0, B): that pair is skipped */
};

/* Loss statistics: LOCAL partial sums over this call's pairs, fp64.  Turning them into
   global means is the caller's SUM all-reduce (one 128-byte message, see below). */
enum {
  ODPO_ST_NPAIRS = 0,      /* number of pairs                                         */
  ODPO_ST_LOSS = 1,        /* sum_p softplus(-z_p) / P_global   (the loss, already a mean) */
  ODPO_ST_NCORRECT = 2,    /* sum_p [z_p > 0]                   (accuracy numerator)  */
  ODPO_ST_Z = 3,           /* sum_p z_p                         (implicit-reward margin) */
  ODPO_ST_RCHOSEN = 4,     /* sum_p beta (S_c - ref_c)          (chosen implicit reward) */
  ODPO_ST_RREJ = 5,        /* sum_p beta (S_r - ref_r)          (rejected implicit reward) */
  ODPO_ST_SCHOSEN = 6,     /* sum_p S_c                                                */
  ODPO_ST_SREJ = 7,        /* sum_p S_r                                                */
  ODPO_ST_NTOK_CHOSEN = 8, /* sum_p #mask tokens of the chosen sequence                */
  ODPO_ST_NTOK_REJ = 9,    /* sum_p #mask tokens of the rejected sequence              */
  ODPO_NSTATS = 10
};
/* Selection statistics (odpo_pair_select), fp64 local partial sums. */
enum {
  ODPO_SEL_MARGIN_SUM = 0, /* sum_p (max - min) shaped reward      */
  ODPO_SEL_NDEGEN = 1,     /* groups with max == min                                 */
  ODPO_SEL_NTRUNC = 2,     /* completions without EOS (penalised)                     */
  ODPO_SEL_NSTATS = 3
};
/* Recommended layout: ONE fp64[16] buffer, loss stats at [0,10), selection stats at
   [10,13), [13,16) zero; a single SUM all-reduce of these 128 bytes gives every global
   statistic. */
#define ODPO_STATS_BUFFER_DOUBLES 16

/* Work schedules of odpo_online_dpo_loss_fwd_bwd_ex. */
enum {
  ODPO_SCHED_AUTO = 0,     /* = TWO_PASS (measured fastest at every BASELINE shape on
                              B200); no co-residency assumption; every
                              schedule gives the same results                          */
  ODPO_SCHED_FUSED = 1,    /* one persistent kernel: forward and backward rows dispatched
                              adaptively (a backward row is taken as soon as its pair's
                              forward pass has completed), per-pair completion counters  */
  ODPO_SCHED_TWO_PASS = 2, /* forward kernel, pair-reduce kernel, backward kernel (2R+1W) */
  ODPO_SCHED_WAVE = 3,     /* (launched cooperatively) one persistent kernel, pairs statically assigned to groups
                              of 2T CTAs (one row per CTA per pair, forward then
                              backward), few enough groups that every in-flight pair
                              stays in L2 (1R+1W at HBM); needs 2T <= resident CTAs and
                              all CTAs co-resident (UNSUPPORTED otherwise).  Measured
                              slower than FUSED on B200          */
  ODPO_SCHED_RESIDENT = 4, /* one persistent CTA per SM; a row's forward pass writes it into a
                              tensor-memory row slot (tcgen05.st) and its backward reads it
                              back (tcgen05.ld), so TMEM-held rows are read from HBM once;
                              rows beyond the TMEM slots are L2-backed (re-streamed for the
                              backward), at most opts->lookahead of them per SM (-1 = 2).
                              Bit-identical to FUSED.  Applies when a row spans <= 8 16-KB
                              chunks (V*elt <= 131072 bytes) and SMs * (TMEM slots + cap)
                              >= 4T; UNSUPPORTED otherwise.  Needs all CTAs co-resident (the
                              GPU not shared with other work).  Measured slower than FUSED
                              on B200; compiled only with
                              -DODPO_EXPERIMENTAL=1, UNSUPPORTED in the default build  */
  ODPO_SCHED_PSYNC = 5,    /* pair-synchronous split-V: every CTA takes the same fixed piece of
                              every pair (the pair's 2T rows flattened and cut into one piece
                              per CTA), forward pieces of pair p + lag run before the backward
                              pieces of pair p, so lag + 1 pairs are live and the backward
                              re-read is served by L2 where they fit (1R+1W at HBM for
                              TLDR-like shapes).  lag = opts->lag_pairs (0 = 4, < 16).
                              Launched cooperatively (all CTAs co-resident or the launch fails:
                              ODPO_ERR_CUDA).  Needs V a multiple of the vector width and a
                              piece of at most one row; UNSUPPORTED otherwise.  Deterministic;
                              row statistics merged in piece order (not FUSED's bits).  */
  ODPO_SCHED_SPLIT = 6     /* factored gradient only (odpo_online_dpo_loss_fwd_bwd_unscaled,
                              odpo_pg_loss_fwd_bwd's single-pass kinds): each row split over a
                              thread-block cluster of up to 8 CTAs, one vocabulary piece per
                              CTA held in registers between its one HBM read and its one HBM
                              write; the CTA partials merged through distributed shared
                              memory.  Needs V * elt <= 256 KB per 8 pieces (bf16 V <=
                              262144); UNSUPPORTED otherwise.  Deterministic; its reduction
                              tree differs from the engine's (results agree to rounding).
                              Measured slower than the row engine on B200 (DESIGN.md
                              section 4); compiled only with -DODPO_EXPERIMENTAL=1,
                              UNSUPPORTED in the default build                          */
};

typedef struct {
  int32_t schedule;     /* ODPO_SCHED_*                                            */
  int32_t lag_pairs;    /* FUSED: cap, in pairs, on how far the forward pass may run ahead of
                           the backward pass (0 = no cap); PSYNC: the lag (0 = 4)     */
  int32_t ctas_per_sm;  /* FUSED: persistent CTAs per SM (0 = auto)               */
  int32_t launches;     /* OUT: number of kernels this call launched               */
  int32_t exp2_split;   /* bf16 only: index of the MUFU/FMA-polynomial exp2 split
                           (-1 = library default)        */
  int32_t lookahead;    /* FUSED: rows a CTA decodes ahead of the row it streams (-1 = default);
                           RESIDENT: L2-backed rows in flight per SM (-1 = default 2)   */
  int32_t row_gap;      /* UNSCALED: forward rows a CTA streams between a row's forward and its
                           backward, 0 or 1 (-1 = default 0); WAVE: pair-steps between a
                           pair's forward and backward rows, 0 or 1 (-1 = default 1)  */
  int32_t engine;       /* row-engine geometry: -1 auto, 0 = 4 consumer warps x 3-stage ring x
                           4 CTAs/SM, 1 = 8 warps x 6 stages x 2 CTAs/SM;
                           geometry 1 requires exp2_split -1 or 0                   */
} odpo_launch_opts;

/*
 * odpo_pair_select -- reward-ranked pair selection (Sec 2.1 "rank them as
 * better (y+) and worse (y-) with the reward model"; App A.1 "the completion
 * with the higher score as the chosen"; Sec 4.2 best/worst of K and the
 * reward margin; PAPER.md:434-435, 518-519 EOS penalty).
 *
 *   rewards      [P][K] f32 device, raw reward-model scores.
 *   has_eos      [P][K] u8 device or NULL (NULL = every completion has EOS).
 *   eos_penalty  shaped score of a completion WITHOUT EOS: it REPLACES the reward (R7).
 *   P >= 0, K >= 2.
 *   chosen[P], rejected[P]  i32 device out: the FIRST index of the max and the LAST index
 *                of the min of the shaped scores (R5), so chosen != rejected always.
 *   pair_rows    [P][2] i32 device out or NULL: (p*K + chosen, p*K + rejected).
 *   reward_margin[P] f32 device out or NULL: max - min (one fp32 subtraction).
 *   sel_stats    [ODPO_SEL_NSTATS] f64 device out or NULL: local sums (overwritten).
 *   status       u32 device or NULL: NONFINITE_REWARD, DEGENERATE_PAIR.
 * One launch.  Bit-exact with the oracle.
 */
odpo_status odpo_pair_select(const float* rewards, const uint8_t* has_eos, float eos_penalty,
                             int64_t P, int32_t K, int32_t* chosen, int32_t* rejected,
                             int32_t* pair_rows, float* reward_margin, double* sel_stats,
                             uint32_t* status, void* stream);

/*
 * odpo_gather_pairs -- compact the selected completions into pair order for the loss call
 * (App A.3: of K completions per prompt only the best and worst are trained on,
 * "we throw out 2 samples").  For d in [0, 2P): destination row d <- source row pair_rows[d]
 * (pair_select's output), so the loss call then takes pair_rows = NULL (rows 2p, 2p+1).
 *
 *   pair_rows   [P][2] i32 device (indices into n_src source rows).
 *   tokens_in / tokens_out   [rows][T] i32 device, mask_in / mask_out [rows][T] u8 device,
 *   ref_in / ref_out         [rows] f32 device; each output (with its input) may be NULL.
 *   status      u32 device or NULL: PAIR_RANGE for an index outside [0, n_src) (that row
 *               is written as zeros).
 * One launch; bit-exact (index work).
 */
odpo_status odpo_gather_pairs(const int32_t* pair_rows, int64_t P, int64_t n_src, int64_t T,
                              const int32_t* tokens_in, const uint8_t* mask_in,
                              const float* ref_in, int32_t* tokens_out, uint8_t* mask_out,
                              float* ref_out, uint32_t* status, void* stream);

/*
 * odpo_seq_logprobs -- log pi(y|x) = sum_t mask[b,t] * log_softmax(invT * logits[b,t,:])[tokens[b,t]]
 * (reading R1: token-wise, pre-shifted, not length-normalised).
 *
 *   logits       [B,T,V] device, dtype dt, strides (stride_b, stride_t) in ELEMENTS, stride_t >= V.
 *   inv_temperature  > 0, finite (R2; 1.0 by default).
 *   seq_logp[B]  f32 device out.
 *   tok_logp[B][T], row_lse[B][T]  f32 device out or NULL (0 where mask = 0).
 *   workspace    device scratch of >= odpo_workspace_bytes(B, T, B/2 + 1) bytes.
 * Single read of the logits: one online log-sum-exp pass per row, then a fixed-order
 * sequence sum.  Bit-identical seq_logp to the fused loss call on the same inputs.
 */
odpo_status odpo_seq_logprobs(const void* logits, odpo_dtype dt, int64_t B, int64_t T, int64_t V,
                              int64_t stride_b, int64_t stride_t, const int32_t* tokens,
                              const uint8_t* mask, float inv_temperature, float* seq_logp,
                              float* tok_logp, float* row_lse, uint32_t* status, void* workspace,
                              size_t workspace_bytes, void* stream);

/*
 * odpo_seq_ppl -- the KL proxy of PAPER.md:121 (Sec 3, "the SFT model's perplexity on the RLHF
 * policy's summaries") and PAPER.md:333 (Sec 5.2, "the perplexity of the base model on the
 * generated completions"), read per completion (R20): with the REFERENCE model's
 * logits, ppl_b = exp(-S_b / n_b), S_b = log pi_ref(y_b|x) (odpo_seq_logprobs), n_b = the
 * number of mask = 1 tokens.
 *
 *   logits .. workspace  as odpo_seq_logprobs (same single-read pass; seq_logp bit-identical).
 *   ppl[B]          f32 device out; an empty completion (n_b = 0, flagged EMPTY_SEQ) gets 1.
 *   ppl_stats[4]    f64 device out: {#completions with n_b > 0, sum_b ppl_b, sum_b S_b,
 *                   sum_b n_b} over the non-empty completions, summed in a fixed order
 *                   (the corpus perplexity is exp(-ppl_stats[2] / ppl_stats[3]); a SUM
 *                   all-reduce of these four doubles gives the global values).
 * Errors: as odpo_seq_logprobs; ppl or ppl_stats NULL -> ODPO_ERR_INVALID_ARG.
 */
odpo_status odpo_seq_ppl(const void* logits, odpo_dtype dt, int64_t B, int64_t T, int64_t V,
                         int64_t stride_b, int64_t stride_t, const int32_t* tokens,
                         const uint8_t* mask, float inv_temperature, float* seq_logp, float* ppl,
                         double* ppl_stats, uint32_t* status, void* workspace,
                         size_t workspace_bytes, void* stream);

/*
 * odpo_online_dpo_loss_fwd_bwd -- Online DPO loss, statistics and dlogits.
 *
 *   policy_logits  [B,T,V] device (as above).
 *   ref_logp[B]    f32 device: log pi_init(y|x) of the same completions (R13).
 *   pair_rows      [P][2] i32 device (chosen row, rejected row) or NULL => rows (2p, 2p+1)
 *                  (then B must equal 2P).  Sequences not referenced by a pair get zero
 *                  gradient.
 *   P_global >= P  pairs in the whole optimiser step across ranks/micro-batches (R3): the
 *                  loss is the MEAN over P_global pairs, so no collective is needed before
 *                  the backward.
 *   beta > 0, inv_temperature > 0 (finite).
 *   dlogits        [B,T,V] device out, same dtype as the logits, strides (dstride_b,
 *                  dstride_t); may EQUAL policy_logits (in place) only with identical
 *                  strides.  dlogits[b,t,:] = coef_b * mask[b,t] * (softmax - onehot(tok)),
 *                  coef_c = +beta sigma(-z) invT / P_global, coef_r = -coef_c.
 *   seq_logp[B]    f32 device out (S_b).
 *   pair_logit[P]  f32 device out or NULL: z_p = beta((S_c - ref_c) - (S_r - ref_r)).
 *   stats          [ODPO_NSTATS] f64 device out: local partial sums (overwritten).
 *   status         u32 device or NULL.
 *   workspace      >= odpo_workspace_bytes(B, T, P) bytes of device scratch.
 * Deterministic: every reduction has a fixed order; no float atomics.
 */
odpo_status odpo_online_dpo_loss_fwd_bwd(const void* policy_logits, odpo_dtype dt, int64_t B,
                                         int64_t T, int64_t V, int64_t stride_b, int64_t stride_t,
                                         const float* ref_logp, const int32_t* tokens,
                                         const uint8_t* mask, const int32_t* pair_rows, int64_t P,
                                         int64_t P_global, float beta, float inv_temperature,
                                         void* dlogits, int64_t dstride_b, int64_t dstride_t,
                                         float* seq_logp, float* pair_logit, double* stats,
                                         uint32_t* status, void* workspace, size_t workspace_bytes,
                                         void* stream);

/* Same as odpo_online_dpo_loss_fwd_bwd with an explicit schedule (opts may be NULL = AUTO);
   opts->launches returns the number of kernels launched. */
odpo_status odpo_online_dpo_loss_fwd_bwd_ex(const void* policy_logits, odpo_dtype dt, int64_t B,
                                            int64_t T, int64_t V, int64_t stride_b,
                                            int64_t stride_t, const float* ref_logp,
                                            const int32_t* tokens, const uint8_t* mask,
                                            const int32_t* pair_rows, int64_t P, int64_t P_global,
                                            float beta, float inv_temperature, void* dlogits,
                                            int64_t dstride_b, int64_t dstride_t, float* seq_logp,
                                            float* pair_logit, double* stats, uint32_t* status,
                                            void* workspace, size_t workspace_bytes,
                                            odpo_launch_opts* opts, void* stream);

/*
 * odpo_online_dpo_loss_fwd_bwd_unscaled -- the same loss, seq_logp, pair_logit, stats and
 * status as odpo_online_dpo_loss_fwd_bwd, with the gradient returned FACTORED per row
 * (performance tier; the gradient of PAPER.md:83's objective):
 *
 *   G          [B,T,V] device out, same dtype as the logits, strides (gstride_b, gstride_t);
 *              may EQUAL policy_logits (in place) only with identical strides.
 *              G[b,t,:] = softmax(invT x[b,t,:]) - onehot(tok[b,t]) for mask = 1 rows of
 *              sequences referenced by a pair, 0 elsewhere.
 *   row_scale  [B][T] f32 device out: coef_b * mask[b,t] (0 for unreferenced sequences), with
 *              coef_c = +beta sigma(-z) invT / P_global, coef_r = -coef_c.
 *
 *   dlogits[b,t,:] = row_scale[b,t] * G[b,t,:]; a consumer such as the LM-head backward GEMM
 *   folds row_scale into its epilogue / prologue.  G does not depend on the pair outcome, so
 *   each row's backward follows its own forward in the same CTA and re-reads the row from L2:
 *   one HBM read and one HBM write of [B,T,V] for every shape.
 *   opts (may be NULL): schedule AUTO (the row engine), SPLIT (ODPO_SCHED_SPLIT: clusters
 *   of CTAs per row, no L2 re-read) or RESIDENT (experimental build); ctas_per_sm,
 *   exp2_split, lookahead, row_gap apply to the engine; opts->launches returns 2.  Other
 *   arguments and errors as odpo_online_dpo_loss_fwd_bwd.
 */
odpo_status odpo_online_dpo_loss_fwd_bwd_unscaled(
    const void* policy_logits, odpo_dtype dt, int64_t B, int64_t T, int64_t V, int64_t stride_b,
    int64_t stride_t, const float* ref_logp, const int32_t* tokens, const uint8_t* mask,
    const int32_t* pair_rows, int64_t P, int64_t P_global, float beta, float inv_temperature,
    void* G, int64_t gstride_b, int64_t gstride_t, float* row_scale, float* seq_logp,
    float* pair_logit, double* stats, uint32_t* status, void* workspace, size_t workspace_bytes,
    odpo_launch_opts* opts, void* stream);

/* Coefficient-variant losses of App B and the Best-of-2 baseline (:209). */
typedef enum {
  ODPO_PG_RLOO = 0,           /* l_p = -1/2 [S1 A1 + S2 A2], A1 = R1 - R2 = -A2 */
  ODPO_PG_COPG = 1,           /* l_p = -1/2 [(S1 - O1) A1 + (S2 - O2) A2]      */
  ODPO_PG_PROX_RLOO = 2,      /* l_p = -1/2 sum_k min(r_k A_k, clip(r_k, 1-eps, 1+eps) A_k),
                                 r = exp(S - O)                                */
  ODPO_PG_BEST_OF_K_SFT = 3   /* l_p = -S1, S1 = the chosen completion            */
} odpo_pg_kind;

/*
 * odpo_pg_loss_fwd_bwd -- the same learner step for the App B losses: S = log pi(y|x) as in
 * odpo_seq_logprobs, the loss averaged over P_global pairs, and
 * dlogits[b,t,:] = coef_b * mask[b,t] * (softmax - onehot(tok)) with coef_b = -(dL/dS_b) invT:
 *   RLOO, CoPG: coef_b = A_b invT / (2 P_global);  SFT: invT / P_global on y1, 0 on y2;
 *   Proximal RLOO: r_b A_b invT / (2 P_global) where min() takes the unclipped term, else 0.
 *
 *   pair_rows  [P][2] (y1, y2) or NULL => (2p, 2p+1); for SFT y1 must be the chosen one
 *              (pair_select's order).
 *   rewards    [B] f32 device: per-sequence (already shaped) rewards R.
 *   old_logp   [B] f32 device: log pi_old(y|x) (CoPG, Proximal RLOO; may be NULL otherwise).
 *   clip_eps   Proximal RLOO clip range, 0 <= eps < 1.
 *   stats      [ODPO_NSTATS] f64 out, per this call: pairs, mean loss, sequences with a nonzero
 *              coefficient, sum r (Proximal RLOO), sum A1, sum |A1|, sum S1, sum S2, tokens of
 *              y1, tokens of y2.
 * RLOO, CoPG and SFT know every coefficient before the forward pass: each row's backward
 * follows its forward in the same CTA (one HBM read and one write of [B,T,V]).  Proximal RLOO
 * needs S first and runs the FUSED (default) or TWO_PASS schedule of the DPO call.
 * Other arguments, ownership and errors as odpo_online_dpo_loss_fwd_bwd.
 */
odpo_status odpo_pg_loss_fwd_bwd(const void* policy_logits, odpo_dtype dt, int64_t B, int64_t T,
                                 int64_t V, int64_t stride_b, int64_t stride_t,
                                 const int32_t* tokens, const uint8_t* mask,
                                 const int32_t* pair_rows, int64_t P, int64_t P_global,
                                 int32_t kind, const float* rewards, const float* old_logp,
                                 float clip_eps, float inv_temperature, void* dlogits,
                                 int64_t dstride_b, int64_t dstride_t, float* seq_logp,
                                 double* stats, uint32_t* status, void* workspace,
                                 size_t workspace_bytes, odpo_launch_opts* opts, void* stream);

/*
 * Vocabulary-parallel loss: the LM head's vocabulary is
 * sharded over W ranks, rank w holding logits[:, :, v0_w : v0_w + V_shard_w] (v0 increasing
 * with w).  Two calls per rank; the 16-byte row partials move between them either through the
 * caller's collective (odpo_vp_row_partials + e.g. an NCCL all_gather, flags = NULL) or INSIDE
 * the kernels over peer memory (odpo_vp_row_partials_put + flags): no host collective.
 *
 * odpo_vp_row_partials -- one read of this rank's shard: for every row with mask = 1,
 *   parts[row] = (m, log1p r, x_tok, owns) with 1 + r = sum over the shard of
 *   exp(invT (x - m)), m the shard maximum, x_tok the sampled token's logit if
 *   v0 <= tok < v0 + V_shard (owns = 1) else 0 (owns = 0); masked rows get (-inf, 0, 0, 0).
 *   parts: [B*T][4] f32 device, 16-byte aligned.  TOKEN_RANGE if tok is outside [0, V_total).
 *
 * odpo_vp_loss_fwd_bwd -- merges parts_all ([W][B*T][4], rank order) into the full-vocabulary
 *   row statistics (lse = invT m* + log1p R, R = r_w* + sum_{w != w*} e^{invT (m_w - m*)}(1+r_w),
 *   w* the first rank holding the maximum), then the same pair reduction and statistics as
 *   odpo_online_dpo_loss_fwd_bwd (identical on every rank: the stats are already global over
 *   the vocabulary group, do not sum them over it), and writes this rank's dlogits shard
 *   coef_b (softmax - onehot) with the global normaliser.  One read of the shard again (2R+1W
 *   per shard).  flags / epoch: NULL for a caller-gathered parts_all; otherwise this rank's
 *   [W] u32 flag words of the in-kernel exchange: the merge kernel first waits (system-scope
 *   acquire, spinning on the device) until flags[q] has reached epoch for every rank q, and
 *   parts_all is this rank's exchange buffer of that epoch (W <= 8).  Other arguments and
 *   errors as odpo_online_dpo_loss_fwd_bwd.
 *
 * odpo_vp_row_partials_put -- odpo_vp_row_partials with the exchange in the kernel: every
 *   row's partial is stored into slot [rank][row] of EVERY rank's buffer
 *   (peer_parts[q] = rank q's [W][B*T][4] f32 buffer for this epoch, mapped into this process:
 *   NVLink P2P on a multi-GPU node, CUDA IPC between processes sharing a GPU), and the last CTA
 *   publishes `epoch` into peer_flags[q][rank] for every q (system-scope release) after a
 *   system fence.  peer_parts / peer_flags are HOST arrays of W device pointers; `done` is this
 *   rank's device u32 CTA counter (0 on entry; the kernel leaves it 0).  Epochs must increase
 *   by one per step; a double-buffered parts region (by epoch parity) is safe because a rank
 *   cannot start step k+2's put before every rank finished step k's merge.  W <= 8.
 *   Errors: INVALID_ARG (null pointers, rank/W), ALIGNMENT, CUDA.
 */
odpo_status odpo_vp_row_partials(const void* logits_shard, odpo_dtype dt, int64_t B, int64_t T,
                                 int64_t V_shard, int64_t stride_b, int64_t stride_t,
                                 int64_t v0, int64_t V_total, const int32_t* tokens,
                                 const uint8_t* mask, float inv_temperature, float* parts,
                                 uint32_t* status, void* workspace, size_t workspace_bytes,
                                 void* stream);
odpo_status odpo_vp_loss_fwd_bwd(const float* parts_all, int32_t W, const void* logits_shard,
                                 odpo_dtype dt, int64_t B, int64_t T, int64_t V_shard,
                                 int64_t stride_b, int64_t stride_t, int64_t v0, int64_t V_total,
                                 const float* ref_logp, const int32_t* tokens,
                                 const uint8_t* mask, const int32_t* pair_rows, int64_t P,
                                 int64_t P_global, float beta, float inv_temperature,
                                 void* dlogits_shard, int64_t dstride_b, int64_t dstride_t,
                                 float* seq_logp, float* pair_logit, double* stats,
                                 const uint32_t* flags, uint32_t epoch, uint32_t* status,
                                 void* workspace, size_t workspace_bytes, void* stream);
odpo_status odpo_vp_row_partials_put(const void* logits_shard, odpo_dtype dt, int64_t B,
                                     int64_t T, int64_t V_shard, int64_t stride_b,
                                     int64_t stride_t, int64_t v0, int64_t V_total,
                                     const int32_t* tokens, const uint8_t* mask,
                                     float inv_temperature, float* const* peer_parts,
                                     uint32_t* const* peer_flags, uint32_t* done, int32_t rank,
                                     int32_t W, uint32_t epoch, uint32_t* status, void* stream);

/*
 * odpo_stats_put / odpo_stats_sum -- the batch-sharded statistics reduction (SURVEY.md §8(e),
 * S6: a SUM over the data-parallel ranks of the 16-double stats buffer) over peer memory instead
 * of a collective, with the exchange buffers of odpo_vp_row_partials_put:
 *   put: stats [16] f64 (this rank's local partials) -> slot [rank][0..16) of every rank's
 *        stats slots (peer_slots[q] = rank q's [W][16] f64 region for this epoch, mapped into this
 *        process), then a system fence and `epoch` into peer_flags[q][rank] (system release).
 *   sum: waits (system acquire) until this rank's flags[q] reached `epoch` for every q, then
 *        out[i] = sum over q = 0..W-1 IN RANK ORDER of slots[q][i]: every rank gets the same bits.
 * peer_slots / peer_flags are HOST arrays of W device pointers; W <= 8.  Errors: INVALID_ARG, CUDA.
 */
odpo_status odpo_stats_put(const double* stats, double* const* peer_slots,
                           uint32_t* const* peer_flags, int32_t rank, int32_t W, uint32_t epoch,
                           void* stream);
odpo_status odpo_stats_sum(const double* slots, const uint32_t* flags, int32_t W, uint32_t epoch,
                           double* out, void* stream);

/* Host-only: device scratch bytes needed by the calls above for B sequences of T tokens
   and P pairs (about 13 bytes per row + 80 bytes per pair + small). */
size_t odpo_workspace_bytes(int64_t B, int64_t T, int64_t P);

/* Host-only: static description of a status code. */
const char* odpo_status_string(odpo_status s);

/* Host-only: library version string. */
const char* odpo_version(void);

/*
 * odpo_lmhead_seq_logprobs -- NEXT-2, forward part: sequence log-probs
 * straight from the LM head (Sec 2.1, with the policy's output layer written
 * out), the [B, T, V] logits never written to memory.
 *
 *   logits[b, t, v] = invT * sum_i hidden[b, t, i] * weight[v, i]
 *   tok_logp[b, t]  = logits[b, t, tokens[b, t]] - logsumexp_v logits[b, t, v]   (mask = 1)
 *   seq_logp[b]     = sum_t mask[b, t] tok_logp[b, t]
 *
 *   hidden     bf16 [B, T, d], contiguous (row b*T + t at hidden + (b*T + t)*d), 16-byte
 *              aligned; d a multiple of 64.
 *   weight     bf16 [V, d], contiguous, 16-byte aligned (the LM head / unembedding).
 *   tokens, mask  int32 / uint8 [B, T].
 *   tok_logp, row_lse  fp32 [B, T] outputs (may be NULL); 0 where mask = 0.
 *   seq_logp   fp32 [B] output.
 *   status     device uint32, OR-ed ODPO_FLAG_* (TOKEN_RANGE, NONFINITE_LOGIT, EMPTY_SEQ).
 *   workspace  >= odpo_lmhead_workspace_bytes(B, T, V) bytes of device scratch.
 * Implementation: tcgen05.mma (bf16 in, fp32 accumulators in TMEM, 128 x 256 tiles) fed by
 * 2-D TMA; the epilogue folds each 256-wide logit tile into the row's online logsumexp.
 * Errors: INVALID_ARG (NULL pointers, non-positive sizes, invT not finite > 0), UNSUPPORTED
 * (d % 64 != 0, B*T or V > 2^31 - 1), ALIGNMENT, WORKSPACE, CUDA (launch or tensor-map
 * encoding failed).
 * Tuning only (environment, read per call): ODPO_LMH_1CTA=1 selects the single-CTA kernel,
 * ODPO_LMH_G=<n> the raster group size (the raster order does not change results).
 */
size_t odpo_lmhead_workspace_bytes(int64_t B, int64_t T, int64_t V);

/*
 * odpo_lmhead_grad -- NEXT-2 backward: the LM-head gradients of the loss whose per-row logit
 * gradient is row_scale * (softmax - onehot) (the factored gradient of
 * odpo_online_dpo_loss_fwd_bwd_unscaled / odpo_online_dpo_loss_from_token_logp):
 *
 *   G[r, v]     = row_scale[r] * (softmax(invT * logits[r, :])[v] - [v == tokens[r]])
 *   dhidden     = G weight          fp32 [R, d] (overwritten)
 *   dweight     = G^T hidden        fp32 [V, d] (overwritten)
 *
 * The logits are recomputed chunk by chunk (chunk_rows rows at a time, rounded up to 256) by
 * the NEXT-2 tcgen05 kernel, whose epilogue writes G (bf16) into `scratch` instead of reducing
 * it; the two GEMMs with G run on the library's own tcgen05 CTA-pair GEMM (bf16 operands
 * staged by TMA, fp32 accumulators in tensor memory; no cuBLAS): dhidden = G W reads W
 * N-major and dweight += G^T H reads G M-major and H N-major straight from their stored
 * layouts (MN-major shared-memory descriptors), so nothing is transposed or copied.
 * Deterministic: every output element is accumulated in a fixed order (chunks in row order,
 * K in order), no atomics.  row_lse is odpo_lmhead_seq_logprobs' row_lse (natural log, invT
 * applied).
 *   hidden bf16 [R, d], weight bf16 [V, d] contiguous, 16-byte aligned, d % 64 == 0.
 *   dhidden, dweight fp32, 16-byte aligned.
 *   scratch >= odpo_lmhead_grad_scratch_bytes(chunk_rows, d, V) bytes (one chunk of G:
 *   about 2 chunk_rows V bytes), 16-byte aligned.
 * Errors: INVALID_ARG, UNSUPPORTED (d % 64, sizes), ALIGNMENT, WORKSPACE, CUDA.
 */
size_t odpo_lmhead_grad_scratch_bytes(int64_t chunk_rows, int64_t d, int64_t V);
odpo_status odpo_lmhead_grad(const void* hidden, const void* weight, int64_t R, int64_t d,
                             int64_t V, const int32_t* tokens, const float* row_lse,
                             const float* row_scale, float inv_temperature, float* dhidden,
                             float* dweight, void* scratch, size_t scratch_bytes,
                             int64_t chunk_rows, void* stream);

/*
 * odpo_lmhead_dpo_step -- NEXT-2 learner step of the LM head with the Online-DPO loss
 * (Sec 2.1) in chunks of whole pairs, the [B, T, V] logits never
 * materialised beyond one chunk.  Per chunk of chunk_pairs pairs:
 *   logits_c = hidden_c W^T          bf16 [2 cp T, V] into scratch (the library's tcgen05 head
 *                                    kernel), its epilogue also folding the stored bf16 logits
 *                                    into one (m, log1p r, x_tok) partial per (row, 256-entry
 *                                    vocabulary tile);
 *   the Online-DPO loss in place over the chunk from those partials (the merge of
 *   odpo_vp_loss_fwd_bwd with one shard per tile: row log-softmax, gather, masked sums, z, loss,
 *   statistics, dlogits = coef (softmax(invT logits) - onehot)) -- the chunk is read once;
 *   dhidden_c = dlogits_c W,  dweight += dlogits_c^T hidden_c   (tcgen05 GEMMs, fp32 out).
 * Three head GEMMs per row (odpo_lmhead_grad's recomputing backward needs four).
 *   hidden bf16 [2P, T, d] with the pair's sequences at rows (2p, 2p+1) (odpo_gather_pairs
 *   compacts a best/worst-of-K selection into this layout), weight bf16 [V, d], d % 64 == 0.
 *   ref_logp [2P] f32, tokens [2P, T] i32, mask [2P, T] u8, P_global >= P, beta, invT > 0.
 *   dhidden fp32 [2P, T, d], dweight fp32 [V, d] (overwritten); seq_logp [2P] f32 out;
 *   pair_logit [P] f32 out or NULL; stats fp64 [>= ODPO_NSTATS] out (the chunks' sums: the
 *   same statistics as the loss call over the whole batch); status as the loss call.
 *   scratch >= odpo_lmhead_dpo_step_scratch_bytes(chunk_pairs, T, V) bytes, 256-byte aligned.
 * The logits are rounded to bf16 (as a materialised bf16 logits tensor would be).
 * Errors: INVALID_ARG, UNSUPPORTED (d % 64, sizes), ALIGNMENT, WORKSPACE, CUDA.
 */
size_t odpo_lmhead_dpo_step_scratch_bytes(int64_t chunk_pairs, int64_t T, int64_t V);
odpo_status odpo_lmhead_dpo_step(const void* hidden, const void* weight, int64_t P, int64_t T,
                                 int64_t d, int64_t V, const float* ref_logp,
                                 const int32_t* tokens, const uint8_t* mask, int64_t P_global,
                                 float beta, float inv_temperature, float* dhidden,
                                 float* dweight, float* seq_logp, float* pair_logit,
                                 double* stats, uint32_t* status, void* scratch,
                                 size_t scratch_bytes, int64_t chunk_pairs, void* stream);

/*
 * odpo_online_dpo_loss_from_token_logp -- the Online-DPO loss (Sec 2.1; S3/S4 of
 * SURVEY.md §8(a)) from per-token policy log-probs, e.g. those odpo_lmhead_seq_logprobs
 * produced without logits.  Same pair reduction (fixed-order sequence sums, z, -log sigma,
 * statistics, coefficients) as odpo_online_dpo_loss_fwd_bwd.
 *   tok_logp   fp32 [B, T] per-token log pi (read where mask = 1 only).
 *   ref_logp, mask, pair_rows, P, P_global, beta, inv_temperature, seq_logp, pair_logit,
 *   stats, status, workspace: as odpo_online_dpo_loss_fwd_bwd (workspace >=
 *   odpo_workspace_bytes(B, T, P)).
 *   row_scale  fp32 [B, T] output (may be NULL): coef_b * mask[b, t], the per-row factor of the
 *              gradient with respect to the logits (d loss / d logits = row_scale * G).
 * Errors: INVALID_ARG, UNSUPPORTED, WORKSPACE, CUDA.
 */
odpo_status odpo_online_dpo_loss_from_token_logp(
    const float* tok_logp, int64_t B, int64_t T, const float* ref_logp, const uint8_t* mask,
    const int32_t* pair_rows, int64_t P, int64_t P_global, float beta, float inv_temperature,
    float* seq_logp, float* pair_logit, double* stats, float* row_scale, uint32_t* status,
    void* workspace, size_t workspace_bytes, void* stream);
odpo_status odpo_lmhead_seq_logprobs(const void* hidden, const void* weight, int64_t B, int64_t T,
                                     int64_t d, int64_t V, const int32_t* tokens,
                                     const uint8_t* mask, float inv_temperature, float* tok_logp,
                                     float* row_lse, float* seq_logp, uint32_t* status,
                                     void* workspace, size_t workspace_bytes, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* ODPO_H */
