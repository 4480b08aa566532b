/*
 * oracle/oracle.c -- the CPU ORACLE for the Online-DPO learner hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load or call this library.  The product
 * path (paper_2410_18252_b200/, libodpo.so) never links, imports or executes it,
 * and this file shares no source, header, table or constant generator with the
 * CUDA path: it re-declares its own enums with the same numeric values.
 *
 * Plain, slow, obviously-correct definitions in IEEE double, compiled with
 * -O2 -ffp-contract=off and without -ffast-math.  Each function cites the passage
 * it follows:
 *
 *   orc_pair_select   PAPER.md:81 (Sec 2.1, "rank them as better (y+) and worse (y-)
 *                     with the reward model"), PAPER.md:400 (App A.1, "the completion
 *                     with the higher score as the chosen"), PAPER.md:282 (Sec 4.2,
 *                     best/worst of K, reward margin), PAPER.md:434-435 / 518-519
 *                     (Penalty Reward Value for completions without an EOS token).
 *   orc_seq_logprobs  PAPER.md:83 (Sec 2.1, the log pi_theta(y|x) inside the Online DPO
 *                     objective) read token-wise: log pi(y|x) = sum_t log softmax(x_t)[y_t]
 *                     (reading R1).
 *   orc_online_dpo_loss_fwd_bwd
 *                     PAPER.md:83 (Online DPO objective
 *                       max E log sigma(beta log pi(y+)/pi_init(y+) - beta log pi(y-)/pi_init(y-)))
 *                     as a mean over pairs of -log sigma(z) (reading R3), and its exact
 *                     gradient w.r.t. the logits, dL/dx = coef_b (softmax - onehot).
 *   orc_pg_loss_fwd_bwd
 *                     the coefficient-variant losses of App B on the same
 *                     token log-probs: RLOO with k = 2, CoPG
 *                     (PAPER.md:716-719), Proximal RLOO and the Best-of-2
 *                     SFT baseline; see that function's comment.
 *   orc_seq_ppl       the KL proxy of PAPER.md:121 (Sec 3) / PAPER.md:333 (Sec 5.2): the
 *                     reference model's per-completion perplexity exp(-S_b / n_b).
 *   orc_online_dpo_loss_fwd_bwd_unscaled
 *                     the same, with the gradient returned factored per row:
 *                     G = softmax - onehot and row_scale = coef_b (dL/dx = row_scale * G).
 *
 * Every step follows the plain definition: y = x * invT; m = max_v y_v;
 * s = sum_v exp(y_v - m) (sequential); logp = (y_tok - m) - log(s); S_b = sum_t logp
 * over mask=1 tokens in t order; z = beta((S_c - ref_c) - (S_r - ref_r));
 * loss_p = softplus(-z); coef_c = beta sigma(-z) invT / P_global, coef_r = -coef_c;
 * g_v = coef_b (exp(y_v - lse) - [v == tok]).
 *
 * Threads (n_threads) only split independent sequences / rows; every sequence and
 * every row is computed by one thread in the fixed order above, and the statistics
 * are summed afterwards in pair order, so results are identical for any n_threads.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* input dtypes (same numeric values as the product header; F64 is oracle-only) */
enum { ORC_F32 = 0, ORC_BF16 = 1, ORC_F64 = 2 };
/* data-dependent status bits */
enum {
  ORC_FLAG_TOKEN_RANGE = 1,
  ORC_FLAG_NONFINITE_LOGIT = 2,
  ORC_FLAG_EMPTY_SEQ = 4,
  ORC_FLAG_NONFINITE_REWARD = 8,
  ORC_FLAG_DUP_ROW = 16,
  ORC_FLAG_DEGENERATE_PAIR = 32,
  ORC_FLAG_PAIR_RANGE = 64
};
/* loss statistics */
enum {
  ORC_ST_NPAIRS = 0, ORC_ST_LOSS, ORC_ST_NCORRECT, ORC_ST_Z, ORC_ST_RCHOSEN, ORC_ST_RREJ,
  ORC_ST_SCHOSEN, ORC_ST_SREJ, ORC_ST_NTOK_CHOSEN, ORC_ST_NTOK_REJ, ORC_NSTATS
};
/* selection statistics */
enum { ORC_SEL_MARGIN_SUM = 0, ORC_SEL_NDEGEN, ORC_SEL_NTRUNC, ORC_SEL_NSTATS };

static double load_x(const void* base, int dtype, int64_t off) {
  if (dtype == ORC_F32) return (double)((const float*)base)[off];
  if (dtype == ORC_F64) return ((const double*)base)[off];
  /* bf16: the 16 stored bits are the high half of an IEEE float */
  uint32_t bits = (uint32_t)((const uint16_t*)base)[off] << 16;
  float f;
  memcpy(&f, &bits, sizeof f);
  return (double)f;
}

/* ------------------------------------------------------------------ pair_select */
int orc_pair_select(const float* rewards, const uint8_t* has_eos, float eos_penalty, int64_t P,
                    int32_t K, int32_t* chosen, int32_t* rejected, int32_t* pair_rows,
                    float* margin, double* sel_stats, uint32_t* status) {
  if (!rewards || !chosen || !rejected || P < 0 || K < 2) return 1;
  uint32_t st = 0;
  double msum = 0.0, ndeg = 0.0, ntrunc = 0.0;
  float* r = (float*)malloc(sizeof(float) * (size_t)K);
  if (!r) return 1;
  for (int64_t p = 0; p < P; ++p) {
    /* 1. shaped reward: the EOS penalty REPLACES the score (reading R7) */
    for (int32_t k = 0; k < K; ++k) {
      int eos = has_eos ? has_eos[p * K + k] != 0 : 1;
      r[k] = eos ? rewards[p * K + k] : eos_penalty;
      if (!eos) ntrunc += 1.0;
      if (!isfinite(r[k])) st |= ORC_FLAG_NONFINITE_REWARD;
    }
    /* 2. chosen = FIRST index attaining the max, rejected = LAST index attaining the min
          (reading R5), using only strict comparisons */
    int32_t best = 0;
    for (int32_t k = 1; k < K; ++k)
      if (r[k] > r[best]) best = k;
    int32_t worst = K - 1;
    for (int32_t k = K - 2; k >= 0; --k)
      if (r[k] < r[worst]) worst = k;
    /* 3. reward margin max - min: one fp32 subtraction */
    float mx = r[best], mn = r[worst];
    float mg = mx - mn;
    if (mx == mn) { st |= ORC_FLAG_DEGENERATE_PAIR; ndeg += 1.0; }
    chosen[p] = best;
    rejected[p] = worst;
    if (pair_rows) {
      pair_rows[2 * p] = (int32_t)(p * K + best);
      pair_rows[2 * p + 1] = (int32_t)(p * K + worst);
    }
    if (margin) margin[p] = mg;
    msum += (double)mg;
  }
  free(r);
  if (sel_stats) {
    sel_stats[ORC_SEL_MARGIN_SUM] = msum;
    sel_stats[ORC_SEL_NDEGEN] = ndeg;
    sel_stats[ORC_SEL_NTRUNC] = ntrunc;
  }
  if (status) *status |= st;
  return 0;
}

/* ------------------------------------------------------------- per-row log-softmax */
typedef struct {
  const void* logits;
  int dtype;
  int64_t B, T, V, sb, stt;
  const int32_t* tokens;
  const uint8_t* mask;
  double invT;
} rows_in;

/* log-softmax of one row at the sampled token; returns 0 on success and fills lse */
static int row_logp(const rows_in* in, int64_t b, int64_t t, double* logp, double* lse,
                    uint32_t* st) {
  int64_t V = in->V;
  int64_t base = b * in->sb + t * in->stt;
  int32_t tok = in->tokens[b * in->T + t];
  double m = -INFINITY;
  for (int64_t v = 0; v < V; ++v) {
    double x = load_x(in->logits, in->dtype, base + v);
    /* reading R14: NaN and +inf are errors; -inf is a legal "impossible token" logit */
    if (isnan(x) || x == INFINITY) *st |= ORC_FLAG_NONFINITE_LOGIT;
    double y = x * in->invT;
    if (y > m) m = y;
  }
  double s = 0.0;
  for (int64_t v = 0; v < V; ++v) s += exp(load_x(in->logits, in->dtype, base + v) * in->invT - m);
  *lse = m + log(s);
  if (tok < 0 || tok >= V) {
    *st |= ORC_FLAG_TOKEN_RANGE;
    *logp = 0.0;
    return 1;
  }
  double ytok = load_x(in->logits, in->dtype, base + tok) * in->invT;
  *logp = (ytok - m) - log(s);
  /* ... but an all -inf row, or a -inf sampled logit, has no finite log-prob (R14) */
  if (!isfinite(m) || !isfinite(*logp)) *st |= ORC_FLAG_NONFINITE_LOGIT;
  return 0;
}

typedef struct {
  const rows_in* in;
  int64_t b0, b1;
  double* S;       /* [B] */
  double* ntok;    /* [B] */
  double* tok_logp;
  double* row_lse;
  uint32_t st;
} seq_job;

static void* seq_worker(void* arg) {
  seq_job* j = (seq_job*)arg;
  const rows_in* in = j->in;
  for (int64_t b = j->b0; b < j->b1; ++b) {
    double S = 0.0, n = 0.0;
    for (int64_t t = 0; t < in->T; ++t) {
      int64_t g = b * in->T + t;
      if (!in->mask[g]) {
        if (j->tok_logp) j->tok_logp[g] = 0.0;
        if (j->row_lse) j->row_lse[g] = 0.0;
        continue;
      }
      double lp, lse;
      row_logp(in, b, t, &lp, &lse, &j->st);
      if (j->tok_logp) j->tok_logp[g] = lp;
      if (j->row_lse) j->row_lse[g] = lse;
      S += lp;
      n += 1.0;
    }
    if (n == 0.0) j->st |= ORC_FLAG_EMPTY_SEQ;
    j->S[b] = S;
    if (j->ntok) j->ntok[b] = n;
  }
  return NULL;
}

static uint32_t run_seqs(const rows_in* in, double* S, double* ntok, double* tok_logp,
                         double* row_lse, int n_threads) {
  if (n_threads < 1) n_threads = 1;
  if (n_threads > in->B) n_threads = (int)(in->B > 0 ? in->B : 1);
  seq_job* jobs = (seq_job*)calloc((size_t)n_threads, sizeof(seq_job));
  pthread_t* th = (pthread_t*)calloc((size_t)n_threads, sizeof(pthread_t));
  for (int i = 0; i < n_threads; ++i) {
    jobs[i].in = in;
    jobs[i].b0 = in->B * i / n_threads;
    jobs[i].b1 = in->B * (i + 1) / n_threads;
    jobs[i].S = S;
    jobs[i].ntok = ntok;
    jobs[i].tok_logp = tok_logp;
    jobs[i].row_lse = row_lse;
    jobs[i].st = 0;
  }
  if (n_threads == 1) {
    seq_worker(&jobs[0]);
  } else {
    for (int i = 0; i < n_threads; ++i) pthread_create(&th[i], NULL, seq_worker, &jobs[i]);
    for (int i = 0; i < n_threads; ++i) pthread_join(th[i], NULL);
  }
  uint32_t st = 0;
  for (int i = 0; i < n_threads; ++i) st |= jobs[i].st;
  free(jobs);
  free(th);
  return st;
}

/* -------------------------------------------------------------------- seq_logprobs */
int orc_seq_logprobs(const void* logits, int dtype, int64_t B, int64_t T, int64_t V,
                     int64_t stride_b, int64_t stride_t, const int32_t* tokens,
                     const uint8_t* mask, float inv_temperature, double* seq_logp,
                     double* tok_logp, double* row_lse, uint32_t* status, int n_threads) {
  if (!logits || !tokens || !mask || !seq_logp || B <= 0 || T <= 0 || V <= 0) return 1;
  rows_in in = {logits, dtype, B, T, V, stride_b, stride_t, tokens, mask, (double)inv_temperature};
  uint32_t st = run_seqs(&in, seq_logp, NULL, tok_logp, row_lse, n_threads);
  if (status) *status |= st;
  return 0;
}

/* ------------------------------------------------------------------ KL proxy (PPL)
 * PAPER.md:121 (Sec 3, Evaluation: "we measure the SFT model's perplexity on the RLHF
 * policy's summaries") and PAPER.md:333 (Sec 5.2, "Final KL is measured using the perplexity
 * of the base model on the generated completions"), read per completion (R20):
 *   ppl_b = exp(-S_b / n_b),  S_b = orc_seq_logprobs' log pi_ref(y_b|x),  n_b = #mask tokens.
 * An empty completion (n_b = 0, flagged EMPTY_SEQ) gets ppl_b = 1 and is left out of
 * ppl_stats = {#completions with n_b > 0, sum_b ppl_b, sum_b S_b, sum_b n_b}
 * (the corpus perplexity is exp(-ppl_stats[2] / ppl_stats[3])). */
int orc_seq_ppl(const void* logits, int dtype, int64_t B, int64_t T, int64_t V, int64_t stride_b,
                int64_t stride_t, const int32_t* tokens, const uint8_t* mask,
                float inv_temperature, double* seq_logp, double* ppl, double* ppl_stats,
                uint32_t* status, int n_threads) {
  if (!logits || !tokens || !mask || !seq_logp || !ppl || B <= 0 || T <= 0 || V <= 0) return 1;
  rows_in in = {logits, dtype, B, T, V, stride_b, stride_t, tokens, mask, (double)inv_temperature};
  double* ntok = (double*)calloc((size_t)B, sizeof(double));
  uint32_t st = run_seqs(&in, seq_logp, ntok, NULL, NULL, n_threads);
  double nseq = 0.0, sp = 0.0, sS = 0.0, sn = 0.0;
  for (int64_t b = 0; b < B; ++b) {
    if (ntok[b] > 0.0) {
      ppl[b] = exp(-seq_logp[b] / ntok[b]);
      nseq += 1.0;
      sp += ppl[b];
      sS += seq_logp[b];
      sn += ntok[b];
    } else {
      ppl[b] = 1.0;
    }
  }
  if (ppl_stats) {
    ppl_stats[0] = nseq;
    ppl_stats[1] = sp;
    ppl_stats[2] = sS;
    ppl_stats[3] = sn;
  }
  free(ntok);
  if (status) *status |= st;
  return 0;
}

/* --------------------------------------------------------- online_dpo_loss_fwd_bwd */
typedef struct {
  const rows_in* in;
  const double* coef;   /* [B] */
  const uint8_t* refd;  /* [B] referenced by a pair */
  const int64_t* rows;  /* rows to emit (NULL = all) */
  int64_t n0, n1;
  int unscaled;         /* emit G = softmax - onehot (without coef_b) */
  double* out;          /* [n][V] */
} grad_job;

static void* grad_worker(void* arg) {
  grad_job* j = (grad_job*)arg;
  const rows_in* in = j->in;
  int64_t V = in->V;
  for (int64_t i = j->n0; i < j->n1; ++i) {
    int64_t g = j->rows ? j->rows[i] : i;
    int64_t b = g / in->T, t = g % in->T;
    double* o = j->out + i * V;
    if (!j->refd[b] || !in->mask[g]) {
      for (int64_t v = 0; v < V; ++v) o[v] = 0.0;
      continue;
    }
    double lp, lse;
    uint32_t st = 0;
    row_logp(in, b, t, &lp, &lse, &st);
    int32_t tok = in->tokens[g];
    int64_t base = b * in->sb + t * in->stt;
    for (int64_t v = 0; v < V; ++v) {
      double y = load_x(in->logits, in->dtype, base + v) * in->invT;
      double gv = exp(y - lse) - (v == tok ? 1.0 : 0.0);
      o[v] = j->unscaled ? gv : j->coef[b] * gv;
    }
  }
  return NULL;
}

static int loss_core(const void* logits, int dtype, int64_t B, int64_t T, int64_t V,
                     int64_t stride_b, int64_t stride_t, const float* ref_logp,
                     const int32_t* tokens, const uint8_t* mask, const int32_t* pair_rows,
                     int64_t P, int64_t P_global, float beta, float inv_temperature,
                     double* dlogits, const int64_t* dl_rows, int64_t n_dl_rows,
                     double* seq_logp, double* z_out, double* stats, uint32_t* status,
                     int n_threads, int unscaled, double* row_scale) {
  if (!logits || !ref_logp || !tokens || !mask || !seq_logp || !stats) return 1;
  if (B <= 0 || T <= 0 || V <= 0 || P <= 0 || P_global < P) return 1;
  if (!pair_rows && B != 2 * P) return 1;
  rows_in in = {logits, dtype, B, T, V, stride_b, stride_t, tokens, mask, (double)inv_temperature};
  double* ntok = (double*)calloc((size_t)B, sizeof(double));
  double* coef = (double*)calloc((size_t)B, sizeof(double));
  uint8_t* refd = (uint8_t*)calloc((size_t)B, 1);
  uint32_t st = run_seqs(&in, seq_logp, ntok, NULL, NULL, n_threads);

  double beta_d = (double)beta, invT = (double)inv_temperature, Pg = (double)P_global;
  double acc[ORC_NSTATS];
  for (int i = 0; i < ORC_NSTATS; ++i) acc[i] = 0.0;
  for (int64_t p = 0; p < P; ++p) {
    int64_t c = pair_rows ? pair_rows[2 * p] : 2 * p;
    int64_t r = pair_rows ? pair_rows[2 * p + 1] : 2 * p + 1;
    if (c < 0 || c >= B || r < 0 || r >= B) {
      st |= ORC_FLAG_PAIR_RANGE;
      if (z_out) z_out[p] = 0.0;
      continue;
    }
    if (c == r || refd[c] || refd[r]) st |= ORC_FLAG_DUP_ROW;
    refd[c] = 1;
    refd[r] = 1;
    double dc = seq_logp[c] - (double)ref_logp[c];
    double dr = seq_logp[r] - (double)ref_logp[r];
    double z = beta_d * (dc - dr);
    double loss_p = fmax(-z, 0.0) + log1p(exp(-fabs(z)));  /* softplus(-z) = -log sigma(z) */
    double sig_neg = 1.0 / (1.0 + exp(z));                 /* sigma(-z) */
    acc[ORC_ST_NPAIRS] += 1.0;
    acc[ORC_ST_LOSS] += loss_p;
    acc[ORC_ST_NCORRECT] += (z > 0.0) ? 1.0 : 0.0;
    acc[ORC_ST_Z] += z;
    acc[ORC_ST_RCHOSEN] += beta_d * dc;
    acc[ORC_ST_RREJ] += beta_d * dr;
    acc[ORC_ST_SCHOSEN] += seq_logp[c];
    acc[ORC_ST_SREJ] += seq_logp[r];
    acc[ORC_ST_NTOK_CHOSEN] += ntok[c];
    acc[ORC_ST_NTOK_REJ] += ntok[r];
    coef[c] = beta_d * sig_neg * invT / Pg;
    coef[r] = -coef[c];
    if (z_out) z_out[p] = z;
  }
  acc[ORC_ST_LOSS] /= Pg;
  for (int i = 0; i < ORC_NSTATS; ++i) stats[i] = acc[i];

  if (dlogits) {
    int64_t n = dl_rows ? n_dl_rows : B * T;
    int nt = n_threads < 1 ? 1 : n_threads;
    if (nt > n) nt = (int)(n > 0 ? n : 1);
    grad_job* jobs = (grad_job*)calloc((size_t)nt, sizeof(grad_job));
    pthread_t* th = (pthread_t*)calloc((size_t)nt, sizeof(pthread_t));
    for (int i = 0; i < nt; ++i) {
      jobs[i].in = &in;
      jobs[i].coef = coef;
      jobs[i].refd = refd;
      jobs[i].rows = dl_rows;
      jobs[i].n0 = n * i / nt;
      jobs[i].n1 = n * (i + 1) / nt;
      jobs[i].unscaled = unscaled;
      jobs[i].out = dlogits;
    }
    if (nt == 1) {
      grad_worker(&jobs[0]);
    } else {
      for (int i = 0; i < nt; ++i) pthread_create(&th[i], NULL, grad_worker, &jobs[i]);
      for (int i = 0; i < nt; ++i) pthread_join(th[i], NULL);
    }
    free(jobs);
    free(th);
  }
  if (row_scale) {
    /* dlogits[b,t,:] = row_scale[b,t] * G[b,t,:] */
    for (int64_t g = 0; g < B * T; ++g) {
      int64_t b = g / T;
      row_scale[g] = (refd[b] && mask[g]) ? coef[b] : 0.0;
    }
  }
  free(ntok);
  free(coef);
  free(refd);
  if (status) *status |= st;
  return 0;
}

int orc_online_dpo_loss_fwd_bwd(const void* logits, int dtype, int64_t B, int64_t T, int64_t V,
                                int64_t stride_b, int64_t stride_t, const float* ref_logp,
                                const int32_t* tokens, const uint8_t* mask,
                                const int32_t* pair_rows, int64_t P, int64_t P_global,
                                float beta, float inv_temperature, double* dlogits,
                                const int64_t* dl_rows, int64_t n_dl_rows, double* seq_logp,
                                double* z_out, double* stats, uint32_t* status, int n_threads) {
  return loss_core(logits, dtype, B, T, V, stride_b, stride_t, ref_logp, tokens, mask, pair_rows,
                   P, P_global, beta, inv_temperature, dlogits, dl_rows, n_dl_rows, seq_logp,
                   z_out, stats, status, n_threads, 0, NULL);
}

/* The same loss with the gradient factored per row (performance tier):
   G[b,t,:] = mask[b,t] * [b referenced] * (softmax(invT x) - onehot(tok)) and
   row_scale[b,t] = mask[b,t] * [b referenced] * coef_b, so dL/dx = row_scale * G. */
int orc_online_dpo_loss_fwd_bwd_unscaled(const void* logits, int dtype, int64_t B, int64_t T,
                                         int64_t V, int64_t stride_b, int64_t stride_t,
                                         const float* ref_logp, const int32_t* tokens,
                                         const uint8_t* mask, const int32_t* pair_rows, int64_t P,
                                         int64_t P_global, float beta, float inv_temperature,
                                         double* G, const int64_t* g_rows, int64_t n_g_rows,
                                         double* row_scale, double* seq_logp, double* z_out,
                                         double* stats, uint32_t* status, int n_threads) {
  return loss_core(logits, dtype, B, T, V, stride_b, stride_t, ref_logp, tokens, mask, pair_rows,
                   P, P_global, beta, inv_temperature, G, g_rows, n_g_rows, seq_logp, z_out,
                   stats, status, n_threads, 1, row_scale);
}

/* ----------------------------------------------------------- coefficient-variant losses
 * Each pair p = (y1, y2) = pair_rows[p] with per-sequence rewards R and advantages
 * A1 = R1 - R2, A2 = R2 - R1 (k = 2).  Losses are MINIMISED, as the negated
 * objectives, averaged over P_global pairs:
 *   kind 0 RLOO       l_p = -1/2 [S1 A1 + S2 A2]                       (
 *                     reading: each sample carries its own leave-one-out advantage)
 *   kind 1 CoPG       l_p = -1/2 [(S1 - O1) A1 + (S2 - O2) A2]
 *   kind 2 Prox RLOO  l_p = -1/2 [min(r1 A1, clip(r1) A1) + min(r2 A2, clip(r2) A2)],
 *                     r = exp(S - O), clip to [1 - eps, 1 + eps]
 *   kind 3 Best-of-2 SFT  l_p = -S1 (y1 = the chosen completion)
 * with S = log pi_theta(y|x) (R1) and O = log pi_old(y|x) (old_logp).  The gradient is
 * dl/dx = coef_b (softmax(invT x) - onehot), coef_b = -(dL/dS_b) invT:
 *   RLOO, CoPG: coef_b = A_b invT / (2 P_global)
 *   Prox: coef_b = r_b A_b invT / (2 P_global) where min() takes the unclipped term
 *         (r A <= clip(r) A), else 0
 *   SFT: coef_1 = invT / P_global, coef_2 = 0.
 * stats[10]: pairs, mean loss, sequences with a nonzero coefficient, sum r (Prox only),
 * sum A1, sum |A1|, sum S1, sum S2, tokens of y1, tokens of y2. */
int orc_pg_loss_fwd_bwd(const void* logits, int dtype, int64_t B, int64_t T, int64_t V,
                        int64_t stride_b, int64_t stride_t, const int32_t* tokens,
                        const uint8_t* mask, const int32_t* pair_rows, int64_t P,
                        int64_t P_global, int kind, const float* rewards,
                        const float* old_logp, float clip_eps, float inv_temperature,
                        double* dlogits, const int64_t* dl_rows, int64_t n_dl_rows,
                        double* seq_logp, double* stats, uint32_t* status, int n_threads) {
  if (!logits || !tokens || !mask || !seq_logp || !stats || !rewards) return 1;
  if (B <= 0 || T <= 0 || V <= 0 || P <= 0 || P_global < P || kind < 0 || kind > 3) return 1;
  if ((kind == 1 || kind == 2) && !old_logp) return 1;
  if (!pair_rows && B != 2 * P) return 1;
  rows_in in = {logits, dtype, B, T, V, stride_b, stride_t, tokens, mask, (double)inv_temperature};
  double* ntok = (double*)calloc((size_t)B, sizeof(double));
  double* coef = (double*)calloc((size_t)B, sizeof(double));
  uint8_t* refd = (uint8_t*)calloc((size_t)B, 1);
  uint32_t st = run_seqs(&in, seq_logp, ntok, NULL, NULL, n_threads);
  double invT = (double)inv_temperature, Pg = (double)P_global, eps = (double)clip_eps;
  double acc[ORC_NSTATS];
  for (int i = 0; i < ORC_NSTATS; ++i) acc[i] = 0.0;
  for (int64_t p = 0; p < P; ++p) {
    int64_t y[2];
    y[0] = pair_rows ? pair_rows[2 * p] : 2 * p;
    y[1] = pair_rows ? pair_rows[2 * p + 1] : 2 * p + 1;
    if (y[0] < 0 || y[0] >= B || y[1] < 0 || y[1] >= B) {
      st |= ORC_FLAG_PAIR_RANGE;
      continue;
    }
    if (y[0] == y[1] || refd[y[0]] || refd[y[1]]) st |= ORC_FLAG_DUP_ROW;
    refd[y[0]] = refd[y[1]] = 1;
    double A[2], loss = 0.0;
    A[0] = (double)rewards[y[0]] - (double)rewards[y[1]];
    A[1] = -A[0];
    for (int k = 0; k < 2; ++k) {
      int64_t b = y[k];
      double S = seq_logp[b];
      double c = 0.0;
      if (kind == 0) {
        loss += -0.5 * S * A[k];
        c = A[k] * invT / (2.0 * Pg);
      } else if (kind == 1) {
        loss += -0.5 * (S - (double)old_logp[b]) * A[k];
        c = A[k] * invT / (2.0 * Pg);
      } else if (kind == 2) {
        double r = exp(S - (double)old_logp[b]);
        double rc = r < 1.0 - eps ? 1.0 - eps : (r > 1.0 + eps ? 1.0 + eps : r);
        double u = r * A[k], v = rc * A[k];
        loss += -0.5 * (u <= v ? u : v);
        c = (u <= v) ? r * A[k] * invT / (2.0 * Pg) : 0.0;
        acc[ORC_ST_Z] += r;
      } else {
        if (k == 0) {
          loss += -S;
          c = invT / Pg;
        }
      }
      coef[b] = c;
      if (c != 0.0) acc[ORC_ST_NCORRECT] += 1.0;
    }
    acc[ORC_ST_NPAIRS] += 1.0;
    acc[ORC_ST_LOSS] += loss;
    acc[ORC_ST_RCHOSEN] += A[0];
    acc[ORC_ST_RREJ] += fabs(A[0]);
    acc[ORC_ST_SCHOSEN] += seq_logp[y[0]];
    acc[ORC_ST_SREJ] += seq_logp[y[1]];
    acc[ORC_ST_NTOK_CHOSEN] += ntok[y[0]];
    acc[ORC_ST_NTOK_REJ] += ntok[y[1]];
  }
  acc[ORC_ST_LOSS] /= Pg;
  for (int i = 0; i < ORC_NSTATS; ++i) stats[i] = acc[i];
  if (dlogits) {
    int64_t n = dl_rows ? n_dl_rows : B * T;
    int nt = n_threads < 1 ? 1 : n_threads;
    if (nt > n) nt = (int)(n > 0 ? n : 1);
    grad_job* jobs = (grad_job*)calloc((size_t)nt, sizeof(grad_job));
    pthread_t* th = (pthread_t*)calloc((size_t)nt, sizeof(pthread_t));
    for (int i = 0; i < nt; ++i) {
      jobs[i].in = &in;
      jobs[i].coef = coef;
      jobs[i].refd = refd;
      jobs[i].rows = dl_rows;
      jobs[i].n0 = n * i / nt;
      jobs[i].n1 = n * (i + 1) / nt;
      jobs[i].unscaled = 0;
      jobs[i].out = dlogits;
    }
    if (nt == 1) {
      grad_worker(&jobs[0]);
    } else {
      for (int i = 0; i < nt; ++i) pthread_create(&th[i], NULL, grad_worker, &jobs[i]);
      for (int i = 0; i < nt; ++i) pthread_join(th[i], NULL);
    }
    free(jobs);
    free(th);
  }
  free(ntok);
  free(coef);
  free(refd);
  if (status) *status |= st;
  return 0;
}
