/* tepai_b200 — C ABI of the B200 (sm_100a) MPS TE-PAI ensemble engine.
 *
 * Plain pointers and sizes only (no torch / CUDA types in the signatures).
 * complex128 buffers are interleaved (re, im) doubles, C-contiguous.
 *
 * Reference interfaces replaced (file:line in /root/reference/pkg/src/tepai):
 *   tb_run_stream     <- _kernel.run_stream(buf, dims, center, ga, gb, pa, pb,
 *                        ang, anchors, chi_cut, floor, counters) -> center
 *                        (_kernel.py:184-215; called from mps._run_lowered,
 *                        mps.py:239-258)
 *   tb_expectation    <- mps.expectation(state, pauli) (mps.py:170-182)
 *   tb_run_ensemble   <- the sample loop of SPEC.md:487-490 + estimator
 *                        accumulation SPEC.md:419-423 (absent in the code;
 *                        SURVEY.md §3.A): run_circuit per checkpoint segment
 *                        (mps.py:276-288) + expectation of Z_j + signed sums
 *   tb_svd            <- the np.linalg.svd(mat, False) call inside
 *                        _split_theta (_kernel.py:117), exposed for unit tests
 *   tb_svd_trunc      <- the same call as consumed by the truncation rule
 *                        (_kernel.py:117-131): only the kept triplets exact
 *
 * Return codes: 0 ok, negative on error; tb_last_error() gives the message.
 */
#ifndef TEPAI_B200_H
#define TEPAI_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TB_OK 0
#define TB_EINVAL (-1)
#define TB_ECUDA (-2)
#define TB_ENOMEM (-3)
#define TB_ENOCONV (-4)

typedef struct tb_ctx tb_ctx;

/* Gate word of the packed stream (one uint32 per applied rotation):
 *   bits  0-7   site a (first support site)
 *   bits  8-15  site b, or 0xFF for a one-site rotation
 *   bits 16-17  Pauli code on a (X=1, Y=2, Z=3)
 *   bits 18-19  Pauli code on b
 *   bit  20     merge_right look-ahead for adjacent two-site gates
 *               (anchors[i] > a, mps.py:219-228 / _kernel.py:202)
 *   bit  21     angle is exactly pi (local Pauli product when pi_local)
 *   bits 22-31  index into the angle table (cos(angle/2), sin(angle/2)) */
#define TB_ONE_SITE 0xFFu

int tb_version(void);
int tb_create(int device, tb_ctx** out);
void tb_destroy(tb_ctx* ctx);
const char* tb_last_error(const tb_ctx* ctx);
/* Number of SMs of the bound device (persistent-grid size). */
int tb_num_sms(const tb_ctx* ctx);
/* Persistent CTAs that run circuits of bond capacity `cap` concurrently:
 * tb_num_sms() for cap > 32; twice that for cap <= 32, where the
 * small-problem engine keeps two circuits resident per SM (TB_SMALL_ENGINE=0
 * disables it).  Size slot pools as a multiple of this. */
int tb_num_ctas(const tb_ctx* ctx, int64_t cap);
/* Read and clear the context's sticky device status word (device-buffer
 * calls do not synchronize, so they report through it): bit 0 = a Jacobi SVD
 * did not converge, bit 2 = a slot was continued (reset = 0) although its
 * state belongs to an older workspace generation. */
int tb_take_status(tb_ctx* ctx, int32_t* status);
/* Diagnostics (collected only when the context was created with TB_PROFILE=1
 * in the environment): clock64 phase counters of the last ensemble launch, summed over
 * CTAs: [0] Jacobi cycles [1] Jacobi calls [2] sweeps [3] centre moves
 * [4] contraction+gate [5] sort+split write-back [6] <Z> sweeps
 * [7] per-sample totals [9..11] cycles/calls/sweeps of 128x128 problems,
 * [16+k] rotations applied in sweep k.  out must hold 64 entries. */
int tb_debug_profile(tb_ctx* ctx, uint64_t* out64);

/* Drop-in for _kernel.run_stream: executes the lowered stream on one MPS.
 * buf: complex128 [n][cap][2][cap] (mutated); dims: int64 [n+1] (mutated);
 * ga/gb/pa/pb/anchors: int64 [n_gates]; ang: float64 [n_gates];
 * counters: float64[4] = {gates, sum k^3, chi_max, discarded}, accumulated
 * exactly like the reference (slot 2 is a running max). */
int tb_run_stream(tb_ctx* ctx, double* buf, int64_t n, int64_t cap, int64_t* dims, int64_t center,
                  const int64_t* ga, const int64_t* gb, const int64_t* pa, const int64_t* pb,
                  const double* ang, const int64_t* anchors, int64_t n_gates, int64_t chi_cut,
                  double svalue_floor, double* counters, int64_t* new_center);

/* <psi|P|psi> by left-to-right transfer contraction; codes: int32 [n], 0=I. */
int tb_expectation(tb_ctx* ctx, const double* buf, int64_t n, int64_t cap, const int64_t* dims,
                   const int32_t* pauli_codes, double* out);

/* Batched <psi_s|P_o|psi_s> for S states and O Pauli strings (transfer
 * contraction as mps.expectation, mps.py:170-182): the one-pass evaluation of
 * a signed mixture's observables (evaluate_observables).
 * bufs: complex128 [S][n][cap][2][cap]; dims: int64 [S][n+1];
 * codes: int32 [O][n] (0=I, 1=X, 2=Y, 3=Z); out: float64 [S][O]. */
int tb_expectation_batch(tb_ctx* ctx, const double* bufs, int64_t n_states, int64_t n, int64_t cap,
                         const int64_t* dims, const int32_t* codes, int64_t n_obs, double* out);

/* Batched thin SVD (unit-test surface of the Jacobi kernel).
 * a: complex128 [batch][m][n] row-major; s: [batch][k]; u: [batch][m][k];
 * vh: [batch][k][n] with k = min(m, n).  Any of u / vh may be NULL. */
int tb_svd(tb_ctx* ctx, const double* a, int64_t batch, int64_t m, int64_t n, double* s, double* u,
           double* vh);

/* Truncated variant: only the kcut largest triplets are needed (the split
 * keeps k <= min(chi_cut, K), _kernel.py:118-131).  s[:kcut], u[:, :kcut] and
 * vh[:kcut] are those of the full SVD, and sum(s^2) is still |a|_F^2; the
 * tail entries are an orthogonal complement that need not be diagonal.
 * kcut <= 0 or >= min(m, n) is the full SVD. */
int tb_svd_trunc(tb_ctx* ctx, const double* a, int64_t batch, int64_t m, int64_t n, int64_t kcut, double* s,
                 double* u, double* vh);

typedef struct tb_ensemble_desc {
  int32_t n;           /* sites */
  int32_t cap;         /* bond capacity = min(chi_cut, 2^(n//2)) (mps.py:187-191) */
  int32_t chi_cut;     /* effective cut (<= cap) */
  int32_t pi_local;    /* 1: pi-angle two-site gates as local Pauli products */
  double svalue_floor; /* relative singular-value floor (_kernel.py:121) */
  int32_t n_samples;
  int32_t n_ckpt;
  int32_t n_obs;
  int32_t n_angles;
  const uint32_t* gates;        /* all samples' packed streams, concatenated */
  const int64_t* gate_offsets;  /* [n_samples+1] */
  const int32_t* ckpt_gate_end; /* [n_samples][n_ckpt] stream position of checkpoint c */
  const int8_t* ckpt_sign;      /* [n_samples][n_ckpt] sign(g) of the prefix, +-1 */
  const double* angle_cs;       /* [n_angles][2] cos(angle/2), sin(angle/2) */
  const double* ckpt_weight;    /* [n_ckpt] ||g||_1 of each prefix (informational) */
  const int32_t* obs_sites;     /* [n_obs] sites j of the <Z_j> observables */
  const double* init_vecs;      /* [n][2] complex128 product-state site vectors */
  /* optional start MPS shared by every sample (hybrid Trotter -> TE-PAI fan-out,
   * SPEC.md:487-495 / mps.py:296-338 snapshots); NULL = product state */
  const double* init_mps;       /* complex128 [n][cap][2][cap] */
  const int32_t* init_dims;     /* [n+1] */
  int32_t init_center;
  int32_t reserved;
} tb_ensemble_desc;

typedef struct tb_ensemble_out {
  double* values;     /* [n_samples][n_ckpt][n_obs] raw <Z_j>, or NULL */
  double* discarded;  /* [n_samples][n_ckpt] cumulative discarded weight, or NULL */
  double* ledger;     /* [n_samples][4] gates, sum k^3, chi_max, discarded, or NULL */
  int64_t* sum_v;     /* [n_ckpt][n_obs] += round(2^40 * sign * <Z>) (accumulated) */
  int64_t* sum_v2;    /* [n_ckpt][n_obs] += round(2^40 * <Z>^2) (accumulated) */
  double* flops;      /* [1] += algorithmic FLOPs (SURVEY.md §8(d) count) */
  float* kernel_ms;   /* [1] device time of the persistent kernel (CUDA events) */
  /* [n_samples] per-sample failure report, or NULL.  A sample whose circuit
   * hits a Jacobi SVD that does not converge (the reference would raise
   * LinAlgError from LAPACK, _kernel.py:117) keeps its raw values, but its
   * checkpoints from that one on are left out of sum_v / sum_v2; excluded[s]
   * is the first such checkpoint, -1 when every checkpoint contributed.  With
   * this array the launch succeeds and the caller drops those rows from its
   * counts; without it the call returns TB_ENOCONV and (host-buffer calls)
   * leaves every caller array untouched.  Device calls: the caller fills it
   * with -1 before the launch. */
  int32_t* excluded;
  /* Optional per-sample final states for the signed mixture:
   * complex128 [n_samples][n][cap][2][cap] (zero-padded), bond dims
   * [n_samples][n+1] and centres [n_samples]; NULL = not retained. */
  double* states;
  int32_t* state_dims;
  int32_t* state_center;
  /* [n_samples] device time (ms) of each sample (queue mode) or of its segment
   * (slot mode): the measured C_circ of the cost report. */
  double* sample_ms;
} tb_ensemble_out;

/* Host-buffer ensemble run: uploads the streams, runs the persistent kernel,
 * downloads results (the end-to-end call). */
int tb_run_ensemble(tb_ctx* ctx, const tb_ensemble_desc* desc, tb_ensemble_out* out);

/* Device-resident variant: every pointer in desc/out is a device pointer
 * (kernel_ms may be a host pointer or NULL); runs on `stream` (cudaStream_t,
 * NULL = legacy default) and does not synchronize unless kernel_ms != NULL. */
int tb_run_ensemble_device(tb_ctx* ctx, const tb_ensemble_desc* desc, tb_ensemble_out* out, void* stream);

/* Continuous batching ("slots"): every slot keeps its MPS resident in HBM
 * between calls.  Each call advances every slot by its own gate-stream
 * segment (base.gates / gate_offsets indexed by slot), optionally restarting
 * it from the product state first (reset[slot] = 1), measures <Z_j> at the
 * segment's checkpoints and adds the signed fixed-point values to estimator
 * row sum_row[slot][c].  The persistent CTAs (min(n_slots, tb_num_ctas()))
 * take slots from an atomic queue, in the order given by `order` (a
 * permutation of the slots, e.g. by decreasing predicted cost; NULL = slot
 * order), so more slots than SMs balance the per-segment work.  The first
 * call for a given (n, cap, n_slots) must reset every slot; any other engine
 * call on the same context (run_stream, run_ensemble, svd) invalidates the
 * slot states.  This is enforced: every slot state carries the workspace
 * generation it was built in, and continuing a slot of an older generation
 * fails the call with TB_EINVAL (status bit 2) instead of reading stale
 * memory.  Give each pipeline its own context to keep the pools apart. */
typedef struct tb_step_desc {
  tb_ensemble_desc base;
  const uint8_t* reset;    /* [n_slots] */
  const int32_t* sum_row;  /* [n_slots][n_ckpt] */
  const int32_t* order;    /* [n_slots] processing order, or NULL */
} tb_step_desc;

/* host buffers; sum_v/sum_v2 hold sum_rows x n_obs entries */
int tb_step(tb_ctx* ctx, const tb_step_desc* desc, tb_ensemble_out* out, int64_t sum_rows);
/* device buffers on `stream` */
int tb_step_device(tb_ctx* ctx, const tb_step_desc* desc, tb_ensemble_out* out, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* TEPAI_B200_H */
