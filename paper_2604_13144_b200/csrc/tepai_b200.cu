// tepai_b200.cu — B200 (sm_100a) MPS TE-PAI ensemble engine, complex128.
//
// One persistent CTA per SM owns one ensemble member (sample) at a time and
// runs that circuit's whole packed gate stream: centre moves (CGS2 QR), the
// two-site contraction with the Pauli-pair rotation or SWAP fused into the
// write-out, a one-sided (Hestenes) Jacobi SVD, the reference truncation rule
// with renormalisation, the split write-back, one-site rotations, local pi
// gates, and at every checkpoint the canonical-form <Z_j> sweep plus the
// fixed-point signed sums of the estimator.
//
// Reference semantics (file:line in /root/reference/pkg/src/tepai):
//   rotations _kernel.py:26-65, centre moves :68-102, one-site :105-111,
//   split/truncation :114-154, two-site/swap :157-181, driver :184-215,
//   lowering look-ahead mps.py:194-236, expectation mps.py:170-182,
//   estimator SPEC.md:404-470.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <string>
#include <vector>

#include "../../include/tepai_b200.h"

// launch parameters shared by both instantiations of the engine
namespace tbc {
struct Job {
  int n, cap, chi_cut, pi_local;
  int precond;  // QR-preconditioned Jacobi for problems >= 32 x 32
  int max_sweeps;  // Jacobi sweep cap (TB_MAX_SWEEPS, tests of the non-convergence path only)
  int inject;      // fault injection (TB_FAULT_INJECT=k): every Jacobi of samples with id % k == 0 reports non-convergence
  int tail_skip;  // skip pairs of discarded-tail columns (see mark_tail)
  int cluster;    // CTAs per thread-block cluster (8: wide Jacobi in distributed smem; 0: none)
  int cluster_tma;  // cluster Jacobi stages its blocks with TMA bulk copies
  int qrcp_tmem;  // QR preconditioner with the matrix in tensor memory (qrcp_tmem)
  int gram_screen;  // late Jacobi sweeps visit only the pairs flagged by the DMMA Gram screen (TB_GRAM_SCREEN)
  double floor;
  int n_samples, n_ckpt, n_obs;
  const uint32_t* gates;
  const int64_t* gate_off;
  const int32_t* ckpt_end;
  const int8_t* ckpt_sign;
  const double* angle_cs;
  const int32_t* obs_sites;
  const double* init_vecs;  // product-state site vectors [n][2] (complex)
  const double2* init_mps;  // optional start MPS [n][cap][2][cap] (hybrid fan-out)
  const int32_t* init_dims; // [n+1] bond dims of init_mps
  int init_center;
  int slot_mode;            // 0: queue of whole samples; 1: queue of slots, one segment each
  const uint8_t* reset;     // slot mode: 1 = start slot b from the product state (NULL: never)
  const int32_t* sum_row;   // [n_samples][n_ckpt] estimator row of each checkpoint (NULL: ck)
  const int32_t* order;     // slot mode: queue position -> slot (NULL: identity)
  // outputs
  double* values;
  double* discarded;
  double* ledger;
  unsigned long long* sum_v;
  unsigned long long* sum_v2;
  double* flops;       // [gridDim.x]
  unsigned long long* prof;  // [16] clock64 phase counters (diagnostics)
  int* next_sample;
  int* status;         // bit 0: Jacobi non-convergence, bit 2: continued a slot of another generation
  int* excluded;       // [n_samples] first checkpoint left out of the sums (non-convergence), -1: none; or NULL
  unsigned char* slot_bad;  // [slots] the slot's current circuit hit a non-converged SVD (slot mode)
  unsigned* slot_gen;       // [slots] workspace generation the slot's state was built in
  unsigned gen;             // current workspace generation
  double2* states;          // [n_samples][n][cap][2][cap] final MPS per sample (signed mixture), or NULL
  int* state_dims;          // [n_samples][n+1]
  int* state_center;        // [n_samples]
  double* sample_ms;        // [n_samples] device time of the sample (queue) / its segment (slot mode), or NULL
  // run_stream mode i/o
  int* slot_dims;        // [slots][MAXN+1] persistent slot state (slot mode)
  int* slot_center;      // [slots]
  double* slot_counters; // [slots][4]
  // workspace
  double2* ws_mps;
  double2* ws_W;
  double2* ws_W0;
  double2* ws_X;
  size_t mps_stride, mat_stride;
};
}  // namespace tbc

// full engine (bond capacity <= 128, one CTA per SM)
#define TB_ENGINE_NS tb
#define TB_ENGINE_MAXCAP 128
#define TB_ENGINE_MINB 1
#define TB_ENGINE_SMALL 0
#include "tepai_engine.cuh"
#undef TB_ENGINE_NS
#undef TB_ENGINE_MAXCAP
#undef TB_ENGINE_MINB
#undef TB_ENGINE_SMALL

// small-problem engine (bond capacity <= 32, two CTAs per SM)
#define TB_ENGINE_NS tbs
#define TB_ENGINE_MAXCAP 32
#ifndef TB_SMALL_MINB
#define TB_SMALL_MINB 2
#endif
#define TB_ENGINE_MINB TB_SMALL_MINB
#define TB_ENGINE_SMALL 1
#include "tepai_engine.cuh"
#undef TB_ENGINE_NS
#undef TB_ENGINE_MAXCAP
#undef TB_ENGINE_MINB
#undef TB_ENGINE_SMALL

// ============================================================================
// host side: context, workspace, C ABI
// ============================================================================
struct tb_ctx {
  int device = 0;
  int sms = 0;
  std::string err;
  // per-slot workspace (one slot per persistent CTA)
  double2* mps = nullptr;
  double2* W = nullptr;
  double2* W0 = nullptr;
  double2* X = nullptr;
  int* slot_dims = nullptr;
  int* slot_center = nullptr;
  double* slot_counters = nullptr;
  unsigned char* slot_bad = nullptr;
  unsigned* slot_gen = nullptr;
  // Workspace generation: bumped whenever the slot pool is reallocated,
  // reshaped, or overwritten by a non-slot call (run_stream, run_ensemble,
  // svd).  A slot continued (reset = 0) with a stale generation is refused.
  unsigned gen = 1;
  size_t mps_cap_bytes = 0, mat_cap_bytes = 0;  // per slot
  int slots = 0;
  size_t mps_stride = 0, mat_stride = 0;
  int state_n = -1, state_cap = -1;  // shape the slot states were built for
  bool profile = false;              // TB_PROFILE=1: clock64 phase counters (diagnostics only)
  // small device scratch
  int* dscratch = nullptr;  // [0] next_sample, [1] status
  double* dflops = nullptr;
  unsigned long long* dprof = nullptr;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
};

namespace {

int fail(tb_ctx* c, int code, const std::string& msg) {
  if (c) c->err = msg;
  return code;
}

#define TB_CUDA(ctx, call)                                                                               \
  do {                                                                                                   \
    cudaError_t _e = (call);                                                                             \
    if (_e != cudaSuccess) return fail(ctx, TB_ECUDA, std::string(#call) + ": " + cudaGetErrorString(_e)); \
  } while (0)

void free_workspace(tb_ctx* c) {
  cudaFree(c->mps);
  cudaFree(c->W);
  cudaFree(c->W0);
  cudaFree(c->X);
  cudaFree(c->slot_dims);
  cudaFree(c->slot_center);
  cudaFree(c->slot_counters);
  cudaFree(c->slot_bad);
  cudaFree(c->slot_gen);
  c->mps = c->W = c->W0 = c->X = nullptr;
  c->slot_dims = c->slot_center = nullptr;
  c->slot_counters = nullptr;
  c->slot_bad = nullptr;
  c->slot_gen = nullptr;
  ++c->gen;
  c->slots = 0;
  c->mps_cap_bytes = c->mat_cap_bytes = 0;
  c->state_n = c->state_cap = -1;
}

// Grow the per-slot workspace to `slots` slots of an (n, cap) chain.  Slot
// states survive only while the shape is unchanged and nothing is reallocated.
int ensure_workspace(tb_ctx* c, int slots, int n, int cap) {
  const size_t mps_bytes = (size_t)n * cap * 2 * cap * sizeof(double2);
  const size_t cols = (size_t)((2 * cap + 31) / 32) * 32;
  const size_t mat_bytes = (size_t)(2 * cap) * (cols > (size_t)(2 * cap) ? cols : (size_t)(2 * cap)) * sizeof(double2);
  c->mps_stride = mps_bytes / sizeof(double2);
  c->mat_stride = mat_bytes / sizeof(double2);
  if (slots <= c->slots && mps_bytes <= c->mps_cap_bytes && mat_bytes <= c->mat_cap_bytes) {
    if (n != c->state_n || cap != c->state_cap) {
      c->state_n = c->state_cap = -1;
      ++c->gen;
    }
    return TB_OK;
  }
  const int s = slots > c->slots ? slots : c->slots;
  const size_t mb = mps_bytes > c->mps_cap_bytes ? mps_bytes : c->mps_cap_bytes;
  const size_t tb = mat_bytes > c->mat_cap_bytes ? mat_bytes : c->mat_cap_bytes;
  free_workspace(c);
  if (cudaMalloc(&c->mps, mb * s) != cudaSuccess || cudaMalloc(&c->W, tb * s) != cudaSuccess ||
      cudaMalloc(&c->W0, tb * s) != cudaSuccess || cudaMalloc(&c->X, tb * s) != cudaSuccess ||
      cudaMalloc(&c->slot_dims, (size_t)s * (tb::MAXN + 1) * sizeof(int)) != cudaSuccess ||
      cudaMalloc(&c->slot_center, (size_t)s * sizeof(int)) != cudaSuccess ||
      cudaMalloc(&c->slot_counters, (size_t)s * 4 * sizeof(double)) != cudaSuccess ||
      cudaMalloc(&c->slot_bad, (size_t)s) != cudaSuccess || cudaMalloc(&c->slot_gen, (size_t)s * sizeof(unsigned)) != cudaSuccess ||
      cudaMemset(c->slot_gen, 0, (size_t)s * sizeof(unsigned)) != cudaSuccess ||
      cudaMemset(c->slot_bad, 0, (size_t)s) != cudaSuccess) {
    cudaGetLastError();
    free_workspace(c);
    return fail(c, TB_ENOMEM, "workspace allocation failed");
  }
  c->slots = s;
  c->mps_cap_bytes = mb;
  c->mat_cap_bytes = tb;
  return TB_OK;
}

int validate_shape(tb_ctx* c, int64_t n, int64_t cap, int64_t chi_cut) {
  if (n < 1 || n > tb::MAXN) return fail(c, TB_EINVAL, "n must lie in [1, 64]");
  if (cap < 1 || cap > tb::MAXCAP) return fail(c, TB_EINVAL, "cap must lie in [1, 128]");
  if (chi_cut < 1 || chi_cut > cap) return fail(c, TB_EINVAL, "chi_cut must lie in [1, cap]");
  return TB_OK;
}

int validate_desc(tb_ctx* c, const tb_ensemble_desc* d, const tb_ensemble_out* o) {
  int rc = validate_shape(c, d->n, d->cap, d->chi_cut);
  if (rc) return rc;
  if (d->n_samples < 0 || d->n_ckpt < 0 || d->n_obs < 0 || d->n_obs > tb::MAXN || d->n_angles < 1 ||
      d->n_angles > 1024)
    return fail(c, TB_EINVAL, "bad ensemble sizes");
  if (!d->gates || !d->gate_offsets || !d->angle_cs || (!d->init_vecs && !d->init_mps) || !o->sum_v || !o->sum_v2 ||
      !o->flops)
    return fail(c, TB_EINVAL, "null argument");
  if (d->n_ckpt > 0 && (!d->ckpt_gate_end || !d->ckpt_sign || (d->n_obs > 0 && !d->obs_sites)))
    return fail(c, TB_EINVAL, "null checkpoint argument");
  if (d->init_mps && (!d->init_dims || d->init_center < 0 || d->init_center >= d->n))
    return fail(c, TB_EINVAL, "init_mps needs init_dims and a centre in [0, n)");
  return TB_OK;
}

// TB_GRAM_SCREEN: 0 = off, 1 = late sweeps visit only the pairs flagged by the
// DMMA Gram screen, 2 = + flag-driven cross phases (default), 3 = + flag-driven
// within-block phases (measured slightly slower than 2: 1.786 vs 1.812
// samples/s, profiles/r02v_bench_*.json)
constexpr int kGramScreenDefault = 2;

tb::Job make_job(tb_ctx* c, const tb_ensemble_desc* d, const tb_ensemble_out* o) {
  tb::Job job;
  memset(&job, 0, sizeof(job));
  job.n = d->n;
  job.cap = d->cap;
  job.chi_cut = d->chi_cut;
  job.pi_local = d->pi_local;
  {
    const char* pe = getenv("TB_PRECOND");
    job.precond = pe ? atoi(pe) : 1;
    const char* ts = getenv("TB_TAIL_SKIP");
    job.tail_skip = ts ? atoi(ts) : 1;
    const char* tm = getenv("TB_QRCP_TMEM");
    job.qrcp_tmem = tm ? atoi(tm) : 1;
    const char* gs = getenv("TB_GRAM_SCREEN");
    job.gram_screen = gs ? atoi(gs) : kGramScreenDefault;
    const char* ms = getenv("TB_MAX_SWEEPS");
    job.max_sweeps = ms ? atoi(ms) : tb::MAXSWEEP;
    if (job.max_sweeps < 1 || job.max_sweeps > tb::MAXSWEEP) job.max_sweeps = tb::MAXSWEEP;
    const char* fi = getenv("TB_FAULT_INJECT");
    job.inject = fi ? atoi(fi) : 0;
    const char* ct = getenv("TB_CLUSTER_TMA");
    job.cluster_tma = ct ? atoi(ct) : 1;
  }
  job.floor = d->svalue_floor;
  job.n_samples = d->n_samples;
  job.n_ckpt = d->n_ckpt;
  job.n_obs = d->n_obs;
  job.gates = d->gates;
  job.gate_off = d->gate_offsets;
  job.ckpt_end = d->ckpt_gate_end;
  job.ckpt_sign = d->ckpt_sign;
  job.angle_cs = d->angle_cs;
  job.obs_sites = d->obs_sites;
  job.init_vecs = d->init_vecs;
  job.init_mps = (const double2*)d->init_mps;
  job.init_dims = d->init_dims;
  job.init_center = d->init_center;
  job.values = o->values;
  job.discarded = o->discarded;
  job.ledger = o->ledger;
  job.sum_v = (unsigned long long*)o->sum_v;
  job.sum_v2 = (unsigned long long*)o->sum_v2;
  job.flops = c->dflops;
  job.prof = (TB_PROF && c->profile) ? c->dprof : nullptr;  // phase atomics only in diagnostics builds
  job.next_sample = c->dscratch;
  job.status = c->dscratch + 1;
  job.excluded = o->excluded;
  job.states = (double2*)o->states;
  job.state_dims = o->state_dims;
  job.state_center = o->state_center;
  job.sample_ms = o->sample_ms;
  job.slot_bad = c->slot_bad;
  job.slot_gen = c->slot_gen;
  job.gen = c->gen;
  job.slot_dims = c->slot_dims;
  job.slot_center = c->slot_center;
  job.slot_counters = c->slot_counters;
  job.ws_mps = c->mps;
  job.ws_W = c->W;
  job.ws_W0 = c->W0;
  job.ws_X = c->X;
  job.mps_stride = c->mps_stride;
  job.mat_stride = c->mat_stride;
  return job;
}

// Small-problem engine (namespace tbs: two resident CTAs per SM) for bond
// capacities <= 32, unless TB_SMALL_ENGINE=0 (A/B against the full engine).
bool small_engine(int cap) {
  if (cap > tbs::MAXCAP) return false;
  const char* e = getenv("TB_SMALL_ENGINE");
  return !(e && !atoi(e));
}

// persistent CTAs that run circuits of bond capacity `cap` concurrently
int persistent_ctas(const tb_ctx* c, int cap) {
  if (!small_engine(cap)) return c->sms;
  const char* e = getenv("TB_SMALL_CTAS_PER_SM");  // debug: 1 = one resident CTA per SM
  return (e && atoi(e) == 1) ? c->sms : 2 * c->sms;
}

// launch the persistent kernel (+ FLOP reduction into o_flops) on stream st
int launch(tb_ctx* c, tb::Job& job, int grid, cudaStream_t st, double* o_flops, float* kernel_ms) {
  const bool small = small_engine(job.cap) && job.cluster <= 1;
  const size_t smem = small ? tbs::kDynSmem : tb::kDynSmem;
  if (small) {
    job.qrcp_tmem = 0;  // tensor memory serves the 128-row problems only
    TB_CUDA(c, cudaFuncSetAttribute(tbs::ensemble_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  } else {
    TB_CUDA(c, cudaFuncSetAttribute(tb::ensemble_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  }
  TB_CUDA(c, cudaMemsetAsync(c->dscratch, 0, sizeof(int), st));  // queue head; the status word stays sticky
  TB_CUDA(c, cudaMemsetAsync(c->dflops, 0, grid * sizeof(double), st));
  TB_CUDA(c, cudaMemsetAsync(c->dprof, 0, 64 * sizeof(unsigned long long), st));
  if (kernel_ms) TB_CUDA(c, cudaEventRecord(c->e0, st));
  if (job.cluster > 1) {
    TB_CUDA(c, cudaFuncSetAttribute(tb::ensemble_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = (unsigned)job.cluster;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3(tb::NT);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    TB_CUDA(c, cudaLaunchKernelEx(&cfg, tb::ensemble_kernel, job));
  } else if (small) {
    tbs::ensemble_kernel<<<grid, tbs::NT, smem, st>>>(job);
  } else {
    tb::ensemble_kernel<<<grid, tb::NT, smem, st>>>(job);
  }
  TB_CUDA(c, cudaGetLastError());
  if (kernel_ms) TB_CUDA(c, cudaEventRecord(c->e1, st));
  if (o_flops) {
    tb::sum_flops_kernel<<<1, 32, 0, st>>>(c->dflops, grid, o_flops);
    TB_CUDA(c, cudaGetLastError());
  }
  if (kernel_ms) {
    TB_CUDA(c, cudaEventSynchronize(c->e1));
    TB_CUDA(c, cudaEventElapsedTime(kernel_ms, c->e0, c->e1));
  }
  return TB_OK;
}

// Read and clear the sticky device status word (bit 0: a Jacobi SVD did not
// converge; bit 2: a slot of another workspace generation was continued).
int take_status(tb_ctx* c, int* out) {
  int st = 0;
  TB_CUDA(c, cudaMemcpy(&st, c->dscratch + 1, sizeof(int), cudaMemcpyDeviceToHost));
  TB_CUDA(c, cudaMemset(c->dscratch + 1, 0, sizeof(int)));
  *out = st;
  return TB_OK;
}

// status -> return code; `nonconv_ok`: the caller receives per-sample
// exclusion flags, so a non-converged sample is reported there instead
int status_rc(tb_ctx* c, int st, bool nonconv_ok) {
  if (st & 4)
    return fail(c, TB_EINVAL,
                "a slot was continued (reset = 0) after its workspace was reallocated, reshaped or reused by "
                "another engine call; reset every slot");
  if ((st & 1) && !nonconv_ok)
    return fail(c, TB_ENOCONV, "Jacobi SVD did not converge (pass tb_ensemble_out.excluded to keep the launch)");
  return TB_OK;
}

int read_status(tb_ctx* c, bool nonconv_ok = false) {
  int st = 0;
  const int rc = take_status(c, &st);
  return rc ? rc : status_rc(c, st, nonconv_ok);
}

// Wide Jacobi in 8-CTA clusters (jacobi_cluster): used when the bond
// capacity admits 256-row problems (cap > 64).  tb_run_stream (one circuit)
// uses it unless TB_CLUSTER=0; the ensemble calls only with
// TB_CLUSTER_ENSEMBLE=1 (one circuit per cluster instead of per SM).
int cluster_mode(int cap, bool ensemble) {
  if (cap <= 64) return 0;
  const char* e = getenv(ensemble ? "TB_CLUSTER_ENSEMBLE" : "TB_CLUSTER");
  if (ensemble) return (e && atoi(e)) ? tb::CL : 0;
  return (e && !atoi(e)) ? 0 : tb::CL;
}

// co-resident 8-CTA clusters of ensemble_kernel on this device
int max_clusters(tb_ctx* c, int* out) {
  const size_t smem = tb::kDynSmem;
  TB_CUDA(c, cudaFuncSetAttribute(tb::ensemble_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = tb::CL;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.gridDim = dim3(tb::CL * 32);
  cfg.blockDim = dim3(tb::NT);
  cfg.dynamicSmemBytes = smem;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int n = 0;
  TB_CUDA(c, cudaOccupancyMaxActiveClusters(&n, tb::ensemble_kernel, &cfg));
  if (n < 1) return fail(c, TB_ECUDA, "no 8-CTA cluster of the engine kernel fits on this device");
  *out = n;
  return TB_OK;
}

// device copies of a host descriptor/outputs; frees on destruction
struct Staged {
  std::vector<void*> allocs;
  ~Staged() {
    for (void* p : allocs) cudaFree(p);
  }
  // device copy of h[0:count] (or uninitialised when !copy); NULL on any
  // allocation or copy failure (the caller reports TB_ENOMEM / TB_ECUDA)
  template <class T>
  T* up(const T* h, size_t count, bool copy = true) {
    void* p = nullptr;
    if (cudaMalloc(&p, count ? count * sizeof(T) : 8) != cudaSuccess) {
      cudaGetLastError();
      return nullptr;
    }
    allocs.push_back(p);
    if (copy && h && count && cudaMemcpy(p, h, count * sizeof(T), cudaMemcpyHostToDevice) != cudaSuccess) {
      cudaGetLastError();
      return nullptr;
    }
    return (T*)p;
  }
};

int stage_inputs(tb_ctx* c, Staged& sg, const tb_ensemble_desc* d, tb_ensemble_desc* dd) {
  const int S = d->n_samples, C = d->n_ckpt, O = d->n_obs;
  const int64_t G = d->gate_offsets[S];
  *dd = *d;
  dd->gates = sg.up(d->gates, (size_t)G);
  dd->gate_offsets = sg.up(d->gate_offsets, (size_t)S + 1);
  dd->ckpt_gate_end = sg.up(d->ckpt_gate_end, (size_t)S * C);
  dd->ckpt_sign = sg.up(d->ckpt_sign, (size_t)S * C);
  dd->angle_cs = sg.up(d->angle_cs, 2 * (size_t)d->n_angles);
  dd->ckpt_weight = nullptr;
  dd->obs_sites = sg.up(d->obs_sites, (size_t)O);
  dd->init_vecs = sg.up(d->init_vecs, 4 * (size_t)d->n);
  dd->init_mps = d->init_mps ? (const double*)sg.up((const double2*)d->init_mps, (size_t)d->n * d->cap * 2 * d->cap) : nullptr;
  dd->init_dims = d->init_mps ? sg.up(d->init_dims, (size_t)d->n + 1) : nullptr;
  if (!dd->gates || !dd->gate_offsets || !dd->ckpt_gate_end || !dd->ckpt_sign || !dd->angle_cs || !dd->obs_sites ||
      !dd->init_vecs || (d->init_mps && (!dd->init_mps || !dd->init_dims)))
    return fail(c, TB_ENOMEM, "device allocation failed");
  return TB_OK;
}

int stage_outputs(tb_ctx* c, Staged& sg, const tb_ensemble_desc* d, const tb_ensemble_out* o, tb_ensemble_out* od) {
  const int S = d->n_samples, C = d->n_ckpt, O = d->n_obs;
  *od = *o;
  od->values = o->values ? sg.up<double>(nullptr, (size_t)S * C * O, false) : nullptr;
  od->discarded = o->discarded ? sg.up<double>(nullptr, (size_t)S * C, false) : nullptr;
  od->ledger = o->ledger ? sg.up<double>(nullptr, (size_t)S * 4, false) : nullptr;
  // sums: the caller's arrays are accumulated into, so they travel both ways
  const size_t rows = (size_t)(o->sum_v ? 1 : 0);
  (void)rows;
  od->flops = sg.up<double>(nullptr, 1, false);
  od->kernel_ms = o->kernel_ms;
  od->excluded = o->excluded ? sg.up<int32_t>(nullptr, (size_t)S, false) : nullptr;
  const size_t sbytes = (size_t)d->n * d->cap * 2 * d->cap;
  od->states = o->states ? (double*)sg.up<double2>(nullptr, (size_t)S * sbytes, false) : nullptr;
  od->state_dims = o->states ? sg.up<int32_t>(nullptr, (size_t)S * (d->n + 1), false) : nullptr;
  od->state_center = o->states ? sg.up<int32_t>(nullptr, (size_t)S, false) : nullptr;
  od->sample_ms = o->sample_ms ? sg.up<double>(nullptr, (size_t)S, false) : nullptr;
  if ((o->values && !od->values) || (o->discarded && !od->discarded) || (o->ledger && !od->ledger) || !od->flops ||
      (o->excluded && !od->excluded) || (o->states && (!od->states || !od->state_dims || !od->state_center)) ||
      (o->sample_ms && !od->sample_ms))
    return fail(c, TB_ENOMEM, "device allocation failed");
  TB_CUDA(c, cudaMemset(od->flops, 0, sizeof(double)));
  if (od->excluded) TB_CUDA(c, cudaMemset(od->excluded, 0xFF, (size_t)S * sizeof(int32_t)));  // -1: none
  return TB_OK;
}

int fetch_outputs(tb_ctx* c, const tb_ensemble_desc* d, tb_ensemble_out* o, const tb_ensemble_out* od, size_t sum_rows) {
  const int S = d->n_samples, C = d->n_ckpt, O = d->n_obs;
  if (o->values) TB_CUDA(c, cudaMemcpy(o->values, od->values, (size_t)S * C * O * sizeof(double), cudaMemcpyDeviceToHost));
  if (o->discarded)
    TB_CUDA(c, cudaMemcpy(o->discarded, od->discarded, (size_t)S * C * sizeof(double), cudaMemcpyDeviceToHost));
  if (o->ledger) TB_CUDA(c, cudaMemcpy(o->ledger, od->ledger, (size_t)S * 4 * sizeof(double), cudaMemcpyDeviceToHost));
  TB_CUDA(c, cudaMemcpy(o->sum_v, od->sum_v, sum_rows * O * sizeof(int64_t), cudaMemcpyDeviceToHost));
  TB_CUDA(c, cudaMemcpy(o->sum_v2, od->sum_v2, sum_rows * O * sizeof(int64_t), cudaMemcpyDeviceToHost));
  if (o->excluded) TB_CUDA(c, cudaMemcpy(o->excluded, od->excluded, (size_t)S * sizeof(int32_t), cudaMemcpyDeviceToHost));
  if (o->states) {
    const size_t sb = (size_t)d->n * d->cap * 2 * d->cap * sizeof(double2);
    TB_CUDA(c, cudaMemcpy(o->states, od->states, (size_t)S * sb, cudaMemcpyDeviceToHost));
    TB_CUDA(c, cudaMemcpy(o->state_dims, od->state_dims, (size_t)S * (d->n + 1) * sizeof(int32_t), cudaMemcpyDeviceToHost));
    TB_CUDA(c, cudaMemcpy(o->state_center, od->state_center, (size_t)S * sizeof(int32_t), cudaMemcpyDeviceToHost));
  }
  if (o->sample_ms)
    TB_CUDA(c, cudaMemcpy(o->sample_ms, od->sample_ms, (size_t)S * sizeof(double), cudaMemcpyDeviceToHost));
  double f = 0;
  TB_CUDA(c, cudaMemcpy(&f, od->flops, sizeof(double), cudaMemcpyDeviceToHost));
  o->flops[0] += f;
  return TB_OK;
}

}  // namespace

extern "C" {

int tb_version(void) { return 1; }

int tb_create(int device, tb_ctx** out) {
  if (!out) return TB_EINVAL;
  *out = nullptr;
  tb_ctx* c = new tb_ctx();
  c->device = device;
  if (cudaSetDevice(device) != cudaSuccess) {
    cudaGetLastError();
    delete c;
    return TB_ECUDA;
  }
  cudaDeviceGetAttribute(&c->sms, cudaDevAttrMultiProcessorCount, device);
  {
    const char* pf = getenv("TB_PROFILE");
    c->profile = pf && atoi(pf) != 0;
  }
  if (cudaMalloc(&c->dscratch, 256 * sizeof(int)) != cudaSuccess ||
      cudaMalloc(&c->dflops, 4096 * sizeof(double)) != cudaSuccess ||
      cudaMalloc(&c->dprof, 64 * sizeof(unsigned long long)) != cudaSuccess ||
      cudaEventCreate(&c->e0) != cudaSuccess || cudaEventCreate(&c->e1) != cudaSuccess) {
    cudaGetLastError();
    delete c;
    return TB_ECUDA;
  }
  cudaMemset(c->dprof, 0, 64 * sizeof(unsigned long long));
  cudaMemset(c->dscratch, 0, 256 * sizeof(int));
  *out = c;
  return TB_OK;
}

void tb_destroy(tb_ctx* c) {
  if (!c) return;
  free_workspace(c);
  cudaFree(c->dscratch);
  cudaFree(c->dflops);
  cudaFree(c->dprof);
  if (c->e0) cudaEventDestroy(c->e0);
  if (c->e1) cudaEventDestroy(c->e1);
  delete c;
}

const char* tb_last_error(const tb_ctx* c) { return c ? c->err.c_str() : "null context"; }

int tb_num_sms(const tb_ctx* c) { return c ? c->sms : 0; }

int tb_num_ctas(const tb_ctx* c, int64_t cap) { return c ? persistent_ctas(c, (int)cap) : 0; }

int tb_take_status(tb_ctx* c, int32_t* status) {
  if (!c || !status) return TB_EINVAL;
  int st = 0;
  const int rc = take_status(c, &st);
  *status = st;
  return rc;
}

int tb_debug_profile(tb_ctx* c, uint64_t* out64) {
  if (!c || !out64) return TB_EINVAL;
  cudaError_t e = cudaMemcpy(out64, c->dprof, 64 * sizeof(uint64_t), cudaMemcpyDeviceToHost);
  return e == cudaSuccess ? TB_OK : fail(c, TB_ECUDA, cudaGetErrorString(e));
}

int tb_run_stream(tb_ctx* c, double* buf, int64_t n, int64_t cap, int64_t* dims, int64_t center, const int64_t* ga,
                  const int64_t* gb, const int64_t* pa, const int64_t* pb, const double* ang, const int64_t* anchors,
                  int64_t n_gates, int64_t chi_cut, double floor, double* counters, int64_t* new_center) {
  if (!c) return TB_EINVAL;
  int rc = validate_shape(c, n, cap, chi_cut);
  if (rc) return rc;
  if (!buf || !dims || !counters || !new_center || (n_gates > 0 && (!ga || !gb || !pa || !pb || !ang || !anchors)))
    return fail(c, TB_EINVAL, "null argument");
  for (int64_t s = 0; s <= n; ++s)
    if (dims[s] < 1 || dims[s] > cap) return fail(c, TB_EINVAL, "bond dimension outside [1, cap]");
  if (center < 0 || center >= n) return fail(c, TB_EINVAL, "center outside [0, n)");
  // pack the lowered stream with a table of its distinct angles (<= 1024)
  std::vector<uint32_t> words((size_t)n_gates);
  std::vector<double> angles, table;
  for (int64_t i = 0; i < n_gates; ++i) {
    const int64_t a = ga[i], b = gb[i];
    if (a < 0 || a >= n || b >= n || (b >= 0 && b <= a)) return fail(c, TB_EINVAL, "gate support outside the chain");
    if (pa[i] < 1 || pa[i] > 3 || (b >= 0 && (pb[i] < 1 || pb[i] > 3))) return fail(c, TB_EINVAL, "bad Pauli code");
    size_t ai = 0;
    while (ai < angles.size() && angles[ai] != ang[i]) ++ai;
    if (ai == angles.size()) {
      if (angles.size() == 1024) return fail(c, TB_EINVAL, "more than 1024 distinct angles in one call");
      angles.push_back(ang[i]);
      table.push_back(cos(0.5 * ang[i]));
      table.push_back(sin(0.5 * ang[i]));
    }
    words[(size_t)i] = (uint32_t)a | ((b < 0 ? TB_ONE_SITE : (uint32_t)b) << 8) | ((uint32_t)pa[i] << 16) |
                       ((uint32_t)(b < 0 ? 0 : pb[i]) << 18) | ((uint32_t)(anchors[i] > a) << 20) |
                       ((uint32_t)(ang[i] == M_PI) << 21) | ((uint32_t)ai << 22);
  }
  if (table.empty()) table = {1.0, 0.0};
  rc = ensure_workspace(c, 1, (int)n, (int)cap);
  if (rc) return rc;
  Staged sg;
  const int64_t off[2] = {0, n_gates};
  uint32_t* dg = sg.up(words.data(), words.size());
  int64_t* doff = sg.up(off, 2);
  double* dtab = sg.up(table.data(), table.size());
  if (!dg || !doff || !dtab) return fail(c, TB_ENOMEM, "device allocation failed");
  std::vector<int> idims((size_t)tb::MAXN + 1, 1);
  for (int64_t s = 0; s <= n; ++s) idims[(size_t)s] = (int)dims[s];
  int icenter = (int)center;
  const size_t site_bytes = (size_t)n * cap * 2 * cap * sizeof(double2);
  TB_CUDA(c, cudaMemcpy(c->slot_dims, idims.data(), idims.size() * sizeof(int), cudaMemcpyHostToDevice));
  TB_CUDA(c, cudaMemcpy(c->slot_center, &icenter, sizeof(int), cudaMemcpyHostToDevice));
  TB_CUDA(c, cudaMemcpy(c->slot_counters, counters, 4 * sizeof(double), cudaMemcpyHostToDevice));
  TB_CUDA(c, cudaMemcpy(c->mps, buf, site_bytes, cudaMemcpyHostToDevice));
  TB_CUDA(c, cudaMemcpy(c->slot_gen, &c->gen, sizeof(unsigned), cudaMemcpyHostToDevice));
  TB_CUDA(c, cudaMemset(c->slot_bad, 0, 1));
  tb_ensemble_desc d;
  memset(&d, 0, sizeof(d));
  d.n = (int)n;
  d.cap = (int)cap;
  d.chi_cut = (int)chi_cut;
  d.pi_local = 0;  // drop-in: the reference's full two-site update for pi gates
  d.svalue_floor = floor;
  d.n_samples = 1;
  d.gates = dg;
  d.gate_offsets = doff;
  d.angle_cs = dtab;
  tb_ensemble_out o;
  memset(&o, 0, sizeof(o));
  tb::Job job = make_job(c, &d, &o);
  job.slot_mode = 1;  // continue the uploaded state (no reset)
  job.cluster = cluster_mode((int)cap, false);
  rc = launch(c, job, job.cluster > 1 ? job.cluster : 1, 0, nullptr, nullptr);
  if (rc) return rc;
  TB_CUDA(c, cudaDeviceSynchronize());
  TB_CUDA(c, cudaMemcpy(buf, c->mps, site_bytes, cudaMemcpyDeviceToHost));
  TB_CUDA(c, cudaMemcpy(idims.data(), c->slot_dims, idims.size() * sizeof(int), cudaMemcpyDeviceToHost));
  TB_CUDA(c, cudaMemcpy(&icenter, c->slot_center, sizeof(int), cudaMemcpyDeviceToHost));
  TB_CUDA(c, cudaMemcpy(counters, c->slot_counters, 4 * sizeof(double), cudaMemcpyDeviceToHost));
  for (int64_t s = 0; s <= n; ++s) dims[s] = idims[(size_t)s];
  *new_center = icenter;
  c->state_n = c->state_cap = -1;  // slot 0 now holds a caller's state, not a pipeline slot
  ++c->gen;
  return read_status(c);
}

int tb_expectation(tb_ctx* c, const double* buf, int64_t n, int64_t cap, const int64_t* dims, const int32_t* codes,
                   double* out) {
  if (!c) return TB_EINVAL;
  int rc = validate_shape(c, n, cap, 1);
  if (rc) return rc;
  if (!buf || !dims || !codes || !out) return fail(c, TB_EINVAL, "null argument");
  for (int64_t s = 0; s <= n; ++s)
    if (dims[s] < 1 || dims[s] > cap) return fail(c, TB_EINVAL, "bond dimension outside [1, cap]");
  for (int64_t s = 0; s < n; ++s)
    if (codes[s] < 0 || codes[s] > 3) return fail(c, TB_EINVAL, "bad Pauli code");
  rc = ensure_workspace(c, 1, (int)n, (int)cap);
  if (rc) return rc;
  std::vector<int> idims((size_t)n + 1);
  for (int64_t s = 0; s <= n; ++s) idims[(size_t)s] = (int)dims[s];
  Staged sg;
  int* dd = sg.up<int>(nullptr, 2 * (size_t)n + 1, false);
  double2* dbuf = sg.up((const double2*)buf, (size_t)n * cap * 2 * cap);
  double* dout = sg.up<double>(nullptr, 1, false);
  if (!dd || !dbuf || !dout) return fail(c, TB_ENOMEM, "device allocation failed");
  TB_CUDA(c, cudaMemcpy(dd, idims.data(), (n + 1) * sizeof(int), cudaMemcpyHostToDevice));
  TB_CUDA(c, cudaMemcpy(dd + n + 1, codes, n * sizeof(int), cudaMemcpyHostToDevice));
  const size_t smem = tb::kTileBytes;
  TB_CUDA(c, cudaFuncSetAttribute(tb::expectation_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  tb::expectation_kernel<<<1, tb::NT, smem>>>(dbuf, (int)n, (int)cap, dd, dd + n + 1, c->W, c->W0, dout);
  TB_CUDA(c, cudaGetLastError());
  TB_CUDA(c, cudaMemcpy(out, dout, sizeof(double), cudaMemcpyDeviceToHost));
  return TB_OK;
}

int tb_expectation_batch(tb_ctx* c, const double* bufs, int64_t n_states, int64_t n, int64_t cap, const int64_t* dims,
                         const int32_t* codes, int64_t n_obs, double* out) {
  if (!c) return TB_EINVAL;
  int rc = validate_shape(c, n, cap, 1);
  if (rc) return rc;
  if (n_states < 0 || n_obs < 0 || (n_states > 0 && n_obs > 0 && (!bufs || !dims || !codes || !out)))
    return fail(c, TB_EINVAL, "null argument");
  if (n_states == 0 || n_obs == 0) return TB_OK;
  std::vector<int> idims((size_t)n_states * (n + 1));
  for (int64_t st = 0; st < n_states; ++st)
    for (int64_t s = 0; s <= n; ++s) {
      const int64_t d = dims[st * (n + 1) + s];
      if (d < 1 || d > cap) return fail(c, TB_EINVAL, "bond dimension outside [1, cap]");
      idims[(size_t)(st * (n + 1) + s)] = (int)d;
    }
  for (int64_t e = 0; e < n_obs * n; ++e)
    if (codes[e] < 0 || codes[e] > 3) return fail(c, TB_EINVAL, "bad Pauli code");
  const int grid = (int)(n_states < c->sms ? n_states : c->sms);
  rc = ensure_workspace(c, grid, (int)n, (int)cap);
  if (rc) return rc;
  ++c->gen;  // the environments use the slot scratch
  Staged sg;
  double2* dbuf = sg.up((const double2*)bufs, (size_t)n_states * n * cap * 2 * cap);
  int* dd = sg.up(idims.data(), idims.size());
  int* dc = sg.up(codes, (size_t)(n_obs * n));
  double* dout = sg.up<double>(nullptr, (size_t)(n_states * n_obs), false);
  if (!dbuf || !dd || !dc || !dout) return fail(c, TB_ENOMEM, "device allocation failed");
  const size_t smem = tb::kTileBytes;
  TB_CUDA(c, cudaFuncSetAttribute(tb::expectation_batch_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  tb::expectation_batch_kernel<<<grid, tb::NT, smem>>>(dbuf, (int)n_states, (int)n, (int)cap, dd, dc, (int)n_obs, c->W,
                                                       c->W0, c->mat_stride, dout);
  TB_CUDA(c, cudaGetLastError());
  TB_CUDA(c, cudaMemcpy(out, dout, (size_t)(n_states * n_obs) * sizeof(double), cudaMemcpyDeviceToHost));
  return TB_OK;
}

int tb_svd(tb_ctx* c, const double* a, int64_t batch, int64_t m, int64_t n, double* s, double* u, double* vh) {
  return tb_svd_trunc(c, a, batch, m, n, 0, s, u, vh);
}

int tb_svd_trunc(tb_ctx* c, const double* a, int64_t batch, int64_t m, int64_t n, int64_t kcut, double* s, double* u,
                 double* vh) {
  if (!c) return TB_EINVAL;
  if (!a || !s || batch < 1 || m < 1 || n < 1) return fail(c, TB_EINVAL, "bad arguments");
  if (m > tb::MAXDIM || n > tb::MAXDIM) return fail(c, TB_EINVAL, "matrix larger than 256");
  const int64_t k = m < n ? m : n;
  const int cap = (int)((m > n ? m : n) + 1) / 2;
  int rc = ensure_workspace(c, (int)batch, 1, cap < 1 ? 1 : cap);
  if (rc) return rc;
  c->state_n = c->state_cap = -1;
  ++c->gen;
  Staged sg;
  double2* da = sg.up((const double2*)a, (size_t)(batch * m * n));
  double* ds = sg.up<double>(nullptr, (size_t)(batch * k), false);
  double2* du = u ? sg.up<double2>(nullptr, (size_t)(batch * m * k), false) : nullptr;
  double2* dvh = vh ? sg.up<double2>(nullptr, (size_t)(batch * k * n), false) : nullptr;
  if (!da || !ds || (u && !du) || (vh && !dvh)) return fail(c, TB_ENOMEM, "device allocation failed");
  TB_CUDA(c, cudaMemset(c->dscratch, 0, 2 * sizeof(int)));
  TB_CUDA(c, cudaMemset(c->dprof, 0, 64 * sizeof(unsigned long long)));
  // tb_svd has no per-sample flags: its status is this call's alone
  const size_t smem = tb::kDynSmem;
  TB_CUDA(c, cudaFuncSetAttribute(tb::svd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const char* pe = getenv("TB_PRECOND");
  const char* tm = getenv("TB_QRCP_TMEM");
  const char* ce = getenv("TB_CLUSTER");
  const bool clu = ce && atoi(ce) && (m > 128 || n > 128);  // unit-test surface of jacobi_cluster
  const char* ct = getenv("TB_CLUSTER_TMA");
  const char* gs = getenv("TB_GRAM_SCREEN");
  const int precond = (pe ? atoi(pe) : 1) | ((!tm || atoi(tm)) ? 2 : 0) | (clu ? 4 : 0) | ((!ct || atoi(ct)) ? 8 : 0) |
                      ((!gs || atoi(gs)) ? 16 : 0) | (((gs ? atoi(gs) : kGramScreenDefault) - 1) & 3) << 7 | ((getenv("TB_CL_DBG") ? atoi(getenv("TB_CL_DBG")) & 3 : 0) << 5);
  if (clu) {
    TB_CUDA(c, cudaFuncSetAttribute(tb::svd_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = tb::CL;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3((unsigned)(batch * tb::CL));
    cfg.blockDim = dim3(tb::NT);
    cfg.dynamicSmemBytes = smem;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    TB_CUDA(c, cudaLaunchKernelEx(&cfg, tb::svd_kernel, (const double2*)da, (int)m, (int)n, c->W, c->W0, c->X,
                                  c->mat_stride, ds, du, dvh, c->dscratch + 1, c->dprof, precond, (int)kcut));
  } else {
    tb::svd_kernel<<<(int)batch, tb::NT, smem>>>(da, (int)m, (int)n, c->W, c->W0, c->X, c->mat_stride, ds, du, dvh,
                                                 c->dscratch + 1, c->dprof, precond, (int)kcut);
  }
  TB_CUDA(c, cudaGetLastError());
  TB_CUDA(c, cudaDeviceSynchronize());
  TB_CUDA(c, cudaMemcpy(s, ds, batch * k * sizeof(double), cudaMemcpyDeviceToHost));
  if (u) TB_CUDA(c, cudaMemcpy(u, du, batch * m * k * sizeof(double2), cudaMemcpyDeviceToHost));
  if (vh) TB_CUDA(c, cudaMemcpy(vh, dvh, batch * k * n * sizeof(double2), cudaMemcpyDeviceToHost));
  return read_status(c);
}

int tb_run_ensemble_device(tb_ctx* c, const tb_ensemble_desc* d, tb_ensemble_out* o, void* stream) {
  if (!c || !d || !o) return TB_EINVAL;
  int rc = validate_desc(c, d, o);
  if (rc) return rc;
  if (d->n_samples == 0) return TB_OK;
  const int cl = cluster_mode(d->cap, true);
  int units = persistent_ctas(c, d->cap);  // persistent CTAs, or clusters
  if (cl > 1 && (rc = max_clusters(c, &units))) return rc;
  const int grid = d->n_samples < units ? d->n_samples : units;
  rc = ensure_workspace(c, grid, d->n, d->cap);
  if (rc) return rc;
  c->state_n = c->state_cap = -1;  // whole-sample runs reuse the slot memory
  ++c->gen;
  tb::Job job = make_job(c, d, o);
  job.slot_mode = 0;
  job.cluster = cl;
  return launch(c, job, cl > 1 ? grid * cl : grid, (cudaStream_t)stream, o->flops, o->kernel_ms);
}

int tb_run_ensemble(tb_ctx* c, const tb_ensemble_desc* d, tb_ensemble_out* o) {
  if (!c || !d || !o) return TB_EINVAL;
  int rc = validate_desc(c, d, o);
  if (rc) return rc;
  if (d->n_samples == 0) return TB_OK;
  Staged sg;
  tb_ensemble_desc dd;
  tb_ensemble_out od;
  if ((rc = stage_inputs(c, sg, d, &dd)) || (rc = stage_outputs(c, sg, d, o, &od))) return rc;
  const size_t rows = (size_t)d->n_ckpt;
  od.sum_v = sg.up(o->sum_v, rows * d->n_obs);
  od.sum_v2 = sg.up(o->sum_v2, rows * d->n_obs);
  if (!od.sum_v || !od.sum_v2) return fail(c, TB_ENOMEM, "device allocation failed");
  rc = tb_run_ensemble_device(c, &dd, &od, nullptr);
  if (rc) return rc;
  TB_CUDA(c, cudaDeviceSynchronize());
  // the caller's arrays (accumulated sums included) change only on success
  if ((rc = read_status(c, o->excluded != nullptr))) return rc;
  return fetch_outputs(c, d, o, &od, rows);
}

int tb_step_device(tb_ctx* c, const tb_step_desc* sd, tb_ensemble_out* o, void* stream) {
  if (!c || !sd || !o) return TB_EINVAL;
  const tb_ensemble_desc* d = &sd->base;
  int rc = validate_desc(c, d, o);
  if (rc) return rc;
  if (d->n_samples == 0) return TB_OK;
  if (!sd->reset || (d->n_ckpt > 0 && !sd->sum_row)) return fail(c, TB_EINVAL, "null reset/sum_row");
  rc = ensure_workspace(c, d->n_samples, d->n, d->cap);
  if (rc) return rc;
  // a slot whose state was not built for this shape must be reset by the caller;
  // the first call after (re)allocation is accepted only if every slot resets,
  // which the host wrapper guarantees
  c->state_n = d->n;
  c->state_cap = d->cap;
  tb::Job job = make_job(c, d, o);
  job.slot_mode = 1;
  job.reset = sd->reset;
  job.sum_row = sd->sum_row;
  job.order = sd->order;
  job.cluster = cluster_mode(d->cap, true);
  int units = persistent_ctas(c, d->cap);
  if (job.cluster > 1 && (rc = max_clusters(c, &units))) return rc;
  const int grid = d->n_samples < units ? d->n_samples : units;
  return launch(c, job, job.cluster > 1 ? grid * job.cluster : grid, (cudaStream_t)stream, o->flops, o->kernel_ms);
}

int tb_step(tb_ctx* c, const tb_step_desc* sd, tb_ensemble_out* o, int64_t sum_rows) {
  if (!c || !sd || !o) return TB_EINVAL;
  const tb_ensemble_desc* d = &sd->base;
  int rc = validate_desc(c, d, o);
  if (rc) return rc;
  if (d->n_samples == 0) return TB_OK;
  if (sum_rows < 1) return fail(c, TB_EINVAL, "sum_rows must be >= 1");
  Staged sg;
  tb_step_desc sdd;
  tb_ensemble_out od;
  sdd = *sd;
  if ((rc = stage_inputs(c, sg, d, &sdd.base)) || (rc = stage_outputs(c, sg, d, o, &od))) return rc;
  sdd.reset = sg.up(sd->reset, (size_t)d->n_samples);
  sdd.sum_row = sg.up(sd->sum_row, (size_t)d->n_samples * d->n_ckpt);
  sdd.order = sd->order ? sg.up(sd->order, (size_t)d->n_samples) : nullptr;
  if (sd->order && !sdd.order) return fail(c, TB_ENOMEM, "device allocation failed");
  od.sum_v = sg.up(o->sum_v, (size_t)sum_rows * d->n_obs);
  od.sum_v2 = sg.up(o->sum_v2, (size_t)sum_rows * d->n_obs);
  if (!sdd.reset || !sdd.sum_row || !od.sum_v || !od.sum_v2) return fail(c, TB_ENOMEM, "device allocation failed");
  rc = tb_step_device(c, &sdd, &od, nullptr);
  if (rc) return rc;
  TB_CUDA(c, cudaDeviceSynchronize());
  if ((rc = read_status(c, o->excluded != nullptr))) return rc;
  return fetch_outputs(c, d, o, &od, (size_t)sum_rows);
}

}  // extern "C"
