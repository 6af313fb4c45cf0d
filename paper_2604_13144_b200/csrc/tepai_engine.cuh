// tepai_engine.cuh — the device side of the engine (everything inside the
// engine namespace).  tepai_b200.cu includes this file TWICE:
//
//   namespace tb   full engine: bond capacity <= 128, one 512-thread CTA per SM
//                  (128 registers per thread, 198 KB of dynamic shared memory);
//   namespace tbs  small-problem engine: bond capacity <= 32 (two-site problems
//                  <= 64 x 64, SURVEY.md configs C1, C2, C4 at chi 16), compiled
//                  with __launch_bounds__(512, 2) and half-height column slots so
//                  that TWO CTAs — two independent circuits — share an SM.  The
//                  small problems are latency-bound, so a second resident
//                  circuit fills the FP64 pipe's idle cycles.  Same code, same
//                  arithmetic, same results; only the chi = 128 / 128-row paths
//                  are compiled out.
//
// Parameters (macros set by the including file): TB_ENGINE_NS, TB_ENGINE_MAXCAP,
// TB_ENGINE_MINB (resident CTAs per SM), TB_ENGINE_SMALL (0/1).
// No include guard on purpose.
namespace TB_ENGINE_NS {

using tbc::Job;
constexpr int NT = 512;        // threads per CTA
constexpr int NWARP = NT / 32;  // warps per CTA
constexpr int MAXCAP = TB_ENGINE_MAXCAP;  // largest supported bond capacity (128; 32 in the small-problem engine)
constexpr int SROWS = TB_ENGINE_SMALL ? 64 : 128;  // rows of a shared-memory column slot
constexpr int MAXDIM = 2 * MAXCAP;
constexpr int MAXN = 64;        // largest supported chain
constexpr int MAXSWEEP = 60;
constexpr int TK = 16;          // GEMM k-chunk
constexpr int TM = 64;          // GEMM output tile
constexpr int TLD = TM + 1;     // padded smem row
constexpr double FIX = 1099511627776.0;  // 2^40 fixed-point unit of the estimator sums

// ----------------------------------------------------------------------------
// complex helpers
// ----------------------------------------------------------------------------
__device__ __forceinline__ double2 cz() { return make_double2(0.0, 0.0); }
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ double2 cconj(double2 a) { return make_double2(a.x, -a.y); }
__device__ __forceinline__ double2 cscale(double2 a, double s) { return make_double2(a.x * s, a.y * s); }
// acc += a * b
__device__ __forceinline__ void cfma(double2& acc, double2 a, double2 b) {
  acc.x = fma(a.x, b.x, acc.x);
  acc.x = fma(-a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y);
  acc.y = fma(a.y, b.x, acc.y);
}
// acc += conj(a) * b
__device__ __forceinline__ void cfmac(double2& acc, double2 a, double2 b) {
  acc.x = fma(a.x, b.x, acc.x);
  acc.x = fma(a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y);
  acc.y = fma(-a.y, b.x, acc.y);
}
__device__ __forceinline__ double abs2(double2 a) { return fma(a.x, a.x, a.y * a.y); }

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// ----------------------------------------------------------------------------
// job description (device side)
// ----------------------------------------------------------------------------

struct Smem {
  int dims[MAXN + 1];
  double sig[MAXDIM];
  double nrm[MAXDIM];
  double dsc[MAXDIM];        // Jacobi column scales (true column = dsc * stored)
  double wbest[2][32];       // per-half-warp pivot candidates (QRCP), double-buffered by step parity in qrcp_mgs
  int qcnt[3 * 32];          // cross-phase Q visit counters (per slot, column)
  unsigned char chg[MAXDIM]; // bit0: rotated in the previous sweep, bit1: in this sweep, bit2: tail column
  int jncol[4];              // live columns per Jacobi block slot
  int wbidx[2][32];
  double nref[MAXDIM];       // QRCP reference norms; after the Jacobi: 1 / sigma of the kept columns
  int qperm[MAXDIM];
  int qpinv[MAXDIM];
  int perm[MAXDIM];
  double2 rco[MAXDIM];
  double red[NWARP * 4];
  double zval[MAXN];
  double counters[4];
  double flops;
  double scale, invsig_tmp;
  double offmax;
  int k;
  int flag;
  int bad;                   // this sample hit a non-converged SVD: its later checkpoints stay out of the sums
  int maxsweep;              // Jacobi sweep cap (MAXSWEEP; lowered only by the failure-path tests)
  int inject;                // fault injection period (samples with index % inject == 0)
  int sweeps;
  int rotcount;
  uint32_t tmem;             // TMEM base address (512 columns, allocated per CTA)
  int tmem_on;               // QRCP in tensor memory (qrcp_tmem)
  int kcut;                  // singular triplets the caller keeps (min(chi_cut, K)); tail pairs beyond are skipped
  uint32_t pbits[SROWS][SROWS / 32];  // Gram screen: bit (i, j) = pair (i, j) is still coupled (see gram_screen)
  int ntail;                 // columns currently marked as tail (chg bit 2)
  int screen_on;             // Gram screen of the late Jacobi sweeps (gram_screen) enabled
  unsigned blkmask;          // Gram screen: bit 4a + b = some pair of column blocks (a <= b) is flagged
  unsigned long long* prof;
  int sample;
  int center;
  // cluster Jacobi (jacobi_cluster): command posted by the leader, reductions
  int cluster;               // CTAs per cluster (0/1: no cluster)
  int cl_op;                 // 1: Jacobi on (cl_W, cl_Mw, cl_Nw), 0: exit
  double2* cl_W;
  int cl_Mw, cl_Nw, cl_maxsweep;
  int cl_flag[2];
  double cl_off[2];
  double cl_part[8];
  int cl_rflag;
  double cl_roff;
  uint16_t cl_sched[16];
  int cl_tma;                // stage the blocks with TMA bulk copies (else plain loads/stores)
  unsigned long long cl_mbar;  // mbarrier of the bulk loads
};

// ----------------------------------------------------------------------------
// CTA-wide reduction of one double
// ----------------------------------------------------------------------------
__device__ double cta_sum(double v, Smem& sm) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) sm.red[w] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x < 32) {
    t = (l < NWARP) ? sm.red[l] : 0.0;
    t = warp_sum(t);
    if (l == 0) sm.red[NWARP] = t;
  }
  __syncthreads();
  t = sm.red[NWARP];
  __syncthreads();
  return t;
}

// ----------------------------------------------------------------------------
// FP64 tensor-core MMA (DMMA): D(8x8) = A(8x4, row) B(4x8, col) + C.
// Fragments (lane l): A[l/4][l%4], B[l%4][l/4], C/D[l/4][2(l%4) + {0,1}].
// ----------------------------------------------------------------------------
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// ----------------------------------------------------------------------------
// Tensor-core variant of cta_gemm (below), used for the two hot GEMMs of the
// two-site update (theta = A.B and the projection Q^H theta).  Same staging
// and interface; the products run on the FP64 tensor cores: each of the 16 warps owns a 16x16 complex block
// (2x2 DMMA tiles), a complex MAC being four real m8n8k4 MMAs
// (re += Ar Br - Ai Bi, im += Ar Bi + Ai Br).  The remaining (small, cold)
// GEMMs stay on the SIMT version: instantiating the DMMA code at every call
// site measurably worsened the register allocation of the QRCP/Jacobi
// functions compiled into the same kernel (QRCP 7.7k -> 9.9k cycles/step).
// ----------------------------------------------------------------------------
template <bool AKF, bool BKF, class LA, class LB, class SC>
__device__ void cta_gemm_tc(int M, int N, int K, LA la, LB lb, SC sc, double2* tile) {
  double2* As = tile;             // [TK][TLD]  (k rows, m cols)
  double2* Bs = tile + TK * TLD;  // [TK][TLD]  (k rows, n cols)
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int wm = (warp >> 2) * 16, wn = (warp & 3) * 16;  // warp block inside the 64x64 tile
  const int fr = lane >> 2, fk = lane & 3;                 // fragment row / k index
  for (int m0 = 0; m0 < M; m0 += TM) {
    for (int n0 = 0; n0 < N; n0 += TM) {
      double cre[2][2][2], cim[2][2][2];
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
          for (int e = 0; e < 2; ++e) cre[i][j][e] = cim[i][j][e] = 0.0;
      for (int k0 = 0; k0 < K; k0 += TK) {
#pragma unroll
        for (int e0 = 0; e0 < TK * TM; e0 += NT) {
          const int e = e0 + tid;
          int mm, kk;
          if (AKF) { kk = e & (TK - 1); mm = e / TK; } else { mm = e & (TM - 1); kk = e / TM; }
          const int gm = m0 + mm, gk = k0 + kk;
          As[kk * TLD + mm] = (gm < M && gk < K) ? la(gm, gk) : cz();
          int nn;
          if (BKF) { kk = e & (TK - 1); nn = e / TK; } else { nn = e & (TM - 1); kk = e / TM; }
          const int gn = n0 + nn, gk2 = k0 + kk;
          Bs[kk * TLD + nn] = (gn < N && gk2 < K) ? lb(gk2, gn) : cz();
        }
        __syncthreads();
        const int ksteps = (min(TK, K - k0) + 3) >> 2;
#pragma unroll 1
        for (int ks = 0; ks < ksteps; ++ks) {
          const int kr = (ks * 4 + fk) * TLD;
          double2 a[2], b[2];
#pragma unroll
          for (int i = 0; i < 2; ++i) a[i] = As[kr + wm + 8 * i + fr];
#pragma unroll
          for (int j = 0; j < 2; ++j) b[j] = Bs[kr + wn + 8 * j + fr];
#pragma unroll
          for (int i = 0; i < 2; ++i) {
            const double nai = -a[i].y;
#pragma unroll
            for (int j = 0; j < 2; ++j) {
              dmma(cre[i][j][0], cre[i][j][1], a[i].x, b[j].x);
              dmma(cre[i][j][0], cre[i][j][1], nai, b[j].y);
              dmma(cim[i][j][0], cim[i][j][1], a[i].x, b[j].y);
              dmma(cim[i][j][0], cim[i][j][1], a[i].y, b[j].x);
            }
          }
        }
        __syncthreads();
      }
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int gm = m0 + wm + 8 * i + fr, gn = n0 + wn + 8 * j + 2 * fk + e;
            if (gm < M && gn < N) sc(gm, gn, make_double2(cre[i][j][e], cim[i][j][e]));
          }
    }
  }
  __syncthreads();
}

// ----------------------------------------------------------------------------
// CTA-level complex GEMM: C(m,n) = sum_k A(m,k) B(k,n), 64x64 output tiles,
// 16-deep k chunks staged in shared memory.  AKF/BKF pick which index is
// contiguous across threads when staging (k-fastest or m/n-fastest) so that
// the global loads coalesce for the operand's real layout.
// ----------------------------------------------------------------------------
template <bool AKF, bool BKF, class LA, class LB, class SC>
__device__ void cta_gemm(int M, int N, int K, LA la, LB lb, SC sc, double2* tile) {
  double2* As = tile;             // [TK][TLD]  (k rows, m cols)
  double2* Bs = tile + TK * TLD;  // [TK][TLD]  (k rows, n cols)
  const int tid = threadIdx.x;
  const int tx = tid & 15, ty = tid >> 4;  // 16 x 32
  for (int m0 = 0; m0 < M; m0 += TM) {
    for (int n0 = 0; n0 < N; n0 += TM) {
      double2 acc[2][4];
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = cz();
      for (int k0 = 0; k0 < K; k0 += TK) {
#pragma unroll
        for (int e0 = 0; e0 < TK * TM; e0 += NT) {
          const int e = e0 + tid;
          int mm, kk;
          if (AKF) { kk = e & (TK - 1); mm = e / TK; } else { mm = e & (TM - 1); kk = e / TM; }
          const int gm = m0 + mm, gk = k0 + kk;
          As[kk * TLD + mm] = (gm < M && gk < K) ? la(gm, gk) : cz();
          int nn;
          if (BKF) { kk = e & (TK - 1); nn = e / TK; } else { nn = e & (TM - 1); kk = e / TM; }
          const int gn = n0 + nn, gk2 = k0 + kk;
          Bs[kk * TLD + nn] = (gn < N && gk2 < K) ? lb(gk2, gn) : cz();
        }
        __syncthreads();
        const int kmax = min(TK, K - k0);
        for (int kk = 0; kk < kmax; ++kk) {
          double2 a0 = As[kk * TLD + ty], a1 = As[kk * TLD + ty + 32];
          double2 b[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) b[j] = Bs[kk * TLD + tx + 16 * j];
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            cfma(acc[0][j], a0, b[j]);
            cfma(acc[1][j], a1, b[j]);
          }
        }
        __syncthreads();
      }
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int gm = m0 + ty + 32 * i, gn = n0 + tx + 16 * j;
          if (gm < M && gn < N) sc(gm, gn, acc[i][j]);
        }
    }
  }
  __syncthreads();
}

// ----------------------------------------------------------------------------
// One-sided (Hestenes) Jacobi on the columns of W (Mw x Nw, column-major,
// ld = Mw).  Parallel round-robin ordering: every round pairs all columns
// once (circle method), one pair per warp; a sweep is Np-1 rounds.  Stops
// after the first sweep without a rotation.  Returns the number of sweeps.
// ----------------------------------------------------------------------------
__device__ __forceinline__ void rr_pair(int r, int p, int Np, int& i, int& j) {
  // circle method, r in [0, Np-1), p in [0, Np/2): no integer division
  const int m = Np - 1;
  if (p == 0) {
    i = m;
    j = r;
  } else {
    i = r + p;
    if (i >= m) i -= m;
    j = r - p;
    if (j < 0) j += m;
  }
}

__device__ int hestenes(double2* W, int Mw, int Nw, Smem& sm) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int Np = Nw + (Nw & 1);
  if (Nw < 2) return 0;
  // off-diagonal threshold ~2 eps sqrt(M): above the rounding noise of a
  // length-M complex dot product, so converged pairs do not re-trigger
  const double tol = fmax(sqrt((double)Mw), 4.0) * 4.440892098500626e-16;
  int sweep = 0;
  for (; sweep < MAXSWEEP; ++sweep) {
    // numerically dead columns (|a|^2 < 1e-28 |A|_F^2, i.e. rounding residue of
    // a rank deficiency) are set exactly to zero; they can never be made
    // orthogonal to the live span and would otherwise rotate forever
    for (int c = warp; c < Nw; c += NWARP) {
      double s = 0.0;
      for (int y = lane; y < Mw; y += 32) s += abs2(W[(size_t)c * Mw + y]);
      s = warp_sum(s);
      if (lane == 0) sm.sig[c] = s;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int c = 0; c < Nw; ++c) t += sm.sig[c];
      sm.scale = t;
      sm.flag = 0;
    }
    __syncthreads();
    const double dead = 1e-28 * sm.scale;
    for (int c = warp; c < Nw; c += NWARP)
      if (sm.sig[c] < dead && sm.sig[c] > 0.0)
        for (int y = lane; y < Mw; y += 32) W[(size_t)c * Mw + y] = cz();
    __syncthreads();
    for (int r = 0; r < Np - 1; ++r) {
      for (int p = warp; p < Np / 2; p += NWARP) {
        int i, j;
        rr_pair(r, p, Np, i, j);
        if (i >= Nw || j >= Nw) continue;
        double2* a = W + (size_t)i * Mw;
        double2* b = W + (size_t)j * Mw;
        double2 av[8], bv[8];
        double al = 0.0, be = 0.0;
        double2 g = cz();
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const int y = lane + 32 * q;
          if (y < Mw) {
            av[q] = a[y];
            bv[q] = b[y];
            al += abs2(av[q]);
            be += abs2(bv[q]);
            cfmac(g, av[q], bv[q]);
          }
        }
        al = warp_sum(al);
        be = warp_sum(be);
        g.x = warp_sum(g.x);
        g.y = warp_sum(g.y);
        const double gab = hypot(g.x, g.y);
        if (!(gab > tol * sqrt(al) * sqrt(be))) continue;
        const double zeta = (be - al) / (2.0 * gab);
        double t;
        if (fabs(zeta) > 1e150) t = 0.5 / zeta;
        else t = copysign(1.0, zeta) / (fabs(zeta) + sqrt(fma(zeta, zeta, 1.0)));
        const double c = 1.0 / sqrt(fma(t, t, 1.0));
        const double s = t * c;
        // e = conj(g)/|g|
        const double2 e = make_double2(g.x / gab, -g.y / gab);
        const double2 se = cscale(e, s), ce = cscale(e, c);
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const int y = lane + 32 * q;
          if (y < Mw) {
            const double2 eb_s = cmul(se, bv[q]);
            const double2 eb_c = cmul(ce, bv[q]);
            a[y] = make_double2(c * av[q].x - eb_s.x, c * av[q].y - eb_s.y);
            b[y] = make_double2(s * av[q].x + eb_c.x, s * av[q].y + eb_c.y);
          }
        }
        if (lane == 0) sm.flag = 1;
      }
      __syncthreads();
    }
    if (sm.flag == 0) break;
    __syncthreads();
  }
  return sweep + 1;
}

// Column norms -> sigma, descending permutation (ties by index).
__device__ void sort_sigma(const double2* W, int Mw, int Nw, Smem& sm) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int c = warp; c < Nw; c += NWARP) {
    double s = 0.0;
    for (int y = lane; y < Mw; y += 32) s += abs2(W[(size_t)c * Mw + y]);
    s = warp_sum(s);
    if (lane == 0) sm.sig[c] = sqrt(s);
  }
  __syncthreads();
  for (int c = threadIdx.x; c < Nw; c += NT) {
    const double v = sm.sig[c];
    int rank = 0;
    for (int d = 0; d < Nw; ++d) {
      const double u = sm.sig[d];
      rank += (u > v) || (u == v && d < c);
    }
    sm.perm[rank] = c;
  }
  __syncthreads();
}

// Phase profiling (clock64 counters summed into Job::prof) is compiled in only
// for diagnostics builds (-DTB_PROF=1, libtepai_b200_prof.so, used by tools/);
// the product library has no clock reads, no profiling atomics and no
// registers held for them in the hot loops.
#ifndef TB_PROF
#define TB_PROF 0
#endif
__device__ __forceinline__ long long prof_clock() { return TB_PROF ? clock64() : 0ll; }
// per-step clocks inside the QRCP loop: a clock64 read per sub-phase costs a
// few % of the loop, so they are compiled in only for phase studies
#ifndef TB_PHASE_CLOCKS
#define TB_PHASE_CLOCKS 0
#endif
__device__ __forceinline__ long long prof_fine() { return TB_PHASE_CLOCKS ? clock64() : 0ll; }

constexpr int JB = 32;  // columns per block

__device__ __forceinline__ double2 lds2(uint32_t a) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts2(uint32_t a, double2 v) {
  asm volatile("st.shared.v2.f64 [%0], {%1, %2};" ::"r"(a), "d"(v.x), "d"(v.y) : "memory");
}

__device__ __forceinline__ int ld_acquire(const int* p) {  // shared, CTA scope
  int v;
  asm volatile("ld.acquire.cta.shared.u32 %0, [%1];" : "=r"(v) : "r"((uint32_t)__cvta_generic_to_shared(p)) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.cta.shared.u32 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(p)), "r"(v) : "memory");
}

// Rotation of one pair in the "tau" form.  With g = a^H b, d = beta - alpha,
// the Jacobi angle is t = 2|g| sgn(d) / (|d| + sqrt(d^2 + 4|g|^2)) and the
// unitary update a' = c (a - t e b), b' = c (b + t conj(e) a), e = conj(g)/|g|,
// c = 1/sqrt(1+t^2).  Writing t e = tau conj(g) with
//   tau = t / |g| = 2 sgn(d) / (|d| + sqrt(d^2 + 4|g|^2))
// removes the normalisation of e (a full-precision rsqrt) from the chain, and
// c = 1/sqrt(1 + tau^2 |g|^2) keeps the transform EXACTLY unitary for any tau:
// tau only sets the angle, so it is evaluated from the MUFU seeds alone
// (~2^-21 relative; the pair's coupling then drops to ~5e-7 of its value
// instead of to rounding, far below the sweep's quadratic rate).  c needs
// full precision (it enters the column scales) and gets two Newton steps.
// About 20 fewer FP64 instructions per pair and half the dependency depth of
// the former (t, c, e) evaluation — the scalar parameter math, executed by
// all 16 lanes of a half, was half of the FP64 pipe's busy time (r02a ncu:
// DMUL 13.2e12 vs DFMA 26.1e12 thread instructions).
struct Rot {
  double c, tau, tg, g2;
  bool rot;
};
__device__ __forceinline__ void atomic_max_pos(double* a, double v) {  // v >= 0
  atomicMax((unsigned long long*)a, (unsigned long long)__double_as_longlong(v));
}

// A pair is left alone when it is orthogonal to relative precision
// (|g|^2 <= tol2 alpha beta); it then gets tau = 0 and c = 1 (the exact identity).
// Branch-free FP64 reciprocal square root for well-scaled positive
// arguments: MUFU seed + Newton steps (2 steps: ~1 ulp).
__device__ __forceinline__ double rsqrt_nr(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double h = 0.5 * x;
  y = y * fma(-h * y, y, 1.5);
  y = y * fma(-h * y, y, 1.5);
  return y;
}

__device__ __forceinline__ Rot rot_params(double gr, double gi, double al, double be, bool valid, double tol2) {
  Rot p;
  p.g2 = fma(gr, gr, gi * gi);
  p.rot = valid && (p.g2 > tol2 * al * be);
  const double d = be - al;
  const double h2 = p.rot ? fma(d, d, 4.0 * p.g2) : 1.0;
  double y, r;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(h2));
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(fabs(d) + h2 * y));
  p.tau = p.rot ? copysign(2.0, d) * r : 0.0;
  p.c = p.rot ? rsqrt_nr(fma(p.tau * p.tau, p.g2, 1.0)) : 1.0;
  p.tg = p.tau * p.g2;  // t |g|: the exact norm transfer alpha' = alpha - t|g|, beta' = beta + t|g|
  return p;
}

// ----------------------------------------------------------------------------
// Half-warp Jacobi (Mw <= 128, Nw <= 128).  A column lives in one half-warp
// (16 lanes x HR rows), so a warp works on two independent pairs whose
// reductions are 4-level butterflies inside each half and whose rotation
// parameters are evaluated by the half that owns the pair — no cross-half
// transposition and no parameter broadcast.  Same block schedule as
// JacobiSmem (3 smem slots + 1 L2 slot of 32 columns); in a cross phase each
// of the 32 half-warps holds one P column in registers and the 32 Q columns
// rotate through the halves (round r: half k takes Q column (k + r) mod 32),
// ordered by per-column counters instead of CTA barriers.
// ----------------------------------------------------------------------------
template <int HR>
struct HCol {
  double2 v[HR];
};

template <int HR>
__device__ __forceinline__ void hcol_lds(HCol<HR>& c, uint32_t a) {
  const uint32_t l = (threadIdx.x & 15) * 16u;
#pragma unroll
  for (int q = 0; q < HR; ++q) c.v[q] = lds2(a + l + 256u * q);
}
template <int HR>
__device__ __forceinline__ void hcol_sts(uint32_t a, const HCol<HR>& c) {
  const uint32_t l = (threadIdx.x & 15) * 16u;
#pragma unroll
  for (int q = 0; q < HR; ++q) sts2(a + l + 256u * q, c.v[q]);
}
template <int HR>
__device__ __forceinline__ void hcol_ldg(HCol<HR>& c, const double2* p, int Mw) {
  const int l = threadIdx.x & 15;
#pragma unroll
  for (int q = 0; q < HR; ++q) {
    const int y = l + 16 * q;
    c.v[q] = (y < Mw) ? p[y] : cz();
  }
}
template <int HR>
__device__ __forceinline__ void hcol_stg(double2* p, const HCol<HR>& c, int Mw) {
  const int l = threadIdx.x & 15;
#pragma unroll
  for (int q = 0; q < HR; ++q) {
    const int y = l + 16 * q;
    if (y < Mw) p[y] = c.v[q];
  }
}

// Scaled ("fast") rotation of one pair.  Columns are stored as a = da * A,
// b = db * B with real scales, and the unitary update
//   a' = c (a - t E b),  b' = c (b + t conj(E) a)
// becomes A' = A - f1 B, B' = B + f2 A with f1 = t E db/da, f2 = t conj(E) da/db
// while the factor c moves into the scales (da' = c da, db' = c db): 8 DFMA
// per complex row pair instead of 12.  B' goes straight to shared memory
// (predicated on `st`); A' is either kept in registers (KEEP_A, the resident
// P column of a cross phase) or stored as well.
template <int HR, bool KEEP_A>
__device__ __forceinline__ void apply_rot_s(HCol<HR>& a, const HCol<HR>& b, uint32_t sa, uint32_t sb, bool st,
                                            double f1r, double f1i, double f2r, double f2i) {
  const uint32_t l = (threadIdx.x & 15) * 16u;
#pragma unroll
  for (int q = 0; q < HR; ++q) {
    const double2 x = a.v[q], y = b.v[q];
    double2 nb, na;
    nb.x = fma(f2r, x.x, fma(-f2i, x.y, y.x));
    nb.y = fma(f2r, x.y, fma(f2i, x.x, y.y));
    na.x = fma(-f1r, y.x, fma(f1i, y.y, x.x));
    na.y = fma(-f1r, y.y, fma(-f1i, y.x, x.y));
    if (st) sts2(sb + l + 256u * q, nb);
    if (KEEP_A) a.v[q] = na;
    else if (st) sts2(sa + l + 256u * q, na);
  }
}

__device__ __forceinline__ double rcp_acc(double x) {  // ~1 ulp
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  y = y * fma(-x, y, 2.0);
  y = y * fma(-x, y, 2.0);
  return y;
}

__device__ __forceinline__ double half_sum(double v) {
  v += __shfl_xor_sync(0xffffffffu, v, 8);
  v += __shfl_xor_sync(0xffffffffu, v, 4);
  v += __shfl_xor_sync(0xffffffffu, v, 2);
  v += __shfl_xor_sync(0xffffffffu, v, 1);
  return v;
}

// Sum of eight values over the 16 lanes of each half-warp, returned to every
// lane of the half: a transposed reduction (8 + 4 + 2 + 1 lane-pair exchanges
// keep halving the values each lane carries, the last step pairs lanes l and
// l ^ 1) and one broadcast shuffle per value — 16 double shuffles instead of
// the 32 of eight separate butterflies, in one dependency chain instead of eight.
__device__ __forceinline__ void half_sum8(double (&v)[8]) {
  const unsigned full = 0xffffffffu;
  const int l = threadIdx.x & 15;
  const bool b3 = l & 8, b2 = l & 4, b1 = l & 2;
  double a[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const double send = b3 ? v[k] : v[k + 4], keep = b3 ? v[k + 4] : v[k];
    a[k] = keep + __shfl_xor_sync(full, send, 8);
  }
  double b[2];
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const double send = b2 ? a[k] : a[k + 2], keep = b2 ? a[k + 2] : a[k];
    b[k] = keep + __shfl_xor_sync(full, send, 4);
  }
  double c = (b1 ? b[1] : b[0]) + __shfl_xor_sync(full, b1 ? b[0] : b[1], 2);
  c += __shfl_xor_sync(full, c, 1);
  // value k now sits on lanes 2k and 2k + 1 of the half (bits 3..1 of the lane)
  const int base = threadIdx.x & 16;
#pragma unroll
  for (int k = 0; k < 8; ++k) v[k] = __shfl_sync(full, c, base | (2 * k));
}

constexpr double kTailTol2 = 1e-8;  // (relative coupling 1e-4)^2 for pairs of two tail columns
#ifndef TB_GRAM_UNROLL
#define TB_GRAM_UNROLL 2  // k-steps of the Gram loop in flight (4: measured)
#endif
constexpr double kScreenOn = 1e-2;  // Gram-screen the next sweep once a sweep's largest rotated coupling^2 is below this

// ----------------------------------------------------------------------------
// Tail skipping for truncated splits.  The caller keeps only the kcut largest
// singular triplets (k <= min(chi_cut, K), _kernel.py:118-131).  Let T be a
// set of small columns whose total weight sum_T |a|^2 is below half of the
// kcut-th largest |a|^2.  Once every pair with at least one column outside T
// has converged, the columns outside T are exact singular vectors, the T block
// is orthogonal to them, and the largest singular value of the T block (at
// most its Frobenius norm) lies below the kcut-th singular value.  The kept
// triplets, the count k and the discarded weight (total - kept, total = the
// Frobenius norm) are therefore those of the full SVD, and T-T pairs need no
// exact orthogonality.  They are still rotated down to a relative coupling of
// 1e-4 (kTailTol2): leaving them fully coupled turns the convergence of the
// kept-tail pairs linear (each kept column would chase a non-orthogonal tail
// basis), while the last orders of magnitude — the late-sweep tail work — are
// skipped.  T is fixed after the first sweep (chg bit 2) and re-checked with
// the converged norms; a failed check clears T and the sweeps go on.
// ----------------------------------------------------------------------------
template <class Live>
__device__ __forceinline__ void tail_rank(const Smem& sm, int ncol, Live live, int c, double a, int& rank,
                                          double& suffix) {
  rank = 0;
  suffix = 0.0;
  for (int j = 0; j < ncol; ++j) {
    if (!live(j)) continue;
    const double b = sm.nrm[j];
    const bool before = b > a || (b == a && j < c);
    rank += before ? 1 : 0;
    suffix += before ? 0.0 : b;
  }
}

// mark T (chg bit 2); returns |T| (CTA-uniform)
template <class Live>
__device__ int mark_tail(Smem& sm, int ncol, Live live) {
  const int c = threadIdx.x;
  const bool me = c < ncol && live(c);
  const int nlive = __syncthreads_count(me);
  if (nlive <= sm.kcut) return 0;
  const double a = me ? sm.nrm[c] : 0.0;
  int rank = 0;
  double suf = 0.0;
  if (me) {
    tail_rank(sm, ncol, live, c, a, rank, suf);
    if (rank == sm.kcut - 1) sm.invsig_tmp = 0.5 * a;
  }
  __syncthreads();
  const bool t = me && rank >= sm.kcut && suf < sm.invsig_tmp;
  if (c < ncol) sm.chg[c] = t ? (sm.chg[c] | 4) : (sm.chg[c] & ~4);
  const int nt = __syncthreads_count(t);
  if (threadIdx.x == 0) sm.ntail = nt;
  return nt;
}

// true when the converged norms still certify T (see above); otherwise T is
// cleared and every column is flagged as changed so that all pairs are swept
template <class Live>
__device__ bool tail_ok(Smem& sm, int ncol, Live live) {
  const int c = threadIdx.x;
  const bool me = c < ncol && live(c);
  if (me) {
    int rank;
    double suf;
    tail_rank(sm, ncol, live, c, sm.nrm[c], rank, suf);
    if (rank == sm.kcut - 1) sm.invsig_tmp = 0.5 * sm.nrm[c];
  }
  const bool t = me && (sm.chg[c] & 4);
  __syncthreads();
  if (threadIdx.x < 32) {
    double st = 0.0;
    for (int j = threadIdx.x; j < ncol; j += 32)
      if (live(j) && (sm.chg[j] & 4)) st += sm.nrm[j];
    st = warp_sum(st);
    if (threadIdx.x == 0) sm.red[0] = (st < sm.invsig_tmp) ? 1.0 : 0.0;
  }
  __syncthreads();
  const bool ok = sm.red[0] != 0.0;
  (void)t;
  if (!ok && c < ncol) sm.chg[c] = (sm.chg[c] & ~4) | 2;
  __syncthreads();
  if (!ok && threadIdx.x == 0) sm.ntail = 0;
  return ok;
}

// one pair per half-warp; `valid` may differ between the halves.  na / nb are
// the TRUE squared norms, da / db the column scales; sa / sb the shared-memory
// homes of the two columns (written only when THIS half rotates).  Returns
// whether this half rotated.  Branches are warp-uniform (a non-rotating half
// applies the exact identity: f1 = f2 = 0, c = 1, and stores nothing).
template <int HR, bool KEEP_A>
__device__ __forceinline__ bool rot_half(HCol<HR>& a, const HCol<HR>& b, uint32_t sa, uint32_t sb, double& na,
                                         double& nb, double& da, double& db, bool valid, double tol2,
                                         double& offmax) {
  // two partial sums: four accumulators shorten the dependent-FMA chain but
  // measured 4% slower overall (register allocation of the cross loop)
  double2 g = cz(), h = cz();
#pragma unroll
  for (int q = 0; q < HR; q += 2) {
    cfmac(g, a.v[q], b.v[q]);
    if (q + 1 < HR) cfmac(h, a.v[q + 1], b.v[q + 1]);
  }
  double gr = g.x + h.x, gi = g.y + h.y;
  gr = half_sum(gr);
  gi = half_sum(gi);
  const double dd = da * db;
  gr *= dd;
  gi *= dd;
  const Rot p = rot_params(gr, gi, na, nb, valid, tol2);
  const bool mine = p.rot;
  if (mine) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(na * nb));
    offmax = fmax(offmax, p.g2 * r);
  }
  const double nan_ = na - p.tg, nbn = nb + p.tg;
  if (__any_sync(0xffffffffu, mine)) {
    // f1 = t e db/da = tau conj(g) db/da, f2 = t conj(e) da/db = tau g da/db
    const double inv = rcp_acc(dd);
    const double r1 = p.tau * db * db * inv, r2 = p.tau * da * da * inv;
    apply_rot_s<HR, KEEP_A>(a, b, sa, sb, mine, gr * r1, -gi * r1, gr * r2, gi * r2);
    da *= p.c;
    db *= p.c;
  }
  const bool fa = mine && nan_ < 0.5 * na, fb = mine && nbn < 0.5 * nb;
  na = nan_;
  nb = nbn;
  if (__any_sync(0xffffffffu, fa || fb)) {  // cancellation: exact norms of the new columns
    const uint32_t l = (threadIdx.x & 15) * 16u;
    double ea = 0.0, eb = 0.0;
#pragma unroll
    for (int q = 0; q < HR; ++q) {
      ea += abs2(KEEP_A ? a.v[q] : lds2(sa + l + 256u * q));
      eb += abs2(lds2(sb + l + 256u * q));
    }
    ea = half_sum(ea) * (da * da);
    eb = half_sum(eb) * (db * db);
    if (fa) na = ea;
    if (fb) nb = eb;
  }
  return mine;
}

template <int HR>
struct JacobiH {
  static constexpr int LD = 16 * HR;        // padded rows per smem column
  static constexpr uint32_t CB = LD * 16u;  // bytes per smem column
  uint32_t base;                            // smem byte address of slot A
  double2* G;                               // global block (columns 96..127, ld = Mw)
  int Mw, nblk;
  double tol2, offmax;
  bool screen;   // this sweep visits only the pairs flagged by gram_screen
  bool swapped;  // slots 0 and 3 have exchanged their contents since the screen was taken

  __device__ uint32_t scol(int s, int c) const { return base + (uint32_t)(s * JB + c) * CB; }

  // ---------------------------------------------------------------------------
  // Gram screen of a late sweep, on the FP64 tensor cores.  From the third
  // sweep on most pairs are already orthogonal to working precision, yet a
  // rotation visit still pays for the column load, the dot product, its
  // butterfly reduction and the rotation parameters only to find that out.
  // Instead, right after refresh_norms (scales folded, exact norms), the whole
  // Gram matrix G = A^H A of the <= 128 column slots is formed with DMMA
  // (mma.sync.m8n8k4.f64: 16x16 complex blocks of 2x2 tiles per warp, upper
  // triangle only, fragments read straight from the Jacobi column slots; the
  // fourth block from its global home), and every pair whose relative
  // coupling |g|^2 / (|a|^2 |b|^2) exceeds half the rotation threshold is
  // flagged in sm.pbits.  The sweep then visits only flagged pairs; an empty
  // screen is the convergence certificate (every pair orthogonal at this very
  // moment — no rotation has happened since the Gram was taken).  Same
  // rotations, same thresholds (tail pairs: kTailTol2), so the computed SVD is
  // that of the unscreened sweep up to the order of negligible rotations.
  // Returns (CTA-uniform) whether any pair is flagged.
  // ---------------------------------------------------------------------------
  __device__ __forceinline__ double2 gram_ld(int col, int row) const {
    if (col < 3 * JB) return lds2(base + (uint32_t)col * CB + 16u * row);
    return (row < Mw) ? G[(size_t)(col - 3 * JB) * Mw + row] : cz();
  }
  __device__ __noinline__ int gram_screen(Smem& sm) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int fr = lane >> 2, fk = lane & 3;
    uint32_t* bits = &sm.pbits[0][0];
    constexpr int WPR = SROWS / 32;  // bitmap words per row
    for (int e = threadIdx.x; e < SROWS * WPR; e += NT) bits[e] = 0u;
    if (threadIdx.x == 0) sm.blkmask = 0u;
    __syncthreads();
    const int nt = 2 * nblk, ntile = nt * (nt + 1) / 2;
    const double thr = 0.5 * tol2;
    bool mine = false;
    unsigned blk = 0u;
    for (int t = warp; t < ntile; t += NWARP) {
      int bi = 0, rem = t;
      while (rem >= nt - bi) {
        rem -= nt - bi;
        ++bi;
      }
      const int bj = bi + rem;
      double cre[2][2][2], cim[2][2][2];
#pragma unroll
      for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int b = 0; b < 2; ++b) cre[a][b][0] = cre[a][b][1] = cim[a][b][0] = cim[a][b][1] = 0.0;
#if TB_GRAM_UNROLL == 4
#pragma unroll 4
#else
#pragma unroll 2
#endif
      for (int k0 = 0; k0 < LD; k0 += 4) {
        const int row = k0 + fk;
        double2 x[2], y[2];
#pragma unroll
        for (int a = 0; a < 2; ++a) x[a] = gram_ld(bi * 16 + 8 * a + fr, row);
#pragma unroll
        for (int b = 0; b < 2; ++b) y[b] = (bi == bj) ? x[b] : gram_ld(bj * 16 + 8 * b + fr, row);
#pragma unroll
        for (int a = 0; a < 2; ++a) {
          const double nxi = -x[a].y;
#pragma unroll
          for (int b = 0; b < 2; ++b) {
            // g = conj(x) y: re = xr yr + xi yi, im = xr yi - xi yr
            dmma(cre[a][b][0], cre[a][b][1], x[a].x, y[b].x);
            dmma(cre[a][b][0], cre[a][b][1], x[a].y, y[b].y);
            dmma(cim[a][b][0], cim[a][b][1], x[a].x, y[b].y);
            dmma(cim[a][b][0], cim[a][b][1], nxi, y[b].x);
          }
        }
      }
#pragma unroll
      for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int b = 0; b < 2; ++b)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int i = bi * 16 + 8 * a + fr, j = bj * 16 + 8 * b + 2 * fk + e;
            if (i < j && (i & (JB - 1)) < sm.jncol[i / JB] && (j & (JB - 1)) < sm.jncol[j / JB]) {
              const double lim = ((sm.chg[i] & sm.chg[j] & 4) ? kTailTol2 : thr) * sm.nrm[i] * sm.nrm[j];
              const double g2 = fma(cre[a][b][e], cre[a][b][e], cim[a][b][e] * cim[a][b][e]);
              if (g2 > lim) {
                atomicOr(&bits[i * WPR + (j >> 5)], 1u << (j & 31));
                atomicOr(&bits[j * WPR + (i >> 5)], 1u << (i & 31));
                blk |= 1u << (4 * (i / JB) + j / JB);
                mine = true;
              }
            }
          }
    }
    blk = __reduce_or_sync(0xffffffffu, blk);
    if (lane == 0 && blk) atomicOr(&sm.blkmask, blk);
    return __syncthreads_or(mine ? 1 : 0);
  }
  // some pair between column blocks a <= b (positions at the sweep's start) needs a visit
  __device__ __forceinline__ bool blk_any(unsigned bm, int a, int b) const { return (bm >> (4 * a + b)) & 1u; }
  // column positions are those of the sweep's start: after the mid-sweep
  // exchange of slots 0 and 3 a position maps back to where the screen saw it
  __device__ __forceinline__ int opos(int c) const {
    return swapped ? (c < JB ? c + 3 * JB : (c >= 3 * JB ? c - 3 * JB : c)) : c;
  }
  __device__ __forceinline__ bool flagged(const Smem& sm, int ci, int cj) const {
    if (!screen) return true;
    ci = opos(ci);
    cj = opos(cj);
    return (sm.pbits[ci][cj >> 5] >> (cj & 31)) & 1u;
  }

  // Round robin inside up to three smem slots.  The slot-rounds are
  // enumerated as m = round * ns + slot and each CTA-wide step takes two of
  // them (halves 0-15: m = 2k, halves 16-31: m = 2k + 1; a slot-round has at
  // most 16 pairs).  For ns >= 2 the two slot-rounds of a step touch
  // different slots, and a slot's consecutive rounds (m, m + ns) always fall
  // in different steps, so one barrier per step orders everything.
  // Within-block phase of a SCREENED sweep: the flagged pairs of the round
  // robin only, ordered by per-column counters instead of one CTA barrier per
  // round.  Half (g, p) (g = hw / 16, p = hw % 16) owns position p of the
  // circle method in the slot-rounds with (round + slot) odd/even = g and walks
  // them in increasing round order; a pair runs once the flagged pairs of BOTH
  // its columns from earlier rounds have released them (a column's counter
  // counts its flagged visits; the number that precede a round is read off the
  // column's bitmap row with the inverse of the circle method).  A column's
  // pairs therefore run in round order, exactly as in within(), and a wait
  // always points to a strictly earlier round, so the walk cannot deadlock;
  // the two halves of a warp advance independently as in cross_screened.
  __device__ __forceinline__ static int rr_round(int i, int j, int Np) {
    const int m = Np - 1;  // odd
    if (i == m) return j;
    if (j == m) return i;
    return ((i + j) * ((m + 1) >> 1)) % m;
  }
  __device__ void within_screened(int s0, int s1, int s2, int ns, Smem& sm) {
    const unsigned full = 0xffffffffu;
    const int hw = threadIdx.x >> 4, hl = threadIdx.x & 15;
    const int base = threadIdx.x & 16, g = hw >> 4, p = hw & 15;
    bool any = false;
    if (threadIdx.x < 3 * 32) sm.qcnt[threadIdx.x] = 0;
    __syncthreads();
    int rounds = 0;
    for (int x = 0; x < ns; ++x) {
      const int nb = sm.jncol[x == 0 ? s0 : (x == 1 ? s1 : s2)];
      rounds = max(rounds, nb + (nb & 1) - 1);
    }
    // scan position: slot-rounds in (round, slot) order
    int r = 0, x = 0;
    bool want = false;
    int s = 0, i = 0, j = 0, nbp = 2;
    auto advance = [&]() {  // next flagged pair of this half at or after (r, x); want = false when exhausted
      want = false;
      while (r < rounds) {
        if (((r + x) & 1) == g) {
          s = (x == 0) ? s0 : (x == 1 ? s1 : s2);
          const int nb = sm.jncol[s];
          nbp = nb + (nb & 1);
          if (r < nbp - 1 && p < nbp / 2) {
            rr_pair(r, p, nbp, i, j);
            if (i < nb && j < nb && flagged(sm, s * JB + i, s * JB + j)) {
              want = true;
              return;
            }
          }
        }
        if (++x == ns) {
          x = 0;
          ++r;
        }
      }
    };
    auto step = [&]() {
      if (++x == ns) {
        x = 0;
        ++r;
      }
    };
    advance();
    while (__any_sync(full, want)) {
      // flagged pairs of column i (and of column j) in earlier rounds: lanes check partners hl and hl + 16
      const int nb = sm.jncol[s];
      int need_i = 0, need_j = 0;
      {
        const int ci = opos(s * JB + i), cj = opos(s * JB + j);
        const unsigned rowi = sm.pbits[ci][ci >> 5], rowj = sm.pbits[cj][cj >> 5];
        bool bi0 = false, bi1 = false, bj0 = false, bj1 = false;
        if (want) {
          const int a = hl, b = hl + 16;
          bi0 = a < nb && a != i && ((rowi >> a) & 1u) && rr_round(i, a, nbp) < r;
          bi1 = b < nb && b != i && ((rowi >> b) & 1u) && rr_round(i, b, nbp) < r;
          bj0 = a < nb && a != j && ((rowj >> a) & 1u) && rr_round(j, a, nbp) < r;
          bj1 = b < nb && b != j && ((rowj >> b) & 1u) && rr_round(j, b, nbp) < r;
        }
        const unsigned hm = 0xFFFFu << base;
        need_i = __popc(__ballot_sync(full, bi0) & hm) + __popc(__ballot_sync(full, bi1) & hm);
        need_j = __popc(__ballot_sync(full, bj0) & hm) + __popc(__ballot_sync(full, bj1) & hm);
      }
      int* cnti = &sm.qcnt[(s < 3 ? s : 0) * 32 + i];
      int* cntj = &sm.qcnt[(s < 3 ? s : 0) * 32 + j];
      int ready = 0;
      if (hl == 0 && want) ready = ld_acquire(cnti) >= need_i && ld_acquire(cntj) >= need_j;
      const bool valid = __shfl_sync(full, ready, base) != 0;
      __syncwarp();
      if (!__any_sync(full, valid)) continue;  // neither half can go yet
      const unsigned ci8 = sm.chg[s * JB + i], cj8 = sm.chg[s * JB + j];
      const bool tt = (ci8 & cj8 & 4) != 0;
      HCol<HR> a, b;
      const uint32_t ai = scol(s, i), aj = scol(s, j);
      hcol_lds(a, ai);
      hcol_lds(b, aj);
      double na = valid ? sm.nrm[s * JB + i] : 0.0, nb2 = valid ? sm.nrm[s * JB + j] : 0.0;
      double da = sm.dsc[s * JB + i], db = sm.dsc[s * JB + j];
      const bool rr = rot_half<HR, false>(a, b, ai, aj, na, nb2, da, db, valid, tt ? kTailTol2 : tol2, offmax);
      if (rr) {
        any = true;
        if (hl == 0) {
          sm.nrm[s * JB + i] = na;
          sm.nrm[s * JB + j] = nb2;
          sm.dsc[s * JB + i] = da;
          sm.dsc[s * JB + j] = db;
          sm.chg[s * JB + i] |= 2;
          sm.chg[s * JB + j] |= 2;
        }
      }
      __syncwarp();  // the half's column stores are ordered before lane 0's releases
      if (valid) {
        if (hl == 0) {
          st_release(cnti, need_i + 1);
          st_release(cntj, need_j + 1);
        }
        step();
        advance();
      }
    }
    __syncthreads();
    if (__any_sync(full, any) && (threadIdx.x & 31) == 0) sm.flag = 1;
    __syncthreads();
  }

  __device__ void within(int s0, int s1, int s2, int ns, Smem& sm) {
    if (screen && sm.screen_on > 2) {
      within_screened(s0, s1, s2, ns, sm);
      return;
    }
    const int hw = threadIdx.x >> 4;  // half-warp id 0..31
    const int hl = threadIdx.x & 15;
    int rounds = 0;
    for (int x = 0; x < ns; ++x) {
      const int nb = sm.jncol[x == 0 ? s0 : (x == 1 ? s1 : s2)];
      rounds = max(rounds, nb + (nb & 1) - 1);
    }
    const int per = ns >= 2 ? 2 : 1;
    const int nsteps = (rounds * ns + per - 1) / per;
    bool any = false;
    for (int k = 0; k < nsteps; ++k) {
      const int m = per * k + (hw >> 4), p = hw & 15;
      const int r = m / ns, x = m - r * ns;
      bool valid = false, tt = false;
      int s = 0, i = 0, j = 0;
      if ((hw >> 4) < per && r < rounds) {
        s = (x == 0) ? s0 : (x == 1 ? s1 : s2);
        const int nb = sm.jncol[s], nbp = nb + (nb & 1);
        if (r < nbp - 1 && p < nbp / 2) {
          rr_pair(r, p, nbp, i, j);
          const unsigned ci = sm.chg[s * JB + i], cj = sm.chg[s * JB + j];
          valid = i < nb && j < nb && ((ci | cj) & 1) && flagged(sm, s * JB + i, s * JB + j);
          tt = (ci & cj & 4) != 0;
        }
      }
      if (__any_sync(0xffffffffu, valid)) {
        // unconditional loads: slot columns past the live count are zeros
        // and a non-rotating half applies the exact identity
        HCol<HR> a, b;
        const uint32_t ai = scol(s, i), aj = scol(s, j);
        hcol_lds(a, ai);
        hcol_lds(b, aj);
        double na = valid ? sm.nrm[s * JB + i] : 0.0, nb2 = valid ? sm.nrm[s * JB + j] : 0.0;
        double da = sm.dsc[s * JB + i], db = sm.dsc[s * JB + j];
        const bool rr = rot_half<HR, false>(a, b, ai, aj, na, nb2, da, db, valid, tt ? kTailTol2 : tol2, offmax);
        if (rr) {
          any = true;
          if (hl == 0) {
            sm.nrm[s * JB + i] = na;
            sm.nrm[s * JB + j] = nb2;
            sm.dsc[s * JB + i] = da;
            sm.dsc[s * JB + j] = db;
            sm.chg[s * JB + i] |= 2;
            sm.chg[s * JB + j] |= 2;
          }
        }
      }
      __syncthreads();
    }
    if (__any_sync(0xffffffffu, any) && (threadIdx.x & 31) == 0) sm.flag = 1;
    __syncthreads();
  }

  // P column of half k (slot sp) against the Q columns of up to three smem
  // slots sq0..sq{S-1}.  Visit (m, x) (round S*m + x): half k takes column
  // (k + m) mod 32 of slot x.  A Q column is therefore touched every S rounds
  // (by halves k, k-1, ...), so with S > 1 the halves may drift apart by S
  // rounds instead of running in lockstep — their latency-bound stretches
  // (reductions, rotation parameters) then overlap other halves' FP64 work.
  __device__ void cross(HCol<HR>& pc, double& np, double& dp, int nP, int sp, int sq0, int sq1, int sq2, int S,
                        Smem& sm) {
    if (screen && sm.screen_on > 1) {
      cross_screened(pc, np, dp, sp, sq0, sq1, sq2, S, sm);
      return;
    }
    const int hw = threadIdx.x >> 4, hl = threadIdx.x & 15;
    const bool vp = hw < nP;
    bool any = false;
    if (threadIdx.x < 3 * 32) sm.qcnt[threadIdx.x] = 0;
    __syncthreads();
    const long long tc0 = prof_clock();
    for (int m = 0; m < 32; ++m) {
      const int c = (hw + m) & 31;  // Q column handled by this half in visit m
      for (int x = 0; x < S; ++x) {
        const int sq = x == 0 ? sq0 : (x == 1 ? sq1 : sq2);
        int* cnt = &sm.qcnt[x * 32 + c];
        if (m > 0) {  // acquire the previous visit's column (lane 0), then share it via the warp barrier
          if (hl == 0)
            while (ld_acquire(cnt) < m) {}
          __syncwarp();
        }
        const unsigned cp = sm.chg[sp * JB + hw], cq = sm.chg[sq * JB + c];
        const bool valid = vp && c < sm.jncol[sq] && ((cp | cq) & 1) && flagged(sm, sp * JB + hw, sq * JB + c);
        const double tl2 = (cp & cq & 4) ? kTailTol2 : tol2;
        if (__any_sync(0xffffffffu, valid)) {
          HCol<HR> q;
          const uint32_t aq = scol(sq, c);
          hcol_lds(q, aq);  // unconditional (see within)
          double nq = valid ? sm.nrm[sq * JB + c] : 0.0, dq = sm.dsc[sq * JB + c];
          const double npo = np;
          const bool rr = rot_half<HR, true>(pc, q, 0u, aq, np, nq, dp, dq, valid, tl2, offmax);
          if (!valid) np = npo;
          if (rr) {
            any = true;
            if (hl == 0) {
              sm.nrm[sq * JB + c] = nq;
              sm.dsc[sq * JB + c] = dq;
              sm.chg[sp * JB + hw] |= 2;
              sm.chg[sq * JB + c] |= 2;
            }
          }
        }
        __syncwarp();  // the half's column stores are ordered before lane 0's release
        if (hl == 0) st_release(cnt, m + 1);
      }
    }
    __syncthreads();
    if (__any_sync(0xffffffffu, any) && (threadIdx.x & 31) == 0) sm.flag = 1;
    if (threadIdx.x == 0 && TB_PROF && sm.prof) atomicAdd(&sm.prof[14], (unsigned long long)(prof_clock() - tc0));
  }

  // Cross phase of a SCREENED sweep: only the flagged pairs are visited, and
  // only they synchronise.  Half k still takes its Q columns in the order of
  // cross() (visit m: column (k + m) mod 32 of each slot), but walks the set
  // bits of its row of the screen bitmap; a column's counter counts its
  // FLAGGED visits, and a visit waits until the flagged visits that precede it
  // in that column's order (halves k+1 .. k+m, read off the column's bitmap
  // row) have released it.  The two halves of a warp advance independently:
  // a half whose next visit is not ready idles for one round (an exact
  // identity inside rot_half) instead of blocking its sibling, so the walk
  // cannot deadlock.  Same pairs, same per-column and per-half order as the
  // unscreened phase restricted to the flagged pairs: deterministic.
  __device__ void cross_screened(HCol<HR>& pc, double& np, double& dp, int sp, int sq0, int sq1, int sq2, int S,
                                 Smem& sm) {
    const unsigned full = 0xffffffffu;
    const int hw = threadIdx.x >> 4, hl = threadIdx.x & 15;
    const int base = threadIdx.x & 16;
    bool any = false;
    if (threadIdx.x < 3 * 32) sm.qcnt[threadIdx.x] = 0;
    __syncthreads();
    const long long tc0 = prof_clock();
    const int po = opos(sp * JB + hw), pw = opos(sp * JB) >> 5;  // my row, and the P block's bitmap word
    // pending visits per slot: bit m <-> column (hw + m) mod 32
    auto pend = [&](int sq) {
      const unsigned row = sm.pbits[po][opos(sq * JB) >> 5];
      return __funnelshift_r(row, row, hw);
    };
    unsigned r0 = pend(sq0), r1 = S > 1 ? pend(sq1) : 0u, r2 = S > 2 ? pend(sq2) : 0u;
    const unsigned cp = sm.chg[sp * JB + hw];
    while (__any_sync(full, (r0 | r1 | r2) != 0u)) {
      int m = 32, x = 0;
      if (r0) m = __ffs((int)r0) - 1;
      if (r1 && __ffs((int)r1) - 1 < m) {
        m = __ffs((int)r1) - 1;
        x = 1;
      }
      if (r2 && __ffs((int)r2) - 1 < m) {
        m = __ffs((int)r2) - 1;
        x = 2;
      }
      const bool want = m < 32;
      const int c = want ? (hw + m) & 31 : 0;
      const int sq = x == 0 ? sq0 : (x == 1 ? sq1 : sq2);
      int* cnt = &sm.qcnt[x * 32 + c];
      // flagged visits of column c that come before mine: halves hw+1 .. hw+m
      int need = 0;
      int ready = 0;
      if (hl == 0 && want) {
        const unsigned col = sm.pbits[opos(sq * JB + c)][pw];
        need = __popc(__funnelshift_r(col, col, (hw + 1) & 31) & ((1u << m) - 1u));
        ready = ld_acquire(cnt) >= need;
      }
      need = __shfl_sync(full, need, base);
      const bool valid = __shfl_sync(full, ready, base) != 0;
      __syncwarp();  // lane 0's acquire is shared with its half before the column loads
      if (!__any_sync(full, valid)) continue;  // neither half can go yet: look again
      if (valid) {
        const unsigned bit = ~(1u << m);
        if (x == 0) r0 &= bit;
        else if (x == 1) r1 &= bit;
        else r2 &= bit;
      }
      const unsigned cq = sm.chg[sq * JB + c];
      const double tl2 = (cp & cq & 4) ? kTailTol2 : tol2;
      HCol<HR> q;
      const uint32_t aq = scol(sq, c);
      hcol_lds(q, aq);  // unconditional: an idle half applies the exact identity
      double nq = valid ? sm.nrm[sq * JB + c] : 0.0, dq = sm.dsc[sq * JB + c];
      const double npo = np;
      const bool rr = rot_half<HR, true>(pc, q, 0u, aq, np, nq, dp, dq, valid, tl2, offmax);
      if (!valid) np = npo;
      if (rr) {
        any = true;
        if (hl == 0) {
          sm.nrm[sq * JB + c] = nq;
          sm.dsc[sq * JB + c] = dq;
          sm.chg[sp * JB + hw] |= 2;
          sm.chg[sq * JB + c] |= 2;
        }
      }
      __syncwarp();  // the half's column stores are ordered before lane 0's release
      if (hl == 0 && valid) st_release(cnt, need + 1);
    }
    __syncthreads();
    if (__any_sync(full, any) && (threadIdx.x & 31) == 0) sm.flag = 1;
    if (threadIdx.x == 0 && TB_PROF && sm.prof) atomicAdd(&sm.prof[14], (unsigned long long)(prof_clock() - tc0));
  }

  __device__ void load_p(HCol<HR>& pc, double& np, double& dp, int s, Smem& sm) {
    const int hw = threadIdx.x >> 4;
    if (s < 3) hcol_lds(pc, scol(s, hw));
    else hcol_ldg(pc, G + (size_t)hw * Mw, Mw);
    np = sm.nrm[s * JB + hw];
    dp = sm.dsc[s * JB + hw];
  }
  __device__ void store_p(const HCol<HR>& pc, double np, double dp, int s, Smem& sm) {
    const int hw = threadIdx.x >> 4;
    if (s < 3) hcol_sts(scol(s, hw), pc);
    else hcol_stg(G + (size_t)hw * Mw, pc, Mw);
    if ((threadIdx.x & 15) == 0) {
      sm.nrm[s * JB + hw] = np;
      sm.dsc[s * JB + hw] = dp;
    }
  }

  // multiply every stored column by its scale and reset the scales to 1
  __device__ void fold_scales(Smem& sm, bool first) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (!first) {
      for (int c = warp; c < JB * nblk; c += NWARP) {
        const double d = sm.dsc[c];
        if (d == 1.0) continue;
        const int s = c / JB, k = c - s * JB;
        if (s < 3) {
          for (int y = lane; y < LD; y += 32) {
            const uint32_t a = scol(s, k) + 16u * y;
            sts2(a, cscale(lds2(a), d));
          }
        } else {
          double2* p = G + (size_t)k * Mw;
          for (int y = lane; y < Mw; y += 32) p[y] = cscale(p[y], d);
        }
      }
    }
    __syncthreads();
    for (int c = threadIdx.x; c < JB * nblk; c += NT) sm.dsc[c] = 1.0;
    __syncthreads();
  }

  // fold the scales into the columns and take exact norms in one pass
  __device__ void refresh_norms(Smem& sm, double tol, bool first) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int c = warp; c < JB * nblk; c += NWARP) {
      const int s = c / JB, k = c - s * JB;
      const double d = first ? 1.0 : sm.dsc[c];
      double acc = 0.0;
      if (s < 3) {
        for (int y = lane; y < LD; y += 32) {
          const uint32_t a = scol(s, k) + 16u * y;
          double2 v = lds2(a);
          if (d != 1.0) {
            v = cscale(v, d);
            sts2(a, v);
          }
          acc += abs2(v);
        }
      } else {
        double2* p = G + (size_t)k * Mw;
        for (int y = lane; y < Mw; y += 32) {
          double2 v = p[y];
          if (d != 1.0) {
            v = cscale(v, d);
            p[y] = v;
          }
          acc += abs2(v);
        }
      }
      acc = warp_sum(acc);
      if (lane == 0) sm.nrm[c] = acc;
    }
    __syncthreads();  // every column folded before the scales are reset
    for (int c = threadIdx.x; c < JB * nblk; c += NT) {
      sm.dsc[c] = 1.0;
      sm.chg[c] = first ? 1 : (((sm.chg[c] >> 1) & 1) | (sm.chg[c] & 4));
    }
    if (threadIdx.x < 32) {
      double t = 0.0;
      for (int c = threadIdx.x; c < JB * nblk; c += 32) t += sm.nrm[c];
      t = warp_sum(t);
      if (threadIdx.x == 0) {
        sm.scale = t;
        sm.flag = 0;
        sm.offmax = 0.0;
      }
    }
    __syncthreads();
    tol2 = tol * tol;
    const double dead = 1e-28 * sm.scale;
    for (int c = warp; c < JB * nblk; c += NWARP) {
      const double v = sm.nrm[c];
      if (v < dead && v > 0.0) {
        const int s = c / JB, k = c - s * JB;
        if (s < 3) {
          for (int y = lane; y < LD; y += 32) sts2(scol(s, k) + 16u * y, cz());
        } else {
          double2* p = G + (size_t)k * Mw;
          for (int y = lane; y < Mw; y += 32) p[y] = cz();
        }
        if (lane == 0) sm.nrm[c] = 0.0;
      }
    }
    __syncthreads();
  }

  __device__ void sweep(Smem& sm) {
    offmax = 0.0;
    swapped = false;
    const int nsm = min(nblk, 3);
    const long long tw0 = prof_clock();
    // screened sweep: whole phases without a flagged pair are skipped
    const unsigned bm = screen ? sm.blkmask : 0xFFFFu;
    if (blk_any(bm, 0, 0) || blk_any(bm, 1, 1) || blk_any(bm, 2, 2)) within(0, 1, 2, nsm, sm);
    if (threadIdx.x == 0 && TB_PROF && sm.prof) atomicAdd(&sm.prof[13], (unsigned long long)(prof_clock() - tw0));
    HCol<HR> pc;
    double np, dp;
    if (nblk == 4) {
      const bool g33 = blk_any(bm, 3, 3), g0x = blk_any(bm, 0, 1) || blk_any(bm, 0, 2);
      if (blk_any(bm, 0, 3) || blk_any(bm, 1, 3) || blk_any(bm, 2, 3) || g33 || g0x) {
      load_p(pc, np, dp, 3, sm);
      cross(pc, np, dp, sm.jncol[3], 3, 0, 1, 2, 3, sm);
      // swap contents of A and G (P holds the current G columns)
      const long long tsw = prof_clock();
      {
        HCol<HR> t;
        double nt, dt;
        load_p(t, nt, dt, 0, sm);
        const int hw = threadIdx.x >> 4;
        unsigned char fa = sm.chg[hw], fg = sm.chg[3 * JB + hw];
        __syncthreads();
        store_p(pc, np, dp, 0, sm);
        store_p(t, nt, dt, 3, sm);
        if ((threadIdx.x & 15) == 0) {
          sm.chg[hw] = fg;
          sm.chg[3 * JB + hw] = fa;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
          const int na = sm.jncol[0];
          sm.jncol[0] = sm.jncol[3];
          sm.jncol[3] = na;
        }
        __syncthreads();
        swapped = true;
      }
      if (threadIdx.x == 0 && TB_PROF && sm.prof) atomicAdd(&sm.prof[27], (unsigned long long)(prof_clock() - tsw));
      if (g33) within(0, 0, 0, 1, sm);  // the former block 3
      if (g0x) {                        // the former block 0 (now in slot 3) against blocks 1, 2
        load_p(pc, np, dp, 3, sm);
        cross(pc, np, dp, sm.jncol[3], 3, 1, 2, 2, 2, sm);
        store_p(pc, np, dp, 3, sm);
        __syncthreads();
      }
      }
      if (blk_any(bm, 1, 2)) {
        load_p(pc, np, dp, 1, sm);
        cross(pc, np, dp, sm.jncol[1], 1, 2, 2, 2, 1, sm);
        store_p(pc, np, dp, 1, sm);
        __syncthreads();
      }
    } else {
      for (int sp = 0; sp + 1 < nsm; ++sp) {
        if (!(blk_any(bm, sp, sp + 1) || blk_any(bm, sp, 2))) continue;
        load_p(pc, np, dp, sp, sm);
        cross(pc, np, dp, sm.jncol[sp], sp, sp + 1, sp + 2, sp + 2, nsm - 1 - sp, sm);
        store_p(pc, np, dp, sp, sm);
        __syncthreads();
      }
    }
    if ((threadIdx.x & 15) == 0 && offmax > 0.0) atomic_max_pos(&sm.offmax, offmax);
  }
};

template <int HR>
__device__ int jacobi_half(double2* W, int Mw, int Nw, Smem& sm, double2* smem) {
  JacobiH<HR> J;
  constexpr int LD = JacobiH<HR>::LD;
  J.Mw = Mw;
  J.nblk = (Nw + JB - 1) / JB;
  J.base = (uint32_t)__cvta_generic_to_shared(smem);
  J.G = W + (size_t)3 * JB * Mw;
  const long long tj0 = prof_clock();
  int start[5];
  start[0] = 0;
  int ncl[4];
  for (int b = 0; b < 4; ++b) {
    ncl[b] = (b < J.nblk) ? (Nw / J.nblk + (b < Nw % J.nblk ? 1 : 0)) : 0;
    start[b + 1] = start[b] + ncl[b];
  }
  __syncthreads();
  if (threadIdx.x < 4) sm.jncol[threadIdx.x] = ncl[threadIdx.x];
#ifndef TB_TOLSCALE
#define TB_TOLSCALE 1.0
#endif
  const double tol = fmax(sqrt((double)Mw), 4.0) * 4.440892098500626e-16 * TB_TOLSCALE;
  const int nsm = min(J.nblk, 3);
  if (J.nblk == 4) {
    // block 3 moves to G (columns 96..127 of W), overlapping its source
    // columns: bounce it through the not yet filled shared-memory slots
    for (int e = threadIdx.x; e < JB * Mw; e += NT) {
      const int k = e / Mw, y = e - k * Mw;
      smem[e] = (k < ncl[3]) ? W[(size_t)(start[3] + k) * Mw + y] : cz();
    }
    __syncthreads();
    for (int e = threadIdx.x; e < JB * Mw; e += NT) J.G[e] = smem[e];
    __syncthreads();
  }
  for (int e = threadIdx.x; e < nsm * JB * LD; e += NT) {
    const int c = e / LD, y = e - c * LD;
    const int sb = c / JB, k = c - sb * JB;
    smem[e] = (k < ncl[sb] && y < Mw) ? W[(size_t)(start[sb] + k) * Mw + y] : cz();
  }
  __syncthreads();
  if (threadIdx.x == 0 && TB_PROF && sm.prof) atomicAdd(&sm.prof[25], (unsigned long long)(prof_clock() - tj0));
  auto live = [&](int c) { return (c & (JB - 1)) < sm.jncol[c / JB]; };
  if (threadIdx.x == 0) sm.ntail = 0;
  int sweep = 0;
  bool conv = false;
  double offprev = 1.0;  // largest relative coupling (squared) rotated in the previous sweep
  J.screen = J.swapped = false;
  for (; sweep < sm.maxsweep; ++sweep) {
    const long long ts0 = prof_clock();
    J.refresh_norms(sm, tol, sweep == 0);
    if (sweep == 1) mark_tail(sm, JB * J.nblk, live);
    if (threadIdx.x == 0 && TB_PROF && sm.prof) atomicAdd(&sm.prof[26], (unsigned long long)(prof_clock() - ts0));
    // late sweeps (the previous one rotated nothing above a relative coupling
    // of kScreenOn): visit only the pairs the tensor-core Gram screen flags
    J.screen = false;
    if (HR >= 4 && sm.screen_on && sweep >= 2 && J.nblk >= 2 && offprev < kScreenOn) {
      const long long tg0 = prof_clock();
      const int any = J.gram_screen(sm);
      if (threadIdx.x == 0 && TB_PROF && sm.prof) {
        atomicAdd(&sm.prof[38], (unsigned long long)(prof_clock() - tg0));
        atomicAdd(&sm.prof[39], 1ull);
      }
      if (!any) {  // every pair orthogonal right now: converged
        if (sm.ntail > 0 && !tail_ok(sm, JB * J.nblk, live)) continue;
        conv = true;
        break;
      }
      J.screen = true;
    }
    J.sweep(sm);
    __syncthreads();
    offprev = sm.offmax;
    if (threadIdx.x == 0 && TB_PROF && sm.prof && Mw == 128 && sweep < 16) {
      atomicAdd(&sm.prof[40 + sweep], (unsigned long long)(prof_clock() - ts0));
      atomicAdd(&sm.prof[56 + min(sweep, 7)], 1ull);
    }
    if (sm.flag == 0 || sm.offmax < 1e-16 * TB_TOLSCALE) {
      if (sm.ntail > 0 && !tail_ok(sm, JB * J.nblk, live)) continue;
      conv = true;
      break;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) sm.sweeps = sweep + 1;
  const long long tw0 = prof_clock();
  J.fold_scales(sm, false);
  for (int e = threadIdx.x; e < nsm * JB * Mw; e += NT) {
    const int c = e / Mw, y = e - c * Mw;
    W[(size_t)c * Mw + y] = smem[(size_t)c * LD + y];
  }
  __syncthreads();
  if (threadIdx.x == 0 && TB_PROF && sm.prof) atomicAdd(&sm.prof[28], (unsigned long long)(prof_clock() - tw0));
  const int neff = (J.nblk == 1) ? Nw : JB * J.nblk;
  return conv ? neff : -neff;
}

#if !TB_ENGINE_SMALL  // chi = 128 paths (wide / cluster Jacobi): not in the small-problem engine
// ----------------------------------------------------------------------------
// Wide Jacobi (Mw <= 256 rows, Nw <= 256 columns: the chi = 128 problems).
// A column is 256 rows = 4 KB, so only one block of 32 columns fits in shared
// memory.  The columns stay in global memory (L2) in blocks of <= 32; a sweep
// takes every block once as the register-resident P block (one column per
// half-warp, 16 lanes x 16 rows) and streams the later blocks through the
// shared-memory slot as Q (same counter-ordered cross phase as JacobiH), plus
// a round robin inside each block.  Shared-memory columns are streamed in
// row chunks (4 rows per lane) so a pair never holds two full columns in
// registers.  Same scaled rotations, convergence test and dead-column rule
// as the half-warp Jacobi.
// ----------------------------------------------------------------------------
struct JacobiW {
  static constexpr int HR = 16, CH = 4;     // rows per lane, rows per streamed chunk
  static constexpr int LD = 16 * HR;        // 256 padded rows per smem column
  static constexpr uint32_t CB = LD * 16u;  // bytes per smem column
  uint32_t base;
  double2* W;
  int Mw, Nw, nblk;
  int start[9], ncl[8];
  double tol2, offmax;

  __device__ uint32_t scol(int c) const { return base + (uint32_t)c * CB; }
  __device__ uint32_t lrow() const { return (threadIdx.x & 15) * 16u; }

  __device__ void stage(int b) {
    const int nc = ncl[b], c0 = start[b];
    for (int e = threadIdx.x; e < JB * LD; e += NT) {
      const int c = e / LD, y = e - c * LD;
      const double2 v = (c < nc && y < Mw) ? W[(size_t)(c0 + c) * Mw + y] : cz();
      sts2(scol(c) + 16u * y, v);
    }
    __syncthreads();
  }
  __device__ void unstage(int b) {
    const int nc = ncl[b], c0 = start[b];
    for (int e = threadIdx.x; e < nc * Mw; e += NT) {
      const int c = e / Mw, y = e - c * Mw;
      W[(size_t)(c0 + c) * Mw + y] = lds2(scol(c) + 16u * y);
    }
    __syncthreads();
  }

  // rotation of the pair (a, b); a in registers (KEEP_A) or in smem at sa,
  // b in smem at sb.  na/nb true squared norms, da/db scales.
  template <bool A_REG>
  __device__ __forceinline__ bool rot(HCol<HR>& a, uint32_t sa, uint32_t sb, double& na, double& nb, double& da,
                                      double& db, bool valid, double tl2) {
    const uint32_t l = lrow();
    double2 g = cz(), h = cz();
#pragma unroll
    for (int q0 = 0; q0 < HR; q0 += CH) {
      double2 x[CH], y[CH];
#pragma unroll
      for (int q = 0; q < CH; ++q) {
        x[q] = A_REG ? a.v[q0 + q] : lds2(sa + l + 256u * (q0 + q));
        y[q] = lds2(sb + l + 256u * (q0 + q));
      }
#pragma unroll
      for (int q = 0; q < CH; q += 2) {
        cfmac(g, x[q], y[q]);
        cfmac(h, x[q + 1], y[q + 1]);
      }
    }
    double gr = half_sum(g.x + h.x), gi = half_sum(g.y + h.y);
    const double dd = da * db;
    gr *= dd;
    gi *= dd;
    const Rot p = rot_params(gr, gi, na, nb, valid, tl2);
    const bool mine = p.rot;
    if (mine) {
      double r;
      asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(na * nb));
      offmax = fmax(offmax, p.g2 * r);
    }
    const double nan_ = na - p.tg, nbn = nb + p.tg;
    if (__any_sync(0xffffffffu, mine)) {
      const double inv = rcp_acc(dd);
      const double r1 = p.tau * db * db * inv, r2 = p.tau * da * da * inv;
      const double f1r = gr * r1, f1i = -gi * r1, f2r = gr * r2, f2i = gi * r2;
#pragma unroll
      for (int q0 = 0; q0 < HR; q0 += CH) {
#pragma unroll
        for (int q = 0; q < CH; ++q) {
          const uint32_t o = l + 256u * (q0 + q);
          const double2 x = A_REG ? a.v[q0 + q] : lds2(sa + o);
          const double2 y = lds2(sb + o);
          double2 nx, ny;
          ny.x = fma(f2r, x.x, fma(-f2i, x.y, y.x));
          ny.y = fma(f2r, x.y, fma(f2i, x.x, y.y));
          nx.x = fma(-f1r, y.x, fma(f1i, y.y, x.x));
          nx.y = fma(-f1r, y.y, fma(-f1i, y.x, x.y));
          if (mine) sts2(sb + o, ny);
          if (A_REG) a.v[q0 + q] = nx;
          else if (mine) sts2(sa + o, nx);
        }
      }
      da *= p.c;
      db *= p.c;
    }
    const bool fa = mine && nan_ < 0.5 * na, fb = mine && nbn < 0.5 * nb;
    na = nan_;
    nb = nbn;
    if (__any_sync(0xffffffffu, fa || fb)) {
      double ea = 0.0, eb = 0.0;
#pragma unroll
      for (int q = 0; q < HR; ++q) {
        ea += abs2(A_REG ? a.v[q] : lds2(sa + l + 256u * q));
        eb += abs2(lds2(sb + l + 256u * q));
      }
      ea = half_sum(ea) * (da * da);
      eb = half_sum(eb) * (db * db);
      if (fa) na = ea;
      if (fb) nb = eb;
    }
    return mine;
  }

  // round robin inside the staged block b (16 pairs per round at most)
  __device__ void within(int b, Smem& sm) {
    const int hw = threadIdx.x >> 4, hl = threadIdx.x & 15;
    const int nb = ncl[b], nbp = nb + (nb & 1), c0 = start[b];
    bool any = false;
    for (int r = 0; r < nbp - 1; ++r) {
      int i = 0, j = 0;
      bool valid = false, tt = false;
      if (hw < nbp / 2) {
        rr_pair(r, hw, nbp, i, j);
        const unsigned ci = sm.chg[c0 + i], cj = sm.chg[c0 + j];
        valid = i < nb && j < nb && ((ci | cj) & 1);
        tt = (ci & cj & 4) != 0;
      }
      if (__any_sync(0xffffffffu, valid)) {
        HCol<HR> dummy;
        double na = valid ? sm.nrm[c0 + i] : 0.0, nb2 = valid ? sm.nrm[c0 + j] : 0.0;
        double da = sm.dsc[c0 + i], db = sm.dsc[c0 + j];
        if (rot<false>(dummy, scol(i), scol(j), na, nb2, da, db, valid, tt ? kTailTol2 : tol2)) {
          any = true;
          if (hl == 0) {
            sm.nrm[c0 + i] = na;
            sm.nrm[c0 + j] = nb2;
            sm.dsc[c0 + i] = da;
            sm.dsc[c0 + j] = db;
            sm.chg[c0 + i] |= 2;
            sm.chg[c0 + j] |= 2;
          }
        }
      }
      __syncthreads();
    }
    if (__any_sync(0xffffffffu, any) && (threadIdx.x & 31) == 0) sm.flag = 1;
  }

  // P block bp (one column per half, in registers) against staged block bq
  __device__ void cross(HCol<HR>& pc, double& np, double& dp, int bp, int bq, Smem& sm) {
    const int hw = threadIdx.x >> 4, hl = threadIdx.x & 15;
    const int nP = ncl[bp], nQ = ncl[bq], p0 = start[bp], q0 = start[bq];
    const bool vp = hw < nP;
    bool any = false;
    if (threadIdx.x < 32) sm.qcnt[threadIdx.x] = 0;
    __syncthreads();
    for (int r = 0; r < 32; ++r) {
      const int c = (hw + r) & 31;
      if (r > 0) {
        if (hl == 0)
          while (ld_acquire(&sm.qcnt[c]) < r) {}
        __syncwarp();
      }
      const unsigned cp = sm.chg[p0 + hw], cq = sm.chg[q0 + c];
      const bool valid = vp && c < nQ && ((cp | cq) & 1);
      const double tl2 = (cp & cq & 4) ? kTailTol2 : tol2;
      if (__any_sync(0xffffffffu, valid)) {
        double nq = valid ? sm.nrm[q0 + c] : 0.0, dq = c < nQ ? sm.dsc[q0 + c] : 1.0;
        const double npo = np;
        const bool rr = rot<true>(pc, 0u, scol(c), np, nq, dp, dq, valid, tl2);
        if (!valid) np = npo;
        if (rr) {
          any = true;
          if (hl == 0) {
            sm.nrm[q0 + c] = nq;
            sm.dsc[q0 + c] = dq;
            sm.chg[p0 + hw] |= 2;
            sm.chg[q0 + c] |= 2;
          }
        }
      }
      __syncwarp();
      if (hl == 0) st_release(&sm.qcnt[c], r + 1);
    }
    __syncthreads();
    if (__any_sync(0xffffffffu, any) && (threadIdx.x & 31) == 0) sm.flag = 1;
  }

  __device__ void fold_and_norms(Smem& sm, double tol, bool first) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int c = warp; c < Nw; c += NWARP) {
      const double d = first ? 1.0 : sm.dsc[c];
      double2* p = W + (size_t)c * Mw;
      double acc = 0.0;
      for (int y = lane; y < Mw; y += 32) {
        double2 v = p[y];
        if (d != 1.0) {
          v = cscale(v, d);
          p[y] = v;
        }
        acc += abs2(v);
      }
      acc = warp_sum(acc);
      if (lane == 0) sm.nrm[c] = acc;
    }
    __syncthreads();  // every column folded before the scales are reset
    for (int c = threadIdx.x; c < Nw; c += NT) {
      sm.dsc[c] = 1.0;
      sm.chg[c] = first ? 1 : (((sm.chg[c] >> 1) & 1) | (sm.chg[c] & 4));
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int c = 0; c < Nw; ++c) t += sm.nrm[c];
      sm.scale = t;
      sm.flag = 0;
      sm.offmax = 0.0;
    }
    __syncthreads();
    tol2 = tol * tol;
    const double dead = 1e-28 * sm.scale;
    for (int c = warp; c < Nw; c += NWARP) {
      const double v = sm.nrm[c];
      if (v < dead && v > 0.0) {
        double2* p = W + (size_t)c * Mw;
        for (int y = lane; y < Mw; y += 32) p[y] = cz();
        if (lane == 0) sm.nrm[c] = 0.0;
      }
    }
    __syncthreads();
  }

  __device__ void sweep(Smem& sm) {
    offmax = 0.0;
    const int hw = threadIdx.x >> 4;
    for (int bp = 0; bp < nblk; ++bp) {
      stage(bp);
      within(bp, sm);
      HCol<HR> pc;
      double np = 0.0, dp = 1.0;
      const bool more = bp + 1 < nblk;
      if (more) {  // P straight from the staged block
        const uint32_t l = lrow();
#pragma unroll
        for (int q = 0; q < HR; ++q) pc.v[q] = lds2(scol(hw) + l + 256u * q);
        if (hw < ncl[bp]) {
          np = sm.nrm[start[bp] + hw];
          dp = sm.dsc[start[bp] + hw];
        }
      }
      __syncthreads();
      unstage(bp);
      if (!more) break;
      for (int bq = bp + 1; bq < nblk; ++bq) {
        stage(bq);
        cross(pc, np, dp, bp, bq, sm);
        unstage(bq);
      }
      if (hw < ncl[bp]) {
        double2* p = W + (size_t)(start[bp] + hw) * Mw;
        const int l = threadIdx.x & 15;
#pragma unroll
        for (int q = 0; q < HR; ++q) {
          const int y = l + 16 * q;
          if (y < Mw) p[y] = pc.v[q];
        }
        if ((threadIdx.x & 15) == 0) {
          sm.nrm[start[bp] + hw] = np;
          sm.dsc[start[bp] + hw] = dp;
        }
      }
      __syncthreads();
    }
    if ((threadIdx.x & 15) == 0 && offmax > 0.0) atomic_max_pos(&sm.offmax, offmax);
  }
};

__device__ int jacobi_wide(double2* W, int Mw, int Nw, Smem& sm, double2* smem) {
  JacobiW J;
  J.W = W;
  J.Mw = Mw;
  J.Nw = Nw;
  J.nblk = (Nw + JB - 1) / JB;
  J.base = (uint32_t)__cvta_generic_to_shared(smem);
  J.start[0] = 0;
  for (int b = 0; b < 8; ++b) {
    J.ncl[b] = (b < J.nblk) ? (Nw / J.nblk + (b >= J.nblk - Nw % J.nblk ? 1 : 0)) : 0;
    J.start[b + 1] = J.start[b] + J.ncl[b];
  }
  const double tol = fmax(sqrt((double)Mw), 4.0) * 4.440892098500626e-16 * TB_TOLSCALE;
  auto live = [](int) { return true; };
  if (threadIdx.x == 0) sm.ntail = 0;
  __syncthreads();
  int sweep = 0;
  bool conv = false;
  for (; sweep < sm.maxsweep; ++sweep) {
    J.fold_and_norms(sm, tol, sweep == 0);
    if (sweep == 1) mark_tail(sm, Nw, live);
    J.sweep(sm);
    __syncthreads();
    if (sm.flag == 0 || sm.offmax < 1e-16 * TB_TOLSCALE) {
      if (sm.ntail > 0 && !tail_ok(sm, Nw, live)) continue;
      conv = true;
      break;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) sm.sweeps = sweep + 1;
  // fold the final scales
  {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int c = warp; c < Nw; c += NWARP) {
      const double d = sm.dsc[c];
      if (d == 1.0) continue;
      double2* p = W + (size_t)c * Mw;
      for (int y = lane; y < Mw; y += 32) p[y] = cscale(p[y], d);
    }
  }
  __syncthreads();
  return conv ? Nw : -Nw;
}

// ----------------------------------------------------------------------------
// Cluster Jacobi: the chi = 128 problems (Mw <= 256 rows x Nw <= 256 columns,
// 1 MB of complex128) held in the DISTRIBUTED shared memory of an 8-CTA
// thread-block cluster instead of streaming through L2 (jacobi_wide).
//
// The columns form 16 blocks of <= 16; CTA r of the cluster homes blocks 2r
// and 2r+1 in its shared memory (256 padded rows x 16 B = 4 KB per column,
// 128 KB per CTA).  A sweep is
//   * a within-block round robin of each CTA's two home blocks (warps 0-7 and
//     8-15, one pair per warp per round), then
//   * the 15 rounds of the circle method over the 16 blocks.  Each round is a
//     perfect matching of the blocks; every CTA takes exactly ONE matched pair
//     (X, Y) in which Y is one of its own home blocks (the matching, seen as a
//     2-regular multigraph on the CTAs, is oriented along its cycles), loads
//     the 16 columns of X into registers (one column per warp, 8 rows per lane)
//     over DSMEM, rotates them against the 16 local columns of Y in 16 rounds
//     (warp w: X_w against Y_(w+r) mod 16), and writes X back to its home CTA.
// A column lives in one whole warp, so a pair's reductions are 5-level
// butterflies and its rotation parameters need no broadcast.  Same scaled
// (tau-form) rotations, pair skipping, dead-column rule and convergence test
// as the single-CTA paths; the per-sweep flag / largest off-diagonal and the
// Frobenius norm are reduced over the cluster in fixed rank order, so every
// CTA takes the same branch and the result is deterministic.
//
// The leader CTA (rank 0) runs the whole circuit; ranks 1..7 wait in
// cluster_follow() for a command posted through the leader's shared memory.
// Replaces the zgesdd of /root/reference/pkg/src/tepai/_kernel.py:117 at
// 2*chi = 256 (SURVEY.md §8 north_star (1)).
// ----------------------------------------------------------------------------
constexpr int CL = 8;            // CTAs per cluster
constexpr int CNB = 2 * CL;      // column blocks
constexpr int CBC = 16;          // max columns per block
constexpr uint32_t CCB = 4096u;  // bytes per shared-memory column (256 rows)

__device__ __forceinline__ int cl_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return (int)r;
}
__device__ __forceinline__ void cl_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t sh_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t cl_map(uint32_t a, int rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
__device__ __forceinline__ double2 ldc2(uint32_t a) {
  double2 v;
  asm volatile("ld.shared::cluster.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ void stc2(uint32_t a, double2 v) {
  asm volatile("st.shared::cluster.v2.f64 [%0], {%1, %2};" ::"r"(a), "d"(v.x), "d"(v.y) : "memory");
}
__device__ __forceinline__ double ldcf(uint32_t a) {
  double v;
  asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ void stcf(uint32_t a, double v) {
  asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(a), "d"(v) : "memory");
}
__device__ __forceinline__ uint32_t ldcu(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared::cluster.u32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ uint64_t ldcl(uint32_t a) {
  uint64_t v;
  asm volatile("ld.shared::cluster.u64 %0, [%1];" : "=l"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t ldcb(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared::cluster.u8 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ void stcb(uint32_t a, uint32_t v) {
  asm volatile("st.shared::cluster.u8 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}

// TMA bulk copies (cp.async.bulk) between global and shared memory, completed
// through an mbarrier (global -> smem) or a bulk group (smem -> global)
__device__ __forceinline__ void mbar_init(uint32_t a, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t a, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(a), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t a, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "TB_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra TB_WAIT_%=;\n}" ::"r"(a),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t mbar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(mbar)
               : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* dst, uint32_t src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(src), "r"(bytes)
               : "memory");
}

// Orientation of round s of the circle method: for CTA `rank`, the visiting
// block X (loaded into registers) and the home block Y, packed X | Y << 8.
__device__ void cluster_schedule(int rank, uint16_t* out) {
  for (int s = 0; s < CNB - 1; ++s) {
    int ea[CL], eb[CL], owner[CL];
    bool done[CL];
    ea[0] = CNB - 1;
    eb[0] = s;
    for (int p = 1; p < CL; ++p) {
      ea[p] = (s + p) % (CNB - 1);
      eb[p] = (s - p + CNB - 1) % (CNB - 1);
    }
    for (int e = 0; e < CL; ++e) {
      owner[e] = -1;
      done[e] = false;
    }
    // every CTA homes two blocks, so the matching is a 2-regular multigraph on
    // the CTAs: walk each cycle, giving every CTA the next unassigned edge
    for (int u0 = 0; u0 < CL; ++u0) {
      int u = u0;
      while (!done[u]) {
        int e = 0;
        while (owner[e] >= 0 || ((ea[e] >> 1) != u && (eb[e] >> 1) != u)) ++e;
        owner[e] = u;
        done[u] = true;
        const int y = ((ea[e] >> 1) == u) ? ea[e] : eb[e];
        const int x = (y == ea[e]) ? eb[e] : ea[e];
        if (u == rank) out[s] = (uint16_t)(x | (y << 8));
        u = x >> 1;
      }
    }
  }
}

struct JacobiC {
  uint32_t base;  // local shared address of home column slot 0
  double2* W;
  int Mw, Nw, rank;
  double tol2, offmax;

  // block b holds columns [start(b), start(b) + ncl(b)), balanced to within one
  __device__ int ncl(int b) const { return Nw / CNB + (b >= CNB - Nw % CNB ? 1 : 0); }
  __device__ int start(int b) const { return b * (Nw / CNB) + max(0, b - (CNB - Nw % CNB)); }

  __device__ uint32_t lcol(int b, int k) const { return base + (uint32_t)((b & 1) * CBC + k) * CCB; }
  __device__ uint32_t lrow() const { return (threadIdx.x & 31) * 16u; }

  // one pair: a in registers (A_REG) or local smem at sa; b in local smem at sb
  template <bool A_REG>
  __device__ __forceinline__ bool rot(HCol<8>& a, uint32_t sa, uint32_t sb, double& na, double& nb, double& da,
                                      double& db) {
    const uint32_t l = lrow();
    double2 x[8], y[8];
    double2 g = cz(), h = cz();
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      x[q] = A_REG ? a.v[q] : lds2(sa + l + 512u * q);
      y[q] = lds2(sb + l + 512u * q);
    }
#pragma unroll
    for (int q = 0; q < 8; q += 2) {
      cfmac(g, x[q], y[q]);
      cfmac(h, x[q + 1], y[q + 1]);
    }
    double gr = g.x + h.x, gi = g.y + h.y;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      gr += __shfl_xor_sync(0xffffffffu, gr, o);
      gi += __shfl_xor_sync(0xffffffffu, gi, o);
    }
    const double dd = da * db;
    gr *= dd;
    gi *= dd;
    const Rot p = rot_params(gr, gi, na, nb, true, tol2);
    if (!p.rot) return false;  // warp-uniform: every lane holds the same sums
    {
      double r;
      asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(na * nb));
      offmax = fmax(offmax, p.g2 * r);
    }
    const double nan_ = na - p.tg, nbn = nb + p.tg;
    const double inv = rcp_acc(dd);
    const double r1 = p.tau * db * db * inv, r2 = p.tau * da * da * inv;
    const double f1r = gr * r1, f1i = -gi * r1, f2r = gr * r2, f2i = gi * r2;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const uint32_t o = l + 512u * q;
      double2 nx, ny;
      ny.x = fma(f2r, x[q].x, fma(-f2i, x[q].y, y[q].x));
      ny.y = fma(f2r, x[q].y, fma(f2i, x[q].x, y[q].y));
      nx.x = fma(-f1r, y[q].x, fma(f1i, y[q].y, x[q].x));
      nx.y = fma(-f1r, y[q].y, fma(-f1i, y[q].x, x[q].y));
      sts2(sb + o, ny);
      if (A_REG) a.v[q] = nx;
      else sts2(sa + o, nx);
    }
    da *= p.c;
    db *= p.c;
    const bool fa = nan_ < 0.5 * na, fb = nbn < 0.5 * nb;
    na = nan_;
    nb = nbn;
    if (fa || fb) {  // cancellation: re-evaluate the transferred norm from the data
      double ea = 0.0, eb = 0.0;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        ea += abs2(A_REG ? a.v[q] : lds2(sa + l + 512u * q));
        eb += abs2(lds2(sb + l + 512u * q));
      }
      ea = warp_sum(ea) * (da * da);
      eb = warp_sum(eb) * (db * db);
      if (fa) na = ea;
      if (fb) nb = eb;
    }
    return true;
  }

  // TMA staging: every home column is one bulk copy of Mw x 16 B straight into
  // its shared-memory slot (rows >= Mw and unused columns are zero-filled by
  // the threads), all completing on one mbarrier
  __device__ void load_home_tma(Smem& sm) {
    const uint32_t mbar = sh_addr(&sm.cl_mbar);
    if (threadIdx.x == 0) mbar_init(mbar, 1);
    for (int s = 0; s < 2; ++s) {
      const int b = 2 * rank + s, nc = ncl(b);
      for (int e = threadIdx.x; e < CBC * 256; e += NT) {
        const int k = e >> 8, y = e & 255;
        if (k >= nc || y >= Mw) sts2(lcol(b, k) + 16u * y, cz());
      }
    }
    // generic-proxy shared-memory traffic (earlier phases, the padding)
    // before the async-proxy writes; W was written by the leader (generic)
    asm volatile("fence.proxy.async.shared::cta;\n\tfence.proxy.async.global;" ::: "memory");
    __syncthreads();
    const int n0 = ncl(2 * rank), n1 = ncl(2 * rank + 1);
    if (threadIdx.x < 32) {
      if (threadIdx.x == 0) mbar_expect_tx(mbar, (uint32_t)((n0 + n1) * Mw * 16));
      __syncwarp();
      const int t = threadIdx.x, s = t >= n0 ? 1 : 0, k = t - s * n0;
      if (t < n0 + n1) {
        const int b = 2 * rank + s;
        bulk_g2s(lcol(b, k), W + (size_t)(start(b) + k) * Mw, (uint32_t)(Mw * 16), mbar);
      }
    }
    mbar_wait(mbar, 0);
  }

  __device__ void store_home_tma(Smem& sm) {
    const int warp = threadIdx.x >> 5;
    for (int t = warp; t < 2 * CBC; t += NWARP) {  // fold the scales in place
      const int b = 2 * rank + t / CBC, k = t % CBC;
      if (k >= ncl(b)) continue;
      const double d = sm.dsc[start(b) + k];
      if (d == 1.0) continue;
      const uint32_t col = lcol(b, k) + lrow();
#pragma unroll
      for (int q = 0; q < 8; ++q) sts2(col + 512u * q, cscale(lds2(col + 512u * q), d));
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    const int n0 = ncl(2 * rank), n1 = ncl(2 * rank + 1);
    if (threadIdx.x < 32) {
      const int t = threadIdx.x, s = t >= n0 ? 1 : 0, k = t - s * n0;
      if (t < n0 + n1) {
        const int b = 2 * rank + s;
        bulk_s2g(W + (size_t)(start(b) + k) * Mw, lcol(b, k), (uint32_t)(Mw * 16));
      }
      asm volatile("cp.async.bulk.commit_group;\n\tcp.async.bulk.wait_group 0;\n\tfence.proxy.async.global;" :::
                       "memory");
    }
  }

  __device__ void load_home() {
    for (int s = 0; s < 2; ++s) {
      const int b = 2 * rank + s, nc = ncl(b), c0 = start(b);
      for (int e = threadIdx.x; e < CBC * 256; e += NT) {
        const int k = e >> 8, y = e & 255;
        const double2 v = (k < nc && y < Mw) ? W[(size_t)(c0 + k) * Mw + y] : cz();
        sts2(lcol(b, k) + 16u * y, v);
      }
    }
    __syncthreads();
  }

  __device__ void store_home(const Smem& sm) {
    for (int s = 0; s < 2; ++s) {
      const int b = 2 * rank + s, nc = ncl(b), c0 = start(b);
      for (int e = threadIdx.x; e < nc * Mw; e += NT) {
        const int k = e / Mw, y = e - k * Mw;
        W[(size_t)(c0 + k) * Mw + y] = cscale(lds2(lcol(b, k) + 16u * y), sm.dsc[c0 + k]);
      }
    }
  }

  // fold the scales of the home columns into their data, refresh their
  // norms, reduce |W|_F^2 over the cluster (fixed rank order) and zero the
  // numerically dead columns
  __device__ void fold_norms(Smem& sm, bool first) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int t = warp; t < 2 * CBC; t += NWARP) {
      const int b = 2 * rank + t / CBC, k = t % CBC;
      if (k >= ncl(b)) continue;
      const int c = start(b) + k;
      const double d = first ? 1.0 : sm.dsc[c];
      const uint32_t col = lcol(b, k) + lrow();
      double acc = 0.0;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        double2 v = lds2(col + 512u * q);
        if (d != 1.0) {
          v = cscale(v, d);
          sts2(col + 512u * q, v);
        }
        acc += abs2(v);
      }
      acc = warp_sum(acc);
      if (lane == 0) {
        sm.nrm[c] = acc;
        sm.dsc[c] = 1.0;
        sm.chg[c] = first ? 1 : ((sm.chg[c] >> 1) & 1);
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      double part = 0.0;
      for (int s = 0; s < 2; ++s)
        for (int k = 0; k < ncl(2 * rank + s); ++k) part += sm.nrm[start(2 * rank + s) + k];
      stcf(cl_map(sh_addr(&sm.cl_part[rank]), 0), part);
      sm.flag = 0;
      sm.offmax = 0.0;
    }
    cl_sync();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int r = 0; r < CL; ++r) t += ldcf(cl_map(sh_addr(&sm.cl_part[r]), 0));
      sm.scale = t;
    }
    __syncthreads();
    const double dead = 1e-28 * sm.scale;
    for (int t = warp; t < 2 * CBC; t += NWARP) {
      const int b = 2 * rank + t / CBC, k = t % CBC;
      if (k >= ncl(b)) continue;
      const int c = start(b) + k;
      const double v = sm.nrm[c];
      if (v < dead && v > 0.0) {
        const uint32_t col = lcol(b, k) + lrow();
#pragma unroll
        for (int q = 0; q < 8; ++q) sts2(col + 512u * q, cz());
        if (lane == 0) sm.nrm[c] = 0.0;
      }
    }
    __syncthreads();
  }

  __device__ void within(Smem& sm) {
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int b = 2 * rank + (w >> 3), p = w & 7;
    const int nb = ncl(b), nbp = nb + (nb & 1), c0 = start(b);
    bool any = false;
    for (int r = 0; r < CBC - 1; ++r) {
      if (r < nbp - 1 && p < nbp / 2) {
        int i, j;
        rr_pair(r, p, nbp, i, j);
        if (i < nb && j < nb && (((sm.chg[c0 + i] | sm.chg[c0 + j]) & 1) || (sm.cl_tma & 4))) {
          double na = sm.nrm[c0 + i], nb2 = sm.nrm[c0 + j], da = sm.dsc[c0 + i], db = sm.dsc[c0 + j];
          HCol<8> unused;
          if (rot<false>(unused, lcol(b, i), lcol(b, j), na, nb2, da, db)) {
            any = true;
            if (lane == 0) {
              sm.nrm[c0 + i] = na;
              sm.nrm[c0 + j] = nb2;
              sm.dsc[c0 + i] = da;
              sm.dsc[c0 + j] = db;
              sm.chg[c0 + i] |= 2;
              sm.chg[c0 + j] |= 2;
            }
          }
        }
      }
      __syncthreads();
    }
    if (any && lane == 0) sm.flag = 1;
  }

  // visiting block X (home CTA X >> 1) against the local home block Y
  __device__ void cross(int X, int Y, Smem& sm) {
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int hx = X >> 1;
    const int nP = ncl(X), nQ = ncl(Y), p0 = start(X), q0 = start(Y);
    const bool vp = w < nP;
    HCol<8> pc;
    double np = 0.0, dp = 1.0;
    uint32_t cp = 0;
    const uint32_t pa = cl_map(lcol(X, w) + lrow(), hx);
    if (vp) {
#pragma unroll
      for (int q = 0; q < 8; ++q) pc.v[q] = ldc2(pa + 512u * q);
      np = ldcf(cl_map(sh_addr(&sm.nrm[p0 + w]), hx));
      dp = ldcf(cl_map(sh_addr(&sm.dsc[p0 + w]), hx));
      cp = ldcb(cl_map(sh_addr(&sm.chg[p0 + w]), hx));
    }
    bool any = false;
    for (int r = 0; r < CBC; ++r) {
      const int c = (w + r) & (CBC - 1);
      if (vp && c < nQ && (((cp | sm.chg[q0 + c]) & 1) || (sm.cl_tma & 4))) {
        double nq = sm.nrm[q0 + c], dq = sm.dsc[q0 + c];
        if (rot<true>(pc, 0u, lcol(Y, c), np, nq, dp, dq)) {
          any = true;
          cp |= 2;
          if (lane == 0) {
            sm.nrm[q0 + c] = nq;
            sm.dsc[q0 + c] = dq;
            sm.chg[q0 + c] |= 2;
          }
        }
      }
      __syncthreads();
    }
    if (vp) {
#pragma unroll
      for (int q = 0; q < 8; ++q) stc2(pa + 512u * q, pc.v[q]);
      if (lane == 0) {
        stcf(cl_map(sh_addr(&sm.nrm[p0 + w]), hx), np);
        stcf(cl_map(sh_addr(&sm.dsc[p0 + w]), hx), dp);
        stcb(cl_map(sh_addr(&sm.chg[p0 + w]), hx), cp);
      }
    }
    if (any && lane == 0) sm.flag = 1;
  }

  // cluster-wide "anything rotated" and largest relative off-diagonal of the
  // sweep; true when the sweep converged
  __device__ bool sweep_end(Smem& sm, int par) {
    if ((threadIdx.x & 31) == 0 && offmax > 0.0) atomic_max_pos(&sm.offmax, offmax);
    __syncthreads();
    if (threadIdx.x == 0) {
      const uint32_t fa = cl_map(sh_addr(&sm.cl_flag[par]), 0), oa = cl_map(sh_addr(&sm.cl_off[par]), 0);
      asm volatile("atom.shared::cluster.or.b32 _, [%0], %1;" ::"r"(fa), "r"(sm.flag) : "memory");
      asm volatile("atom.shared::cluster.max.u64 _, [%0], %1;" ::"r"(oa),
                   "l"((unsigned long long)__double_as_longlong(sm.offmax))
                   : "memory");
    }
    cl_sync();
    if (threadIdx.x == 0) {
      sm.cl_rflag = (int)ldcu(cl_map(sh_addr(&sm.cl_flag[par]), 0));
      sm.cl_roff = ldcf(cl_map(sh_addr(&sm.cl_off[par]), 0));
      if (rank == 0) {  // the other parity is next read after >= 1 more cluster barrier
        sm.cl_flag[par ^ 1] = 0;
        sm.cl_off[par ^ 1] = 0.0;
      }
    }
    __syncthreads();
    // Converged only after a sweep without a rotation.  The single-CTA paths
    // also stop once the largest rotated coupling^2 of a sweep is below 1e-16
    // (quadratic convergence); with that shortcut the cluster sweeps stopped
    // one sweep early in about one run out of three (orthogonality 1e-11 ..
    // 1e-7 instead of 1e-14, profiles/r02m_dbg_cluster.log), so it is off here
    // unless asked for (debug switch bit 1 of cl_tma, TB_CL_DBG=1).
    return sm.cl_rflag == 0 || ((sm.cl_tma & 2) && sm.cl_roff < 1e-16 * TB_TOLSCALE);
  }
};

// All CTAs of the cluster call this with the same arguments; returns Nw
// (converged) or -Nw, with the rotated columns (scales folded) back in W.
__device__ __noinline__ int jacobi_cluster(double2* W, int Mw, int Nw, int maxsweep, Smem& sm, double2* smem) {
  JacobiC J;
  J.W = W;
  J.Mw = Mw;
  J.Nw = Nw;
  J.rank = cl_rank();
  J.base = sh_addr(smem);
  const double tol = fmax(sqrt((double)Mw), 4.0) * 4.440892098500626e-16 * TB_TOLSCALE;
  J.tol2 = tol * tol;
  if (threadIdx.x == 0) cluster_schedule(J.rank, sm.cl_sched);
  if (sm.cl_tma & 1) J.load_home_tma(sm);
  else J.load_home();
  int sweep = 0;
  bool conv = false;
  for (; sweep < maxsweep; ++sweep) {
    J.fold_norms(sm, sweep == 0);
    J.offmax = 0.0;
    J.within(sm);
    cl_sync();
    for (int s = 0; s < CNB - 1; ++s) {
      const int xy = sm.cl_sched[s];
      J.cross(xy & 0xff, xy >> 8, sm);
      cl_sync();
    }
    if (J.sweep_end(sm, sweep & 1)) {
      conv = true;
      break;
    }
  }
  if (threadIdx.x == 0) sm.sweeps = sweep + 1;
  if (sm.cl_tma & 1) J.store_home_tma(sm);
  else J.store_home(sm);
  __threadfence();
  cl_sync();
  return conv ? Nw : -Nw;
}

// leader side: post the command, then take part as rank 0
__device__ int jacobi_cluster_lead(double2* W, int Mw, int Nw, Smem& sm, double2* smem) {
  if (threadIdx.x == 0) {
    sm.cl_op = 1;
    sm.cl_W = W;
    sm.cl_Mw = Mw;
    sm.cl_Nw = Nw;
    sm.cl_maxsweep = sm.maxsweep;
    sm.cl_flag[0] = sm.cl_flag[1] = 0;
    sm.cl_off[0] = sm.cl_off[1] = 0.0;
  }
  // W (global) as this CTA wrote it, before the followers load their blocks.
  // The followers read it through the async proxy (TMA bulk loads): the
  // WRITER orders its generic-proxy stores before them (without this fence a
  // follower's bulk load could return the buffer's previous contents)
  asm volatile("fence.proxy.async.global;" ::: "memory");
  __threadfence();
  __syncthreads();
  cl_sync();
  return jacobi_cluster(W, Mw, Nw, sm.maxsweep, sm, smem);
}

// ranks 1..7: serve the leader's cluster Jacobi calls until it posts op 0
__device__ void cluster_follow(Smem& sm, double2* smem) {
  for (;;) {
    cl_sync();
    if (threadIdx.x == 0) {
      sm.cl_op = (int)ldcu(cl_map(sh_addr(&sm.cl_op), 0));
      sm.cl_W = (double2*)ldcl(cl_map(sh_addr(&sm.cl_W), 0));
      sm.cl_Mw = (int)ldcu(cl_map(sh_addr(&sm.cl_Mw), 0));
      sm.cl_Nw = (int)ldcu(cl_map(sh_addr(&sm.cl_Nw), 0));
      sm.cl_maxsweep = (int)ldcu(cl_map(sh_addr(&sm.cl_maxsweep), 0));
      sm.cl_tma = (int)ldcu(cl_map(sh_addr(&sm.cl_tma), 0));
    }
    __syncthreads();
    if (sm.cl_op == 0) {
      cl_sync();  // the leader's shared memory stays alive until every follower read op 0
      return;
    }
    jacobi_cluster(sm.cl_W, sm.cl_Mw, sm.cl_Nw, sm.cl_maxsweep, sm, smem);
  }
}

// leader side: release the followers (end of the kernel)
__device__ void cluster_release(Smem& sm) {
  if (threadIdx.x == 0) sm.cl_op = 0;
  __syncthreads();
  cl_sync();
  cl_sync();
}

#endif  // !TB_ENGINE_SMALL

// dispatcher: returns the number of (possibly padded) result columns in W;
// sets status bit 0 on non-convergence
__device__ int jacobi(double2* W, int Mw, int Nw, Smem& sm, double2* smem, int* status) {
  int neff;
  if (Nw < 2) return Nw;
  if (Mw <= 16 && Nw <= 128) neff = jacobi_half<1>(W, Mw, Nw, sm, smem);
  else if (Mw <= 32 && Nw <= 128) neff = jacobi_half<2>(W, Mw, Nw, sm, smem);
  else if (Mw <= 64 && Nw <= 128) neff = jacobi_half<4>(W, Mw, Nw, sm, smem);
#if !TB_ENGINE_SMALL
  else if (Mw <= 128 && Nw <= 128) neff = jacobi_half<8>(W, Mw, Nw, sm, smem);
  else if (Mw <= 256 && Nw <= 256)
    neff = sm.cluster > 1 ? jacobi_cluster_lead(W, Mw, Nw, sm, smem) : jacobi_wide(W, Mw, Nw, sm, smem);
#endif
  else {
    const int sw = hestenes(W, Mw, Nw, sm);
    neff = (sw > MAXSWEEP) ? -Nw : Nw;
  }
  // fault injection (tests of the exclusion path): a CTA-uniform decision
  if (sm.inject > 0 && sm.sample % sm.inject == 0 && neff > 0) neff = -neff;
  if (neff < 0) {
    if (threadIdx.x == 0) {
      atomicOr(status, 1);
      sm.bad = 1;
    }
    neff = -neff;
  }
  return neff;
}

// ----------------------------------------------------------------------------
// Column-pivoted QR preconditioner (Businger-Golub pivoting, modified
// Gram-Schmidt updates; only R is kept).  For the left singular vectors of W
// (Mw x Nw) factor Y = W^H (Nw x Mw): Y Pi = Q R, so W = Pi L Q^H with
// L = R^H (Mw x r, lower trapezoidal), and the left singular vectors of W are
// Pi times those of L.  One-sided Jacobi on L converges in a few sweeps
// (Drmac-Veselic preconditioning) instead of the ~15 it needs on W.
//
// Y (global, col-major, ld = Nw) is staged as: columns < 96 in the three
// smem slots, columns 96..127 in registers (2 per warp).  R goes to global
// (row-major, ld = Mw, indexed by the ORIGINAL column), the pivot order to
// sm.qperm.  Returns the numerical rank r (residual columns below the dead
// threshold end the factorisation).
// ----------------------------------------------------------------------------
template <int HR>
__device__ int qrcp_mgs(const double2* Y, int Nw, int Mw, double2* R, Smem& sm, double2* smem) {
  // half-warp column layout: half k (0..31) owns smem columns k, k+32, k+64 and
  // keeps column 96+k in registers
  constexpr int LD = 16 * HR;
  constexpr uint32_t CB = LD * 16u;
  const int hw = threadIdx.x >> 4, hl = threadIdx.x & 15, lane = threadIdx.x & 31;
  const uint32_t base = (uint32_t)__cvta_generic_to_shared(smem);
  const uint32_t qaddr = base + 3u * JB * CB;  // q buffer after the slots
  const int nsm = min(Mw, 3 * JB);
  for (int e = threadIdx.x; e < nsm * LD; e += NT) {
    const int c = e / LD, y = e - c * LD;
    smem[e] = (y < Nw) ? Y[(size_t)c * Nw + y] : cz();
  }
  HCol<HR> g;
  const int cg = 3 * JB + hw;
  hcol_ldg(g, Y + (size_t)cg * Nw, cg < Mw ? Nw : 0);
  __syncthreads();
  // exact norms
  for (int k = 0; k < 3; ++k) {
    const int c = hw + 32 * k;
    double acc = 0.0;
    if (c < nsm) {
      HCol<HR> v;
      hcol_lds(v, base + (uint32_t)c * CB);
#pragma unroll
      for (int q = 0; q < HR; ++q) acc += abs2(v.v[q]);
    }
    acc = half_sum(acc);
    if (hl == 0 && c < nsm) sm.nrm[c] = sm.nref[c] = acc;
  }
  {
    double acc = 0.0;
#pragma unroll
    for (int q = 0; q < HR; ++q) acc += abs2(g.v[q]);
    acc = half_sum(acc);
    if (hl == 0 && cg < Mw) sm.nrm[cg] = sm.nref[cg] = acc;
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    double t = 0.0;
    for (int c = threadIdx.x; c < Mw; c += 32) t += sm.nrm[c];
    t = warp_sum(t);
    if (threadIdx.x == 0) sm.scale = 1e-28 * t;  // dead threshold on residual norm^2
  }
  // per-half pivot candidate over the owned columns (lanes 0-3 of the half)
  auto local_best = [&](int buf) {
    const int c = (hl < 3) ? hw + 32 * hl : cg;
    const bool ok = hl < 4 && c < Mw && (hl == 3 || c < nsm);
    double best = ok ? sm.nrm[c] : -1.0;
    int bi = ok ? c : -1;
#pragma unroll
    for (int o = 2; o > 0; o >>= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, best, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ob > best || (ob == best && oi >= 0 && (bi < 0 || oi < bi))) { best = ob; bi = oi; }
    }
    if (hl == 0) {
      sm.wbest[buf][hw] = best;
      sm.wbidx[buf][hw] = bi;
    }
  };
  local_best(0);
  __syncthreads();
  const double dead = sm.scale;
  const int rmax = min(Mw, Nw);
  int j = 0;
  long long tq0 = prof_fine(), tq1 = 0, tq2 = 0, tq3 = 0, tqa = 0, tqb = 0, tqc = 0, tqd = 0;
  for (; j < rmax; ++j) {
    const long long tt0 = prof_fine();
    // global pivot (every warp): largest residual.  Key = high word of the
    // (non-negative) norm with its 7 low bits replaced by 127 - column, so one
    // redux.max picks the largest norm (to ~1e-6 relative; near-ties go to the
    // lowest index, which is immaterial for the preconditioner)
    // The candidates of step j live in buffer j & 1 and those of step j + 1 go
    // to the other one: a step has a single barrier (at its end), so a half
    // that finishes its updates early writes its next candidate while a slower
    // warp may not have read this step's yet.  With one buffer that warp could
    // pick a different pivot than the rest of the CTA (seen on the GPU with
    // two resident CTAs per SM: run-to-run differences at rounding level and
    // sporadic faults on 32x32 problems).
    const int wi = sm.wbidx[j & 1][lane];
    const double wv = sm.wbest[j & 1][lane];
    const unsigned key = (wi >= 0 && wv > dead) ? ((unsigned)__double2hiint(wv) & 0xFFFFFF80u) | (unsigned)(127 - wi) : 0u;
    const unsigned kmax = __reduce_max_sync(0xffffffffu, key);
    if (kmax == 0u) break;
    const int p = 127 - (int)(kmax & 127u);
    const long long tt1 = prof_fine();
    tqa += tt1 - tt0;
    // Every half normalises the pivot column itself (bit-identical results),
    // reading it straight from its shared-memory home; only a register-held
    // pivot (columns >= 96) is first published through the q buffer, which
    // costs the one extra barrier.  The owner half never touches column p in
    // this step, so the reads need no other ordering than the barrier that
    // closed the previous step.
    const bool regp = p >= 3 * JB;
    const int owner = regp ? (p - 3 * JB) : (p & 31);
    uint32_t src = base + (uint32_t)p * CB;
    if (regp) {
      if (hw == owner) hcol_sts(qaddr, g);
      __syncthreads();
      src = qaddr;
    }
    const long long tt2 = prof_fine();
    HCol<HR> qv;
    hcol_lds(qv, src);
    {
      double nn = 0.0;
#pragma unroll
      for (int q = 0; q < HR; ++q) nn += abs2(qv.v[q]);
      nn = half_sum(nn);
      const double inv = rsqrt_nr(nn), rn = nn * inv;
#pragma unroll
      for (int q = 0; q < HR; ++q) qv.v[q] = cscale(qv.v[q], inv);
      if (hw == owner && hl == 0) {
        R[(size_t)j * Mw + p] = make_double2(rn, 0.0);
        sm.qperm[j] = p;
      }
    }
    const long long tt3 = prof_fine();
    tqb += tt2 - tt1;
    tqc += tt3 - tt2;
    // MGS update of one column per half: r = q^H y, y -= r q
    auto upd = [&](HCol<HR>& y, int c, bool valid) {
      double2 d = cz(), e = cz();
#pragma unroll
      for (int q = 0; q < HR; q += 2) {
        cfmac(d, qv.v[q], y.v[q]);
        if (q + 1 < HR) cfmac(e, qv.v[q + 1], y.v[q + 1]);
      }
      d.x = half_sum(d.x + e.x);
      d.y = half_sum(d.y + e.y);
      if (!valid) d = cz();
#pragma unroll
      for (int q = 0; q < HR; ++q) {
        // y -= d q as four fused multiply-adds (no DMUL/DADD pairs)
        y.v[q].x = fma(-d.x, qv.v[q].x, fma(d.y, qv.v[q].y, y.v[q].x));
        y.v[q].y = fma(-d.x, qv.v[q].y, fma(-d.y, qv.v[q].x, y.v[q].y));
      }
      double nr = valid ? sm.nrm[c] - abs2(d) : 0.0;
      const bool f = valid && nr < 1e-2 * sm.nref[c];
      if (__any_sync(0xffffffffu, f)) {  // cancellation: exact norm
        double acc = 0.0;
#pragma unroll
        for (int q = 0; q < HR; ++q) acc += abs2(y.v[q]);
        acc = half_sum(acc);
        if (f) nr = acc;
      }
      if (hl == 0 && valid) {
        sm.nrm[c] = nr;
        if (f) sm.nref[c] = nr;
        R[(size_t)j * Mw + c] = d;
      }
    };
#pragma unroll 1
    for (int k = 0; k < 3; ++k) {
      const int c = hw + 32 * k;
      const bool valid = c < nsm && c != p && sm.nrm[c] >= 0.0;
      if (!__any_sync(0xffffffffu, valid)) continue;
      HCol<HR> y;
      if (valid) hcol_lds(y, base + (uint32_t)c * CB);
      else {
#pragma unroll
        for (int q = 0; q < HR; ++q) y.v[q] = cz();
      }
      upd(y, c, valid);
      if (valid) hcol_sts(base + (uint32_t)c * CB, y);
    }
    {
      const bool valid = cg < Mw && cg != p && sm.nrm[cg] >= 0.0;
      if (__any_sync(0xffffffffu, valid)) upd(g, cg, valid);
    }
    if (hw == owner && hl == 0) sm.nrm[p] = -1.0;
    __syncwarp();
    local_best((j + 1) & 1);
    const long long tt4 = prof_fine();
    __syncthreads();
    tqd += tt4 - tt3;
    tq1 += prof_fine() - tt4;
  }
  if (threadIdx.x == 0 && TB_PROF && sm.prof) {
    atomicAdd(&sm.prof[15], (unsigned long long)j);
    atomicAdd(&sm.prof[32], (unsigned long long)tqa);   // pivot selection
    atomicAdd(&sm.prof[33], (unsigned long long)tqb);   // register-pivot publication (incl. its barrier)
    atomicAdd(&sm.prof[34], (unsigned long long)tqc);   // pivot load + normalisation
    atomicAdd(&sm.prof[35], (unsigned long long)tqd);   // update + local best
    atomicAdd(&sm.prof[36], (unsigned long long)tq1);   // barrier 2 wait
    atomicAdd(&sm.prof[37], (unsigned long long)(prof_fine() - tq0));
  }
  (void)tq2; (void)tq3;
  // complete the permutation with the numerically dead columns
  if (threadIdx.x == 0) {
    int k = j;
    for (int c = 0; c < Mw; ++c)
      if (sm.nrm[c] >= 0.0) sm.qperm[k++] = c;
    for (int k2 = 0; k2 < Mw; ++k2) sm.qpinv[sm.qperm[k2]] = k2;
  }
  __syncthreads();
  return j;
}

#if !TB_ENGINE_SMALL  // tensor-memory QRCP (128-row problems only)
// TMEM allocation of the whole 512-column tensor memory of the SM (one CTA
// per SM); qrcp_tmem is its only user.
__device__ __forceinline__ void tmem_alloc(Smem& sm) {
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(&sm.tmem)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
}
__device__ __forceinline__ void tmem_free(Smem& sm) {
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(sm.tmem));
}

// ----------------------------------------------------------------------------
// TMEM-resident column-pivoted MGS (same algorithm, layout and outputs as
// qrcp_mgs<8>).  The smem version is bound by shared-memory bandwidth: every
// live column is loaded and stored once per step (4 KB each, ~3k of its ~7.5k
// cycles per step at 128 B/clk).  Here the columns live in tensor memory,
// which streams at ~470 B/clk (ld) / ~970 B/clk (st) per SM on this B200
// (tools/tmem_bw.cu).  Half-warp k owns columns k + 32 t (t = 0..3) exactly as
// in qrcp_mgs: lane l of the half holds rows l + 16 q, i.e. TMEM lane
// 32 (w & 3) + l' (l' = lane in the warp), words 128 (w >> 2) + 32 t + 4 q —
// the four warps of a lane quadrant split its 512 words, so all 128 columns
// fit.  tcgen05.ld/st are warp-collective, so both halves of a warp move
// their column t together.  The pivot column is published through a 2 KB
// shared-memory buffer (one extra barrier per step).
// ----------------------------------------------------------------------------
__device__ __forceinline__ void tm_ld32(uint32_t a, uint32_t (&v)[32]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];" : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31]) : "r"(a) : "memory");
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tm_st32(uint32_t a, const uint32_t (&v)[32]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};" :: "r"(a), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]), "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31]) : "memory");
}
__device__ __forceinline__ void tm_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ double2 tm_c(const uint32_t (&v)[32], int r) {
  return make_double2(__hiloint2double((int)v[4 * r + 1], (int)v[4 * r]), __hiloint2double((int)v[4 * r + 3], (int)v[4 * r + 2]));
}
__device__ __forceinline__ void tm_put(uint32_t (&v)[32], int r, double2 e) {
  v[4 * r] = (uint32_t)__double2loint(e.x);
  v[4 * r + 1] = (uint32_t)__double2hiint(e.x);
  v[4 * r + 2] = (uint32_t)__double2loint(e.y);
  v[4 * r + 3] = (uint32_t)__double2hiint(e.y);
}

__device__ __forceinline__ void tm_ld_col(uint32_t a, HCol<8>& c) {
  uint32_t v[32];
  tm_ld32(a, v);
#pragma unroll
  for (int q = 0; q < 8; ++q) c.v[q] = tm_c(v, q);
}
__device__ __forceinline__ void tm_st_col(uint32_t a, const HCol<8>& c) {
  uint32_t v[32];
#pragma unroll
  for (int q = 0; q < 8; ++q) tm_put(v, q, c.v[q]);
  tm_st32(a, v);
}

__device__ __noinline__ int qrcp_tmem(const double2* Y, int Nw, int Mw, double2* R, Smem& sm, double2* smem) {
  constexpr int HR = 8;
  const int hw = threadIdx.x >> 4, hl = threadIdx.x & 15, lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint32_t qaddr = (uint32_t)__cvta_generic_to_shared(smem);
  const uint32_t tcol = sm.tmem + ((uint32_t)(32 * (w & 3)) << 16) + 128u * (uint32_t)(w >> 2);
  // stage column hw + 32 t into word block t, exact norms
#pragma unroll 1
  for (int t = 0; t < 4; ++t) {
    const int c = hw + 32 * t;
    HCol<HR> v;
    hcol_ldg(v, Y + (size_t)c * Nw, c < Mw ? Nw : 0);
    double acc = 0.0;
#pragma unroll
    for (int q = 0; q < HR; ++q) acc += abs2(v.v[q]);
    acc = half_sum(acc);
    if (hl == 0 && c < Mw) sm.nrm[c] = sm.nref[c] = acc;
    tm_st_col(tcol + 32u * t, v);
  }
  tm_wait_st();
  __syncthreads();
  if (threadIdx.x < 32) {
    double t = 0.0;
    for (int c = threadIdx.x; c < Mw; c += 32) t += sm.nrm[c];
    t = warp_sum(t);
    if (threadIdx.x == 0) sm.scale = 1e-28 * t;  // dead threshold on residual norm^2
  }
  auto local_best = [&]() {
    const int c = hw + 32 * hl;
    const bool ok = hl < 4 && c < Mw;
    double best = ok ? sm.nrm[c] : -1.0;
    int bi = ok ? c : -1;
#pragma unroll
    for (int o = 2; o > 0; o >>= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, best, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ob > best || (ob == best && oi >= 0 && (bi < 0 || oi < bi))) { best = ob; bi = oi; }
    }
    if (hl == 0) {
      sm.wbest[0][hw] = best;
      sm.wbidx[0][hw] = bi;
    }
  };
  local_best();
  __syncthreads();
  const double dead = sm.scale;
  const int rmax = min(Mw, Nw);
  int j = 0;
  for (; j < rmax; ++j) {
    const int wi = sm.wbidx[0][lane];
    const double wv = sm.wbest[0][lane];
    const unsigned key = (wi >= 0 && wv > dead) ? ((unsigned)__double2hiint(wv) & 0xFFFFFF80u) | (unsigned)(127 - wi) : 0u;
    const unsigned kmax = __reduce_max_sync(0xffffffffu, key);
    if (kmax == 0u) break;
    const int p = 127 - (int)(kmax & 127u);
    const int owner = p & 31, tp = p >> 5;
    if ((owner >> 1) == w) {  // the owner's warp loads (warp-collective), the owner half publishes
      HCol<HR> v;
      tm_ld_col(tcol + 32u * tp, v);
      if (hw == owner) hcol_sts(qaddr, v);
    }
    __syncthreads();
    HCol<HR> qv;
    hcol_lds(qv, qaddr);
    {
      double nn = 0.0;
#pragma unroll
      for (int q = 0; q < HR; ++q) nn += abs2(qv.v[q]);
      nn = half_sum(nn);
      const double inv = rsqrt_nr(nn), rn = nn * inv;
#pragma unroll
      for (int q = 0; q < HR; ++q) qv.v[q] = cscale(qv.v[q], inv);
      if (hw == owner && hl == 0) {
        R[(size_t)j * Mw + p] = make_double2(rn, 0.0);
        sm.qperm[j] = p;
      }
    }
    // MGS update of one column per half: r = q^H y, y -= r q.  An invalid
    // column applies d = 0 and is stored back unchanged.  (Two columns at a
    // time, to interleave their reductions, spilled in the hot loop: 16.4k
    // instead of 5.8k cycles per step.)
    auto dotp = [&](const HCol<HR>& y) {
      double2 d = cz(), e = cz();
#pragma unroll
      for (int q = 0; q < HR; q += 2) {
        cfmac(d, qv.v[q], y.v[q]);
        cfmac(e, qv.v[q + 1], y.v[q + 1]);
      }
      return cadd(d, e);
    };
    auto apply = [&](HCol<HR>& y, int c, bool valid, double2 d) {
      if (!valid) d = cz();
#pragma unroll
      for (int q = 0; q < HR; ++q) {
        // y -= d q as four fused multiply-adds (no DMUL/DADD pairs)
        y.v[q].x = fma(-d.x, qv.v[q].x, fma(d.y, qv.v[q].y, y.v[q].x));
        y.v[q].y = fma(-d.x, qv.v[q].y, fma(-d.y, qv.v[q].x, y.v[q].y));
      }
      double nr = valid ? sm.nrm[c] - abs2(d) : 0.0;
      const bool f = valid && nr < 1e-2 * sm.nref[c];
      if (__any_sync(0xffffffffu, f)) {  // cancellation: exact norm
        double acc = 0.0;
#pragma unroll
        for (int q = 0; q < HR; ++q) acc += abs2(y.v[q]);
        acc = half_sum(acc);
        if (f) nr = acc;
      }
      if (hl == 0 && valid) {
        sm.nrm[c] = nr;
        if (f) sm.nref[c] = nr;
        R[(size_t)j * Mw + c] = d;
      }
    };
    // Two passes over the half's four columns: every dot product first
    // (partial sums only), ONE transposed reduction of the eight partials,
    // then the updates, re-reading each column from tensor memory (which
    // streams far faster than the reductions' latency) instead of holding
    // it.  The four per-column reduction chains no longer serialise.
    bool vt[4];
    double part[8];
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const int c = hw + 32 * t;
      vt[t] = c < Mw && c != p && sm.nrm[c] >= 0.0;
      double2 d = cz();
      if (__any_sync(0xffffffffu, vt[t])) {
        HCol<HR> y;
        tm_ld_col(tcol + 32u * t, y);
        d = dotp(y);
      }
      part[2 * t] = d.x;
      part[2 * t + 1] = d.y;
    }
    half_sum8(part);
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      if (!__any_sync(0xffffffffu, vt[t])) continue;
      HCol<HR> y;
      tm_ld_col(tcol + 32u * t, y);
      apply(y, hw + 32 * t, vt[t], make_double2(part[2 * t], part[2 * t + 1]));
      tm_st_col(tcol + 32u * t, y);
    }
    tm_wait_st();
    if (hw == owner && hl == 0) sm.nrm[p] = -1.0;
    __syncwarp();
    local_best();
    __syncthreads();
  }
  if (threadIdx.x == 0 && TB_PROF && sm.prof) atomicAdd(&sm.prof[15], (unsigned long long)j);
  // complete the permutation with the numerically dead columns
  if (threadIdx.x == 0) {
    int k = j;
    for (int c = 0; c < Mw; ++c)
      if (sm.nrm[c] >= 0.0) sm.qperm[k++] = c;
    for (int k2 = 0; k2 < Mw; ++k2) sm.qpinv[sm.qperm[k2]] = k2;
  }
  __syncthreads();
  return j;
}

#endif  // !TB_ENGINE_SMALL

// L = R^H in pivoted row order: L[k][i] = conj(R[i][perm[k]]) for k >= i
// (Mw x r, column-major into W)
__device__ void build_l(const double2* R, int Mw, int r, double2* W, const Smem& sm) {
  for (int e = threadIdx.x; e < Mw * r; e += NT) {
    const int i = e / Mw, k = e - i * Mw;
    W[e] = (k >= i) ? cconj(R[(size_t)i * Mw + sm.qperm[k]]) : cz();
  }
  __syncthreads();
}

template <int HR>
__device__ int precond_jacobi_t(double2* W, double2* X, int Mw, int Nw, Smem& sm, double2* smem, int* status) {
  const long long t0 = prof_clock();
#if TB_ENGINE_SMALL
  const int r = qrcp_mgs<HR>(W, Nw, Mw, X, sm, smem);
#else
  const int r = (sm.tmem_on && HR == 8) ? qrcp_tmem(W, Nw, Mw, X, sm, smem) : qrcp_mgs<HR>(W, Nw, Mw, X, sm, smem);
#endif
  if (threadIdx.x == 0 && TB_PROF && sm.prof) {
    atomicAdd(&sm.prof[12], (unsigned long long)(prof_clock() - t0));
    atomicAdd(&sm.prof[8], 1ull);
  }
  const int K = min(Mw, Nw);
  int neff = 0;
  if (r > 0) {
    const long long tb0 = prof_clock();
    build_l(X, Mw, r, W, sm);
    if (threadIdx.x == 0 && TB_PROF && sm.prof) atomicAdd(&sm.prof[24], (unsigned long long)(prof_clock() - tb0));
    neff = jacobi(W, Mw, r, sm, smem, status);
  }
  // the numerically dead directions are exact zero columns
  if (neff < K) {
    for (int e = threadIdx.x; e < (K - neff) * Mw; e += NT) W[(size_t)neff * Mw + e] = cz();
    __syncthreads();
  }
  return max(neff, K);
}

#if !TB_ENGINE_SMALL
// Y = W^H is in W (ld = Nw); returns Neff, W = rotated columns of L (ld = Mw),
// rows in pivoted order (sm.qpinv maps an original row to its position)
// Column-pivoted MGS QR for the wide problems (Y: Nw <= 256 rows x Mw <= 256
// columns, col-major, ld = Nw, in global memory).  Same algorithm and outputs
// as qrcp_mgs (R row-major by original column, sm.qperm / sm.qpinv, returns
// the numerical rank), but the columns stay in global memory (L2): half-warp
// k owns columns k, k+32, ..., a column is 16 lanes x 16 rows in registers
// while it is updated, and q is streamed from shared memory.
__device__ int qrcp_wide(double2* Y, int Nw, int Mw, double2* R, Smem& sm, double2* smem) {
  constexpr int HR = 16;
  const int hw = threadIdx.x >> 4, hl = threadIdx.x & 15, lane = threadIdx.x & 31;
  const uint32_t qaddr = (uint32_t)__cvta_generic_to_shared(smem);
  const uint32_t l = hl * 16u;
  const int nown = (Mw - hw + 31) / 32;  // columns owned by this half
  for (int k = 0; k < 8; ++k) {
    const int c = hw + 32 * k;
    double acc = 0.0;
    if (k < nown) {
      HCol<HR> v;
      hcol_ldg(v, Y + (size_t)c * Nw, Nw);
#pragma unroll
      for (int q = 0; q < HR; ++q) acc += abs2(v.v[q]);
    }
    acc = half_sum(acc);
    if (hl == 0 && k < nown) sm.nrm[c] = sm.nref[c] = acc;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int c = 0; c < Mw; ++c) t += sm.nrm[c];
    sm.scale = 1e-28 * t;
  }
  auto local_best = [&]() {  // lanes 0-7 of a half hold its candidates
    const int c = hw + 32 * (hl & 7);
    const bool ok = hl < 8 && (hl & 7) < nown;
    double best = ok ? sm.nrm[c] : -1.0;
    int bi = ok ? c : -1;
#pragma unroll
    for (int o = 4; o > 0; o >>= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, best, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ob > best || (ob == best && oi >= 0 && (bi < 0 || oi < bi))) { best = ob; bi = oi; }
    }
    if (hl == 0) {
      sm.wbest[0][hw] = best;
      sm.wbidx[0][hw] = bi;
    }
  };
  local_best();
  __syncthreads();
  const double dead = sm.scale;
  const int rmax = min(Mw, Nw);
  int j = 0;
  for (; j < rmax; ++j) {
    // global pivot: same packed-key redux as qrcp_mgs (8 index bits here)
    const int wi = sm.wbidx[0][lane];
    const double wv = sm.wbest[0][lane];
    const unsigned key =
        (wi >= 0 && wv > dead) ? ((unsigned)__double2hiint(wv) & 0xFFFFFF00u) | (unsigned)(255 - wi) : 0u;
    const unsigned kmax = __reduce_max_sync(0xffffffffu, key);
    if (kmax == 0u) break;
    const int p = 255 - (int)(kmax & 255u);
    const int owner = p & 31;
    if ((owner >> 1) == (threadIdx.x >> 5)) {
      const bool me = hw == owner;
      HCol<HR> v;
      hcol_ldg(v, Y + (size_t)p * Nw, Nw);
      double nn = 0.0;
#pragma unroll
      for (int q = 0; q < HR; ++q) nn += abs2(v.v[q]);
      nn = half_sum(nn);
      const double rn = sqrt(nn), inv = 1.0 / rn;
      if (me) {
#pragma unroll
        for (int q = 0; q < HR; ++q) sts2(qaddr + l + 256u * q, cscale(v.v[q], inv));
        if (hl == 0) {
          R[(size_t)j * Mw + p] = make_double2(rn, 0.0);
          sm.qperm[j] = p;
          sm.nrm[p] = -1.0;
        }
      }
    }
    __syncthreads();
#pragma unroll 1
    for (int k = 0; k < 8; ++k) {
      const int c = hw + 32 * k;
      const bool valid = k < nown && sm.nrm[c] >= 0.0;
      if (!__any_sync(0xffffffffu, valid)) continue;
      HCol<HR> y;
      if (valid) hcol_ldg(y, Y + (size_t)c * Nw, Nw);
      else {
#pragma unroll
        for (int q = 0; q < HR; ++q) y.v[q] = cz();
      }
      double2 d = cz(), e = cz();
#pragma unroll
      for (int q = 0; q < HR; q += 2) {
        cfmac(d, lds2(qaddr + l + 256u * q), y.v[q]);
        cfmac(e, lds2(qaddr + l + 256u * (q + 1)), y.v[q + 1]);
      }
      d.x = half_sum(d.x + e.x);
      d.y = half_sum(d.y + e.y);
      if (!valid) d = cz();
#pragma unroll
      for (int q = 0; q < HR; ++q) {
        const double2 qq = lds2(qaddr + l + 256u * q);
        // y -= d q as four fused multiply-adds (no DMUL/DADD pairs)
        y.v[q].x = fma(-d.x, qq.x, fma(d.y, qq.y, y.v[q].x));
        y.v[q].y = fma(-d.x, qq.y, fma(-d.y, qq.x, y.v[q].y));
      }
      double nr = valid ? sm.nrm[c] - abs2(d) : 0.0;
      const bool f = valid && nr < 1e-2 * sm.nref[c];
      if (__any_sync(0xffffffffu, f)) {
        double acc = 0.0;
#pragma unroll
        for (int q = 0; q < HR; ++q) acc += abs2(y.v[q]);
        acc = half_sum(acc);
        if (f) nr = acc;
      }
      if (valid) {
        hcol_stg(Y + (size_t)c * Nw, y, Nw);
        if (hl == 0) {
          sm.nrm[c] = nr;
          if (f) sm.nref[c] = nr;
          R[(size_t)j * Mw + c] = d;
        }
      }
    }
    __syncwarp();
    local_best();
    __syncthreads();
  }
  if (threadIdx.x == 0 && TB_PROF && sm.prof) atomicAdd(&sm.prof[15], (unsigned long long)j);
  if (threadIdx.x == 0) {
    int k = j;
    for (int c = 0; c < Mw; ++c)
      if (sm.nrm[c] >= 0.0) sm.qperm[k++] = c;
    for (int k2 = 0; k2 < Mw; ++k2) sm.qpinv[sm.qperm[k2]] = k2;
  }
  __syncthreads();
  return j;
}

__device__ int precond_jacobi_wide(double2* W, double2* X, int Mw, int Nw, Smem& sm, double2* smem, int* status) {
  const long long t0 = prof_clock();
  const int r = qrcp_wide(W, Nw, Mw, X, sm, smem);
  if (threadIdx.x == 0 && TB_PROF && sm.prof) {
    atomicAdd(&sm.prof[12], (unsigned long long)(prof_clock() - t0));
    atomicAdd(&sm.prof[8], 1ull);
  }
  const int K = min(Mw, Nw);
  int neff = 0;
  if (r > 0) {
    build_l(X, Mw, r, W, sm);
    neff = jacobi(W, Mw, r, sm, smem, status);
  }
  if (neff < K) {
    for (int e = threadIdx.x; e < (K - neff) * Mw; e += NT) W[(size_t)neff * Mw + e] = cz();
    __syncthreads();
  }
  return max(neff, K);
}

#endif  // !TB_ENGINE_SMALL

__device__ int precond_jacobi(double2* W, double2* X, int Mw, int Nw, Smem& sm, double2* smem, int* status) {
#if !TB_ENGINE_SMALL
  if (Nw > 128 || Mw > 128) return precond_jacobi_wide(W, X, Mw, Nw, sm, smem, status);
#endif
  if (Nw <= 16) return precond_jacobi_t<1>(W, X, Mw, Nw, sm, smem, status);
  if (Nw <= 32) return precond_jacobi_t<2>(W, X, Mw, Nw, sm, smem, status);
#if TB_ENGINE_SMALL
  return precond_jacobi_t<4>(W, X, Mw, Nw, sm, smem, status);
#else
  if (Nw <= 64) return precond_jacobi_t<4>(W, X, Mw, Nw, sm, smem, status);
  return precond_jacobi_t<8>(W, X, Mw, Nw, sm, smem, status);
#endif
}

// ----------------------------------------------------------------------------
// Per-CTA sample context
// ----------------------------------------------------------------------------
__device__ __forceinline__ void prof_add(const Job& jb, int slot, long long v) {
  if (TB_PROF && threadIdx.x == 0 && jb.prof) atomicAdd(&jb.prof[slot], (unsigned long long)v);
}

constexpr int kTileElems = 2 * TK * TLD;                                // GEMM staging tiles
constexpr int kQrSmemElems = (3 * JB + 1) * SROWS - kTileElems;           // rest of the dynamic smem

struct Ctx {
  const Job* job;
  double2* mps;
  double2* W;
  double2* W0;
  double2* X;
  double2* tile;
  int cap;
  __device__ double2* site(int s) const { return mps + (size_t)s * cap * 2 * cap; }
};

// ----------------------------------------------------------------------------
// Two-site update at bond (s, s+1): contraction, gate or swap, SVD split.
// kind: 0 = Pauli-pair rotation, 1 = swap.  (_kernel.py:114-181)
// ----------------------------------------------------------------------------
__device__ void two_site(const Ctx& cx, Smem& sm, int s, int kind, int pa, int pb, double cth, double sth,
                         bool merge_right) {
  const Job& jb = *cx.job;
  const int cap = cx.cap;
  const int cl = sm.dims[s], cm = sm.dims[s + 1], cr = sm.dims[s + 2];
  const int M = 2 * cl, N = 2 * cr;
  const int Mw = merge_right ? M : N, Nw = merge_right ? N : M;
  double2* A = cx.site(s);
  double2* B = cx.site(s + 1);
  double2* W = cx.W;
  double2* W0 = cx.W0;
  const long long t0 = prof_clock();

  // QR-preconditioned path for sizeable problems: W holds Y = W_jac^H, i.e.
  // theta is written in the opposite orientation (see precond_jacobi)
  const bool pre = jb.precond && Mw >= 32 && Nw >= 32;
  const bool orient = pre ? !merge_right : merge_right;  // true: col-major theta
  const int ldw = orient ? M : N;

  // theta = A (2cl x cm) . B (cm x 2cr), written into W.  A swap (_kernel.py:
  // 171-181) only exchanges the physical legs, theta'[(l,j),(i,r)] =
  // theta[(l,i),(j,r)], so the GEMM epilogue writes it straight to its
  // permuted place in both W and W0; a gate needs the pass below.
  const bool swap = kind == 1;
  cta_gemm_tc<true, false>(
      M, N, cm, [&](int m, int k) { return A[(size_t)m * cap + k]; },
      [&](int k, int n) {
        const int j = n >= cr ? 1 : 0;  // n < 2 cr
        return B[(size_t)(k * 2 + j) * cap + (n - j * cr)];
      },
      [&](int m, int n, double2 v) {
        int row = m, col = n;
        if (swap) {
          const int j = n >= cr ? 1 : 0, r = n - j * cr;
          row = (m & ~1) | j;
          col = (m & 1) * cr + r;
          W0[merge_right ? (size_t)col * Mw + row : (size_t)row * Mw + col] = merge_right ? v : cconj(v);
        }
        if (orient) W[(size_t)col * ldw + row] = v;
        else W[(size_t)row * ldw + col] = cconj(v);
      },
      cx.tile);
  const long long tg = prof_clock();
  prof_add(jb, 30, tg - t0);

  // gate on the physical pair, fused into the (W, W0) write-out
  const int fa = (pa == 3) ? 0 : 1, fb = (pb == 3) ? 0 : 1;
  for (int e = swap ? cl * cr : threadIdx.x; e < cl * cr; e += NT) {
    // consecutive threads walk the contiguous index of W's layout
    int l, r;
    if (orient) { r = e / cl; l = e - r * cl; }
    else { l = e / cr; r = e - l * cr; }
    double2 t[2][2];
    size_t idx[2][2];
    size_t idw[2][2];
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int row = l * 2 + i, col = j * cr + r;
        idx[i][j] = merge_right ? (size_t)col * Mw + row : (size_t)row * Mw + col;
        idw[i][j] = orient ? (size_t)col * ldw + row : (size_t)row * ldw + col;
        const double2 v = W[idw[i][j]];
        t[i][j] = orient ? v : cconj(v);
      }
    double2 o[2][2];
    if (kind == 1) {
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) o[i][j] = t[j][i];
    } else {
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          // phase of Pa(i, i^fa) * Pb(j, j^fb)
          double2 ph = make_double2(1.0, 0.0);
          if (pa == 2) ph = make_double2(0.0, i == 0 ? -1.0 : 1.0);
          else if (pa == 3 && i == 1) ph = make_double2(-1.0, 0.0);
          if (pb == 2) ph = cmul(ph, make_double2(0.0, j == 0 ? -1.0 : 1.0));
          else if (pb == 3 && j == 1) ph = make_double2(-ph.x, -ph.y);
          // w = -i * sth * ph
          const double2 w = make_double2(sth * ph.y, -sth * ph.x);
          const double2 other = t[i ^ fa][j ^ fb];
          double2 v = make_double2(cth * t[i][j].x, cth * t[i][j].y);
          v = cadd(v, cmul(w, other));
          o[i][j] = v;
        }
    }
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        W[idw[i][j]] = orient ? o[i][j] : cconj(o[i][j]);
        W0[idx[i][j]] = merge_right ? o[i][j] : cconj(o[i][j]);
      }
  }
  __syncthreads();

  const long long t1 = prof_clock();
  prof_add(jb, 31, t1 - tg);
  if (threadIdx.x == 0) {
    sm.sweeps = 0;
    sm.kcut = jb.tail_skip ? min(jb.chi_cut, min(M, N)) : MAXDIM;
  }
  const int Neff = pre ? precond_jacobi(W, cx.X, Mw, Nw, sm, cx.tile, jb.status) : jacobi(W, Mw, Nw, sm, cx.tile, jb.status);
  if (!pre) {
    for (int y = threadIdx.x; y < Mw; y += NT) sm.qpinv[y] = y;
    __syncthreads();
  }
  const long long t2 = prof_clock();
  prof_add(jb, 4, t1 - t0);
  prof_add(jb, 0, t2 - t1);
  prof_add(jb, 1, 1);
  prof_add(jb, 2, sm.sweeps);
  if (Mw == 128 && Nw == 128) {
    prof_add(jb, 9, t2 - t1);
    prof_add(jb, 10, 1);
    prof_add(jb, 11, sm.sweeps);
  }
  const long long tss = prof_clock();
  sort_sigma(W, Mw, Neff, sm);
  prof_add(jb, 29, prof_clock() - tss);

  // truncation rule + renormalisation (_kernel.py:118-131)
  if (threadIdx.x == 0) {
    const int K = min(M, N);
    const int kmax = min(jb.chi_cut, K);
    const double smax = sm.sig[sm.perm[0]];
    int k = 0;
    for (int i = 0; i < kmax; ++i) k += (sm.sig[sm.perm[i]] > smax * jb.floor) ? 1 : 0;
    if (k == 0) k = 1;
    double total = 0.0, kept = 0.0;
    for (int i = 0; i < K; ++i) {
      const double v = sm.sig[sm.perm[i]];
      total += v * v;
    }
    for (int i = 0; i < k; ++i) {
      const double v = sm.sig[sm.perm[i]];
      kept += v * v;
    }
    sm.counters[3] += (total - kept) / total;
    sm.scale = 1.0 / sqrt(kept);
    sm.k = k;
    sm.counters[0] += 1.0;
    sm.counters[1] += (double)k * (double)k * (double)k;
    if (k > sm.counters[2]) sm.counters[2] = k;
    const double Mx = max(M, N), Kx = min(M, N);
    sm.flops += 32.0 * cl * cm * cr + 4.0 * (6.0 * Mx * Kx * Kx + 20.0 * Kx * Kx * Kx);
  }
  __syncthreads();
  const int k = sm.k;
  const double scale = sm.scale;
  for (int c = threadIdx.x; c < k; c += NT) sm.nref[c] = 1.0 / sm.sig[sm.perm[c]];
  __syncthreads();
  // isometric factor Q[:, c] = W[:, perm c] / sigma
  for (int e = threadIdx.x; e < k * Mw; e += NT) {
    const int c = e / Mw, y = e - c * Mw;
    const int pc = sm.perm[c];
    const double2 q = cscale(W[(size_t)pc * Mw + sm.qpinv[y]], sm.nref[c]);
    if (merge_right) {
      A[(size_t)y * cap + c] = q;  // site s [(l,i)][c]
    } else {
      const int j = y / cr, r = y - j * cr;
      B[(size_t)(c * 2 + j) * cap + r] = cconj(q);  // site s+1 [c][(j,r)]
    }
  }
  // weighted factor P = Q^H W0 (k x Nw), scaled by 1/sqrt(kept)
  cta_gemm_tc<true, true>(
      k, Nw, Mw,
      [&](int c, int y) { return cscale(cconj(W[(size_t)sm.perm[c] * Mw + sm.qpinv[y]]), sm.nref[c]); },
      [&](int y, int x) { return W0[(size_t)x * Mw + y]; },
      [&](int c, int x, double2 v) {
        if (merge_right) {
          const int j = x / cr, r = x - j * cr;
          B[(size_t)(c * 2 + j) * cap + r] = cscale(v, scale);
        } else {
          A[(size_t)x * cap + c] = cscale(cconj(v), scale);
        }
      },
      cx.tile);
  if (threadIdx.x == 0) sm.dims[s + 1] = k;
  __syncthreads();
  prof_add(jb, 5, prof_clock() - t2);
}

// ----------------------------------------------------------------------------
// CGS2 QR of the columns of W (Mx x Nx, column-major): Q overwrites W, R
// (Nx x Nx, row-major) goes to R.  Numerically dependent columns (residual
// below 1e-13 of the column) become zero columns with a zero R row — the
// zero-padding the reference lacks when 2*cl < cr (_kernel.py:75/87).
// ----------------------------------------------------------------------------
__device__ void cgs2_qr(double2* W, int Mx, int Nx, double2* R, Smem& sm) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int e = threadIdx.x; e < Nx * Nx; e += NT) R[e] = cz();
  __syncthreads();
  for (int j = 0; j < Nx; ++j) {
    double2* wj = W + (size_t)j * Mx;
    // original column norm (for the dependence test)
    double n0 = 0.0;
    if (warp == 0) {
      for (int y = lane; y < Mx; y += 32) n0 += abs2(wj[y]);
      n0 = warp_sum(n0);
      if (lane == 0) sm.red[NWARP + 1] = n0;
    }
    for (int pass = 0; pass < 2; ++pass) {
      for (int i = warp; i < j; i += NWARP) {
        const double2* wi = W + (size_t)i * Mx;
        double2 d = cz();
        for (int y = lane; y < Mx; y += 32) cfmac(d, wi[y], wj[y]);
        d.x = warp_sum(d.x);
        d.y = warp_sum(d.y);
        if (lane == 0) sm.rco[i] = d;
      }
      __syncthreads();
      for (int y = threadIdx.x; y < Mx; y += NT) {
        double2 v = wj[y];
        for (int i = 0; i < j; ++i) {
          const double2 r = sm.rco[i];
          const double2 q = W[(size_t)i * Mx + y];
          v = csub(v, cmul(r, q));
        }
        wj[y] = v;
      }
      for (int i = threadIdx.x; i < j; i += NT) R[(size_t)i * Nx + j] = cadd(R[(size_t)i * Nx + j], sm.rco[i]);
      __syncthreads();
    }
    double nr = 0.0;
    if (warp == 0) {
      for (int y = lane; y < Mx; y += 32) nr += abs2(wj[y]);
      nr = warp_sum(nr);
      if (lane == 0) sm.red[NWARP + 2] = nr;
    }
    __syncthreads();
    const double nrm = sqrt(sm.red[NWARP + 2]);
    const bool dep = !(nrm > 1e-13 * sqrt(sm.red[NWARP + 1])) || nrm == 0.0;
    const double inv = dep ? 0.0 : 1.0 / nrm;
    for (int y = threadIdx.x; y < Mx; y += NT) wj[y] = cscale(wj[y], inv);
    if (threadIdx.x == 0) R[(size_t)j * Nx + j] = make_double2(dep ? 0.0 : nrm, 0.0);
    __syncthreads();
  }
}

// centre c -> c+1 (_kernel.py:68-77)
__device__ void move_right(const Ctx& cx, Smem& sm, int c) {
  const int cap = cx.cap;
  const int cl = sm.dims[c], cr = sm.dims[c + 1], cr2 = sm.dims[c + 2];
  const int Mx = 2 * cl, Nx = cr, N2 = 2 * cr2;
  double2* S = cx.site(c);
  double2* T = cx.site(c + 1);
  // the QR runs in shared memory when the site matrix fits beside the GEMM tiles
  double2* W = (Mx * Nx <= kQrSmemElems) ? cx.tile + kTileElems : cx.W;
  double2* R = cx.X;
  double2* T0 = cx.W0;
  for (int e = threadIdx.x; e < Mx * Nx; e += NT) {
    const int y = e / Nx, r = e - y * Nx;
    W[(size_t)r * Mx + y] = S[(size_t)y * cap + r];
  }
  for (int e = threadIdx.x; e < Nx * N2; e += NT) {
    const int m = e / N2, x = e - m * N2;
    const int j = x / cr2, r = x - j * cr2;
    T0[e] = T[(size_t)(m * 2 + j) * cap + r];
  }
  __syncthreads();
  cgs2_qr(W, Mx, Nx, R, sm);
  for (int e = threadIdx.x; e < Mx * Nx; e += NT) {
    const int y = e / Nx, r = e - y * Nx;
    S[(size_t)y * cap + r] = W[(size_t)r * Mx + y];
  }
  cta_gemm<true, false>(
      Nx, N2, Nx, [&](int m, int q) { return R[(size_t)m * Nx + q]; }, [&](int q, int x) { return T0[(size_t)q * N2 + x]; },
      [&](int m, int x, double2 v) {
        const int j = x / cr2, r = x - j * cr2;
        T[(size_t)(m * 2 + j) * cap + r] = v;
      },
      cx.tile);
  if (threadIdx.x == 0) {
    const double K = Nx, Mm = Mx;
    sm.flops += 16.0 * K * K * (Mm - K / 3.0) + 8.0 * K * K * N2;
  }
}

// centre c -> c-1 (_kernel.py:80-90)
__device__ void move_left(const Ctx& cx, Smem& sm, int c) {
  const int cap = cx.cap;
  const int cl = sm.dims[c], cr = sm.dims[c + 1], clm = sm.dims[c - 1];
  const int Mx = 2 * cr, Nx = cl, Mp = 2 * clm;
  double2* S = cx.site(c);
  double2* T = cx.site(c - 1);
  // the QR runs in shared memory when the site matrix fits beside the GEMM tiles
  double2* W = (Mx * Nx <= kQrSmemElems) ? cx.tile + kTileElems : cx.W;
  double2* R = cx.X;
  double2* T0 = cx.W0;
  for (int e = threadIdx.x; e < Nx * Mx; e += NT) {
    const int l = e / Mx, x = e - l * Mx;
    const int j = x / cr, r = x - j * cr;
    W[(size_t)l * Mx + x] = cconj(S[(size_t)(l * 2 + j) * cap + r]);
  }
  for (int e = threadIdx.x; e < Mp * Nx; e += NT) {
    const int y = e / Nx, m = e - y * Nx;
    T0[e] = T[(size_t)y * cap + m];
  }
  __syncthreads();
  cgs2_qr(W, Mx, Nx, R, sm);
  for (int e = threadIdx.x; e < Nx * Mx; e += NT) {
    const int l = e / Mx, x = e - l * Mx;
    const int j = x / cr, r = x - j * cr;
    S[(size_t)(l * 2 + j) * cap + r] = cconj(W[(size_t)l * Mx + x]);
  }
  cta_gemm<true, true>(
      Mp, Nx, Nx, [&](int y, int m) { return T0[(size_t)y * Nx + m]; },
      [&](int m, int l) { return cconj(R[(size_t)l * Nx + m]); },
      [&](int y, int l, double2 v) { T[(size_t)y * cap + l] = v; }, cx.tile);
  if (threadIdx.x == 0) {
    const double K = Nx, Mm = Mx;
    sm.flops += 16.0 * K * K * (Mm - K / 3.0) + 8.0 * K * K * Mp;
  }
}

__device__ void ensure_center(const Ctx& cx, Smem& sm, int s) {
  const long long t0 = prof_clock();
  const bool moved = sm.center < s || sm.center > s + 1;
  while (sm.center < s) {
    move_right(cx, sm, sm.center);
    if (threadIdx.x == 0) sm.center += 1;
    __syncthreads();
  }
  while (sm.center > s + 1) {
    move_left(cx, sm, sm.center);
    if (threadIdx.x == 0) sm.center -= 1;
    __syncthreads();
  }
  if (moved) prof_add(*cx.job, 3, prof_clock() - t0);
}

// one-site rotation exp(-i angle/2 P) (_kernel.py:105-111); with pauli=true
// applies phase * P instead (exact local pi gates).
__device__ void one_site(const Ctx& cx, Smem& sm, int s, int p, double c, double sn, bool pauli, double2 phase) {
  const int cap = cx.cap;
  const int cl = sm.dims[s], cr = sm.dims[s + 1];
  double2* T = cx.site(s);
  for (int e = threadIdx.x; e < cl * cr; e += NT) {
    const int l = e / cr, r = e - l * cr;
    double2* p0 = T + (size_t)(l * 2) * cap + r;
    double2* p1 = p0 + cap;
    const double2 t0 = *p0, t1 = *p1;
    double2 n0, n1;
    if (pauli) {
      if (p == 1) { n0 = t1; n1 = t0; }
      else if (p == 2) { n0 = make_double2(t1.y, -t1.x); n1 = make_double2(-t0.y, t0.x); }
      else { n0 = t0; n1 = make_double2(-t1.x, -t1.y); }
      n0 = cmul(phase, n0);
      n1 = cmul(phase, n1);
    } else if (p == 3) {
      n0 = cmul(make_double2(c, -sn), t0);
      n1 = cmul(make_double2(c, sn), t1);
    } else if (p == 1) {
      // c t - i s (X t)
      n0 = make_double2(c * t0.x + sn * t1.y, c * t0.y - sn * t1.x);
      n1 = make_double2(c * t1.x + sn * t0.y, c * t1.y - sn * t0.x);
    } else {
      // -i s Y = [[0, -s], [s, 0]]
      n0 = make_double2(c * t0.x - sn * t1.x, c * t0.y - sn * t1.y);
      n1 = make_double2(c * t1.x + sn * t0.x, c * t1.y + sn * t0.y);
    }
    *p0 = n0;
    *p1 = n1;
  }
  __syncthreads();
}

// ----------------------------------------------------------------------------
// canonical-form <Z_j> for every site (no change to the state): right
// environments from the centre leftwards, left environments rightwards.
// ----------------------------------------------------------------------------
__device__ void measure_z(const Ctx& cx, Smem& sm) {
  const Job& jb = *cx.job;
  const int n = jb.n, cap = cx.cap, c = sm.center;
  double2* E = cx.X;   // environment (<= cap x cap)
  double2* F = cx.W0;  // intermediate (<= 2cap x cap)
  {
    const int cl = sm.dims[c], cr = sm.dims[c + 1];
    const double2* T = cx.site(c);
    double acc = 0.0;
    for (int e = threadIdx.x; e < cl * cr; e += NT) {
      const int l = e / cr, r = e - l * cr;
      acc += abs2(T[(size_t)(l * 2) * cap + r]) - abs2(T[(size_t)(l * 2 + 1) * cap + r]);
    }
    acc = cta_sum(acc, sm);
    if (threadIdx.x == 0) sm.zval[c] = acc;
  }
  // leftwards
  if (c > 0) {
    const int cl = sm.dims[c], cr = sm.dims[c + 1];
    const double2* T = cx.site(c);
    cta_gemm<true, true>(
        cl, cl, 2 * cr,
        [&](int l, int q) {
          const int i = q / cr, r = q - i * cr;
          return T[(size_t)(l * 2 + i) * cap + r];
        },
        [&](int q, int l2) {
          const int i = q / cr, r = q - i * cr;
          return cconj(T[(size_t)(l2 * 2 + i) * cap + r]);
        },
        [&](int a, int b, double2 v) { E[(size_t)a * cl + b] = v; }, cx.tile);
    for (int k = c - 1; k >= 0; --k) {
      const int kl = sm.dims[k], km = sm.dims[k + 1];
      const double2* Tk = cx.site(k);
      cta_gemm<true, false>(
          2 * kl, km, km, [&](int y, int m) { return Tk[(size_t)y * cap + m]; },
          [&](int m, int m2) { return E[(size_t)m * km + m2]; },
          [&](int y, int m2, double2 v) { F[(size_t)y * km + m2] = v; }, cx.tile);
      double acc = 0.0;
      for (int e = threadIdx.x; e < 2 * kl * km; e += NT) {
        const int y = e / km, m = e - y * km;
        const double2 f = F[e];
        const double2 t = Tk[(size_t)y * cap + m];
        const double re = f.x * t.x + f.y * t.y;
        acc += (y & 1) ? -re : re;
      }
      acc = cta_sum(acc, sm);
      if (threadIdx.x == 0) sm.zval[k] = acc;
      if (k > 0) {
        cta_gemm<true, true>(
            kl, kl, 2 * km,
            [&](int l, int q) {
              const int i = q / km, m = q - i * km;
              return F[(size_t)(l * 2 + i) * km + m];
            },
            [&](int q, int l2) {
              const int i = q / km, m = q - i * km;
              return cconj(Tk[(size_t)(l2 * 2 + i) * cap + m]);
            },
            [&](int a, int b, double2 v) { E[(size_t)a * kl + b] = v; }, cx.tile);
      }
    }
  }
  // rightwards
  if (c < n - 1) {
    const int cl = sm.dims[c], cr = sm.dims[c + 1];
    const double2* T = cx.site(c);
    cta_gemm<false, false>(
        cr, cr, 2 * cl, [&](int r, int q) { return cconj(T[(size_t)q * cap + r]); },
        [&](int q, int r2) { return T[(size_t)q * cap + r2]; },
        [&](int a, int b, double2 v) { E[(size_t)a * cr + b] = v; }, cx.tile);
    for (int k = c + 1; k < n; ++k) {
      const int kl = sm.dims[k], kr = sm.dims[k + 1];
      const double2* Tk = cx.site(k);
      const int K2 = 2 * kr;
      cta_gemm<true, false>(
          kl, K2, kl, [&](int l, int l2) { return E[(size_t)l * kl + l2]; },
          [&](int l2, int q) {
            const int i = q / kr, r = q - i * kr;
            return Tk[(size_t)(l2 * 2 + i) * cap + r];
          },
          [&](int l, int q, double2 v) { F[(size_t)l * K2 + q] = v; }, cx.tile);
      double acc = 0.0;
      for (int e = threadIdx.x; e < kl * K2; e += NT) {
        const int l = e / K2, q = e - l * K2;
        const int i = q / kr, r = q - i * kr;
        const double2 h = F[e];
        const double2 t = Tk[(size_t)(l * 2 + i) * cap + r];
        const double re = t.x * h.x + t.y * h.y;
        acc += i ? -re : re;
      }
      acc = cta_sum(acc, sm);
      if (threadIdx.x == 0) sm.zval[k] = acc;
      if (k < n - 1) {
        cta_gemm<false, false>(
            kr, kr, 2 * kl, [&](int r, int q) { return cconj(Tk[(size_t)q * cap + r]); },
            [&](int q, int r2) {
              const int l = q >> 1, i = q & 1;
              return F[(size_t)l * K2 + i * kr + r2];
            },
            [&](int a, int b, double2 v) { E[(size_t)a * kr + b] = v; }, cx.tile);
      }
    }
  }
  __syncthreads();
}

__device__ void record_checkpoint(const Ctx& cx, Smem& sm, int sample, int ck) {
  const Job& jb = *cx.job;
  const long long t0 = prof_clock();
  measure_z(cx, sm);
  prof_add(jb, 6, prof_clock() - t0);
  const double sign = jb.ckpt_sign ? (double)jb.ckpt_sign[(size_t)sample * jb.n_ckpt + ck] : 1.0;
  // a sample whose circuit hit a non-converged SVD keeps its raw values but
  // contributes nothing from that checkpoint on; the caller learns which
  // checkpoint through `excluded` and drops it from that row's count
  const bool bad = sm.bad != 0;
  // (one CTA owns the sample and records its checkpoints in order: the first
  // excluded checkpoint is the first write over the caller's -1)
  if (bad && threadIdx.x == 0 && jb.excluded && jb.excluded[sample] < 0) jb.excluded[sample] = ck;
  for (int o = threadIdx.x; o < jb.n_obs; o += NT) {
    const double z = sm.zval[jb.obs_sites[o]];
    if (jb.values) jb.values[((size_t)sample * jb.n_ckpt + ck) * jb.n_obs + o] = z;
    if (bad) continue;
    const double v = sign * z;
    const long long qv = llrint(v * FIX);
    const long long qv2 = llrint(z * z * FIX);
    const size_t row = jb.sum_row ? (size_t)jb.sum_row[(size_t)sample * jb.n_ckpt + ck] : (size_t)ck;
    atomicAdd(&jb.sum_v[row * jb.n_obs + o], (unsigned long long)qv);
    atomicAdd(&jb.sum_v2[row * jb.n_obs + o], (unsigned long long)qv2);
  }
  if (threadIdx.x == 0 && jb.discarded) jb.discarded[(size_t)sample * jb.n_ckpt + ck] = sm.counters[3];
  __syncthreads();
}

// ----------------------------------------------------------------------------
// the persistent ensemble kernel
// ----------------------------------------------------------------------------
__global__ void __launch_bounds__(NT, TB_ENGINE_MINB) ensemble_kernel(const __grid_constant__ Job job) {
  extern __shared__ double2 dyn_smem[];
  __shared__ Smem sm;
  const int cap = job.cap, n = job.n;
  Ctx cx;
  cx.job = &job;
  cx.cap = cap;
  // cluster launch: rank 0 of each cluster runs circuits, ranks 1..7 only
  // serve its wide Jacobi calls (cluster_follow)
#if TB_ENGINE_SMALL
  const int wid = blockIdx.x;
#else
  const int wid = job.cluster > 1 ? blockIdx.x / job.cluster : blockIdx.x;
  if (job.cluster > 1) {
    if (threadIdx.x == 0) sm.cluster = job.cluster;
    cl_sync();  // every CTA of the cluster is running before any DSMEM access
    if (cl_rank() != 0) {
      cluster_follow(sm, dyn_smem);
      return;
    }
  }
#endif
  cx.mps = job.ws_mps + job.mps_stride * wid;
  cx.W = job.ws_W + job.mat_stride * wid;
  cx.W0 = job.ws_W0 + job.mat_stride * wid;
  cx.X = job.ws_X + job.mat_stride * wid;
  cx.tile = dyn_smem;
  if (threadIdx.x == 0) {
    sm.cluster = job.cluster;
    sm.cl_tma = job.cluster_tma;
    sm.flops = 0.0;
    sm.prof = job.prof;
    sm.tmem_on = job.qrcp_tmem;
    sm.screen_on = job.gram_screen;
    sm.bad = 0;
    sm.maxsweep = job.max_sweeps;
    sm.inject = job.inject;
  }
#if !TB_ENGINE_SMALL
  if (job.qrcp_tmem) tmem_alloc(sm);
#endif
  for (int iter = 0;; ++iter) {
    // both modes take work items from an atomic queue: whole samples (queue
    // mode) or slots, each advanced by one checkpoint segment (slot mode).
    // More slots than CTAs balance the per-segment work (a segment's cost
    // varies with its ring-gate count) instead of waiting for the slowest.
    if (threadIdx.x == 0) {
      const int q = atomicAdd(job.next_sample, 1);
      sm.sample = (q < job.n_samples && job.slot_mode && job.order) ? job.order[q] : q;
    }
    __syncthreads();
    const int sample = sm.sample;
    if (sample >= job.n_samples) break;
    // a slot's MPS and bookkeeping live with the slot, not with the CTA
    if (job.slot_mode) cx.mps = job.ws_mps + job.mps_stride * (size_t)sample;
    int* sdims = job.slot_dims + (size_t)sample * (MAXN + 1);
    // --- initial state: product state, or the slot's persistent state
    const bool fresh = !job.slot_mode || (job.reset && job.reset[sample]);
    if (job.slot_mode && !fresh && job.slot_gen[sample] != job.gen) {
      // the slot's state was built in another workspace generation (the pool
      // was reallocated or reshaped, or another engine call reused it): refuse
      // to continue it rather than read stale memory
      if (threadIdx.x == 0) atomicOr(job.status, 4);
      __syncthreads();
      continue;
    }
    if (threadIdx.x == 0) sm.bad = (job.slot_mode && !fresh) ? (int)job.slot_bad[sample] : 0;
    if (fresh && job.init_mps) {
      // hybrid fan-out: every sample starts from the broadcast snapshot
      for (int e = threadIdx.x; e < n + 1; e += NT) sm.dims[e] = job.init_dims[e];
      __syncthreads();
      for (int s = 0; s < n; ++s) {
        const int cl = sm.dims[s], cr = sm.dims[s + 1];
        const double2* src = job.init_mps + (size_t)s * cap * 2 * cap;
        double2* dst = cx.site(s);
        for (int e = threadIdx.x; e < cl * 2 * cr; e += NT) {
          const int row = e / cr, r = e - row * cr;
          dst[(size_t)row * cap + r] = src[(size_t)row * cap + r];
        }
      }
      if (threadIdx.x == 0) {
        sm.center = job.init_center;
        int mx = 1;
        for (int q = 0; q <= n; ++q) mx = max(mx, sm.dims[q]);
        sm.counters[0] = sm.counters[1] = sm.counters[3] = 0.0;
        sm.counters[2] = mx;
      }
    } else if (fresh) {
      for (int e = threadIdx.x; e < n + 1; e += NT) sm.dims[e] = 1;
      for (int e = threadIdx.x; e < n * 2; e += NT) {
        const int s = e >> 1, i = e & 1;
        cx.site(s)[(size_t)i * cap] = make_double2(job.init_vecs[4 * s + 2 * i], job.init_vecs[4 * s + 2 * i + 1]);
      }
      if (threadIdx.x == 0) {
        sm.center = 0;
        sm.counters[0] = sm.counters[1] = sm.counters[3] = 0.0;
        sm.counters[2] = 1.0;
      }
    } else {
      for (int e = threadIdx.x; e < n + 1; e += NT) sm.dims[e] = sdims[e];
      if (threadIdx.x == 0) {
        sm.center = job.slot_center[sample];
        for (int q = 0; q < 4; ++q) sm.counters[q] = job.slot_counters[(size_t)sample * 4 + q];
      }
    }
    __syncthreads();
    const long long tstart = prof_clock();
    unsigned long long ns0 = 0;
    if (job.sample_ms && threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ns0));
    const int64_t g0 = job.gate_off[sample], g1 = job.gate_off[sample + 1];
    int ck = 0;
    for (int64_t gi = g0; gi < g1; ++gi) {
      while (ck < job.n_ckpt && job.ckpt_end[(size_t)sample * job.n_ckpt + ck] <= (int)(gi - g0)) {
        record_checkpoint(cx, sm, sample, ck);
        ++ck;
      }
      const uint32_t w = job.gates[gi];
      const int a = w & 0xFF, b = (w >> 8) & 0xFF, pa = (w >> 16) & 3, pb = (w >> 18) & 3;
      const bool mr = (w >> 20) & 1, is_pi = (w >> 21) & 1;
      const int ai = w >> 22;
      const double c = job.angle_cs[2 * ai], s = job.angle_cs[2 * ai + 1];
      if (b == TB_ONE_SITE) {
        one_site(cx, sm, a, pa, c, s, false, cz());
        if (threadIdx.x == 0) sm.counters[0] += 1.0;
        __syncthreads();
      } else if (is_pi && job.pi_local) {
        one_site(cx, sm, a, pa, 0, 0, true, make_double2(0.0, -1.0));
        one_site(cx, sm, b, pb, 0, 0, true, make_double2(1.0, 0.0));
        if (threadIdx.x == 0) sm.counters[0] += 1.0;
        __syncthreads();
      } else if (b == a + 1) {
        ensure_center(cx, sm, a);
        two_site(cx, sm, a, 0, pa, pb, c, s, mr);
        if (threadIdx.x == 0) sm.center = mr ? a + 1 : a;
        __syncthreads();
      } else {
        for (int q = b - 1; q > a; --q) {
          ensure_center(cx, sm, q);
          two_site(cx, sm, q, 1, 0, 0, 0, 0, false);
          if (threadIdx.x == 0) sm.center = q;
          __syncthreads();
        }
        two_site(cx, sm, a, 0, pa, pb, c, s, true);
        if (threadIdx.x == 0) sm.center = a + 1;
        __syncthreads();
        for (int q = a + 1; q < b; ++q) {
          two_site(cx, sm, q, 1, 0, 0, 0, 0, true);
          if (threadIdx.x == 0) sm.center = q + 1;
          __syncthreads();
        }
      }
    }
    while (ck < job.n_ckpt) {
      record_checkpoint(cx, sm, sample, ck);
      ++ck;
    }
    prof_add(job, 7, prof_clock() - tstart);
    if (job.states) {
      // retain the final MPS (zero-padded to cap x 2 x cap per site) for the
      // signed-mixture post-processing
      double2* dst = job.states + (size_t)sample * n * cap * 2 * cap;
      for (int st = 0; st < n; ++st) {
        const double2* src = cx.site(st);
        const int cl = sm.dims[st], cr = sm.dims[st + 1];
        for (int e = threadIdx.x; e < cap * 2 * cap; e += NT) {
          const int row = e / cap, r = e - row * cap;
          dst[(size_t)st * cap * 2 * cap + e] = ((row >> 1) < cl && r < cr) ? src[e] : cz();
        }
      }
      for (int e = threadIdx.x; e <= n; e += NT) job.state_dims[(size_t)sample * (n + 1) + e] = sm.dims[e];
      if (threadIdx.x == 0) job.state_center[sample] = sm.center;
    }
    if (job.sample_ms && threadIdx.x == 0) {
      unsigned long long ns1;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ns1));
      job.sample_ms[sample] = 1e-6 * (double)(ns1 - ns0);
    }
    if (threadIdx.x == 0) {
      if (job.ledger)
        for (int q = 0; q < 4; ++q) job.ledger[(size_t)sample * 4 + q] = sm.counters[q];
      if (job.slot_mode) {
        job.slot_center[sample] = sm.center;
        for (int q = 0; q < 4; ++q) job.slot_counters[(size_t)sample * 4 + q] = sm.counters[q];
        job.slot_bad[sample] = (unsigned char)sm.bad;
        job.slot_gen[sample] = job.gen;
      }
    }
    if (job.slot_mode)
      for (int e = threadIdx.x; e < n + 1; e += NT) sdims[e] = sm.dims[e];
    __syncthreads();
  }
  if (threadIdx.x == 0) job.flops[blockIdx.x] += sm.flops;
#if !TB_ENGINE_SMALL
  if (job.qrcp_tmem) tmem_free(sm);
  if (job.cluster > 1) cluster_release(sm);
#endif
}

#if !TB_ENGINE_SMALL  // single-state kernels: only in the full engine
// ----------------------------------------------------------------------------
// transfer-contraction expectation of a general Pauli string (mps.py:170-182)
// ----------------------------------------------------------------------------
__device__ double transfer_expect(const double2* buf, int n, int cap, const Smem& sm, const int* codes, double2* E,
                                  double2* F, double2* tile) {
  if (threadIdx.x == 0) E[0] = make_double2(1.0, 0.0);
  __syncthreads();
  for (int k = 0; k < n; ++k) {
    const int kl = sm.dims[k], kr = sm.dims[k + 1], K2 = 2 * kr;
    const double2* T = buf + (size_t)k * cap * 2 * cap;
    const int p = codes[k];
    // F[l][(i,r)] = sum_l2 E[l][l2] T[l2][i][r], then P on i
    cta_gemm<true, false>(
        kl, K2, kl, [&](int l, int l2) { return E[(size_t)l * kl + l2]; },
        [&](int l2, int q) {
          const int i = q / kr, r = q - i * kr;
          return T[(size_t)(l2 * 2 + i) * cap + r];
        },
        [&](int l, int q, double2 v) { F[(size_t)l * K2 + q] = v; }, tile);
    if (p != 0) {
      for (int e = threadIdx.x; e < kl * kr; e += NT) {
        const int l = e / kr, r = e - l * kr;
        double2* f0 = F + (size_t)l * K2 + r;
        double2* f1 = f0 + kr;
        const double2 a = *f0, b = *f1;
        if (p == 1) { *f0 = b; *f1 = a; }
        else if (p == 2) { *f0 = make_double2(b.y, -b.x); *f1 = make_double2(-a.y, a.x); }
        else { *f1 = make_double2(-b.x, -b.y); }
      }
      __syncthreads();
    }
    cta_gemm<false, false>(
        kr, kr, 2 * kl,
        [&](int r, int q) {
          const int l = q >> 1, i = q & 1;
          return cconj(T[(size_t)(l * 2 + i) * cap + r]);
        },
        [&](int q, int r2) {
          const int l = q >> 1, i = q & 1;
          return F[(size_t)l * K2 + i * kr + r2];
        },
        [&](int a, int b, double2 v) { E[(size_t)a * kr + b] = v; }, tile);
  }
  const double v = E[0].x;
  __syncthreads();
  return v;
}

__global__ void __launch_bounds__(NT, 1) expectation_kernel(const double2* buf, int n, int cap, const int* dims,
                                                            const int* codes, double2* E, double2* F, double* out) {
  extern __shared__ double2 dyn_smem[];
  __shared__ Smem sm;
  for (int e = threadIdx.x; e < n + 1; e += NT) sm.dims[e] = dims[e];
  __syncthreads();
  const double v = transfer_expect(buf, n, cap, sm, codes, E, F, dyn_smem);
  if (threadIdx.x == 0) out[0] = v;
}

// Batched transfer-contraction expectations (the signed-mixture post-processing
// of SPEC.md:413-417): states [S][n][cap][2][cap] with dims [S][n+1], Pauli
// strings codes [O][n]; out [S][O].  Persistent CTAs stride over the states;
// each CTA uses its own slice of the W / W0 scratch for the environments.
__global__ void __launch_bounds__(NT, 1) expectation_batch_kernel(const double2* bufs, int S, int n, int cap,
                                                                  const int* dims, const int* codes, int O,
                                                                  double2* Ew, double2* Fw, size_t mat_stride,
                                                                  double* out) {
  extern __shared__ double2 dyn_smem[];
  __shared__ Smem sm;
  double2* E = Ew + mat_stride * blockIdx.x;
  double2* F = Fw + mat_stride * blockIdx.x;
  for (int st = blockIdx.x; st < S; st += gridDim.x) {
    __syncthreads();
    for (int e = threadIdx.x; e < n + 1; e += NT) sm.dims[e] = dims[(size_t)st * (n + 1) + e];
    __syncthreads();
    const double2* buf = bufs + (size_t)st * n * cap * 2 * cap;
    for (int o = 0; o < O; ++o) {
      const double v = transfer_expect(buf, n, cap, sm, codes + (size_t)o * n, E, F, dyn_smem);
      if (threadIdx.x == 0) out[(size_t)st * O + o] = v;
    }
  }
}

// ----------------------------------------------------------------------------
// batched thin SVD (unit-test surface of the Jacobi path)
// ----------------------------------------------------------------------------
__global__ void __launch_bounds__(NT, 1) svd_kernel(const double2* a, int m, int n, double2* Wg, double2* W0g,
                                                    double2* Xg, size_t mat_stride, double* s, double2* u,
                                                    double2* vh, int* status, unsigned long long* prof, int precond,
                                                    int kcut) {
  extern __shared__ double2 dyn_smem[];
  __shared__ Smem sm;
  const bool clu = (precond >> 2) & 1;  // 8-CTA clusters: one matrix per cluster
  const int b = clu ? blockIdx.x / CL : blockIdx.x;
  const int K = min(m, n);
  if (clu) {
    cl_sync();
    if (cl_rank() != 0) {
      cluster_follow(sm, dyn_smem);
      return;
    }
  }
  if (threadIdx.x == 0) {
    sm.cluster = clu ? CL : 0;
    sm.cl_tma = ((precond >> 3) & 1) | (((precond >> 5) & 3) << 1);  // bits 1, 2: debug switches
    sm.prof = prof;
    sm.kcut = (kcut > 0 && kcut < K) ? kcut : MAXDIM;
    sm.tmem_on = (precond >> 1) & 1;
    sm.screen_on = ((precond >> 4) & 1) ? 1 + ((precond >> 7) & 3) : 0;  // 0 off, 1..3 (see TB_GRAM_SCREEN)
    sm.maxsweep = MAXSWEEP;
    sm.inject = 0;
    sm.sample = 0;
  }
  if (precond & 2) tmem_alloc(sm);
  double2* W = Wg + mat_stride * b;
  double2* W0 = W0g + mat_stride * b;
  double2* X = Xg + mat_stride * b;
  const double2* A = a + (size_t)b * m * n;
  const bool pre = (precond & 1) && m >= 32 && n >= 32;
  // left singular vectors of A (m x n): columns of W = A, or Y = A^H when preconditioned
  for (int e = threadIdx.x; e < m * n; e += NT) {
    const int y = e / n, c = e - y * n;
    if (pre) W[(size_t)y * n + c] = cconj(A[e]);
    else W[(size_t)c * m + y] = A[e];
    W0[(size_t)c * m + y] = A[e];
  }
  __syncthreads();
  const int Neff = pre ? precond_jacobi(W, X, m, n, sm, dyn_smem, status) : jacobi(W, m, n, sm, dyn_smem, status);
  if (!pre)
    for (int y = threadIdx.x; y < m; y += NT) sm.qpinv[y] = y;
  __syncthreads();
  if (threadIdx.x == 0 && prof) {
    atomicAdd(&prof[1], 1ull);
    atomicAdd(&prof[2], (unsigned long long)sm.sweeps);
  }
  sort_sigma(W, m, Neff, sm);
  for (int i = threadIdx.x; i < K; i += NT) s[(size_t)b * K + i] = sm.sig[sm.perm[i]];
  if (u)
    for (int e = threadIdx.x; e < m * K; e += NT) {
      const int y = e / K, c = e - y * K;
      const int pc = sm.perm[c];
      const double sg = sm.sig[pc];
      u[(size_t)b * m * K + e] = sg > 0 ? cscale(W[(size_t)pc * m + sm.qpinv[y]], 1.0 / sg) : cz();
    }
  if (vh)
    cta_gemm<true, true>(
        K, n, m,
        [&](int c, int y) {
          const int pc = sm.perm[c];
          const double sg = sm.sig[pc];
          return sg > 0 ? cscale(cconj(W[(size_t)pc * m + sm.qpinv[y]]), 1.0 / (sg * sg)) : cz();
        },
        [&](int y, int x) { return W0[(size_t)x * m + y]; },
        [&](int c, int x, double2 v) { vh[(size_t)b * K * n + (size_t)c * n + x] = v; }, dyn_smem);
  if (precond & 2) tmem_free(sm);
  if (clu) cluster_release(sm);
}

#endif  // !TB_ENGINE_SMALL

constexpr size_t kTileBytes = 2 * TK * TLD * sizeof(double2);
constexpr size_t kDynSmem = (3 * JB + 1) * SROWS * sizeof(double2);  // Jacobi/QRCP slots + q buffer; tiles alias
static_assert(kDynSmem >= kTileBytes, "tile buffer aliases the Jacobi slots");

#if !TB_ENGINE_SMALL
__global__ void sum_flops_kernel(const double* f, int n, double* out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double s = 0;
    for (int i = 0; i < n; ++i) s += f[i];
    out[0] += s;
  }
}
#endif

}  // namespace TB_ENGINE_NS
