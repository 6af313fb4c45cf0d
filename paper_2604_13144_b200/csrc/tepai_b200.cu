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
#include <string.h>

#include <string>
#include <vector>

#include "../../include/tepai_b200.h"

namespace tb {

constexpr int NT = 512;        // threads per CTA
constexpr int NWARP = NT / 32;  // warps per CTA
constexpr int MAXCAP = 128;     // largest supported bond capacity
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
struct Job {
  int n, cap, chi_cut, pi_local;
  double floor;
  int n_samples, n_ckpt, n_obs;
  const uint32_t* gates;
  const int64_t* gate_off;
  const int32_t* ckpt_end;
  const int8_t* ckpt_sign;
  const double* angle_cs;
  const int32_t* obs_sites;
  const double* init_vecs;  // NULL => state preloaded in slot 0 (run_stream mode)
  // outputs
  double* values;
  double* discarded;
  double* ledger;
  unsigned long long* sum_v;
  unsigned long long* sum_v2;
  double* flops;       // [gridDim.x]
  int* next_sample;
  int* status;         // bit 0: Jacobi non-convergence, bit 1: bad dims
  // run_stream mode i/o
  int* io_dims;        // [n+1]
  int* io_center;
  double* io_counters; // [4] in/out
  // workspace
  double2* ws_mps;
  double2* ws_W;
  double2* ws_W0;
  double2* ws_X;
  size_t mps_stride, mat_stride;
};

struct Smem {
  int dims[MAXN + 1];
  double sig[MAXDIM];
  int perm[MAXDIM];
  double2 rco[MAXDIM];
  double red[NWARP * 4];
  double zval[MAXN];
  double counters[4];
  double flops;
  double scale, invsig_tmp;
  int k;
  int flag;
  int sample;
  int center;
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
  const int m = Np - 1;
  if (p == 0) { i = m; j = r; }
  else { i = (r + p) % m; j = (r - p + m) % m; }
}

__device__ int hestenes(double2* W, int Mw, int Nw, Smem& sm) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int Np = Nw + (Nw & 1);
  if (Nw < 2) return 0;
  const double tol = sqrt((double)Mw) * 1.1102230246251565e-16;
  int sweep = 0;
  for (; sweep < MAXSWEEP; ++sweep) {
    if (threadIdx.x == 0) sm.flag = 0;
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

// ----------------------------------------------------------------------------
// Per-CTA sample context
// ----------------------------------------------------------------------------
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

  // theta = A (2cl x cm) . B (cm x 2cr), written into W in the Jacobi orientation
  cta_gemm<true, false>(
      M, N, cm, [&](int m, int k) { return A[(size_t)m * cap + k]; },
      [&](int k, int n) {
        const int j = n / cr, r = n - j * cr;
        return B[(size_t)(k * 2 + j) * cap + r];
      },
      [&](int m, int n, double2 v) {
        if (merge_right) W[(size_t)n * Mw + m] = v;
        else W[(size_t)m * Mw + n] = cconj(v);
      },
      cx.tile);

  // gate / swap on the physical pair, fused into the (W, W0) write-out
  const int fa = (pa == 3) ? 0 : 1, fb = (pb == 3) ? 0 : 1;
  for (int e = threadIdx.x; e < cl * cr; e += NT) {
    const int l = e / cr, r = e - (e / cr) * cr;
    double2 t[2][2];
    size_t idx[2][2];
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int row = l * 2 + i, col = j * cr + r;
        idx[i][j] = merge_right ? (size_t)col * Mw + row : (size_t)row * Mw + col;
        const double2 v = W[idx[i][j]];
        t[i][j] = merge_right ? v : cconj(v);
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
        const double2 v = merge_right ? o[i][j] : cconj(o[i][j]);
        W[idx[i][j]] = v;
        W0[idx[i][j]] = v;
      }
  }
  __syncthreads();

  const int sweeps = hestenes(W, Mw, Nw, sm);
  if (sweeps > MAXSWEEP && threadIdx.x == 0) atomicOr(jb.status, 1);
  sort_sigma(W, Mw, Nw, sm);

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
  // isometric factor Q[:, c] = W[:, perm c] / sigma
  for (int e = threadIdx.x; e < k * Mw; e += NT) {
    const int c = e / Mw, y = e - c * Mw;
    const int pc = sm.perm[c];
    const double2 q = cscale(W[(size_t)pc * Mw + y], 1.0 / sm.sig[pc]);
    if (merge_right) {
      A[(size_t)y * cap + c] = q;  // site s [(l,i)][c]
    } else {
      const int j = y / cr, r = y - j * cr;
      B[(size_t)(c * 2 + j) * cap + r] = cconj(q);  // site s+1 [c][(j,r)]
    }
  }
  // weighted factor P = Q^H W0 (k x Nw), scaled by 1/sqrt(kept)
  cta_gemm<true, true>(
      k, Nw, Mw,
      [&](int c, int y) {
        const int pc = sm.perm[c];
        return cscale(cconj(W[(size_t)pc * Mw + y]), 1.0 / sm.sig[pc]);
      },
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
  double2* W = cx.W;
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
  double2* W = cx.W;
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
  measure_z(cx, sm);
  const double sign = jb.ckpt_sign ? (double)jb.ckpt_sign[(size_t)sample * jb.n_ckpt + ck] : 1.0;
  for (int o = threadIdx.x; o < jb.n_obs; o += NT) {
    const double z = sm.zval[jb.obs_sites[o]];
    if (jb.values) jb.values[((size_t)sample * jb.n_ckpt + ck) * jb.n_obs + o] = z;
    const double v = sign * z;
    const long long qv = llrint(v * FIX);
    const long long qv2 = llrint(z * z * FIX);
    atomicAdd(&jb.sum_v[(size_t)ck * jb.n_obs + o], (unsigned long long)qv);
    atomicAdd(&jb.sum_v2[(size_t)ck * jb.n_obs + o], (unsigned long long)qv2);
  }
  if (threadIdx.x == 0 && jb.discarded) jb.discarded[(size_t)sample * jb.n_ckpt + ck] = sm.counters[3];
  __syncthreads();
}

// ----------------------------------------------------------------------------
// the persistent ensemble kernel
// ----------------------------------------------------------------------------
__global__ void __launch_bounds__(NT, 1) ensemble_kernel(const __grid_constant__ Job job) {
  extern __shared__ double2 dyn_smem[];
  __shared__ Smem sm;
  const int cap = job.cap, n = job.n;
  Ctx cx;
  cx.job = &job;
  cx.cap = cap;
  cx.mps = job.ws_mps + job.mps_stride * blockIdx.x;
  cx.W = job.ws_W + job.mat_stride * blockIdx.x;
  cx.W0 = job.ws_W0 + job.mat_stride * blockIdx.x;
  cx.X = job.ws_X + job.mat_stride * blockIdx.x;
  cx.tile = dyn_smem;
  if (threadIdx.x == 0) sm.flops = 0.0;
  for (;;) {
    if (threadIdx.x == 0) sm.sample = atomicAdd(job.next_sample, 1);
    __syncthreads();
    const int sample = sm.sample;
    if (sample >= job.n_samples) break;
    // --- initial state
    if (job.init_vecs) {
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
      for (int e = threadIdx.x; e < n + 1; e += NT) sm.dims[e] = job.io_dims[e];
      if (threadIdx.x == 0) {
        sm.center = *job.io_center;
        for (int q = 0; q < 4; ++q) sm.counters[q] = job.io_counters[q];
      }
    }
    __syncthreads();
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
    if (threadIdx.x == 0) {
      if (job.ledger)
        for (int q = 0; q < 4; ++q) job.ledger[(size_t)sample * 4 + q] = sm.counters[q];
      if (!job.init_vecs) {
        *job.io_center = sm.center;
        for (int q = 0; q < 4; ++q) job.io_counters[q] = sm.counters[q];
      }
    }
    if (!job.init_vecs)
      for (int e = threadIdx.x; e < n + 1; e += NT) job.io_dims[e] = sm.dims[e];
    __syncthreads();
  }
  if (threadIdx.x == 0) job.flops[blockIdx.x] += sm.flops;
}

// ----------------------------------------------------------------------------
// transfer-contraction expectation of a general Pauli string (mps.py:170-182)
// ----------------------------------------------------------------------------
__global__ void __launch_bounds__(NT, 1) expectation_kernel(const double2* buf, int n, int cap, const int* dims,
                                                            const int* codes, double2* E, double2* F, double* out) {
  extern __shared__ double2 dyn_smem[];
  __shared__ Smem sm;
  for (int e = threadIdx.x; e < n + 1; e += NT) sm.dims[e] = dims[e];
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
        [&](int l, int q, double2 v) { F[(size_t)l * K2 + q] = v; }, dyn_smem);
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
        [&](int a, int b, double2 v) { E[(size_t)a * kr + b] = v; }, dyn_smem);
  }
  if (threadIdx.x == 0) out[0] = E[0].x;
}

// ----------------------------------------------------------------------------
// batched thin SVD (unit-test surface of the Jacobi path)
// ----------------------------------------------------------------------------
__global__ void __launch_bounds__(NT, 1) svd_kernel(const double2* a, int m, int n, double2* Wg, double2* W0g,
                                                    size_t mat_stride, double* s, double2* u, double2* vh,
                                                    int* status) {
  extern __shared__ double2 dyn_smem[];
  __shared__ Smem sm;
  const int b = blockIdx.x;
  const int K = min(m, n);
  double2* W = Wg + mat_stride * b;
  double2* W0 = W0g + mat_stride * b;
  const double2* A = a + (size_t)b * m * n;
  // orthogonalise columns of A (m x n): W[c][y] = A[y][c]
  for (int e = threadIdx.x; e < m * n; e += NT) {
    const int y = e / n, c = e - y * n;
    W[(size_t)c * m + y] = A[e];
    W0[(size_t)c * m + y] = A[e];
  }
  __syncthreads();
  const int sweeps = hestenes(W, m, n, sm);
  if (sweeps > MAXSWEEP && threadIdx.x == 0) atomicOr(status, 1);
  sort_sigma(W, m, n, sm);
  for (int i = threadIdx.x; i < K; i += NT) s[(size_t)b * K + i] = sm.sig[sm.perm[i]];
  if (u)
    for (int e = threadIdx.x; e < m * K; e += NT) {
      const int y = e / K, c = e - y * K;
      const int pc = sm.perm[c];
      const double sg = sm.sig[pc];
      u[(size_t)b * m * K + e] = sg > 0 ? cscale(W[(size_t)pc * m + y], 1.0 / sg) : cz();
    }
  if (vh)
    cta_gemm<true, true>(
        K, n, m,
        [&](int c, int y) {
          const int pc = sm.perm[c];
          const double sg = sm.sig[pc];
          return sg > 0 ? cscale(cconj(W[(size_t)pc * m + y]), 1.0 / (sg * sg)) : cz();
        },
        [&](int y, int x) { return W0[(size_t)x * m + y]; },
        [&](int c, int x, double2 v) { vh[(size_t)b * K * n + (size_t)c * n + x] = v; }, dyn_smem);
}

constexpr size_t kTileBytes = 2 * TK * TLD * sizeof(double2);

__global__ void sum_flops_kernel(const double* f, int n, double* out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double s = 0;
    for (int i = 0; i < n; ++i) s += f[i];
    out[0] += s;
  }
}

}  // namespace tb

// ============================================================================
// host side: context, workspace, C ABI
// ============================================================================
struct tb_ctx {
  int device = 0;
  int sms = 0;
  std::string err;
  // workspace
  double2* mps = nullptr;
  double2* W = nullptr;
  double2* W0 = nullptr;
  double2* X = nullptr;
  size_t mps_cap_bytes = 0, mat_cap_bytes = 0;  // per slot
  int slots = 0;
  size_t mps_stride = 0, mat_stride = 0;
  // small device scratch
  int* dscratch = nullptr;  // [0] next_sample, [1] status, [2] center, [3..] dims
  double* dflops = nullptr;
  double* dcounters = nullptr;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
};

namespace {

int fail(tb_ctx* c, int code, const std::string& msg) {
  if (c) c->err = msg;
  return code;
}

#define TB_CUDA(ctx, call)                                                                      \
  do {                                                                                          \
    cudaError_t _e = (call);                                                                    \
    if (_e != cudaSuccess) return fail(ctx, TB_ECUDA, std::string(#call) + ": " + cudaGetErrorString(_e)); \
  } while (0)

int ensure_workspace(tb_ctx* c, int slots, int n, int cap) {
  const size_t mps_bytes = (size_t)n * cap * 2 * cap * sizeof(double2);
  const size_t mat_bytes = (size_t)(2 * cap) * (2 * cap) * sizeof(double2);
  if (slots <= c->slots && mps_bytes <= c->mps_cap_bytes && mat_bytes <= c->mat_cap_bytes) {
    c->mps_stride = mps_bytes / sizeof(double2);
    c->mat_stride = mat_bytes / sizeof(double2);
    return TB_OK;
  }
  cudaFree(c->mps);
  cudaFree(c->W);
  cudaFree(c->W0);
  cudaFree(c->X);
  c->mps = c->W = c->W0 = c->X = nullptr;
  const int s = slots > c->slots ? slots : c->slots;
  const size_t mb = mps_bytes > c->mps_cap_bytes ? mps_bytes : c->mps_cap_bytes;
  const size_t tb = mat_bytes > c->mat_cap_bytes ? mat_bytes : c->mat_cap_bytes;
  if (cudaMalloc(&c->mps, mb * s) != cudaSuccess || cudaMalloc(&c->W, tb * s) != cudaSuccess ||
      cudaMalloc(&c->W0, tb * s) != cudaSuccess || cudaMalloc(&c->X, tb * s) != cudaSuccess) {
    cudaGetLastError();
    c->slots = 0;
    c->mps_cap_bytes = c->mat_cap_bytes = 0;
    return fail(c, TB_ENOMEM, "workspace allocation failed");
  }
  c->slots = s;
  c->mps_cap_bytes = mb;
  c->mat_cap_bytes = tb;
  c->mps_stride = mps_bytes / sizeof(double2);
  c->mat_stride = mat_bytes / sizeof(double2);
  return TB_OK;
}

int validate_shape(tb_ctx* c, int64_t n, int64_t cap, int64_t chi_cut) {
  if (n < 1 || n > tb::MAXN) return fail(c, TB_EINVAL, "n must lie in [1, 64]");
  if (cap < 1 || cap > tb::MAXCAP) return fail(c, TB_EINVAL, "cap must lie in [1, 128]");
  if (chi_cut < 1) return fail(c, TB_EINVAL, "chi_cut must be >= 1");
  return TB_OK;
}

int launch_ensemble(tb_ctx* c, tb::Job& job, int grid, cudaStream_t st, float* kernel_ms) {
  const size_t smem = tb::kTileBytes;
  TB_CUDA(c, cudaFuncSetAttribute(tb::ensemble_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  if (kernel_ms) TB_CUDA(c, cudaEventRecord(c->e0, st));
  tb::ensemble_kernel<<<grid, tb::NT, smem, st>>>(job);
  TB_CUDA(c, cudaGetLastError());
  if (kernel_ms) {
    TB_CUDA(c, cudaEventRecord(c->e1, st));
    TB_CUDA(c, cudaEventSynchronize(c->e1));
    TB_CUDA(c, cudaEventElapsedTime(kernel_ms, c->e0, c->e1));
  }
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
  if (cudaMalloc(&c->dscratch, 256 * sizeof(int)) != cudaSuccess ||
      cudaMalloc(&c->dflops, 4096 * sizeof(double)) != cudaSuccess ||
      cudaMalloc(&c->dcounters, 8 * sizeof(double)) != cudaSuccess ||
      cudaEventCreate(&c->e0) != cudaSuccess || cudaEventCreate(&c->e1) != cudaSuccess) {
    cudaGetLastError();
    delete c;
    return TB_ECUDA;
  }
  *out = c;
  return TB_OK;
}

void tb_destroy(tb_ctx* c) {
  if (!c) return;
  cudaFree(c->mps);
  cudaFree(c->W);
  cudaFree(c->W0);
  cudaFree(c->X);
  cudaFree(c->dscratch);
  cudaFree(c->dflops);
  cudaFree(c->dcounters);
  if (c->e0) cudaEventDestroy(c->e0);
  if (c->e1) cudaEventDestroy(c->e1);
  delete c;
}

const char* tb_last_error(const tb_ctx* c) { return c ? c->err.c_str() : "null context"; }

int tb_num_sms(const tb_ctx* c) { return c ? c->sms : 0; }

int tb_run_stream(tb_ctx* c, double* buf, int64_t n, int64_t cap, int64_t* dims, int64_t center, const int64_t* ga,
                  const int64_t* gb, const int64_t* pa, const int64_t* pb, const double* ang, const int64_t* anchors,
                  int64_t n_gates, int64_t chi_cut, double floor, double* counters, int64_t* new_center) {
  if (!c) return TB_EINVAL;
  int rc = validate_shape(c, n, cap, chi_cut);
  if (rc) return rc;
  if (chi_cut > cap) return fail(c, TB_EINVAL, "chi_cut exceeds the buffer capacity");
  if (!buf || !dims || !counters || !new_center || (n_gates > 0 && (!ga || !gb || !pa || !pb || !ang || !anchors)))
    return fail(c, TB_EINVAL, "null argument");
  for (int64_t s = 0; s <= n; ++s)
    if (dims[s] < 1 || dims[s] > cap) return fail(c, TB_EINVAL, "bond dimension outside [1, cap]");
  if (center < 0 || center >= n) return fail(c, TB_EINVAL, "center outside [0, n)");
  // pack the lowered stream (angle table of distinct angles, <= 1024)
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
    uint32_t w = (uint32_t)a | ((b < 0 ? TB_ONE_SITE : (uint32_t)b) << 8) | ((uint32_t)pa[i] << 16) |
                 ((uint32_t)(b < 0 ? 0 : pb[i]) << 18) | ((uint32_t)(anchors[i] > a) << 20) |
                 ((uint32_t)(ang[i] == M_PI) << 21) | ((uint32_t)ai << 22);
    words[(size_t)i] = w;
  }
  if (table.empty()) table = {1.0, 0.0};
  rc = ensure_workspace(c, 1, (int)n, (int)cap);
  if (rc) return rc;
  uint32_t* dg = nullptr;
  int64_t* doff = nullptr;
  double* dtab = nullptr;
  const size_t gbytes = words.size() * sizeof(uint32_t) + 4;
  TB_CUDA(c, cudaMalloc(&dg, gbytes));
  TB_CUDA(c, cudaMalloc(&doff, 2 * sizeof(int64_t)));
  TB_CUDA(c, cudaMalloc(&dtab, table.size() * sizeof(double)));
  int64_t off[2] = {0, n_gates};
  std::vector<int> idims((size_t)n + 1);
  for (int64_t s = 0; s <= n; ++s) idims[(size_t)s] = (int)dims[s];
  int hs[2] = {0, 0};
  int icenter = (int)center;
  cudaMemcpy(dg, words.data(), words.size() * sizeof(uint32_t), cudaMemcpyHostToDevice);
  cudaMemcpy(doff, off, sizeof(off), cudaMemcpyHostToDevice);
  cudaMemcpy(dtab, table.data(), table.size() * sizeof(double), cudaMemcpyHostToDevice);
  cudaMemcpy(c->dscratch, hs, sizeof(hs), cudaMemcpyHostToDevice);
  cudaMemcpy(c->dscratch + 2, &icenter, sizeof(int), cudaMemcpyHostToDevice);
  cudaMemcpy(c->dscratch + 3, idims.data(), idims.size() * sizeof(int), cudaMemcpyHostToDevice);
  cudaMemcpy(c->dcounters, counters, 4 * sizeof(double), cudaMemcpyHostToDevice);
  cudaMemset(c->dflops, 0, sizeof(double));
  const size_t site_bytes = (size_t)n * cap * 2 * cap * sizeof(double2);
  cudaMemcpy(c->mps, buf, site_bytes, cudaMemcpyHostToDevice);
  TB_CUDA(c, cudaGetLastError());

  tb::Job job;
  memset(&job, 0, sizeof(job));
  job.n = (int)n;
  job.cap = (int)cap;
  job.chi_cut = (int)chi_cut;
  job.pi_local = 0;  // drop-in: the reference's full update for pi gates
  job.floor = floor;
  job.n_samples = 1;
  job.gates = dg;
  job.gate_off = doff;
  job.angle_cs = dtab;
  job.next_sample = c->dscratch;
  job.status = c->dscratch + 1;
  job.io_center = c->dscratch + 2;
  job.io_dims = c->dscratch + 3;
  job.io_counters = c->dcounters;
  job.flops = c->dflops;
  job.ws_mps = c->mps;
  job.ws_W = c->W;
  job.ws_W0 = c->W0;
  job.ws_X = c->X;
  job.mps_stride = c->mps_stride;
  job.mat_stride = c->mat_stride;
  rc = launch_ensemble(c, job, 1, 0, nullptr);
  if (rc == TB_OK) {
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) rc = fail(c, TB_ECUDA, std::string("kernel: ") + cudaGetErrorString(e));
  }
  if (rc == TB_OK) {
    cudaMemcpy(buf, c->mps, site_bytes, cudaMemcpyDeviceToHost);
    cudaMemcpy(hs, c->dscratch, sizeof(hs), cudaMemcpyDeviceToHost);
    cudaMemcpy(&icenter, c->dscratch + 2, sizeof(int), cudaMemcpyDeviceToHost);
    cudaMemcpy(idims.data(), c->dscratch + 3, idims.size() * sizeof(int), cudaMemcpyDeviceToHost);
    cudaMemcpy(counters, c->dcounters, 4 * sizeof(double), cudaMemcpyDeviceToHost);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) rc = fail(c, TB_ECUDA, cudaGetErrorString(e));
    for (int64_t s = 0; s <= n; ++s) dims[s] = idims[(size_t)s];
    *new_center = icenter;
    if (rc == TB_OK && (hs[1] & 1)) rc = fail(c, TB_ENOCONV, "Jacobi SVD did not converge");
  }
  cudaFree(dg);
  cudaFree(doff);
  cudaFree(dtab);
  return rc;
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
  int* dd = nullptr;
  TB_CUDA(c, cudaMalloc(&dd, (2 * n + 1) * sizeof(int)));
  cudaMemcpy(dd, idims.data(), (n + 1) * sizeof(int), cudaMemcpyHostToDevice);
  cudaMemcpy(dd + n + 1, codes, n * sizeof(int), cudaMemcpyHostToDevice);
  cudaMemcpy(c->mps, buf, (size_t)n * cap * 2 * cap * sizeof(double2), cudaMemcpyHostToDevice);
  const size_t smem = tb::kTileBytes;
  cudaFuncSetAttribute(tb::expectation_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  tb::expectation_kernel<<<1, tb::NT, smem>>>(c->mps, (int)n, (int)cap, dd, dd + n + 1, c->W, c->W0, c->dflops);
  cudaError_t e = cudaDeviceSynchronize();
  if (e == cudaSuccess) e = cudaMemcpy(out, c->dflops, sizeof(double), cudaMemcpyDeviceToHost);
  cudaFree(dd);
  if (e != cudaSuccess) return fail(c, TB_ECUDA, std::string("expectation: ") + cudaGetErrorString(e));
  return TB_OK;
}

int tb_svd(tb_ctx* c, const double* a, int64_t batch, int64_t m, int64_t n, double* s, double* u, double* vh) {
  if (!c) return TB_EINVAL;
  if (!a || !s || batch < 1 || m < 1 || n < 1) return fail(c, TB_EINVAL, "bad arguments");
  if (m > tb::MAXDIM || n > tb::MAXDIM) return fail(c, TB_EINVAL, "matrix larger than 256");
  const int64_t k = m < n ? m : n;
  const int cap = (int)((m > n ? m : n) + 1) / 2;
  int rc = ensure_workspace(c, (int)batch, 1, cap < 1 ? 1 : cap);
  if (rc) return rc;
  double2 *da = nullptr, *du = nullptr, *dvh = nullptr;
  double* ds = nullptr;
  TB_CUDA(c, cudaMalloc(&da, batch * m * n * sizeof(double2)));
  TB_CUDA(c, cudaMalloc(&ds, batch * k * sizeof(double)));
  if (u) TB_CUDA(c, cudaMalloc(&du, batch * m * k * sizeof(double2)));
  if (vh) TB_CUDA(c, cudaMalloc(&dvh, batch * k * n * sizeof(double2)));
  cudaMemcpy(da, a, batch * m * n * sizeof(double2), cudaMemcpyHostToDevice);
  cudaMemset(c->dscratch, 0, 2 * sizeof(int));
  const size_t smem = tb::kTileBytes;
  cudaFuncSetAttribute(tb::svd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  tb::svd_kernel<<<(int)batch, tb::NT, smem>>>(da, (int)m, (int)n, c->W, c->W0, c->mat_stride, ds, du, dvh,
                                               c->dscratch + 1);
  cudaError_t e = cudaDeviceSynchronize();
  int st[2] = {0, 0};
  if (e == cudaSuccess) {
    cudaMemcpy(s, ds, batch * k * sizeof(double), cudaMemcpyDeviceToHost);
    if (u) cudaMemcpy(u, du, batch * m * k * sizeof(double2), cudaMemcpyDeviceToHost);
    if (vh) cudaMemcpy(vh, dvh, batch * k * n * sizeof(double2), cudaMemcpyDeviceToHost);
    e = cudaMemcpy(st, c->dscratch, sizeof(st), cudaMemcpyDeviceToHost);
  }
  cudaFree(da);
  cudaFree(ds);
  cudaFree(du);
  cudaFree(dvh);
  if (e != cudaSuccess) return fail(c, TB_ECUDA, std::string("svd: ") + cudaGetErrorString(e));
  if (st[1] & 1) return fail(c, TB_ENOCONV, "Jacobi SVD did not converge");
  return TB_OK;
}

int tb_run_ensemble_device(tb_ctx* c, const tb_ensemble_desc* d, tb_ensemble_out* o, void* stream) {
  if (!c || !d || !o) return TB_EINVAL;
  int rc = validate_shape(c, d->n, d->cap, d->chi_cut);
  if (rc) return rc;
  if (d->chi_cut > d->cap) return fail(c, TB_EINVAL, "chi_cut exceeds cap");
  if (d->n_samples < 0 || d->n_ckpt < 0 || d->n_obs < 0 || d->n_obs > tb::MAXN)
    return fail(c, TB_EINVAL, "bad ensemble sizes");
  if (!d->gates || !d->gate_offsets || !d->angle_cs || !d->init_vecs || !o->sum_v || !o->sum_v2 || !o->flops)
    return fail(c, TB_EINVAL, "null argument");
  if (d->n_ckpt > 0 && (!d->ckpt_gate_end || !d->ckpt_sign || (d->n_obs > 0 && !d->obs_sites)))
    return fail(c, TB_EINVAL, "null checkpoint argument");
  if (d->n_samples == 0) return TB_OK;
  const int grid = d->n_samples < c->sms ? d->n_samples : c->sms;
  rc = ensure_workspace(c, grid, d->n, d->cap);
  if (rc) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  TB_CUDA(c, cudaMemsetAsync(c->dscratch, 0, 2 * sizeof(int), st));
  TB_CUDA(c, cudaMemsetAsync(c->dflops, 0, grid * sizeof(double), st));
  tb::Job job;
  memset(&job, 0, sizeof(job));
  job.n = d->n;
  job.cap = d->cap;
  job.chi_cut = d->chi_cut;
  job.pi_local = d->pi_local;
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
  job.values = o->values;
  job.discarded = o->discarded;
  job.ledger = o->ledger;
  job.sum_v = (unsigned long long*)o->sum_v;
  job.sum_v2 = (unsigned long long*)o->sum_v2;
  job.flops = c->dflops;
  job.next_sample = c->dscratch;
  job.status = c->dscratch + 1;
  job.ws_mps = c->mps;
  job.ws_W = c->W;
  job.ws_W0 = c->W0;
  job.ws_X = c->X;
  job.mps_stride = c->mps_stride;
  job.mat_stride = c->mat_stride;
  rc = launch_ensemble(c, job, grid, st, o->kernel_ms);
  if (rc) return rc;
  tb::sum_flops_kernel<<<1, 32, 0, st>>>(c->dflops, grid, o->flops);
  TB_CUDA(c, cudaGetLastError());
  return TB_OK;
}

}  // extern "C"

extern "C" int tb_run_ensemble(tb_ctx* c, const tb_ensemble_desc* d, tb_ensemble_out* o) {
  if (!c || !d || !o) return TB_EINVAL;
  if (d->n_samples <= 0) return TB_OK;
  const int S = d->n_samples, C = d->n_ckpt, O = d->n_obs;
  const int64_t G = d->gate_offsets[S];
  std::vector<void*> allocs;
  auto dalloc = [&](size_t bytes) -> void* {
    void* p = nullptr;
    if (cudaMalloc(&p, bytes ? bytes : 8) != cudaSuccess) return nullptr;
    allocs.push_back(p);
    return p;
  };
  auto cleanup = [&]() {
    for (void* p : allocs) cudaFree(p);
  };
  tb_ensemble_desc dd = *d;
  tb_ensemble_out od = *o;
  uint32_t* g = (uint32_t*)dalloc(G * sizeof(uint32_t));
  int64_t* off = (int64_t*)dalloc((S + 1) * sizeof(int64_t));
  int32_t* ce = (int32_t*)dalloc((size_t)S * C * sizeof(int32_t));
  int8_t* cs = (int8_t*)dalloc((size_t)S * C);
  double* ang = (double*)dalloc(2 * d->n_angles * sizeof(double));
  int32_t* obs = (int32_t*)dalloc(O * sizeof(int32_t));
  double* iv = (double*)dalloc(4 * d->n * sizeof(double));
  double* vals = o->values ? (double*)dalloc((size_t)S * C * O * sizeof(double)) : nullptr;
  double* disc = o->discarded ? (double*)dalloc((size_t)S * C * sizeof(double)) : nullptr;
  double* led = o->ledger ? (double*)dalloc((size_t)S * 4 * sizeof(double)) : nullptr;
  int64_t* sv = (int64_t*)dalloc((size_t)C * O * sizeof(int64_t));
  int64_t* sv2 = (int64_t*)dalloc((size_t)C * O * sizeof(int64_t));
  double* fl = (double*)dalloc(sizeof(double));
  if (!g || !off || !ce || !cs || !ang || !obs || !iv || !sv || !sv2 || !fl || (o->values && !vals) ||
      (o->discarded && !disc) || (o->ledger && !led)) {
    cleanup();
    return fail(c, TB_ENOMEM, "device allocation failed");
  }
  cudaMemcpy(g, d->gates, G * sizeof(uint32_t), cudaMemcpyHostToDevice);
  cudaMemcpy(off, d->gate_offsets, (S + 1) * sizeof(int64_t), cudaMemcpyHostToDevice);
  if (C) {
    cudaMemcpy(ce, d->ckpt_gate_end, (size_t)S * C * sizeof(int32_t), cudaMemcpyHostToDevice);
    cudaMemcpy(cs, d->ckpt_sign, (size_t)S * C, cudaMemcpyHostToDevice);
  }
  cudaMemcpy(ang, d->angle_cs, 2 * d->n_angles * sizeof(double), cudaMemcpyHostToDevice);
  if (O) cudaMemcpy(obs, d->obs_sites, O * sizeof(int32_t), cudaMemcpyHostToDevice);
  cudaMemcpy(iv, d->init_vecs, 4 * d->n * sizeof(double), cudaMemcpyHostToDevice);
  cudaMemcpy(sv, o->sum_v, (size_t)C * O * sizeof(int64_t), cudaMemcpyHostToDevice);
  cudaMemcpy(sv2, o->sum_v2, (size_t)C * O * sizeof(int64_t), cudaMemcpyHostToDevice);
  cudaMemset(fl, 0, sizeof(double));
  dd.gates = g;
  dd.gate_offsets = off;
  dd.ckpt_gate_end = ce;
  dd.ckpt_sign = cs;
  dd.angle_cs = ang;
  dd.obs_sites = obs;
  dd.init_vecs = iv;
  od.values = vals;
  od.discarded = disc;
  od.ledger = led;
  od.sum_v = sv;
  od.sum_v2 = sv2;
  od.flops = fl;
  int rc = tb_run_ensemble_device(c, &dd, &od, nullptr);
  if (rc == TB_OK) {
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) rc = fail(c, TB_ECUDA, std::string("ensemble kernel: ") + cudaGetErrorString(e));
  }
  if (rc == TB_OK) {
    if (vals) cudaMemcpy(o->values, vals, (size_t)S * C * O * sizeof(double), cudaMemcpyDeviceToHost);
    if (disc) cudaMemcpy(o->discarded, disc, (size_t)S * C * sizeof(double), cudaMemcpyDeviceToHost);
    if (led) cudaMemcpy(o->ledger, led, (size_t)S * 4 * sizeof(double), cudaMemcpyDeviceToHost);
    cudaMemcpy(o->sum_v, sv, (size_t)C * O * sizeof(int64_t), cudaMemcpyDeviceToHost);
    cudaMemcpy(o->sum_v2, sv2, (size_t)C * O * sizeof(int64_t), cudaMemcpyDeviceToHost);
    double f = 0;
    cudaMemcpy(&f, fl, sizeof(double), cudaMemcpyDeviceToHost);
    if (o->flops) o->flops[0] += f;
    int st[2] = {0, 0};
    cudaMemcpy(st, c->dscratch, sizeof(st), cudaMemcpyDeviceToHost);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) rc = fail(c, TB_ECUDA, cudaGetErrorString(e));
    else if (st[1] & 1) rc = fail(c, TB_ENOCONV, "Jacobi SVD did not converge");
  }
  cleanup();
  return rc;
}
