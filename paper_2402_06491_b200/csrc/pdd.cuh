// pdd.cuh — probabilistic domain decomposition downstream (NEXT row f1,
// DESIGN.md §11): the interface values produced by the tree walk are turned
// into Dirichlet data and four fully decoupled subdomain solves
// ("Interpolation" and "Local solver", 1007-1012).
//
//   pdd_spline_s_kernel + pdd_spline_t_kernel: the tensor-product not-a-knot
//     cubic spline in (s, t) of each line's nodal table,
//     evaluated at every grid node s_i for every time step t_n.
//   pdd_adi_kernel: one CTA per subdomain (the paper's "each subdomain ...
//     assigned to different processors" — here an SM each), the whole time
//     march in shared memory: Strang splitting with RK4 half reactions and a
//     Peaceman–Rachford ADI diffusion step (Crank–Nicolson per direction,
//     PAPER.md:971-973), Dirichlet data carried through the same splitting.
//
// Geometry (square [lo, hi]^2 split at mid = (lo + hi)/2): grid nodes
// x_i = lo + i h, i = 0..n, h = (hi - lo)/n, n even, m = n/2 cells per
// subdomain side.  Lines: 0 interface x = mid (s = y), 1 interface y = mid
// (s = x), 2 edge x = lo, 3 edge x = hi (s = y), 4 edge y = lo, 5 edge y = hi
// (s = x).  Nodal table V[line][k][j] at s_j = lo + j (hi - lo)/(ns - 1),
// t_k = k T/(nt - 1).  Boundary table W[line][step][i] at (s = x_i, t_step).
#pragma once
#include <cstdint>
#include <cooperative_groups.h>

namespace rtk {

constexpr int kPddMaxNodes = 64;    // ns, nt <= 64

// Second derivatives of the not-a-knot cubic spline through y[0..n) on a
// uniform grid (n >= 4).  With M0 = 2M1 - M2 and M_{n-1} = 2M_{n-2} - M_{n-3}
// (third derivative continuous at x_1, x_{n-2}) the first and last interior
// C² equations reduce to 6 M_1 = r_1 and 6 M_{n-2} = r_{n-2}; the rest is the
// tridiagonal (1, 4, 1) system, r_i = 6 (y_{i+1} - 2 y_i + y_{i-1}) / h².
// y and M are strided (element i at y[i*ys], M[i*ms]); M doubles as the
// Thomas sweep's d' storage, and the factors c'_i (the same for every system
// of size n) come precomputed in cp — no local arrays.
__device__ inline void nak_m(const double* y, int ys, int n, double h, double* M, int ms,
                             const double* cp) {
  const double s = 6.0 / (h * h);
  const double m1 = (y[2 * ys] - 2.0 * y[ys] + y[0]) * s / 6.0;
  const double mn = (y[(n - 1) * ys] - 2.0 * y[(n - 2) * ys] + y[(n - 3) * ys]) * s / 6.0;
  // interior unknowns M_2..M_{n-3} (Thomas; d'_i stored in M_i)
  const int a = 2, b = n - 3;
  double prev = 0.0;
  for (int i = a; i <= b; ++i) {
    double r = (y[(i + 1) * ys] - 2.0 * y[i * ys] + y[(i - 1) * ys]) * s;
    if (i == a) r -= m1;
    if (i == b) r -= mn;
    const double den = (i == a) ? 4.0 : 4.0 - cp[i - 1];
    prev = (i == a) ? r / den : (r - prev) / den;
    M[i * ms] = prev;
  }
  double nxt = 0.0;
  for (int i = b; i >= a; --i) {
    nxt = (i == b) ? M[i * ms] : M[i * ms] - cp[i] * nxt;
    M[i * ms] = nxt;
  }
  M[ms] = m1;
  M[(n - 2) * ms] = mn;
  M[0] = 2.0 * m1 - M[2 * ms];
  M[(n - 1) * ms] = 2.0 * mn - M[(n - 3) * ms];
}

// c'_i = 1/den_i of nak_m's Thomas sweep for a system of n nodes (i = 2..n-3)
__device__ inline void nak_factors(int n, double* cp) {
  for (int i = 2; i <= n - 3; ++i) cp[i] = 1.0 / ((i == 2) ? 4.0 : 4.0 - cp[i - 1]);
}

__device__ inline double nak_at(const double* y, int ys, const double* M, int ms, int n, double x0,
                                double h, double x) {
  int j = static_cast<int>(floor((x - x0) / h));
  j = j < 0 ? 0 : (j > n - 2 ? n - 2 : j);
  const double a = x0 + j * h, b = a + h;
  const double Mj = M[j * ms], Mj1 = M[(j + 1) * ms], yj = y[j * ys], yj1 = y[(j + 1) * ys];
  return Mj * (b - x) * (b - x) * (b - x) / (6.0 * h) +
         Mj1 * (x - a) * (x - a) * (x - a) / (6.0 * h) +
         (yj / h - Mj * h / 6.0) * (b - x) + (yj1 / h - Mj1 * h / 6.0) * (x - a);
}

struct PddGeom {
  double lo, hi, h, T, dt;
  int n, m, ns, nt, n_steps;
};

// Interpolation, two passes with no local memory:
// pdd_spline_s_kernel: one thread per (line, time level k): the spline in s
//   of V[line][k][·] — its second derivatives Ms[line][k][·];
// pdd_spline_t_kernel: one thread per (line, grid node i): A[k] = that
//   spline at s = x_i for every level, the spline in t through A (second
//   derivatives in At), evaluated at every time step into W[line][step][i].
//   A and At are [line][k][i] (coalesced across the threads i).
__global__ void pdd_spline_s_kernel(const double* __restrict__ V, double* __restrict__ Ms, PddGeom G,
                                    int n_lines) {
  __shared__ double cp[kPddMaxNodes];
  if (threadIdx.x == 0) nak_factors(G.ns, cp);
  __syncthreads();
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= n_lines * G.nt) return;
  const double hs = (G.hi - G.lo) / (G.ns - 1);
  nak_m(V + static_cast<int64_t>(q) * G.ns, 1, G.ns, hs, Ms + static_cast<int64_t>(q) * G.ns, 1, cp);
}

__global__ void pdd_spline_t_kernel(const double* __restrict__ V, const double* __restrict__ Ms,
                                    double* __restrict__ A, double* __restrict__ At,
                                    double* __restrict__ W, PddGeom G, int n_lines) {
  __shared__ double cp[kPddMaxNodes];
  if (threadIdx.x == 0) nak_factors(G.nt, cp);
  __syncthreads();
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  const int n1 = G.n + 1;
  if (q >= n_lines * n1) return;
  const int line = q / n1, i = q - line * n1;
  const double x = G.lo + i * G.h;
  const double hs = (G.hi - G.lo) / (G.ns - 1), ht = G.T / (G.nt - 1);
  const int64_t vb = static_cast<int64_t>(line) * G.nt * G.ns;
  double* Al = A + static_cast<int64_t>(line) * G.nt * n1 + i;       // A[line][k][i]
  double* Atl = At + static_cast<int64_t>(line) * G.nt * n1 + i;
  for (int k = 0; k < G.nt; ++k)              // splines in s at every time node
    Al[static_cast<int64_t>(k) * n1] = nak_at(V + vb + k * G.ns, 1, Ms + vb + k * G.ns, 1, G.ns, G.lo, hs, x);
  nak_m(Al, n1, G.nt, ht, Atl, n1, cp);      // then the spline in t at s = x_i
  double* Wl = W + static_cast<int64_t>(line) * (G.n_steps + 1) * n1 + i;
  for (int st = 0; st <= G.n_steps; ++st)
    Wl[static_cast<int64_t>(st) * n1] = nak_at(Al, n1, Atl, n1, G.nt, 0.0, ht, st * G.dt);
}

struct PddEq {
  double b[9];
  int degree;
  int init_kind;
  double amp, inv_scale, inv_scale2, D;
};

// f(u) by Horner over all nine coefficients (b_k = 0 above the degree; the
// leading zeros add exact zeros): unrolled, the coefficients read from the
// kernel's constant parameters — no dynamically indexed local copy
__device__ __forceinline__ double pdd_f(const PddEq& E, double u) {
  double r = E.b[8];
#pragma unroll
  for (int k = 7; k >= 0; --k) r = fma(r, u, E.b[k]);
  return r;
}

__device__ inline double pdd_rk4(const PddEq& E, double u, double hh) {
  const double k1 = pdd_f(E, u);
  const double k2 = pdd_f(E, u + 0.5 * hh * k1);
  const double k3 = pdd_f(E, u + 0.5 * hh * k2);
  const double k4 = pdd_f(E, u + hh * k3);
  return u + hh / 6.0 * (k1 + 2.0 * k2 + 2.0 * k3 + k4);
}

__device__ inline double pdd_g(const PddEq& E, double x, double y) {
  const double r2 = x * x + y * y;
  switch (E.init_kind) {
    case 0: return E.amp;
    case 1: return E.amp * 0.5 * (1.0 + tanh(x * E.inv_scale));
    case 2: return E.amp * exp(-r2 * E.inv_scale2);
    default: return E.amp / (1.0 + r2 * E.inv_scale2);
  }
}

constexpr int kPcrLevels = 6;   // cyclic reduction for up to 64 unknowns per line

// shared memory of pdd_adi_kernel: u, u* [(m+1)²], edges [8][m+1], Thomas
// factors [2][m+1], PCR multipliers [6][128] + [64], the next edge data
// [4][m+1], PCR scratch [3][64]
__host__ __device__ constexpr int pdd_smem_doubles(int m) {
  return 2 * (m + 1) * (m + 1) + 8 * (m + 1) + 2 * (m + 1) + kPcrLevels * 128 + 64 + 4 * (m + 1);
}
__host__ __device__ constexpr int pdd_smem_bytes(int m) {
  return (pdd_smem_doubles(m) + 3 * 64) * 8;   // + pcr_factors' scratch
}

// Elimination multipliers of parallel cyclic reduction for the constant
// tridiagonal matrix tridiag(a, b, a) of size n <= 64 (every line of every
// step shares it): at level lv (stride δ = 2^lv) equation i becomes
// d_i − k1_i d_{i−δ} − k2_i d_{i+δ} with k1_i = a_i/b_{i−δ}, k2_i = c_i/b_{i+δ}
// (0 outside [0, n)), and a, b, c updated as the reduction prescribes; after
// the last level x_i = d_i / b_i.  Written to pk [level][k1 | k2][64] and
// [64] 1/b; uses 3 x 64 doubles of scratch.  Block-wide (barriers inside).
__device__ inline void pcr_factors(int n, double a0, double b0, double* pk, double* scr) {
  double* A = scr;
  double* B = scr + 64;
  double* C = scr + 128;
  const int i = threadIdx.x;
  double a = 0.0, b = 1.0, c = 0.0;
  if (i < n) {
    a = i > 0 ? a0 : 0.0;
    b = b0;
    c = i + 1 < n ? a0 : 0.0;
  }
  for (int lv = 0; lv < kPcrLevels; ++lv) {
    const int dl = 1 << lv;
    if (i < 64) { A[i] = a; B[i] = b; C[i] = c; }
    __syncthreads();
    if (i < 64) {
      double k1 = 0.0, k2 = 0.0, na = 0.0, nc = 0.0, nb = b;
      if (i < n && i - dl >= 0) { k1 = a / B[i - dl]; na = -A[i - dl] * k1; nb -= C[i - dl] * k1; }
      if (i < n && i + dl < n) { k2 = c / B[i + dl]; nc = -C[i + dl] * k2; nb -= A[i + dl] * k2; }
      pk[lv * 128 + i] = k1;
      pk[lv * 128 + 64 + i] = k2;
      a = na; b = nb; c = nc;
    }
    __syncthreads();
  }
  if (i < 64) pk[kPcrLevels * 128 + i] = 1.0 / b;
  __syncthreads();
}

// One CTA per subdomain q = qx + 2 qy.  Shared memory: u, u* [(m+1)^2] with
// index [i][j] = (x_i, y_j) of the subdomain, the four edges' bB and bM
// [4][m+1], the Thomas factors of (I - r/2 δ²) [m].  Writes its nodes of the
// global field F[(n+1)^2] (index [i][j] global).
__global__ void pdd_adi_kernel(const double* __restrict__ W, double* __restrict__ F, PddGeom G,
                               const __grid_constant__ PddEq E) {
  extern __shared__ double sm[];
  const int m = G.m, mm = m + 1;
  const int qx = blockIdx.x & 1, qy = blockIdx.x >> 1;
  double* u = sm;                    // [mm][mm]
  double* us = u + mm * mm;          // [mm][mm]
  double* eB = us + mm * mm;         // [4][mm] edges: 0 x0, 1 x1, 2 y0, 3 y1
  double* eM = eB + 4 * mm;          // [4][mm]
  double* cp = eM + 4 * mm;          // [mm] Thomas: c'_i
  double* piv = cp + mm;             // [mm] Thomas: 1/(b - a c'_{i-1})
  double* pk = piv + mm;             // PCR: [kPcrLevels][2][64] k1, k2 per level, [64] 1/b
  double* wN = pk + kPcrLevels * 128 + 64;   // [4][mm] W(t_{n+1}) on the four edges
  const int tid = threadIdx.x, nth = blockDim.x;
  const int nu = m - 1;              // interior unknowns per line
  const bool pcr = nu <= 64;         // warp-per-line cyclic reduction (else Thomas)
  const int i0 = qx * m, j0 = qy * m;             // global offsets
  // edge lines of this subdomain (see the header)
  const int lx0 = qx == 0 ? 2 : 0, lx1 = qx == 0 ? 0 : 3;
  const int ly0 = qy == 0 ? 4 : 1, ly1 = qy == 0 ? 1 : 5;
  const int64_t lstride = static_cast<int64_t>(G.n_steps + 1) * (G.n + 1);
  auto Wat = [&](int line, int st, int gi) -> double {
    return W[line * lstride + static_cast<int64_t>(st) * (G.n + 1) + gi];
  };
  const double r = E.D * G.dt / (G.h * G.h);
  if (tid == 0) {                     // Thomas factors of tridiag(-r/2, 1 + r, -r/2), size m-1
    for (int k = 1; k <= m - 1; ++k) {
      const double den = (k == 1) ? 1.0 + r : 1.0 + r - (-0.5 * r) * cp[k - 1];
      piv[k] = 1.0 / den;
      cp[k] = (-0.5 * r) * piv[k];
    }
  }
  if (pcr) pcr_factors(nu, -0.5 * r, 1.0 + r, pk, sm + pdd_smem_doubles(m));   // (+ scratch)
  // the edge data of the step's end, W(t_{n+1}): edge e = tid / mm (0 x0,
  // 1 x1, 2 y0, 3 y1), loaded at the step's start (the latency overlaps the
  // first reaction) and used twice — bB and the new boundary
  auto w_next = [&](int n) -> double {
    if (tid >= 4 * mm) return 0.0;
    const int e = tid / mm, k = tid - e * mm;
    const int line = e == 0 ? lx0 : (e == 1 ? lx1 : (e == 2 ? ly0 : ly1));
    return Wat(line, n + 1, (e < 2 ? j0 : i0) + k);
  };
  // pointwise reaction R_{dt/2} on the whole subdomain, four independent
  // points per thread in flight (the RK4 stages are a serial chain)
  auto react = [&](double* w, double hh) {
    for (int q0 = tid; q0 < mm * mm; q0 += 4 * nth) {
      double v[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) v[c] = q0 + c * nth < mm * mm ? w[q0 + c * nth] : 0.0;
#pragma unroll
      for (int c = 0; c < 4; ++c) v[c] = pdd_rk4(E, v[c], hh);
#pragma unroll
      for (int c = 0; c < 4; ++c)
        if (q0 + c * nth < mm * mm) w[q0 + c * nth] = v[c];
    }
  };
  for (int q = tid; q < mm * mm; q += nth) {      // u(x, y, 0) = g
    const int i = q / mm, j = q - i * mm;
    u[q] = pdd_g(E, G.lo + (i0 + i) * G.h, G.lo + (j0 + j) * G.h);
  }
  __syncthreads();
  // one line's solve of (I - r/2 δ²) w = d by cyclic reduction in a warp:
  // lane l holds unknowns l and l + 32; the elimination multipliers depend
  // only on the (constant) matrix, so they come precomputed (pcr_factors)
  const int lane = tid & 31, warp = tid >> 5, nwarp = nth >> 5;
  auto pcr_solve = [&](double& d0, double& d1) {
    // levels with compile-time strides; a level whose stride reaches nu is
    // a no-op (its multipliers are 0) and is skipped
#pragma unroll
    for (int lv = 0; lv < kPcrLevels; ++lv) {
      constexpr int kW = 32;
      const int dl = 1 << lv;
      if (dl >= nu) break;                        // (uniform)
      const double* k1 = pk + lv * 128;
      const double* k2 = k1 + 64;
      double lo0, lo1, hi0, hi1;
      if (dl < kW) {
        const double a0 = __shfl_up_sync(0xffffffffu, d0, dl), a1 = __shfl_up_sync(0xffffffffu, d1, dl);
        const double w0 = __shfl_down_sync(0xffffffffu, d0, dl), w1 = __shfl_down_sync(0xffffffffu, d1, dl);
        const double c0 = __shfl_sync(0xffffffffu, d0, (lane - dl) & 31);   // e1's lower across the halves
        const double c1 = __shfl_sync(0xffffffffu, d1, (lane + dl) & 31);   // e0's upper across the halves
        const bool dn = lane >= dl, up = lane + dl < kW;
        lo0 = dn ? a0 : 0.0;
        lo1 = dn ? a1 : c0;
        hi0 = up ? w0 : c1;
        hi1 = up ? w1 : 0.0;
      } else {                                   // dl = 32: e0 <-> e1 of the same lane
        lo0 = 0.0; lo1 = d0; hi0 = d1; hi1 = 0.0;
      }
      // (multipliers are 0 where the neighbour is outside [0, nu))
      d0 = fma(-k2[lane], hi0, fma(-k1[lane], lo0, d0));
      d1 = fma(-k2[lane + 32], hi1, fma(-k1[lane + 32], lo1, d1));
    }
    d0 *= pk[kPcrLevels * 128 + lane];
    d1 *= pk[kPcrLevels * 128 + lane + 32];
  };
  auto impose = [&](double* w, int st) {           // boundary = W at step st
    for (int k = tid; k < mm; k += nth) {
      w[0 * mm + k] = Wat(lx0, st, j0 + k);
      w[m * mm + k] = Wat(lx1, st, j0 + k);
    }
    __syncthreads();
    for (int k = tid; k < mm; k += nth) {
      w[k * mm + 0] = Wat(ly0, st, i0 + k);
      w[k * mm + m] = Wat(ly1, st, i0 + k);
    }
    __syncthreads();
  };
  impose(u, 0);
  // bM's edge value of u after the first reaction: edge e = tid / mm
  auto u_edge = [&](const double* w) -> double {
    const int e = tid / mm, k = tid - e * mm;
    return e == 0 ? w[k] : (e == 1 ? w[m * mm + k] : (e == 2 ? w[k * mm] : w[k * mm + m]));
  };
  double w_ahead = w_next(0);                       // W(t_1), one step ahead
  for (int n = 0; n < G.n_steps; ++n) {
    // bB = R_{-dt/2} W(t_{n+1}) — independent of u: one edge value per
    // thread, computed alongside the first reaction; W(t_{n+2}) is loaded a
    // whole step before its use (its latency hidden behind the step)
    const double wv = w_ahead;
    if (n + 1 < G.n_steps) w_ahead = w_next(n + 1);
    const double bv = tid < 4 * mm ? pdd_rk4(E, wv, -0.5 * G.dt) : 0.0;
    react(u, 0.5 * G.dt);                                                   // -> bA
    __syncthreads();
    if (tid < 4 * mm) {                                                     // bM = (bA + bB)/2
      wN[tid] = wv;
      eB[tid] = bv;
      eM[tid] = 0.5 * (u_edge(u) + bv);
    }
    __syncthreads();
    // x-sweep: row j (thread), unknowns i = 1..m-1:
    // (I - r/2 δx²) u* = (I + r/2 δy²) u with u* = bM on the x edges
    auto dx = [&](int i, int j) -> double {
      double d = u[i * mm + j] + 0.5 * r * (u[i * mm + j - 1] - 2.0 * u[i * mm + j] + u[i * mm + j + 1]);
      if (i == 1) d += 0.5 * r * eM[0 * mm + j];
      if (i == m - 1) d += 0.5 * r * eM[1 * mm + j];
      return d;
    };
    if (pcr) {
      for (int j = 1 + warp; j <= m - 1; j += nwarp) {   // a warp per row
        double d0 = lane < nu ? dx(lane + 1, j) : 0.0;
        double d1 = lane + 32 < nu ? dx(lane + 33, j) : 0.0;
        pcr_solve(d0, d1);
        if (lane < nu) us[(lane + 1) * mm + j] = d0;
        if (lane + 32 < nu) us[(lane + 33) * mm + j] = d1;
      }
    } else {
      for (int j = 1 + tid; j <= m - 1; j += nth) {
        double prev = 0.0;
        for (int i = 1; i <= m - 1; ++i) {
          prev = (i == 1) ? dx(i, j) * piv[i] : (dx(i, j) - (-0.5 * r) * prev) * piv[i];
          us[i * mm + j] = prev;                    // forward pass: d'_i
        }
        for (int i = m - 2; i >= 1; --i) us[i * mm + j] -= cp[i] * us[(i + 1) * mm + j];
      }
    }
    for (int k = tid; k < mm; k += nth) {           // u* boundary = bM
      us[0 * mm + k] = eM[0 * mm + k];
      us[m * mm + k] = eM[1 * mm + k];
    }
    __syncthreads();
    for (int k = tid; k < mm; k += nth) {
      us[k * mm + 0] = eM[2 * mm + k];
      us[k * mm + m] = eM[3 * mm + k];
    }
    __syncthreads();
    // y-sweep: column i (thread), unknowns j = 1..m-1:
    // (I - r/2 δy²) v = (I + r/2 δx²) u* with v = bB on the y edges
    auto dy = [&](int i, int j) -> double {
      double d = us[i * mm + j] + 0.5 * r * (us[(i - 1) * mm + j] - 2.0 * us[i * mm + j] + us[(i + 1) * mm + j]);
      if (j == 1) d += 0.5 * r * eB[2 * mm + i];
      if (j == m - 1) d += 0.5 * r * eB[3 * mm + i];
      return d;
    };
    if (pcr) {
      for (int i = 1 + warp; i <= m - 1; i += nwarp) {   // a warp per column
        double d0 = lane < nu ? dy(i, lane + 1) : 0.0;
        double d1 = lane + 32 < nu ? dy(i, lane + 33) : 0.0;
        pcr_solve(d0, d1);
        if (lane < nu) u[i * mm + lane + 1] = d0;
        if (lane + 32 < nu) u[i * mm + lane + 33] = d1;
      }
    } else {
      for (int i = 1 + tid; i <= m - 1; i += nth) {
        double prev = 0.0;
        for (int j = 1; j <= m - 1; ++j) {
          prev = (j == 1) ? dy(i, j) * piv[j] : (dy(i, j) - (-0.5 * r) * prev) * piv[j];
          u[i * mm + j] = prev;
        }
        for (int j = m - 2; j >= 1; --j) u[i * mm + j] -= cp[j] * u[i * mm + j + 1];
      }
    }
    __syncthreads();
    for (int k = tid; k < mm; k += nth) {           // v boundary = bB
      u[0 * mm + k] = eB[0 * mm + k];
      u[m * mm + k] = eB[1 * mm + k];
    }
    __syncthreads();
    for (int k = tid; k < mm; k += nth) {
      u[k * mm + 0] = eB[2 * mm + k];
      u[k * mm + m] = eB[3 * mm + k];
    }
    __syncthreads();
    react(u, 0.5 * G.dt);
    __syncthreads();
    for (int k = tid; k < mm; k += nth) {          // boundary = W(t_{n+1})
      u[0 * mm + k] = wN[0 * mm + k];
      u[m * mm + k] = wN[1 * mm + k];
    }
    __syncthreads();
    for (int k = tid; k < mm; k += nth) {
      u[k * mm + 0] = wN[2 * mm + k];
      u[k * mm + m] = wN[3 * mm + k];
    }
    __syncthreads();
  }
  for (int q = tid; q < mm * mm; q += nth) {
    const int i = q / mm, j = q - i * mm;
    F[static_cast<int64_t>(i0 + i) * (G.n + 1) + (j0 + j)] = u[q];
  }
}


// The same local solver with each subdomain spread over a thread-block
// CLUSTER of kPddCluster CTAs (one SM each; 4 x 8 = 32 SMs instead of 4),
// for lines of up to 64 unknowns.  Every CTA keeps full copies of u and u*
// in its shared memory; CTA c of a cluster owns the rows j ≡ c (mod C) (the
// reactions and the x-direction line solves) and the columns i ≡ c (the
// y-direction line solves), and writes every value it computes into all C
// copies through distributed shared memory (st.shared::cluster), one cluster
// barrier after each of the four phases of a step.  The edge data, their
// R_{±dt/2} transforms and the line-solve multipliers are computed by every
// CTA redundantly (identical arithmetic), and the new step's boundary values
// W(t_{n+1}) are folded into the first reaction of the next step, so no
// phase writes a value another CTA may still be reading.  The arithmetic of
// every value is the single-CTA kernel's: the fields agree bit for bit.
constexpr int kPddCluster = 8;

__host__ __device__ constexpr int pdd_cluster_smem_doubles(int m) {
  return 2 * (m + 1) * (m + 1) + 8 * (m + 1) + kPcrLevels * 128 + 64 + 8 * (m + 1);
}
__host__ __device__ constexpr int pdd_cluster_smem_bytes(int m) {
  return (pdd_cluster_smem_doubles(m) + 3 * 64) * 8;
}

__global__ void pdd_adi_cluster_kernel(const double* __restrict__ W, double* __restrict__ F, PddGeom G,
                                       const __grid_constant__ PddEq E) {
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  extern __shared__ double sm[];
  const int C = static_cast<int>(cl.num_blocks());
  const int crank = static_cast<int>(cl.block_rank());
  const int sub = blockIdx.x / C;                 // subdomain q = qx + 2 qy
  const int m = G.m, mm = m + 1, nu = m - 1;
  const int qx = sub & 1, qy = sub >> 1;
  double* u = sm;                    // [mm][mm] full copy
  double* us = u + mm * mm;          // [mm][mm] full copy
  double* eB = us + mm * mm;         // [4][mm]
  double* eM = eB + 4 * mm;          // [4][mm]
  double* pk = eM + 4 * mm;          // PCR multipliers [6][128] + [64]
  double* wN = pk + kPcrLevels * 128 + 64;   // [4][mm] W(t_{n+1})
  double* wB = wN + 4 * mm;                  // [4][mm] W(t_n): this step's boundary
  const int tid = threadIdx.x, nth = blockDim.x;
  const int lane = tid & 31, warp = tid >> 5, nwarp = nth >> 5;
  const int i0 = qx * m, j0 = qy * m;
  const int lx0 = qx == 0 ? 2 : 0, lx1 = qx == 0 ? 0 : 3;
  const int ly0 = qy == 0 ? 4 : 1, ly1 = qy == 0 ? 1 : 5;
  const int64_t lstride = static_cast<int64_t>(G.n_steps + 1) * (G.n + 1);
  auto Wat = [&](int line, int st, int gi) -> double {
    return W[line * lstride + static_cast<int64_t>(st) * (G.n + 1) + gi];
  };
  auto w_at = [&](int st) -> double {            // edge e = tid / mm of W(t_st)
    if (tid >= 4 * mm) return 0.0;
    const int e = tid / mm, k = tid - e * mm;
    const int line = e == 0 ? lx0 : (e == 1 ? lx1 : (e == 2 ? ly0 : ly1));
    return Wat(line, st, (e < 2 ? j0 : i0) + k);
  };
  const double r = E.D * G.dt / (G.h * G.h);
  pcr_factors(nu, -0.5 * r, 1.0 + r, pk, sm + pdd_cluster_smem_doubles(m));
  // remote copies: the same offset in every CTA of the cluster
  auto put = [&](double* base, int off, double v) {
    for (int c = 0; c < C; ++c) cl.map_shared_rank(base, c)[off] = v;
  };
  // the value at (i, j) at the start of a step: the boundary is W(t_n) (the
  // y-edges over the x-edges at the corners, as the single-CTA impose)
  auto start_val = [&](int i, int j) -> double {
    if (j == 0) return wB[2 * mm + i];
    if (j == m) return wB[3 * mm + i];
    if (i == 0) return wB[0 * mm + j];
    if (i == m) return wB[1 * mm + j];
    return u[i * mm + j];
  };
  {                                              // u(x, y, 0) = g; W(t_0)
    const double w0 = w_at(0);
    for (int q = tid; q < mm * mm; q += nth) {
      const int i = q / mm, j = q - i * mm;
      u[q] = pdd_g(E, G.lo + (i0 + i) * G.h, G.lo + (j0 + j) * G.h);
    }
    if (tid < 4 * mm) wB[tid] = w0;
  }
  cl.sync();
  auto pcr_solve = [&](double& d0, double& d1) {
#pragma unroll
    for (int lv = 0; lv < kPcrLevels; ++lv) {
      const int dl = 1 << lv;
      if (dl >= nu) break;
      const double* k1 = pk + lv * 128;
      const double* k2 = k1 + 64;
      double lo0, lo1, hi0, hi1;
      if (dl < 32) {
        const double a0 = __shfl_up_sync(0xffffffffu, d0, dl), a1 = __shfl_up_sync(0xffffffffu, d1, dl);
        const double w0 = __shfl_down_sync(0xffffffffu, d0, dl), w1 = __shfl_down_sync(0xffffffffu, d1, dl);
        const double c0 = __shfl_sync(0xffffffffu, d0, (lane - dl) & 31);
        const double c1 = __shfl_sync(0xffffffffu, d1, (lane + dl) & 31);
        const bool dn = lane >= dl, up = lane + dl < 32;
        lo0 = dn ? a0 : 0.0;
        lo1 = dn ? a1 : c0;
        hi0 = up ? w0 : c1;
        hi1 = up ? w1 : 0.0;
      } else {
        lo0 = 0.0; lo1 = d0; hi0 = d1; hi1 = 0.0;
      }
      d0 = fma(-k2[lane], hi0, fma(-k1[lane], lo0, d0));
      d1 = fma(-k2[lane + 32], hi1, fma(-k1[lane + 32], lo1, d1));
    }
    d0 *= pk[kPcrLevels * 128 + lane];
    d1 *= pk[kPcrLevels * 128 + lane + 32];
  };
  // owned points (i, j), j ≡ crank (mod C): four in flight per thread
  const int nrow = (mm - crank + C - 1) / C;     // owned rows j = crank + C t
  auto react_owned = [&](bool from_start, double hh) {
    const int npt = nrow * mm;
    if (npt <= nth) {                            // one point per thread
      if (tid < npt) {
        const int i = tid % mm, j = crank + C * (tid / mm);
        put(u, i * mm + j, pdd_rk4(E, from_start ? start_val(i, j) : u[i * mm + j], hh));
      }
      return;
    }
    for (int q0 = tid; q0 < npt; q0 += 4 * nth) {
      double v[4];
      int ii[4], jj[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int q = q0 + c * nth;
        ii[c] = q % mm;
        jj[c] = crank + C * (q / mm);
        v[c] = q < npt ? (from_start ? start_val(ii[c], jj[c]) : u[ii[c] * mm + jj[c]]) : 0.0;
      }
#pragma unroll
      for (int c = 0; c < 4; ++c) v[c] = pdd_rk4(E, v[c], hh);
#pragma unroll
      for (int c = 0; c < 4; ++c)
        if (q0 + c * nth < npt) put(u, ii[c] * mm + jj[c], v[c]);
    }
  };
  auto u_edge = [&](const double* w) -> double {
    const int e = tid / mm, k = tid - e * mm;
    return e == 0 ? w[k] : (e == 1 ? w[m * mm + k] : (e == 2 ? w[k * mm] : w[k * mm + m]));
  };
  double w_ahead = w_at(1);                          // W(t_1), one step ahead
  for (int n = 0; n < G.n_steps; ++n) {
    const double wv = w_ahead;
    if (n + 1 < G.n_steps) w_ahead = w_at(n + 2);
    const double bv = tid < 4 * mm ? pdd_rk4(E, wv, -0.5 * G.dt) : 0.0;   // bB (every CTA)
    react_owned(true, 0.5 * G.dt);                // bA (boundary W(t_n) folded in)
    cl.sync();
    if (tid < 4 * mm) {                           // bM = (bA + bB)/2
      wN[tid] = wv;
      eB[tid] = bv;
      eM[tid] = 0.5 * (u_edge(u) + bv);
    }
    __syncthreads();
    // x-sweep, owned rows j: (I - r/2 δx²) u* = (I + r/2 δy²) u, u* = bM on the x edges
    auto dx = [&](int i, int j) -> double {
      double d = u[i * mm + j] + 0.5 * r * (u[i * mm + j - 1] - 2.0 * u[i * mm + j] + u[i * mm + j + 1]);
      if (i == 1) d += 0.5 * r * eM[0 * mm + j];
      if (i == m - 1) d += 0.5 * r * eM[1 * mm + j];
      return d;
    };
    for (int t = warp; ; t += nwarp) {
      const int j = crank + C * t;
      if (j > m - 1) break;
      if (j < 1) continue;
      double d0 = lane < nu ? dx(lane + 1, j) : 0.0;
      double d1 = lane + 32 < nu ? dx(lane + 33, j) : 0.0;
      pcr_solve(d0, d1);
      if (lane < nu) put(us, (lane + 1) * mm + j, d0);
      if (lane + 32 < nu) put(us, (lane + 33) * mm + j, d1);
    }
    for (int k = tid; k < mm; k += nth) {         // u* boundary = bM (every CTA)
      us[0 * mm + k] = eM[0 * mm + k];
      us[m * mm + k] = eM[1 * mm + k];
    }
    __syncthreads();
    for (int k = tid; k < mm; k += nth) {
      us[k * mm + 0] = eM[2 * mm + k];
      us[k * mm + m] = eM[3 * mm + k];
    }
    cl.sync();
    // y-sweep, owned columns i: (I - r/2 δy²) v = (I + r/2 δx²) u*, v = bB on the y edges
    auto dy = [&](int i, int j) -> double {
      double d = us[i * mm + j] + 0.5 * r * (us[(i - 1) * mm + j] - 2.0 * us[i * mm + j] + us[(i + 1) * mm + j]);
      if (j == 1) d += 0.5 * r * eB[2 * mm + i];
      if (j == m - 1) d += 0.5 * r * eB[3 * mm + i];
      return d;
    };
    for (int t = warp; ; t += nwarp) {
      const int i = crank + C * t;
      if (i > m - 1) break;
      if (i < 1) continue;
      double d0 = lane < nu ? dy(i, lane + 1) : 0.0;
      double d1 = lane + 32 < nu ? dy(i, lane + 33) : 0.0;
      pcr_solve(d0, d1);
      if (lane < nu) put(u, i * mm + lane + 1, d0);
      if (lane + 32 < nu) put(u, i * mm + lane + 33, d1);
    }
    for (int k = tid; k < mm; k += nth) {         // v boundary = bB (every CTA)
      u[0 * mm + k] = eB[0 * mm + k];
      u[m * mm + k] = eB[1 * mm + k];
    }
    __syncthreads();
    for (int k = tid; k < mm; k += nth) {
      u[k * mm + 0] = eB[2 * mm + k];
      u[k * mm + m] = eB[3 * mm + k];
    }
    cl.sync();
    react_owned(false, 0.5 * G.dt);
    if (tid < 4 * mm) wB[tid] = wN[tid];          // the next step's boundary: W(t_{n+1})
    cl.sync();
  }
  // the field at T with the final boundary W(t_N), owned rows
  for (int q = tid; q < nrow * mm; q += nth) {
    const int i = q % mm, j = crank + C * (q / mm);
    F[static_cast<int64_t>(i0 + i) * (G.n + 1) + (j0 + j)] = start_val(i, j);
  }
}

}  // namespace rtk
