// workloads/gen.cpp — seeded synthetic problem generator (shared INPUT module).
//
// This module builds the linear systems both the oracle (oracle/) and the CUDA
// path (paper_0812_2769_b200/) are run on.  It holds none of the method's
// arithmetic (no GS scaling, no Krylov step): it only discretises the PDEs of the
// paper's setup and of BASELINE.json's configs into CSR form.
//
//   Discretisation  PAPER.md:281-294 (§2.1 "Setup of the numerical experiments"):
//     central differences with half-point coefficients a_{i±1/2,j},
//     equally spaced grid, u^0 = 0.
//   Readings:
//     M1  N interior points per axis, h = 1/(N+1), node I (0-based) at (I+1)h.
//     M2  operator is h^2-scaled (entries O(k)).
//     M3  k sampled at face midpoints; coordinates on the doubled lattice
//         m/(2(N+1)) so interface tests are exact integer comparisons.
//     M4  C5: node-centred k, face value = harmonic mean, boundary face = node k.
//     M5  convection b·grad u at the node: centred +-b h/2 or 1st-order upwind;
//         P1 keeps the paper's conservative d(du)/dx form.
//     M8  structural pattern (computed zeros kept), x fastest, ascending columns.
//     M9  Dirichlet unknowns eliminated; P4 RHS from u=1 on z=0.
//     M10 x* = 2U-1 from a counter-based SplitMix64, b = A x* (BASELINE configs).
//     M11-M16 per-config fields.
//
// Build: g++ -O2 -fopenmp -ffp-contract=off -shared -fPIC (see __graft_entry__.build).
#include <cstdint>
#include <cstring>
#include <cmath>
#include <vector>
#include <algorithm>
#include <functional>

namespace {

// ---- counter-based SplitMix64 (M10/M15): value = mix(seed, stream, i) ------------
inline uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
inline uint64_t h64(uint64_t seed, uint64_t stream, uint64_t i) {
  // base depends on (seed, stream); i enters linearly with an odd multiplier, so
  // for fixed (seed, stream) the map i -> h64 is a bijection on 2^64 (M14).
  uint64_t base = mix64(seed * 0x9E3779B97F4A7C15ULL + stream * 0xD1B54A32D192ED03ULL + 0x632BE59BD9B4E019ULL);
  return mix64(base + (i + 1) * 0x9E3779B97F4A7C15ULL);
}
inline double u01(uint64_t seed, uint64_t stream, uint64_t i) {  // [0,1)
  return (double)(h64(seed, stream, i) >> 11) * 0x1.0p-53;
}
inline double u01_open(uint64_t seed, uint64_t stream, uint64_t i) {  // (0,1]
  return (double)((h64(seed, stream, i) >> 11) + 1) * 0x1.0p-53;
}

enum Scheme { CENTRED = 0, UPWIND = 1, CONSERVATIVE = 2 };

struct Problem {
  int dim = 2;
  int N = 0;
  int Nz = 0;  // planes in z (3D); N except for the stacked-slab variant (cfg 24)
  Scheme scheme = CENTRED;
  // k at a face midpoint given by doubled-lattice coords (mx, my, mz); a point
  // has coordinate m / (2(N+1)).  Used when node_k is empty.
  std::function<double(int64_t, int64_t, int64_t)> kface;
  // optional node-centred k (C5, M4): size N^dim, harmonic faces.
  std::vector<double> node_k;
  // velocity at a node (coordinates in [0,1]); returns components in v[3].
  std::function<void(double, double, double, double*)> vel;
  // P4: u = 1 on z = 0 plane (M9); otherwise homogeneous Dirichlet.
  bool bc_z0_one = false;
};

inline int64_t nrows(const Problem& P) {
  int64_t N = P.N;
  return P.dim == 2 ? N * N : N * N * P.Nz;
}

// number of structural neighbours of node (I,J,K) inside the grid
inline int row_len(const Problem& P, int64_t I, int64_t J, int64_t K) {
  int N = P.N;
  int c = 1;
  c += (I > 0) + (I < N - 1) + (J > 0) + (J < N - 1);
  if (P.dim == 3) c += (K > 0) + (K < P.Nz - 1);
  return c;
}

// Assemble one row (h^2-scaled, §2.1 stencil).  Writes entries in ascending
// column order.  Returns the entry count and the boundary RHS contribution.
int assemble_row(const Problem& P, int64_t I, int64_t J, int64_t K,
                 int32_t* col, double* val, double* rhs_bc) {
  const int N = P.N;
  const int64_t NN = (int64_t)N * N;
  const double h = 1.0 / (N + 1);
  const int64_t r = I + (int64_t)N * J + NN * K;
  // slot order: D(-z) S(-y) W(-x) C E(+x) N(+y) U(+z)
  double off[7] = {0, 0, 0, 0, 0, 0, 0};
  double diag = 0.0;
  int64_t idx[3] = {I, J, K};
  // node coordinates on the doubled lattice
  int64_t m[3] = {2 * (I + 1), 2 * (J + 1), 2 * (K + 1)};
  auto face_k = [&](int axis, int side) -> double {
    if (!P.node_k.empty()) {
      // M4: harmonic mean of the two node values; boundary face takes the node's k
      double k1 = P.node_k[r];
      int64_t nb[3] = {idx[0], idx[1], idx[2]};
      nb[axis] += side;
      if (nb[axis] < 0 || nb[axis] >= N) return k1;
      double k2 = P.node_k[nb[0] + (int64_t)N * nb[1] + NN * nb[2]];
      return 2.0 * k1 * k2 / (k1 + k2);
    }
    int64_t fm[3] = {m[0], m[1], m[2]};
    fm[axis] += side;  // face midpoint = node +- h/2
    return P.kface(fm[0], fm[1], P.dim == 3 ? fm[2] : 0);
  };
  // slot indices for axis minus/plus
  const int minus_slot[3] = {2, 1, 0};
  const int plus_slot[3] = {4, 5, 6};
  double xyz[3] = {(I + 1) * h, (J + 1) * h, P.dim == 3 ? (K + 1) * h : 0.0};
  double v[3] = {0, 0, 0};
  P.vel(xyz[0], xyz[1], xyz[2], v);
  for (int a = 0; a < P.dim; ++a) {
    double km = face_k(a, -1), kp = face_k(a, +1);
    diag += km;
    diag += kp;
    off[minus_slot[a]] -= km;
    off[plus_slot[a]] -= kp;
  }
  for (int a = 0; a < P.dim; ++a) {
    if (P.scheme == CENTRED) {
      double c = v[a] * h * 0.5;
      off[plus_slot[a]] += c;
      off[minus_slot[a]] -= c;
    } else if (P.scheme == UPWIND) {
      double c = v[a] * h;
      if (v[a] > 0) { diag += c; off[minus_slot[a]] -= c; }
      else if (v[a] < 0) { diag -= c; off[plus_slot[a]] += c; }
    } else {  // CONSERVATIVE: d(beta u)/dx with beta at the neighbour nodes
      double xp[3] = {xyz[0], xyz[1], xyz[2]}, xm[3] = {xyz[0], xyz[1], xyz[2]};
      xp[a] += h; xm[a] -= h;
      double vp[3], vm[3];
      P.vel(xp[0], xp[1], xp[2], vp);
      P.vel(xm[0], xm[1], xm[2], vm);
      off[plus_slot[a]] += vp[a] * h * 0.5;
      off[minus_slot[a]] -= vm[a] * h * 0.5;
    }
  }
  off[3] = diag;
  *rhs_bc = 0.0;
  int cnt = 0;
  auto put = [&](bool inside, int64_t c, double a) {
    if (inside) { col[cnt] = (int32_t)c; val[cnt] = a; ++cnt; }
  };
  if (P.dim == 3) {
    put(K > 0, r - NN, off[0]);
    if (K == 0 && P.bc_z0_one) *rhs_bc = -off[0];  // u = 1 on z = 0 (M9)
  }
  put(J > 0, r - N, off[1]);
  put(I > 0, r - 1, off[2]);
  put(true, r, off[3]);
  put(I < N - 1, r + 1, off[4]);
  put(J < N - 1, r + N, off[5]);
  if (P.dim == 3) put(K < P.Nz - 1, r + NN, off[6]);
  return cnt;
}

// ---- configuration table ----------------------------------------------------------
// cfg ids: 1..5 = BASELINE configs C1..C5; 11 = paper P1 (a=b=param inside
// (1/4,3/4)^2, else 1); 12 = P1 continuous (a=b=param everywhere);
// 14 = paper P4 (a = param inside (1/3,2/3)^3); 20/21 = 2D/3D Laplacian (k=1, no
// convection; closed-form eigenvectors).
bool make_problem(int cfg, int N, uint64_t seed, double param, Problem& P) {
  P.N = N;
  P.Nz = N;
  switch (cfg) {
    case 1: {  // C1: 2D, k=1e4 strictly inside (1/4,3/4)^2, b=(10,10), centred
      P.dim = 2; P.scheme = CENTRED;
      int64_t L = 2 * (int64_t)(N + 1);
      P.kface = [L](int64_t mx, int64_t my, int64_t) {
        bool in = (L < 4 * mx) && (4 * mx < 3 * L) && (L < 4 * my) && (4 * my < 3 * L);
        return in ? 1e4 : 1.0;
      };
      P.vel = [](double, double, double, double* v) { v[0] = 10; v[1] = 10; v[2] = 0; };
      return true;
    }
    case 2: {  // C2: 2D upwind, 8x8 blocks from {1,1e3,1e6}, b=(50x,-50y) (M6, M16)
      P.dim = 2; P.scheme = UPWIND;
      std::vector<double> blk(64);
      const double vals[3] = {1.0, 1e3, 1e6};
      for (int i = 0; i < 64; ++i) {
        int c = (int)(u01(seed, 2, i) * 3.0);
        if (c > 2) c = 2;
        blk[i] = vals[c];
      }
      int64_t N1 = N + 1;
      P.kface = [blk, N1](int64_t mx, int64_t my, int64_t) {
        int64_t bx = std::min<int64_t>(7, (4 * mx) / N1);  // floor(8 x), x = mx/(2(N+1))
        int64_t by = std::min<int64_t>(7, (4 * my) / N1);
        return blk[by * 8 + bx];
      };
      P.vel = [](double x, double y, double, double* v) { v[0] = 50.0 * x; v[1] = -50.0 * y; v[2] = 0; };
      return true;
    }
    case 3: {  // C3: 3D centred, 40 spheres r~U[0.03,0.12], k=1e5 inside (M11)
      P.dim = 3; P.scheme = CENTRED;
      std::vector<double> sph(160);
      for (int s = 0; s < 40; ++s) {
        sph[4 * s + 0] = u01(seed, 3, 4 * s + 0);
        sph[4 * s + 1] = u01(seed, 3, 4 * s + 1);
        sph[4 * s + 2] = u01(seed, 3, 4 * s + 2);
        sph[4 * s + 3] = 0.03 + 0.09 * u01(seed, 3, 4 * s + 3);
      }
      double inv = 1.0 / (2.0 * (N + 1));
      P.kface = [sph, inv](int64_t mx, int64_t my, int64_t mz) {
        double x = mx * inv, y = my * inv, z = mz * inv;
        for (int s = 0; s < 40; ++s) {
          double dx = x - sph[4 * s], dy = y - sph[4 * s + 1], dz = z - sph[4 * s + 2];
          double r = sph[4 * s + 3];
          if (dx * dx + dy * dy + dz * dz < r * r) return 1e5;
        }
        return 1.0;
      };
      P.vel = [](double, double, double, double* v) { v[0] = 20; v[1] = 40; v[2] = 60; };
      return true;
    }
    case 4: {  // C4: 3D upwind, 5 z-slabs, 4 distinct cuts in [1,N-1] (M12)
      P.dim = 3; P.scheme = UPWIND;
      std::vector<int64_t> cuts;
      for (uint64_t t = 0; cuts.size() < 4 && t < 100000; ++t) {
        int64_t c = 1 + (int64_t)(h64(seed, 4, t) % (uint64_t)(N - 1));
        if (std::find(cuts.begin(), cuts.end(), c) == cuts.end()) cuts.push_back(c);
      }
      std::sort(cuts.begin(), cuts.end());
      const double kv[5] = {1.0, 1e2, 1e4, 1e-2, 1e6};
      std::vector<double> kvv(kv, kv + 5);
      P.kface = [cuts, kvv](int64_t, int64_t, int64_t mz) {
        // 1-based node c and c+1 are separated by the face at doubled coord 2c+1;
        // half-open membership: a face on a boundary takes the upper slab.
        int s = 0;
        for (int64_t c : cuts) s += (2 * c + 1 <= mz);
        return kvv[s];
      };
      P.vel = [](double, double, double, double* v) { v[0] = 30; v[1] = 0; v[2] = -30; };
      return true;
    }
    case 24: {  // C4 stacked: G = param copies of C4's layered medium in z (weak scaling,
      // DESIGN.md §8).  N x N x (G N) nodes, the same h, velocity and slab cuts; a face
      // takes the slab of its block's local doubled coordinate (the face between two
      // blocks is the upper block's bottom face; the top face of the last block keeps
      // C4's top slab), so G = 1 is exactly C4.
      const int G = param >= 1 ? (int)param : 1;
      if (!make_problem(4, N, seed, 0.0, P)) return false;
      P.Nz = N * G;
      auto k4 = P.kface;
      const int64_t twoN = 2 * (int64_t)N;
      P.kface = [k4, twoN, G](int64_t mx, int64_t my, int64_t mz) {
        const int64_t g = std::min<int64_t>(G - 1, (mz - 1) / twoN);
        return k4(mx, my, mz - g * twoN);
      };
      return true;
    }
    case 5: {  // C5: 2D centred, log-uniform k via Gaussian-copula field (M13)
      P.dim = 2; P.scheme = CENTRED;
      const int64_t n = (int64_t)N * N;
      std::vector<double> g(n), tmp(n);
      const double two_pi = 6.283185307179586;
      #pragma omp parallel for schedule(static)
      for (int64_t i = 0; i < n; ++i) {
        double a = u01_open(seed, 5, 2 * i), b = u01(seed, 5, 2 * i + 1);
        g[i] = std::sqrt(-2.0 * std::log(a)) * std::cos(two_pi * b);
      }
      const int sigma = 16, R = 4 * sigma;
      std::vector<double> w(2 * R + 1);
      double ws = 0;
      for (int t = -R; t <= R; ++t) { w[t + R] = std::exp(-0.5 * (double)t * t / ((double)sigma * sigma)); ws += w[t + R]; }
      for (auto& x : w) x /= ws;
      // separable periodic filter: x then y
      #pragma omp parallel for schedule(static)
      for (int64_t J = 0; J < N; ++J)
        for (int64_t I = 0; I < N; ++I) {
          double acc = 0;
          for (int t = -R; t <= R; ++t) acc += w[t + R] * g[((I + t) % N + N) % N + J * N];
          tmp[I + J * N] = acc;
        }
      #pragma omp parallel for schedule(static)
      for (int64_t J = 0; J < N; ++J)
        for (int64_t I = 0; I < N; ++I) {
          double acc = 0;
          for (int t = -R; t <= R; ++t) acc += w[t + R] * tmp[I + (((J + t) % N + N) % N) * N];
          g[I + J * N] = acc;
        }
      double mean = 0, var = 0;
      for (int64_t i = 0; i < n; ++i) mean += g[i];
      mean /= (double)n;
      for (int64_t i = 0; i < n; ++i) var += (g[i] - mean) * (g[i] - mean);
      double sd = std::sqrt(var / (double)n);
      P.node_k.resize(n);
      #pragma omp parallel for schedule(static)
      for (int64_t i = 0; i < n; ++i) {
        double z = (g[i] - mean) / sd;
        double u = 0.5 * std::erfc(-z / std::sqrt(2.0));
        P.node_k[i] = std::pow(10.0, -3.0 + 8.0 * u);
      }
      P.vel = [](double, double, double, double* v) { v[0] = 5; v[1] = 5; v[2] = 0; };
      return true;
    }
    case 11: case 12: {  // paper P1, conservative convection
      P.dim = 2; P.scheme = CONSERVATIVE;
      int64_t L = 2 * (int64_t)(N + 1);
      double a_in = param > 0 ? param : 1e3;
      bool cont = (cfg == 12);
      P.kface = [L, a_in, cont](int64_t mx, int64_t my, int64_t) {
        if (cont) return a_in;
        bool in = (L < 4 * mx) && (4 * mx < 3 * L) && (L < 4 * my) && (4 * my < 3 * L);
        return in ? a_in : 1.0;
      };
      // d = 10(x+y), e = 10(x-y)
      P.vel = [](double x, double y, double, double* v) { v[0] = 10.0 * (x + y); v[1] = 10.0 * (x - y); v[2] = 0; };
      return true;
    }
    case 14: case 15: {  // paper P4: a = D inside (1/3,2/3)^3
      // 14: d=e=f=100, D = param; 15: D = 1e4, d=e=f = param (Table "limit",
      // PAPER.md:1099-1147, convection sweep 100/200/500/1000)
      P.dim = 3; P.scheme = CENTRED; P.bc_z0_one = true;
      int64_t L = 2 * (int64_t)(N + 1);
      double D = (cfg == 14 && param > 0) ? param : 1e4;
      const double cv = (cfg == 15 && param > 0) ? param : 100.0;
      P.kface = [L, D](int64_t mx, int64_t my, int64_t mz) {
        auto in = [L](int64_t m) { return (L < 3 * m) && (3 * m < 2 * L); };
        return (in(mx) && in(my) && in(mz)) ? D : 1.0;
      };
      P.vel = [cv](double, double, double, double* v) { v[0] = cv; v[1] = cv; v[2] = cv; };
      return true;
    }
    case 20: case 21: {  // Laplacian, k = 1, no convection
      P.dim = (cfg == 20) ? 2 : 3; P.scheme = CENTRED;
      P.kface = [](int64_t, int64_t, int64_t) { return 1.0; };
      P.vel = [](double, double, double, double* v) { v[0] = v[1] = v[2] = 0; };
      return true;
    }
    default:
      return false;
  }
}

}  // namespace

extern "C" {

// Sizes of the stacked-slab system (cfg 24): N x N x (G N) nodes.
int gen_dims_stacked(int N, int G, int64_t* n, int64_t* nnz) {
  if (N < 2 || G < 1) return -1;
  const int64_t NN = (int64_t)N * N, Nz = (int64_t)N * G;
  *n = NN * Nz;
  *nnz = 7 * NN * Nz - 4 * (int64_t)N * Nz - 2 * NN;
  return 0;
}

// Sizes of the system for (cfg, N).  Returns 0, or -1 for an unknown cfg.
int gen_dims(int cfg, int N, int64_t* n, int64_t* nnz) {
  Problem P;
  P.N = N;
  if (cfg == 1 || cfg == 2 || cfg == 5 || cfg == 11 || cfg == 12 || cfg == 20) P.dim = 2;
  else if (cfg == 3 || cfg == 4 || cfg == 14 || cfg == 15 || cfg == 21) P.dim = 3;
  else return -1;
  if (N < 2) return -1;
  int64_t NN = N;
  *n = P.dim == 2 ? NN * NN : NN * NN * NN;
  *nnz = P.dim == 2 ? 5 * NN * NN - 4 * NN : 7 * NN * NN * NN - 6 * NN * NN;
  return 0;
}

// Fill the CSR system.  row_ptr[n+1], col[nnz], val[nnz], xstar[n], b[n], perm[n]
// (perm may be null; it receives pi with new_index = pi[old_index], identity
// except for cfg 5).  b = A x* (plain ascending sum) for the BASELINE configs; for
// P1 b = A e and x* = e; for P4 b comes from the boundary data
// and x* = 0 (unknown).
int gen_fill(int cfg, int N, uint64_t seed, double param, int32_t* row_ptr, int32_t* col,
             double* val, double* xstar, double* b, int32_t* perm) {
  Problem P;
  if (!make_problem(cfg, N, seed, param, P)) return -1;
  const int64_t n = nrows(P);
  const int64_t NN = (int64_t)N * N;
  // row pointers from the structural pattern
  row_ptr[0] = 0;
  for (int64_t r = 0; r < n; ++r) {
    int64_t I = r % N, J = (r / N) % N, K = r / NN;
    row_ptr[r + 1] = row_ptr[r] + row_len(P, I, J, P.dim == 3 ? K : 0);
  }
  std::vector<double> rhs_bc(n, 0.0);
  #pragma omp parallel for schedule(static)
  for (int64_t r = 0; r < n; ++r) {
    int64_t I = r % N, J = (r / N) % N, K = P.dim == 3 ? r / NN : 0;
    assemble_row(P, I, J, K, col + row_ptr[r], val + row_ptr[r], &rhs_bc[r]);
  }
  // x*
  const bool is_p1 = (cfg == 11 || cfg == 12), is_p4 = (cfg == 14 || cfg == 15);
  #pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i)
    xstar[i] = is_p1 ? 1.0 : (is_p4 ? 0.0 : 2.0 * u01(seed, 1, i) - 1.0);

  if (cfg == 5 && !(param < 0)) {  // param < 0: unpermuted (tests)
    // M14: pi = rank of h64(seed, 6, i); A' = P A P^T, columns re-sorted.
    std::vector<std::pair<uint64_t, int32_t>> key(n);
    for (int64_t i = 0; i < n; ++i) key[i] = {h64(seed, 6, i), (int32_t)i};
    std::sort(key.begin(), key.end());
    std::vector<int32_t> pi(n);
    for (int64_t k = 0; k < n; ++k) pi[key[k].second] = (int32_t)k;
    std::vector<int32_t> inv(n);
    for (int64_t i = 0; i < n; ++i) inv[pi[i]] = (int32_t)i;
    const int64_t nnz = row_ptr[n];
    std::vector<int32_t> rp2(n + 1), c2(nnz);
    std::vector<double> v2(nnz), xs2(n);
    rp2[0] = 0;
    for (int64_t k = 0; k < n; ++k) rp2[k + 1] = rp2[k] + (row_ptr[inv[k] + 1] - row_ptr[inv[k]]);
    #pragma omp parallel for schedule(static)
    for (int64_t k = 0; k < n; ++k) {
      int64_t old = inv[k];
      int32_t s = row_ptr[old], e = row_ptr[old + 1];
      std::vector<std::pair<int32_t, double>> ent;
      ent.reserve(e - s);
      for (int32_t q = s; q < e; ++q) ent.push_back({pi[col[q]], val[q]});
      std::sort(ent.begin(), ent.end(), [](const auto& a, const auto& b2) { return a.first < b2.first; });
      for (size_t q = 0; q < ent.size(); ++q) { c2[rp2[k] + q] = ent[q].first; v2[rp2[k] + q] = ent[q].second; }
      xs2[k] = xstar[old];
    }
    std::memcpy(row_ptr, rp2.data(), sizeof(int32_t) * (n + 1));
    std::memcpy(col, c2.data(), sizeof(int32_t) * nnz);
    std::memcpy(val, v2.data(), sizeof(double) * nnz);
    std::memcpy(xstar, xs2.data(), sizeof(double) * n);
    if (perm) std::memcpy(perm, pi.data(), sizeof(int32_t) * n);
  } else if (perm) {
    for (int64_t i = 0; i < n; ++i) perm[i] = (int32_t)i;
  }
  // right-hand side
  #pragma omp parallel for schedule(static)
  for (int64_t r = 0; r < n; ++r) {
    if (is_p4) { b[r] = rhs_bc[r]; continue; }
    double acc = 0.0;
    for (int32_t q = row_ptr[r]; q < row_ptr[r + 1]; ++q) acc = std::fma(val[q], xstar[col[q]], acc);
    b[r] = acc;
  }
  return 0;
}

// Rows [lo, hi) of the system (global column indices, row_ptr[0] = 0), x* and b = A x*
// on those rows — what one rank of a row-block sharded solve needs,
// without building the rest.  Any config but C5 (whose permutation is global) and
// the paper's P-workloads (b from boundary data).  Row for row identical to gen_fill.
int gen_fill_rows(int cfg, int N, uint64_t seed, double param, int64_t lo, int64_t hi, int32_t* row_ptr,
                  int32_t* col, double* val, double* xstar, double* b) {
  if (cfg == 5 || cfg == 11 || cfg == 12 || cfg == 14 || cfg == 15) return -1;
  Problem P;
  if (!make_problem(cfg, N, seed, param, P)) return -1;
  const int64_t n = nrows(P);
  if (lo < 0 || hi > n || lo > hi) return -1;
  const int64_t NN = (int64_t)N * N, m = hi - lo;
  row_ptr[0] = 0;
  for (int64_t q = 0; q < m; ++q) {
    const int64_t r = lo + q;
    int64_t I = r % N, J = (r / N) % N, K = P.dim == 3 ? r / NN : 0;
    row_ptr[q + 1] = row_ptr[q] + row_len(P, I, J, K);
  }
  #pragma omp parallel for schedule(static)
  for (int64_t q = 0; q < m; ++q) {
    const int64_t r = lo + q;
    int64_t I = r % N, J = (r / N) % N, K = P.dim == 3 ? r / NN : 0;
    double bc = 0.0;
    assemble_row(P, I, J, K, col + row_ptr[q], val + row_ptr[q], &bc);
  }
  #pragma omp parallel for schedule(static)
  for (int64_t q = 0; q < m; ++q) {
    xstar[q] = 2.0 * u01(seed, 1, lo + q) - 1.0;
    double acc = 0.0;
    for (int32_t k = row_ptr[q]; k < row_ptr[q + 1]; ++k)
      acc = std::fma(val[k], 2.0 * u01(seed, 1, col[k]) - 1.0, acc);
    b[q] = acc;
  }
  return 0;
}

// Raw access to the counter generator (tests / seeded vectors for kernels).
void gen_uniform(uint64_t seed, uint64_t stream, int64_t n, double lo, double hi, double* out) {
  #pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) out[i] = lo + (hi - lo) * u01(seed, stream, i);
}

}  // extern "C"
