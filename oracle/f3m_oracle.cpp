// =====================================================================================
//  F^3M ORACLE  --  TEST INFRASTRUCTURE ONLY
// =====================================================================================
//  A plain, slow, obviously-correct, single-threaded fp64 CPU implementation of the
//  F^3M approximate kernel matrix-vector product (arXiv 2202.01085, /root/reference/
//  PAPER.md) and of the exact direct KMVM.  It follows App. F Algorithm 1
//   step by step, with the readings listed in DESIGN.md
//  ("Readings of the paper", R1..R24; they are SURVEY.md 8(c) Q1..Q24).
//
//  * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
//    reference leg may load this library.  The product (paper_2202_01085_b200/) never
//    does; the two share no code, header, table or constant generator.
//  * fp64 throughout: inputs are fp32 values converted exactly to fp64 by the caller.
//  * Build: g++ -O2 -ffp-contract=off -fno-fast-math -shared -fPIC (no OpenMP, no SIMD
//    intrinsics).  std::stable_sort gives the unique stable permutation.
//  * Parity status of every function is stated in DESIGN.md ("Oracle pins").  No
//    function here is "parity unpinned": each is pinned in tests/test_oracle_*.py to
//    closed forms, the paper's worked formulas, brute force or invariants.
// =====================================================================================
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <map>
#include <string>
#include <vector>

namespace {

// status codes (numerically the same meaning as SPEC exit codes S:611; defined here
// independently of include/f3m.h)
enum { ORC_OK = 0, ORC_INVALID_INPUT = 2, ORC_RESOURCE = 3, ORC_INTERNAL = 4,
       ORC_INVALID_SPEC = 5, ORC_GRID_TOO_LARGE = 6 };

// configuration flags (ablations)
enum { ORC_EXACT = 1, ORC_NO_SMOOTH = 2, ORC_NO_ADAPTIVE = 4, ORC_NO_SMALL = 8,
       ORC_NO_DROP = 16, ORC_MAXNORM = 32, ORC_KEEP_EMPTY = 64 };

// pair tags
enum { TAG_NEAR = 0, TAG_FAR = 1, TAG_FAR_DROPPED = 2, TAG_SMOOTH = 3, TAG_SMALL = 4 };

const int MAXLEV = 64;
thread_local std::string g_err;

// ---- Sec. 3 "Lagrange interpolation": Chebyshev nodes of the 2nd
// kind s_i = cos(i*pi/r), i = 0..r, with r = P-1 (reading R2: P nodes per dimension).
std::vector<double> cheb_nodes(int P) {
  std::vector<double> s(P);
  const double r = (double)(P - 1);
  for (int i = 0; i < P; ++i) s[i] = std::cos((double)i * M_PI / r);
  return s;
}

// ---- App. C: w_i = (-1)^i delta_i, delta = 1/2 at both ends.
std::vector<double> bary_weights(int P) {
  std::vector<double> w(P);
  for (int i = 0; i < P; ++i) {
    double d = (i == 0 || i == P - 1) ? 0.5 : 1.0;
    w[i] = (i % 2 == 0) ? d : -d;
  }
  return w;
}

// ---- App. C: barycentric Lagrange basis, second form.
//   L_i(t) = (w_i/(t-s_i)) / sum_j (w_j/(t-s_j));  L_i(s_j) = delta_ij at a node.
void bary_basis(int P, const double* s, const double* w, double t, double* L) {
  for (int i = 0; i < P; ++i) {
    if (t == s[i]) {  // singular case: exact node hit
      for (int j = 0; j < P; ++j) L[j] = (j == i) ? 1.0 : 0.0;
      return;
    }
  }
  double den = 0.0;
  for (int j = 0; j < P; ++j) den += w[j] / (t - s[j]);
  for (int i = 0; i < P; ++i) L[i] = (w[i] / (t - s[i])) / den;
}

// ---- Sec. 5: Gaussian kernel exp(-||x-y||^2 / (2 gamma^2)).
inline double gauss(const double* x, const double* y, int D, double gamma) {
  double d2 = 0.0;
  for (int d = 0; d < D; ++d) {
    double diff = x[d] - y[d];
    d2 += diff * diff;
  }
  return std::exp(-d2 / (2.0 * gamma * gamma));
}

// ---- Sec. 1 "Notations": v_i = sum_j k(x_i, y_j) b_j, j ascending.
void direct(const double* X, int64_t nx, const double* Y, int64_t ny, int D, const double* b,
            double gamma, double* v) {
  for (int64_t i = 0; i < nx; ++i) {
    double acc = 0.0;
    for (int64_t j = 0; j < ny; ++j) acc += gauss(X + i * D, Y + j * D, D, gamma) * b[j];
    v[i] = acc;
  }
}

struct Box {
  uint64_t key;          // order-key prefix at this depth (nested Morton, reading R13)
  int64_t start, count;  // interval [start, start+count) of the sorted order (Sec. 4.1)
  int64_t cell[7];       // integer cell coordinates i_{p,d} at this depth
  int64_t child0 = 0, nchild = 0;  // children (indices into the next depth's box array)
};

struct Side {
  int64_t n = 0;
  const double* pts = nullptr;  // row-major n x D
  double alpha[7] = {0};
  std::vector<uint64_t> key;       // order key per ORIGINAL point index
  std::vector<int64_t> cellT;      // leaf cells c_d(T) per original point, n x D
  std::vector<int64_t> perm;       // sorted position -> original index (pi)
  std::vector<std::vector<Box>> lev;  // lev[t], t = 0..T
};

struct Pair { int64_t p, q; };

struct Charges {  // stage-1/2 records kept for the per-kernel parity tests
  int t, P;
  int64_t m = 0;   // nodes per box (P^D, or |H| of a sparse grid)
  int q = 0;       // sparse-grid level (0: tensor grid of P nodes per dimension)
  std::vector<uint64_t> src_key;   std::vector<double> W;  // [nsrc x m]
  std::vector<uint64_t> tgt_key;   std::vector<double> U;  // [ntgt x m]
};

struct Result {
  int D = 0;
  double E = 0.0;
  int t_star = 0, T_sort = 0, depth_reached = 0;
  double alphaX[7] = {0}, alphaY[7] = {0};
  std::vector<double> v;
  Side X, Y;
  bool aliased = false;
  // per depth t (1-based) stats
  int64_t M[MAXLEV] = {0}, expanded[MAXLEV] = {0}, m_far[MAXLEV] = {0},
          m_far_dropped[MAXLEV] = {0}, m_smooth[MAXLEV] = {0}, m_small[MAXLEV] = {0},
          m_near[MAXLEV] = {0}, boxes_x[MAXLEV] = {0}, boxes_y[MAXLEV] = {0},
          empty_x[MAXLEV] = {0}, empty_y[MAXLEV] = {0}, pfar[MAXLEV] = {0};
  int64_t n_near_flushed = 0;
  // all classified pairs per depth: (key_p, key_q, tag)
  std::vector<std::vector<uint64_t>> pk, qk;
  std::vector<std::vector<int32_t>> tag;
  std::vector<Charges> charges;
};

// ---- Sec. 4.2 box index on one coordinate, reading R12:
//   u = (x - alpha)/E (IEEE fp64, correctly rounded), c(t) = min(floor(u 2^t), 2^t - 1).
inline int64_t cell_of(double x, double alpha, double E, int T) {
  double u = (x - alpha) / E;
  double f = std::floor(std::ldexp(u, T));
  int64_t c = (int64_t)f;
  int64_t cmax = ((int64_t)1 << T) - 1;
  return c > cmax ? cmax : c;
}

// nested Morton order key (reading R13): K = sum_{s=1..T} l_s 2^{D(T-s)},
// l_s = sum_d 2^{d-1} bit(c_d(T), T-s)   (dimension 1 is the least significant bit).
uint64_t order_key(const int64_t* c, int D, int T) {
  uint64_t K = 0;
  for (int s = 1; s <= T; ++s) {
    uint64_t l = 0;
    for (int d = 0; d < D; ++d) l |= (uint64_t)((c[d] >> (T - s)) & 1) << d;
    K = (K << D) | l;
  }
  return K;
}

// Steps 4-5 of the oracle algorithm: keys, stable counting permutation (Sec. 4.1 steps
// 1-2, made stable per reading R13), and the box tables of every depth
// (empty boxes never appear: only runs of present keys are boxes, Sec. 4.2).
void build_side(Side& S, int D, double E, int T) {
  const int64_t n = S.n;
  S.key.assign(n, 0);
  S.cellT.assign(n * D, 0);
  for (int64_t i = 0; i < n; ++i) {
    for (int d = 0; d < D; ++d) S.cellT[i * D + d] = cell_of(S.pts[i * D + d], S.alpha[d], E, T);
    S.key[i] = order_key(&S.cellT[i * D], D, T);
  }
  S.perm.resize(n);
  for (int64_t i = 0; i < n; ++i) S.perm[i] = i;
  std::stable_sort(S.perm.begin(), S.perm.end(),
                   [&](int64_t a, int64_t b) { return S.key[a] < S.key[b]; });
  S.lev.assign(T + 1, {});
  for (int t = 0; t <= T; ++t) {
    const int sh = D * (T - t);
    std::vector<Box>& L = S.lev[t];
    for (int64_t i = 0; i < n; ++i) {
      const int64_t o = S.perm[i];
      const uint64_t pre = (sh >= 64) ? 0 : (S.key[o] >> sh);
      if (L.empty() || L.back().key != pre) {
        Box bx;
        bx.key = pre;
        bx.start = i;
        bx.count = 0;
        for (int d = 0; d < 7; ++d) bx.cell[d] = 0;
        for (int d = 0; d < D; ++d) bx.cell[d] = S.cellT[o * D + d] >> (T - t);
        L.push_back(bx);
      }
      L.back().count++;
    }
  }
  for (int t = 0; t < T; ++t) {
    std::vector<Box>& P = S.lev[t];
    const std::vector<Box>& C = S.lev[t + 1];
    int64_t j = 0;
    for (size_t p = 0; p < P.size(); ++p) {
      P[p].child0 = j;
      while (j < (int64_t)C.size() && (C[j].key >> D) == P[p].key) ++j;
      P[p].nchild = j - P[p].child0;
    }
  }
}

// FFM-style box tables (the FFM(GPU) ablation of Tables 5-6; Fig. 5,
// PAPER.md:183-189): no empty-box removal -- every depth holds all 2^{D t} cells in key order,
// empty ones with count 0, and a divided box has all 2^D children.  The points' order (pi) is
// unchanged; empty boxes only add (zero-valued) interactions.
void keep_empty_boxes(Side& S, int D, int T) {
  for (int t = 0; t <= T; ++t) {
    const std::vector<Box> L0 = S.lev[t];
    const int64_t nb = (int64_t)1 << (D * t);
    std::vector<Box> L(nb);
    size_t j = 0;
    int64_t pos = 0;
    for (int64_t k = 0; k < nb; ++k) {
      Box& bx = L[k];
      bx.key = (uint64_t)k;
      for (int d = 0; d < 7; ++d) bx.cell[d] = 0;
      for (int s = 0; s < t; ++s) {
        const uint64_t g = ((uint64_t)k >> (D * (t - 1 - s))) & (((uint64_t)1 << D) - 1);
        for (int d = 0; d < D; ++d) bx.cell[d] = (bx.cell[d] << 1) | (int64_t)((g >> d) & 1);
      }
      if (j < L0.size() && L0[j].key == (uint64_t)k) {
        bx.start = L0[j].start;
        bx.count = L0[j].count;
        pos = bx.start + bx.count;
        ++j;
      } else {
        bx.start = pos;
        bx.count = 0;
      }
      bx.child0 = k << D;
      bx.nchild = (t < T) ? ((int64_t)1 << D) : 0;
    }
    S.lev[t].swap(L);
  }
}

// tensor-product basis L_k(x) = prod_d L_{k_d}(tau_d) (Sec. 3), k = sum_d k_d P^d
void tensor_basis(int D, int P, const double* s, const double* w, const double* tau, double* out) {
  std::vector<double> L1(D * P);
  for (int d = 0; d < D; ++d) bary_basis(P, s, w, tau[d], &L1[d * P]);
  int64_t m = 1;
  for (int d = 0; d < D; ++d) m *= P;
  for (int64_t k = 0; k < m; ++k) {
    int64_t r = k;
    double prod = 1.0;
    for (int d = 0; d < D; ++d) {
      prod *= L1[d * P + (r % P)];
      r /= P;
    }
    out[k] = prod;
  }
}

// box-local coordinate tau = 2(x - alpha)/l - (2i + 1) in [-1, 1] (Fig. 4 step 1 "normalize
// the data between [-1,1]", geometric cell per reading R15).
inline double local_coord(double x, double alpha, double l, int64_t i) {
  return (2.0 * (x - alpha)) / l - (double)(2 * i + 1);
}

// node coordinate n = c + (l/2) s with c = alpha + (i + 1/2) l (reading R15)
inline double node_coord(double alpha, int64_t i, double l, double s) {
  double c = alpha + ((double)i + 0.5) * l;
  return c + (l / 2.0) * s;
}

struct Params {
  int D, P;
  double gamma, eta;
  int64_t rho, zeta;
  int max_depth;
  unsigned flags;
  int64_t node_cap;
  int64_t n_eval;  // > 0: subset-target mode, v only for the original rows i < n_eval (Sec. 5
                   // error protocol evaluates the first rows); the tree, every
                   // charge and every pair list are those of the full problem
  int sparse_level;  // > 0: Smolyak sparse grid of this level instead of the P^D tensor grid
};

inline bool evaluated(const Params& prm, int64_t orig_row) { return prm.n_eval <= 0 || orig_row < prm.n_eval; }

// ---- Smolyak sparse grids (Sec. 4.2 "Sparse grids": "we implement sparse grids
// [Smolyak] to allow for a finer selection of interpolation nodes"; construction per SPEC S:128
// and reading R27 of DESIGN.md -- the paper gives none).  1-D nested Chebyshev (Clenshaw-Curtis)
// levels: level 0 = {0}, level j >= 1 = the 2^j + 1 Chebyshev points cos(k pi / 2^j).  The
// interpolant of level q in D dimensions is the combination technique
//     A(q, D) = sum_{j >= 0, q - D + 1 <= |j|_1 <= q} (-1)^(q - |j|_1) C(D - 1, q - |j|_1) (x)_d U^(j_d),
// U^(j) the 1-D Lagrange interpolant on level j.  Because the levels are nested, every node of a
// term grid is a node of the finest 1-D grid (2^q + 1 points); the sparse node set H is the union
// of the term grids, ordered by the linear index sum_d h_d (2^q + 1)^d of the finest-grid
// coordinates h_d, and the sparse basis function of node h is
//     Phi_h(x) = sum_{terms j with h in grid_j} c_j prod_d L^(j_d)_{k_d}(x_d),   h_d = k_d 2^(q - j_d)
// (h_d = 2^(q-1) for the single level-0 node).  Far field: the kernel is interpolated in x and y
// with A(q, D), i.e. the three stages of Sec. 3 with L_k replaced by Phi_h and the nodes H.
struct SparseGrid {
  int D = 0, q = 0, n1 = 0;                    // n1 = 2^q + 1 finest 1-D points
  std::vector<std::vector<int>> terms;         // multi-indices j
  std::vector<double> coef;                    // combination coefficients c_j
  std::vector<std::vector<int64_t>> nodes;     // H: finest-grid coordinates, ascending linear index
  std::vector<double> s1;                      // finest 1-D node coordinates
};

inline int level_points(int j) { return j == 0 ? 1 : (1 << j) + 1; }

inline double binom(int n, int k) {
  double r = 1.0;
  for (int i = 1; i <= k; ++i) r = r * (double)(n - k + i) / (double)i;
  return r;
}

SparseGrid make_sparse_grid(int D, int q) {
  SparseGrid g;
  g.D = D;
  g.q = q;
  g.n1 = (1 << q) + 1;
  g.s1 = cheb_nodes(g.n1);
  std::vector<int> j(D, 0);
  std::map<int64_t, std::vector<int64_t>> hset;  // linear index -> coordinates
  while (true) {
    int sum = 0;
    for (int d = 0; d < D; ++d) sum += j[d];
    if (sum <= q && sum >= q - D + 1) {
      const double c = ((q - sum) % 2 ? -1.0 : 1.0) * binom(D - 1, q - sum);
      g.terms.push_back(j);
      g.coef.push_back(c);
      std::vector<int64_t> k(D, 0);
      while (true) {
        std::vector<int64_t> h(D);
        int64_t lin = 0, mul = 1;
        for (int d = 0; d < D; ++d) {
          h[d] = j[d] == 0 ? (int64_t)1 << (q - 1) : k[d] << (q - j[d]);
          lin += h[d] * mul;
          mul *= g.n1;
        }
        hset[lin] = h;
        int d = 0;
        while (d < D && ++k[d] == level_points(j[d])) k[d++] = 0;
        if (d == D) break;
      }
    }
    int d = 0;
    while (d < D && ++j[d] > q) j[d++] = 0;
    if (d == D) break;
  }
  for (auto& kv : hset) g.nodes.push_back(kv.second);
  return g;
}

// Phi_h(tau) for every h in H (out has |H| entries)
void sparse_basis(const SparseGrid& g, const double* tau, double* out) {
  const int D = g.D;
  const int64_t m = (int64_t)g.nodes.size();
  std::map<int64_t, int64_t> pos;
  for (int64_t i = 0; i < m; ++i) {
    int64_t lin = 0, mul = 1;
    for (int d = 0; d < D; ++d) { lin += g.nodes[i][d] * mul; mul *= g.n1; }
    pos[lin] = i;
  }
  for (int64_t i = 0; i < m; ++i) out[i] = 0.0;
  // 1-D bases of every level and dimension
  std::vector<std::vector<std::vector<double>>> L(D, std::vector<std::vector<double>>(g.q + 1));
  for (int d = 0; d < D; ++d)
    for (int lv = 0; lv <= g.q; ++lv) {
      if (lv == 0) { L[d][lv] = {1.0}; continue; }
      const int P = level_points(lv);
      std::vector<double> s = cheb_nodes(P), w = bary_weights(P);
      L[d][lv].resize(P);
      bary_basis(P, s.data(), w.data(), tau[d], L[d][lv].data());
    }
  for (size_t t = 0; t < g.terms.size(); ++t) {
    const std::vector<int>& j = g.terms[t];
    std::vector<int64_t> k(D, 0);
    while (true) {
      double prod = g.coef[t];
      int64_t lin = 0, mul = 1;
      for (int d = 0; d < D; ++d) {
        prod *= L[d][j[d]][k[d]];
        const int64_t h = j[d] == 0 ? (int64_t)1 << (g.q - 1) : k[d] << (g.q - j[d]);
        lin += h * mul;
        mul *= g.n1;
      }
      out[pos[lin]] += prod;
      int d = 0;
      while (d < D && ++k[d] == level_points(j[d])) k[d++] = 0;
      if (d == D) break;
    }
  }
}

// the level used for a far-field group under the adaptive rule's min(r, 3^D) branch (reading
// R27): the largest level <= q whose node set has at most 3^D nodes (at least level 1)
int sparse_level_3d(int D, int q) {
  int64_t cap = 1;
  for (int d = 0; d < D; ++d) cap *= 3;
  int best = 1;
  for (int lv = 1; lv <= q; ++lv)
    if ((int64_t)make_sparse_grid(D, lv).nodes.size() <= cap) best = lv;
  return best;
}

// Far field of one depth with the sparse grid of level q (the three stages of far_field below
// with Phi_h and the nodes H, reading R27)
void far_field_sparse(Result& R, const Params& prm, int t, int q, const std::vector<Pair>& pairs,
                      const double* b, double* vsorted_x);

// Far-field three-stage compute for one depth and one node count P' (Sec. 3
// "v = L_X^T (K (L_Y b)) ... first computing v1, then v2 and lastly v"; Fig. 4):
//   stage 1  v1: W_q = L_Y b for every source box of the list,
//   stage 2  v2: U_p = sum_{(p,q) in list} K(nodes_p, nodes_q) W_q,
//   stage 3  v : v_x += sum_k L_k(x) U_p[k] for x in box p.
void far_field(Result& R, const Params& prm, int t, int Pn, const std::vector<Pair>& pairs,
               const double* b, double* vsorted_x) {
  if (pairs.empty()) return;
  const int D = prm.D;
  const double l = std::ldexp(R.E, -t);
  const std::vector<double> s = cheb_nodes(Pn), w = bary_weights(Pn);
  int64_t m = 1;
  for (int d = 0; d < D; ++d) m *= Pn;
  const std::vector<Box>& BX = R.X.lev[t];
  const std::vector<Box>& BY = R.Y.lev[t];
  Charges rec;
  rec.t = t;
  rec.P = Pn;
  rec.m = m;
  // stage 1 (once per (depth, source box, P'), identical to Prop. 2's per-pair form)
  std::map<int64_t, int64_t> slot;
  for (const Pair& pr : pairs) {
    if (slot.count(pr.q)) continue;
    const int64_t sq = (int64_t)slot.size();
    slot[pr.q] = sq;
    const Box& q = BY[pr.q];
    std::vector<double> Wq(m, 0.0), Lk(m), tau(D);
    for (int64_t j = q.start; j < q.start + q.count; ++j) {
      const int64_t o = R.Y.perm[j];
      for (int d = 0; d < D; ++d) tau[d] = local_coord(R.Y.pts[o * D + d], R.alphaY[d], l, q.cell[d]);
      tensor_basis(D, Pn, s.data(), w.data(), tau.data(), Lk.data());
      for (int64_t k = 0; k < m; ++k) Wq[k] += Lk[k] * b[o];
    }
    rec.src_key.push_back(q.key);
    rec.W.insert(rec.W.end(), Wq.begin(), Wq.end());
  }
  // stage 2 + 3, per target box (pairs are sorted by p)
  size_t a = 0;
  std::vector<double> np(D), nq(D), Lk(m), tau(D);
  while (a < pairs.size()) {
    size_t e = a;
    while (e < pairs.size() && pairs[e].p == pairs[a].p) ++e;
    const Box& p = BX[pairs[a].p];
    std::vector<double> U(m, 0.0);
    // stage 2 for every target box of the list (with F3M_KEEP_EMPTY that includes empty boxes,
    // whose interactions FFM(GPU) computes, reading R28); subset-target mode skips boxes without
    // an evaluated target (their locals reach no output)
    bool any_eval = prm.n_eval <= 0;
    for (int64_t i = p.start; i < p.start + p.count && !any_eval; ++i) any_eval = evaluated(prm, R.X.perm[i]);
    for (size_t r = a; r < e && any_eval; ++r) {
      const Box& q = BY[pairs[r].q];
      const double* Wq = &rec.W[slot[pairs[r].q] * m];
      for (int64_t k = 0; k < m; ++k) {
        int64_t rk = k;
        for (int d = 0; d < D; ++d) {
          np[d] = node_coord(R.alphaX[d], p.cell[d], l, s[rk % Pn]);
          rk /= Pn;
        }
        double acc = 0.0;
        for (int64_t j = 0; j < m; ++j) {
          int64_t rj = j;
          for (int d = 0; d < D; ++d) {
            nq[d] = node_coord(R.alphaY[d], q.cell[d], l, s[rj % Pn]);
            rj /= Pn;
          }
          acc += gauss(np.data(), nq.data(), D, prm.gamma) * Wq[j];
        }
        U[k] += acc;
      }
    }
    for (int64_t i = p.start; i < p.start + p.count; ++i) {
      const int64_t o = R.X.perm[i];
      if (!evaluated(prm, o)) continue;
      for (int d = 0; d < D; ++d) tau[d] = local_coord(R.X.pts[o * D + d], R.alphaX[d], l, p.cell[d]);
      tensor_basis(D, Pn, s.data(), w.data(), tau.data(), Lk.data());
      double acc = 0.0;
      for (int64_t k = 0; k < m; ++k) acc += Lk[k] * U[k];
      vsorted_x[i] += acc;
    }
    rec.tgt_key.push_back(p.key);
    rec.U.insert(rec.U.end(), U.begin(), U.end());
    a = e;
  }
  R.charges.push_back(std::move(rec));
}

void far_field_sparse(Result& R, const Params& prm, int t, int q, const std::vector<Pair>& pairs,
                      const double* b, double* vsorted_x) {
  if (pairs.empty()) return;
  const int D = prm.D;
  const double l = std::ldexp(R.E, -t);
  const SparseGrid sg = make_sparse_grid(D, q);
  const int64_t m = (int64_t)sg.nodes.size();
  const std::vector<Box>& BX = R.X.lev[t];
  const std::vector<Box>& BY = R.Y.lev[t];
  Charges rec;
  rec.t = t;
  rec.P = sg.n1;
  rec.m = m;
  rec.q = q;
  // stage 1 (once per (depth, source box, P'), identical to Prop. 2's per-pair form)
  std::map<int64_t, int64_t> slot;
  for (const Pair& pr : pairs) {
    if (slot.count(pr.q)) continue;
    const int64_t sq = (int64_t)slot.size();
    slot[pr.q] = sq;
    const Box& q = BY[pr.q];
    std::vector<double> Wq(m, 0.0), Lk(m), tau(D);
    for (int64_t j = q.start; j < q.start + q.count; ++j) {
      const int64_t o = R.Y.perm[j];
      for (int d = 0; d < D; ++d) tau[d] = local_coord(R.Y.pts[o * D + d], R.alphaY[d], l, q.cell[d]);
      sparse_basis(sg, tau.data(), Lk.data());
      for (int64_t k = 0; k < m; ++k) Wq[k] += Lk[k] * b[o];
    }
    rec.src_key.push_back(q.key);
    rec.W.insert(rec.W.end(), Wq.begin(), Wq.end());
  }
  // stage 2 + 3, per target box (pairs are sorted by p)
  size_t a = 0;
  std::vector<double> np(D), nq(D), Lk(m), tau(D);
  while (a < pairs.size()) {
    size_t e = a;
    while (e < pairs.size() && pairs[e].p == pairs[a].p) ++e;
    const Box& p = BX[pairs[a].p];
    std::vector<double> U(m, 0.0);
    // stage 2 for every target box of the list (with F3M_KEEP_EMPTY that includes empty boxes,
    // whose interactions FFM(GPU) computes, reading R28); subset-target mode skips boxes without
    // an evaluated target (their locals reach no output)
    bool any_eval = prm.n_eval <= 0;
    for (int64_t i = p.start; i < p.start + p.count && !any_eval; ++i) any_eval = evaluated(prm, R.X.perm[i]);
    for (size_t r = a; r < e && any_eval; ++r) {
      const Box& q = BY[pairs[r].q];
      const double* Wq = &rec.W[slot[pairs[r].q] * m];
      for (int64_t k = 0; k < m; ++k) {
        for (int d = 0; d < D; ++d) np[d] = node_coord(R.alphaX[d], p.cell[d], l, sg.s1[sg.nodes[k][d]]);
        double acc = 0.0;
        for (int64_t j = 0; j < m; ++j) {
          for (int d = 0; d < D; ++d) nq[d] = node_coord(R.alphaY[d], q.cell[d], l, sg.s1[sg.nodes[j][d]]);
          acc += gauss(np.data(), nq.data(), D, prm.gamma) * Wq[j];
        }
        U[k] += acc;
      }
    }
    for (int64_t i = p.start; i < p.start + p.count; ++i) {
      const int64_t o = R.X.perm[i];
      if (!evaluated(prm, o)) continue;
      for (int d = 0; d < D; ++d) tau[d] = local_coord(R.X.pts[o * D + d], R.alphaX[d], l, p.cell[d]);
      sparse_basis(sg, tau.data(), Lk.data());
      double acc = 0.0;
      for (int64_t k = 0; k < m; ++k) acc += Lk[k] * U[k];
      vsorted_x[i] += acc;
    }
    rec.tgt_key.push_back(p.key);
    rec.U.insert(rec.U.end(), U.begin(), U.end());
    a = e;
  }
  R.charges.push_back(std::move(rec));
}

// exact box-pair sum (Sec. 3 Eq. (1)), sources j ascending in sorted
// order (= original order inside a box, because the permutation is stable)
void direct_pair(Result& R, const Params& prm, const Box& p, const Box& q, const double* b,
                 double* vsorted_x) {
  const int D = prm.D;
  for (int64_t i = p.start; i < p.start + p.count; ++i) {
    if (!evaluated(prm, R.X.perm[i])) continue;
    const double* x = R.X.pts + R.X.perm[i] * D;
    double acc = 0.0;
    for (int64_t j = q.start; j < q.start + q.count; ++j) {
      const int64_t o = R.Y.perm[j];
      acc += gauss(x, R.Y.pts + o * D, D, prm.gamma) * b[o];
    }
    vsorted_x[i] += acc;
  }
}

int run(const double* X, int64_t nx, const double* Y, int64_t ny, const double* b,
        const Params& prm, Result& R) {
  const int D = prm.D;
  // ---- step 1: validation
  if (D < 1 || D > 7) { g_err = "D must be in [1,7]"; return ORC_INVALID_INPUT; }
  if (nx < 1 || ny < 1) { g_err = "empty input"; return ORC_INVALID_INPUT; }
  for (int64_t i = 0; i < nx * D; ++i)
    if (!std::isfinite(X[i])) { g_err = "non-finite coordinate in X"; return ORC_INVALID_INPUT; }
  if (Y)
    for (int64_t i = 0; i < ny * D; ++i)
      if (!std::isfinite(Y[i])) { g_err = "non-finite coordinate in Y"; return ORC_INVALID_INPUT; }
  if (!(prm.gamma > 0.0) || !std::isfinite(prm.gamma)) { g_err = "gamma must be > 0"; return ORC_INVALID_SPEC; }
  if (prm.P < 2) { g_err = "P must be >= 2"; return ORC_INVALID_SPEC; }
  if (!(prm.eta > 0.0)) { g_err = "eta must be > 0"; return ORC_INVALID_SPEC; }
  if (prm.rho < 0 || prm.zeta < 1) { g_err = "rho >= 0 and zeta >= 1 required"; return ORC_INVALID_SPEC; }
  if (prm.sparse_level < 0 || prm.sparse_level > 6) { g_err = "sparse level must be in [0, 6]"; return ORC_INVALID_SPEC; }
  if (prm.sparse_level > 0) {  // |H| <= node cap
    if ((double)make_sparse_grid(D, prm.sparse_level).nodes.size() > (double)prm.node_cap) {
      g_err = "grid too large";
      return ORC_GRID_TOO_LARGE;
    }
  } else {  // P^D <= node cap (Sec. 5 "a cap at r = 2048")
    double m = 1;
    for (int d = 0; d < D; ++d) m *= prm.P;
    if (m > (double)prm.node_cap) { g_err = "grid too large"; return ORC_GRID_TOO_LARGE; }
  }
  R.D = D;
  R.aliased = (Y == nullptr);
  if (R.aliased) { Y = X; ny = nx; }
  R.v.assign(nx, 0.0);

  // ---- step 2: enclosing cube (Sec. 3 "Enclosing"), reading R14
  double E = 0.0;
  for (int d = 0; d < D; ++d) {
    double mnx = X[d], mxx = X[d], mny = Y[d], mxy = Y[d];
    for (int64_t i = 0; i < nx; ++i) { mnx = std::min(mnx, X[i * D + d]); mxx = std::max(mxx, X[i * D + d]); }
    for (int64_t i = 0; i < ny; ++i) { mny = std::min(mny, Y[i * D + d]); mxy = std::max(mxy, Y[i * D + d]); }
    R.alphaX[d] = mnx;
    R.alphaY[d] = mny;
    E = std::max(E, std::max(mxx - mnx, mxy - mny));
  }
  R.E = E;
  const int64_t nx_eval = prm.n_eval > 0 ? std::min(prm.n_eval, nx) : nx;
  if (E == 0.0 || (prm.flags & ORC_EXACT)) {  // S:271 degenerate cube / exact mode
    direct(X, nx_eval, Y, ny, D, b, prm.gamma, R.v.data());
    return ORC_OK;
  }

  // ---- step 3: level scalars (readings R3, R5), computed in this exact operation order
  const int tcap = 63 / D;
  int tstar = tcap;
  for (int t = 1; t <= tcap; ++t) {
    const double l = std::ldexp(E, -t);
    const double st = ((D * l) * l) / ((4.0 * prm.gamma) * prm.gamma);
    if (st <= prm.eta) { tstar = t; break; }
  }
  R.t_star = tstar;
  int T = std::min(tstar, tcap);
  if (prm.max_depth >= 0) T = std::min(T, prm.max_depth);
  R.T_sort = T;
  if (T < 1) {  // no division allowed: everything is near field
    direct(X, nx_eval, Y, ny, D, b, prm.gamma, R.v.data());
    return ORC_OK;
  }

  // ---- steps 4-5: keys, stable permutation, box tables
  R.X.n = nx; R.X.pts = X;
  R.Y.n = ny; R.Y.pts = Y;
  for (int d = 0; d < D; ++d) { R.X.alpha[d] = R.alphaX[d]; R.Y.alpha[d] = R.alphaY[d]; }
  build_side(R.X, D, E, T);
  build_side(R.Y, D, E, T);
  if (prm.flags & ORC_KEEP_EMPTY) {
    if ((int64_t)D * T > 24) { g_err = "keep-empty (FFM) mode needs D * T_sort <= 24"; return ORC_RESOURCE; }
    keep_empty_boxes(R.X, D, T);
    keep_empty_boxes(R.Y, D, T);
  }

  std::vector<double> vs(nx, 0.0);  // accumulated in X-sorted order, sigma applied at the end
  R.pk.assign(T + 1, {});
  R.qk.assign(T + 1, {});
  R.tag.assign(T + 1, {});

  // ---- step 6: Algorithm 1
  int t = 0;
  std::vector<Pair> near = {{0, 0}};
  auto maxbox = [&](const Side& S, bool xside) {
    int64_t mb = 0;
    for (const Pair& pr : near) mb = std::max(mb, S.lev[t][xside ? pr.p : pr.q].count);
    return mb;
  };
  while (!near.empty() && maxbox(R.X, true) > prm.zeta && maxbox(R.Y, false) > prm.zeta && t < T) {
    ++t;
    const double l = std::ldexp(E, -t);
    const double st = ((D * l) * l) / ((4.0 * prm.gamma) * prm.gamma);
    const double qt = (l * l) / ((2.0 * prm.gamma) * prm.gamma);
    int Pfar;  // adaptive far-field rule (Sec. 4.3), reading R2/R5
    if (qt <= 0.01) Pfar = std::min(prm.P, 3);
    else if (qt <= 5.0) Pfar = prm.P;
    else Pfar = 0;
    if (prm.flags & ORC_NO_ADAPTIVE) Pfar = prm.P;
    if ((prm.flags & ORC_NO_DROP) && Pfar == 0) Pfar = prm.P;
    R.pfar[t] = Pfar;
    const bool smooth_level = !(prm.flags & ORC_NO_SMOOTH) && (st <= prm.eta);
    double delta[7];
    for (int d = 0; d < D; ++d) delta[d] = R.aliased ? 0.0 : (R.alphaX[d] - R.alphaY[d]) / l;

    const std::vector<Box>& PX = R.X.lev[t - 1];
    const std::vector<Box>& PY = R.Y.lev[t - 1];
    const std::vector<Box>& CX = R.X.lev[t];
    const std::vector<Box>& CY = R.Y.lev[t];
    // active (divided) boxes: the boxes occurring in I_near (reading R9)
    {
      std::vector<char> ax(PX.size(), 0), ay(PY.size(), 0);
      for (const Pair& pr : near) { ax[pr.p] = 1; ay[pr.q] = 1; }
      for (size_t i = 0; i < PX.size(); ++i)
        if (ax[i]) { R.boxes_x[t] += PX[i].nchild; R.empty_x[t] += ((int64_t)1 << D) - PX[i].nchild; }
      for (size_t i = 0; i < PY.size(); ++i)
        if (ay[i]) { R.boxes_y[t] += PY[i].nchild; R.empty_y[t] += ((int64_t)1 << D) - PY[i].nchild; }
    }
    // divide I_near (Fig. 6): sorted by construction
    std::vector<Pair> cand;
    size_t a = 0;
    while (a < near.size()) {
      size_t e = a;
      while (e < near.size() && near[e].p == near[a].p) ++e;
      const Box& p = PX[near[a].p];
      for (int64_t pc = p.child0; pc < p.child0 + p.nchild; ++pc)
        for (size_t r = a; r < e; ++r) {
          const Box& q = PY[near[r].q];
          for (int64_t qc = q.child0; qc < q.child0 + q.nchild; ++qc) cand.push_back({pc, qc});
        }
      a = e;
    }
    R.expanded[t] = (int64_t)near.size() << (2 * D);
    R.M[t] = (int64_t)cand.size();
    // classify, precedence far > smooth > small > near (reading R11)
    std::vector<Pair> farl, smoothl, nextnear;
    for (const Pair& pr : cand) {
      const Box& p = CX[pr.p];
      const Box& q = CY[pr.q];
      double dist2 = 0.0, distmax = 0.0;
      for (int d = 0; d < D; ++d) {
        const double o = (double)(p.cell[d] - q.cell[d]) + delta[d];
        dist2 += o * o;
        distmax = std::max(distmax, std::fabs(o));
      }
      // ||c_p - c_q|| >= 2l (Sec. 3); the max-norm variant
      // does not call corner-touching boxes far at D >= 4
      const bool is_far = (prm.flags & ORC_MAXNORM) ? distmax >= 2.0 : dist2 >= 4.0;
      int tg;
      if (is_far) tg = (Pfar > 0) ? TAG_FAR : TAG_FAR_DROPPED;
      else if (smooth_level) tg = TAG_SMOOTH;                             // Sec. 4.3 O(1) bound
      else if (!(prm.flags & ORC_NO_SMALL) && p.count + q.count <= prm.rho) tg = TAG_SMALL;  // Sec. 4.2
      else tg = TAG_NEAR;
      R.pk[t].push_back(p.key);
      R.qk[t].push_back(q.key);
      R.tag[t].push_back(tg);
      switch (tg) {
        case TAG_FAR: R.m_far[t]++; farl.push_back(pr); break;
        case TAG_FAR_DROPPED: R.m_far[t]++; R.m_far_dropped[t]++; break;  // "throw away" (Alg. 1)
        case TAG_SMOOTH: R.m_smooth[t]++; smoothl.push_back(pr); break;
        case TAG_SMALL: R.m_small[t]++; direct_pair(R, prm, p, q, b, vs.data()); break;
        default: R.m_near[t]++; nextnear.push_back(pr); break;
      }
    }
    // FarFieldCompute on I_far (with P_far) and I_smooth (with P, reading R6)
    if (prm.sparse_level > 0) {  // reading R27: the grid level replaces P; "min(r, 3^D)" -> q3
      const int q = prm.sparse_level;
      const int qf = (Pfar == prm.P) ? q : (Pfar > 0 ? sparse_level_3d(D, q) : 0);
      if (qf == q) {
        std::vector<Pair> both;
        std::merge(farl.begin(), farl.end(), smoothl.begin(), smoothl.end(), std::back_inserter(both),
                   [](const Pair& u, const Pair& w) { return u.p < w.p || (u.p == w.p && u.q < w.q); });
        far_field_sparse(R, prm, t, q, both, b, vs.data());
      } else {
        far_field_sparse(R, prm, t, qf, farl, b, vs.data());
        far_field_sparse(R, prm, t, q, smoothl, b, vs.data());
      }
    } else if (Pfar == prm.P) {
      std::vector<Pair> both;  // same node count: one three-stage pass over the merged sorted list
      std::merge(farl.begin(), farl.end(), smoothl.begin(), smoothl.end(), std::back_inserter(both),
                 [](const Pair& u, const Pair& w) { return u.p < w.p || (u.p == w.p && u.q < w.q); });
      far_field(R, prm, t, prm.P, both, b, vs.data());
    } else {
      far_field(R, prm, t, Pfar, farl, b, vs.data());
      far_field(R, prm, t, prm.P, smoothl, b, vs.data());
    }
    near.swap(nextnear);
  }
  R.depth_reached = t;
  // NearFieldCompute on the remaining I_near
  R.n_near_flushed = (int64_t)near.size();
  for (const Pair& pr : near) direct_pair(R, prm, R.X.lev[t][pr.p], R.Y.lev[t][pr.q], b, vs.data());
  // ---- step 7: sigma restores the input order (Sec. 3)
  for (int64_t i = 0; i < nx; ++i) R.v[R.X.perm[i]] = vs[i];
  return ORC_OK;
}

}  // namespace

extern "C" {

const char* orc_last_error(void) { return g_err.c_str(); }

int orc_cheb_nodes(int P, double* s) {
  if (P < 2) return ORC_INVALID_SPEC;
  std::vector<double> v = cheb_nodes(P);
  std::memcpy(s, v.data(), sizeof(double) * P);
  return ORC_OK;
}

int orc_bary_weights(int P, double* w) {
  if (P < 2) return ORC_INVALID_SPEC;
  std::vector<double> v = bary_weights(P);
  std::memcpy(w, v.data(), sizeof(double) * P);
  return ORC_OK;
}

int orc_basis(int P, double t, double* L) {
  if (P < 2) return ORC_INVALID_SPEC;
  std::vector<double> s = cheb_nodes(P), w = bary_weights(P);
  bary_basis(P, s.data(), w.data(), t, L);
  return ORC_OK;
}

int orc_tensor_basis(int D, int P, const double* tau, double* out) {
  if (P < 2 || D < 1 || D > 7) return ORC_INVALID_SPEC;
  std::vector<double> s = cheb_nodes(P), w = bary_weights(P);
  tensor_basis(D, P, s.data(), w.data(), tau, out);
  return ORC_OK;
}

// Smolyak sparse grid of level q (reading R27): node count, nodes (finest-grid coordinates,
// [|H| x D] int64) and the basis Phi_h(tau) at one point ([|H|])
int64_t orc_sparse_size(int D, int q) {
  if (D < 1 || D > 7 || q < 1 || q > 6) return -1;
  return (int64_t)make_sparse_grid(D, q).nodes.size();
}
int orc_sparse_nodes(int D, int q, int64_t* out) {
  if (D < 1 || D > 7 || q < 1 || q > 6) return ORC_INVALID_SPEC;
  const SparseGrid g = make_sparse_grid(D, q);
  for (size_t i = 0; i < g.nodes.size(); ++i)
    for (int d = 0; d < D; ++d) out[i * D + d] = g.nodes[i][d];
  return ORC_OK;
}
int orc_sparse_basis(int D, int q, const double* tau, double* out) {
  if (D < 1 || D > 7 || q < 1 || q > 6) return ORC_INVALID_SPEC;
  sparse_basis(make_sparse_grid(D, q), tau, out);
  return ORC_OK;
}

// Sec. 4.2 paper box id beta = sum_d 2^{t(d-1)} c_d(t) for one point
int64_t orc_box_index(const double* x, int D, int t, double E, const double* alpha) {
  int64_t beta = 0;
  for (int d = 0; d < D; ++d) beta += cell_of(x[d], alpha[d], E, t) << (t * d);
  return beta;
}

int orc_direct(const double* X, int64_t nx, const double* Y, int64_t ny, int D, const double* b,
               double gamma, double* v) {
  if (D < 1 || D > 7 || nx < 0 || ny < 0) { g_err = "bad shape"; return ORC_INVALID_INPUT; }
  if (!(gamma > 0.0)) { g_err = "gamma must be > 0"; return ORC_INVALID_SPEC; }
  direct(X, nx, Y ? Y : X, Y ? ny : nx, D, b, gamma, v);
  return ORC_OK;
}

int orc_f3m_run(const double* X, int64_t nx, const double* Y, int64_t ny, int D, const double* b,
                double gamma, int P, double eta, int64_t rho, int64_t zeta, int max_depth,
                unsigned flags, int64_t node_cap, int64_t n_eval, int sparse_level, void** handle) {
  *handle = nullptr;
  Params prm{D, P, gamma, eta, rho, zeta, max_depth, flags, node_cap, n_eval, sparse_level};
  Result* R = new Result();
  int st;
  try {
    st = run(X, nx, Y, ny, b, prm, *R);
  } catch (const std::bad_alloc&) {
    g_err = "out of memory";
    st = ORC_RESOURCE;
  }
  if (st != ORC_OK) { delete R; return st; }
  *handle = R;
  return ORC_OK;
}

// ---- Full-size helpers (fp32 inputs converted exactly to fp64 point by point, so that a
// 1e9-point problem needs no fp64 copy).  Same arithmetic as steps 2, 4 and stage 1 above.
// Step 2: alpha[d] = min, E = max_d (max - min) of one point set.
int orc_cube_f32(const float* X, int64_t n, int D, double* alpha, double* E) {
  if (D < 1 || D > 7 || n < 1) { g_err = "bad shape"; return ORC_INVALID_INPUT; }
  double e = 0.0;
  for (int d = 0; d < D; ++d) {
    double mn = (double)X[d], mx = (double)X[d];
    for (int64_t i = 0; i < n; ++i) { mn = std::min(mn, (double)X[i * D + d]); mx = std::max(mx, (double)X[i * D + d]); }
    alpha[d] = mn;
    e = std::max(e, mx - mn);
  }
  *E = e;
  return ORC_OK;
}

// Step 4 (reading R12/R13): order key of every point at depth T (D T <= 32).
int orc_keys_f32(const float* X, int64_t n, int D, int T, double E, const double* alpha, uint32_t* key) {
  if (D < 1 || D > 7 || D * T > 32) { g_err = "keys need D*T <= 32"; return ORC_INVALID_INPUT; }
  int64_t c[7];
  for (int64_t i = 0; i < n; ++i) {
    for (int d = 0; d < D; ++d) c[d] = cell_of((double)X[i * D + d], alpha[d], E, T);
    key[i] = (uint32_t)order_key(c, D, T);
  }
  return ORC_OK;
}

// Stage 1 for ONE source box (Sec. 3 "v1 = L_Y b"): W[k] = sum over the points
// whose depth-t cell (c_d(T) >> (T - t), as in build_side) equals cell[] of b L_k(y), points in
// ascending original order (= the stable sorted order inside the box).
int orc_s2m_box_f32(const float* X, const float* b, int64_t n, int D, int P, int T, int t, double E,
                    const double* alpha, const int64_t* cell, double* W) {
  if (D < 1 || D > 7 || P < 2 || t < 1 || t > T) { g_err = "bad arguments"; return ORC_INVALID_INPUT; }
  const std::vector<double> s = cheb_nodes(P), w = bary_weights(P);
  int64_t m = 1;
  for (int d = 0; d < D; ++d) m *= P;
  const double l = std::ldexp(E, -t);
  std::vector<double> Lk(m), tau(D), y(D);
  for (int64_t k = 0; k < m; ++k) W[k] = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    bool in = true;
    for (int d = 0; d < D && in; ++d) {
      y[d] = (double)X[i * D + d];
      in = (cell_of(y[d], alpha[d], E, T) >> (T - t)) == cell[d];
    }
    if (!in) continue;
    for (int d = 0; d < D; ++d) tau[d] = local_coord(y[d], alpha[d], l, cell[d]);
    tensor_basis(D, P, s.data(), w.data(), tau.data(), Lk.data());
    for (int64_t k = 0; k < m; ++k) W[k] += Lk[k] * (double)b[i];
  }
  return ORC_OK;
}

void orc_free(void* h) { delete static_cast<Result*>(h); }

int orc_get_v(void* h, double* v) {
  Result* R = static_cast<Result*>(h);
  std::memcpy(v, R->v.data(), sizeof(double) * R->v.size());
  return ORC_OK;
}

// scalars: [E, t_star, T_sort, depth_reached, alphaX[0..6], alphaY[0..6], n_near_flushed]
int orc_get_scalars(void* h, double* out) {
  Result* R = static_cast<Result*>(h);
  out[0] = R->E; out[1] = R->t_star; out[2] = R->T_sort; out[3] = R->depth_reached;
  for (int d = 0; d < 7; ++d) { out[4 + d] = R->alphaX[d]; out[11 + d] = R->alphaY[d]; }
  out[18] = (double)R->n_near_flushed;
  return ORC_OK;
}

int64_t orc_num_points(void* h, int side) {
  Result* R = static_cast<Result*>(h);
  return side == 0 ? R->X.n : R->Y.n;
}

int orc_get_keys(void* h, int side, uint64_t* keys) {
  Result* R = static_cast<Result*>(h);
  const Side& S = side == 0 ? R->X : R->Y;
  std::memcpy(keys, S.key.data(), sizeof(uint64_t) * S.key.size());
  return ORC_OK;
}

int orc_get_perm(void* h, int side, int64_t* perm) {
  Result* R = static_cast<Result*>(h);
  const Side& S = side == 0 ? R->X : R->Y;
  std::memcpy(perm, S.perm.data(), sizeof(int64_t) * S.perm.size());
  return ORC_OK;
}

// stats[k][t] for k in {M, expanded, m_far, m_far_dropped, m_smooth, m_small, m_near,
// boxes_x, boxes_y, empty_x, empty_y, pfar}, t = 0..63  -> out[12*64]
int orc_get_stats(void* h, int64_t* out) {
  Result* R = static_cast<Result*>(h);
  const int64_t* arrs[12] = {R->M, R->expanded, R->m_far, R->m_far_dropped, R->m_smooth, R->m_small,
                             R->m_near, R->boxes_x, R->boxes_y, R->empty_x, R->empty_y, R->pfar};
  for (int k = 0; k < 12; ++k) std::memcpy(out + k * MAXLEV, arrs[k], sizeof(int64_t) * MAXLEV);
  return ORC_OK;
}

int64_t orc_num_boxes(void* h, int side, int t) {
  Result* R = static_cast<Result*>(h);
  const Side& S = side == 0 ? R->X : R->Y;
  if (t < 0 || t >= (int)S.lev.size()) return -1;
  return (int64_t)S.lev[t].size();
}

int orc_get_boxes(void* h, int side, int t, uint64_t* key, int64_t* start, int64_t* count) {
  Result* R = static_cast<Result*>(h);
  const Side& S = side == 0 ? R->X : R->Y;
  const std::vector<Box>& L = S.lev[t];
  for (size_t i = 0; i < L.size(); ++i) { key[i] = L[i].key; start[i] = L[i].start; count[i] = L[i].count; }
  return ORC_OK;
}

int64_t orc_num_pairs(void* h, int t) {
  Result* R = static_cast<Result*>(h);
  if (t < 0 || t >= (int)R->tag.size()) return 0;
  return (int64_t)R->tag[t].size();
}

int orc_get_pairs(void* h, int t, uint64_t* kp, uint64_t* kq, int32_t* tag) {
  Result* R = static_cast<Result*>(h);
  for (size_t i = 0; i < R->tag[t].size(); ++i) { kp[i] = R->pk[t][i]; kq[i] = R->qk[t][i]; tag[i] = R->tag[t][i]; }
  return ORC_OK;
}

int orc_num_charge_sets(void* h) { return (int)static_cast<Result*>(h)->charges.size(); }

// info: [t, P, nsrc, ntgt]
int orc_charge_info(void* h, int i, int64_t* info) {
  const Charges& C = static_cast<Result*>(h)->charges[i];
  info[0] = C.t; info[1] = C.P; info[2] = (int64_t)C.src_key.size(); info[3] = (int64_t)C.tgt_key.size();
  info[4] = C.m; info[5] = C.q;
  return ORC_OK;
}

int orc_get_charges(void* h, int i, uint64_t* src_key, double* W, uint64_t* tgt_key, double* U) {
  const Charges& C = static_cast<Result*>(h)->charges[i];
  std::memcpy(src_key, C.src_key.data(), sizeof(uint64_t) * C.src_key.size());
  std::memcpy(W, C.W.data(), sizeof(double) * C.W.size());
  std::memcpy(tgt_key, C.tgt_key.data(), sizeof(uint64_t) * C.tgt_key.size());
  std::memcpy(U, C.U.data(), sizeof(double) * C.U.size());
  return ORC_OK;
}

}  // extern "C"
