// Host engine + C ABI of libf3m.so (include/f3m.h).
//
// Orchestrates App. F Algorithm 1 on one B200:
//   a1 enclosing cube  -> k_bbox
//   a2-a3 keys + stable counting sort (Sec. 4.1-4.2) -> k_count / k_scan / k_scatter
//   a4 box tables per depth (empty boxes never materialised)
//   a5 interaction division + classification (Fig. 6, Sec. 3, 4.2, 4.3) -- host, exact
//      integer/fp64 decisions in the operation order of DESIGN.md "Readings"
//   a6-a8 S2M / M2L / L2T per (depth, node count) (Sec. 3, Fig. 4)
//   a9 small + final near pairs, exact (Sec. 3 Eq. (1), Sec. 4.2, Alg. 1 last line)
//   a10 sigma: v[i] = vs[sigma[i]]
// No computation of the method runs on the host except the O(boxes + pairs) tree logic.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <map>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/f3m.h"
#include "f3m_internal.h"

namespace f3m {

thread_local std::string g_err;

struct Fail {
  f3m_status st;
  std::string msg;
};

#define CK(expr)                                                                                     \
  do {                                                                                               \
    cudaError_t e__ = (expr);                                                                        \
    if (e__ != cudaSuccess)                                                                          \
      throw Fail{e__ == cudaErrorMemoryAllocation ? F3M_ERR_RESOURCE : F3M_ERR_CUDA,                 \
                 std::string(#expr) + ": " + cudaGetErrorString(e__)};                               \
  } while (0)

// ---------------------------------------------------------------------------------------
// workspace: stream-ordered device allocations released at scope exit
// ---------------------------------------------------------------------------------------
class Workspace {
 public:
  Workspace(cudaStream_t st, const f3m_allocator* a) : st_(st), alloc_(a) {
    static std::once_flag once;
    std::call_once(once, [] {
      int dev = 0;
      cudaGetDevice(&dev);
      cudaMemPool_t pool;
      if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t thr = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
      }
    });
  }
  ~Workspace() { release(); }
  void release() {
    for (void* p : ptrs_) {
      if (alloc_ && alloc_->free) alloc_->free(alloc_->ctx, p, st_);
      else cudaFreeAsync(p, st_);
    }
    ptrs_.clear();
  }
  template <class T>
  T* get(size_t count, const char* what, int depth = -1) {
    if (count == 0) count = 1;
    size_t bytes = count * sizeof(T);
    bytes = (bytes + 255) / 256 * 256;
    void* p = nullptr;
    if (alloc_ && alloc_->alloc) {
      p = alloc_->alloc(alloc_->ctx, bytes, st_);
    } else if (cudaMallocAsync(&p, bytes, st_) != cudaSuccess) {
      cudaGetLastError();
      p = nullptr;
    }
    if (!p) {
      char buf[256];
      snprintf(buf, sizeof buf, "device allocation of %zu bytes for %s failed (depth %d)", bytes, what, depth);
      throw Fail{F3M_ERR_RESOURCE, buf};
    }
    ptrs_.push_back(p);
    return static_cast<T*>(p);
  }
  template <class T>
  T* upload(const std::vector<T>& v, const char* what, int depth = -1) {
    T* d = get<T>(v.size(), what, depth);
    if (!v.empty()) CK(cudaMemcpyAsync(d, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, st_));
    return d;
  }

 private:
  cudaStream_t st_;
  const f3m_allocator* alloc_;
  std::vector<void*> ptrs_;
};

// ---------------------------------------------------------------------------------------
// configuration
// ---------------------------------------------------------------------------------------
// ---------------------------------------------------------------------------------------
// Smolyak sparse grids (Sec. 4.2 "Sparse grids"; reading R27 of DESIGN.md).
// Level-q grid in D dimensions over nested Chebyshev (Clenshaw-Curtis) levels: level 0 = {0},
// level j >= 1 = the 2^j + 1 points cos(k pi / 2^j); H = union of the tensor grids of the
// combination technique's terms |j| <= q, as coordinates on the finest 1-D grid (2^q + 1
// points), ordered by ascending linear index sum_d h_d (2^q + 1)^d.  The interpolant spans
// prod_d T_{k_d} for k in K_q = { k : k_d <= deg(j_d) for some |j| = q } (deg(0) = 0,
// deg(j) = 2^j), |K_q| = |H|, and its cardinal functions are Phi_h = sum_k A[h][k] T_k with
// A = (V^T)^-1, V[h][k] = T_k(node_h) (fp64 Gauss-Jordan on the host, once per (D, q)).
// ---------------------------------------------------------------------------------------
struct SparseGrid {
  int D = 0, q = 0, n1 = 0;
  int64_t m = 0;
  std::vector<uint8_t> nodes;   // [m][D] finest-grid coordinates of H
  std::vector<uint2> fac;       // [m] per k: 4 x u16 offsets d n1 + k_d of its factors (0: T_0 = 1)
  std::vector<double> Vinv, VinvT;
  uint8_t* d_nodes = nullptr;
  uint2* d_fac = nullptr;
  double* d_Vinv = nullptr;     // matT of W = A M   (A = Vinv^T)
  double* d_VinvT = nullptr;    // matT of Ut = A^T U
};

static void sparse_enum_levels(int D, int q, const std::function<void(const std::vector<int>&)>& fn) {
  std::vector<int> j(D, 0);
  while (true) {
    int sum = 0;
    for (int d = 0; d < D; ++d) sum += j[d];
    if (sum <= q) fn(j);
    int d = 0;
    while (d < D && ++j[d] > q) j[d++] = 0;
    if (d == D) break;
  }
}

static std::vector<std::vector<int>> sparse_node_set(int D, int q) {
  const int64_t n1 = ((int64_t)1 << q) + 1;
  std::map<int64_t, std::vector<int>> hs;
  sparse_enum_levels(D, q, [&](const std::vector<int>& j) {
    std::vector<int> k(D, 0);
    while (true) {
      std::vector<int> h(D);
      int64_t lin = 0, mul = 1;
      for (int d = 0; d < D; ++d) {
        h[d] = j[d] == 0 ? (1 << (q - 1)) : (k[d] << (q - j[d]));
        lin += h[d] * mul;
        mul *= n1;
      }
      hs[lin] = h;
      int d = 0;
      while (d < D && ++k[d] == (j[d] == 0 ? 1 : (1 << j[d]) + 1)) k[d++] = 0;
      if (d == D) break;
    }
  });
  std::vector<std::vector<int>> out;
  for (auto& kv : hs) out.push_back(kv.second);
  return out;
}

static int64_t sparse_grid_size(int D, int q) { return (int64_t)sparse_node_set(D, q).size(); }

static const SparseGrid& sparse_grid(int D, int q) {
  static std::mutex mu;
  static std::map<int, SparseGrid*> cache;
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache.find(D * 16 + q);
  if (it != cache.end()) return *it->second;
  SparseGrid* g = new SparseGrid();
  g->D = D;
  g->q = q;
  g->n1 = (1 << q) + 1;
  const std::vector<std::vector<int>> H = sparse_node_set(D, q);
  const int64_t m = (int64_t)H.size();
  g->m = m;
  std::map<std::vector<int>, int> kset;  // K_q, lexicographic
  sparse_enum_levels(D, q, [&](const std::vector<int>& j) {
    int sum = 0;
    for (int d = 0; d < D; ++d) sum += j[d];
    if (sum != q) return;
    std::vector<int> k(D, 0);
    while (true) {
      kset[k] = 0;
      int d = 0;
      while (d < D && ++k[d] > (j[d] == 0 ? 0 : (1 << j[d]))) k[d++] = 0;
      if (d == D) break;
    }
  });
  if ((int64_t)kset.size() != m) throw Fail{F3M_ERR_INTERNAL, "sparse grid: |K_q| != |H|"};
  std::vector<std::vector<int>> K;
  for (auto& kv : kset) K.push_back(kv.first);
  const double pi = 3.14159265358979323846;
  // V[h][k] = prod_d T_{k_d}(cos(h_d pi / 2^q)) = prod_d cos(k_d h_d pi / 2^q)
  std::vector<double> V((size_t)m * m), I((size_t)m * m, 0.0);
  for (int64_t h = 0; h < m; ++h)
    for (int64_t k = 0; k < m; ++k) {
      double v = 1.0;
      for (int d = 0; d < D; ++d) v *= std::cos((double)K[k][d] * (double)H[h][d] * pi / (double)(1 << q));
      V[h * m + k] = v;
    }
  for (int64_t i = 0; i < m; ++i) I[i * m + i] = 1.0;
  for (int64_t c = 0; c < m; ++c) {  // Gauss-Jordan with partial pivoting: I <- V^-1
    int64_t piv = c;
    for (int64_t r = c + 1; r < m; ++r)
      if (std::fabs(V[r * m + c]) > std::fabs(V[piv * m + c])) piv = r;
    if (std::fabs(V[piv * m + c]) < 1e-300) throw Fail{F3M_ERR_INTERNAL, "sparse grid: singular node matrix"};
    if (piv != c)
      for (int64_t k = 0; k < m; ++k) { std::swap(V[c * m + k], V[piv * m + k]); std::swap(I[c * m + k], I[piv * m + k]); }
    const double inv = 1.0 / V[c * m + c];
    for (int64_t k = 0; k < m; ++k) { V[c * m + k] *= inv; I[c * m + k] *= inv; }
    for (int64_t r = 0; r < m; ++r) {
      if (r == c) continue;
      const double f = V[r * m + c];
      if (f == 0.0) continue;
      for (int64_t k = 0; k < m; ++k) { V[r * m + k] -= f * V[c * m + k]; I[r * m + k] -= f * I[c * m + k]; }
    }
  }
  g->Vinv = I;
  g->VinvT.resize((size_t)m * m);
  for (int64_t a = 0; a < m; ++a)
    for (int64_t b = 0; b < m; ++b) g->VinvT[b * m + a] = I[a * m + b];
  g->nodes.resize((size_t)m * D);
  for (int64_t h = 0; h < m; ++h)
    for (int d = 0; d < D; ++d) g->nodes[h * D + d] = (uint8_t)H[h][d];
  g->fac.resize(m);
  for (int64_t k = 0; k < m; ++k) {
    uint32_t o[4] = {0, 0, 0, 0};
    int nf = 0;
    for (int d = 0; d < D; ++d)
      if (K[k][d] > 0) {
        if (nf >= 4) throw Fail{F3M_ERR_INTERNAL, "sparse grid: more than 4 factors"};
        o[nf++] = (uint32_t)(d * g->n1 + K[k][d]);
      }
    g->fac[k] = make_uint2(o[0] | (o[1] << 16), o[2] | (o[3] << 16));
  }
  auto up = [](const void* src, size_t bytes) {
    void* p = nullptr;
    if (cudaMalloc(&p, bytes) != cudaSuccess) throw Fail{F3M_ERR_RESOURCE, "sparse grid tables: cudaMalloc"};
    if (cudaMemcpy(p, src, bytes, cudaMemcpyHostToDevice) != cudaSuccess) throw Fail{F3M_ERR_CUDA, "sparse grid tables: cudaMemcpy"};
    return p;
  };
  g->d_nodes = (uint8_t*)up(g->nodes.data(), g->nodes.size());
  g->d_fac = (uint2*)up(g->fac.data(), sizeof(uint2) * g->fac.size());
  g->d_Vinv = (double*)up(g->Vinv.data(), sizeof(double) * g->Vinv.size());
  g->d_VinvT = (double*)up(g->VinvT.data(), sizeof(double) * g->VinvT.size());
  cache[D * 16 + q] = g;
  return *g;
}

// the level of a far group under the adaptive rule's min(r, 3^D) branch (reading R27): the
// largest level <= q whose grid has at most 3^D nodes (at least 1)
static int sparse_level_3d(int D, int q) {
  int64_t cap = 1;
  for (int d = 0; d < D; ++d) cap *= 3;
  int best = 1;
  for (int lv = 1; lv <= q; ++lv)
    if (sparse_grid_size(D, lv) <= cap) best = lv;
  return best;
}

struct Cfg {
  int D, P;
  int q = 0;  // Smolyak sparse-grid level (0: tensor grid), reading R27
  int64_t m;
  double gamma, eta;
  int64_t rho, zeta;
  int max_depth;
  uint32_t flags;
};

static Cfg resolve(int D, const f3m_kernel* k, const f3m_config* c) {
  if (D < 1 || D > 7) throw Fail{F3M_ERR_INVALID_INPUT, "D must be in [1, 7]"};
  if (!k) throw Fail{F3M_ERR_INVALID_SPEC, "kernel spec is NULL"};
  if (k->kind != F3M_KERNEL_GAUSSIAN) throw Fail{F3M_ERR_INVALID_SPEC, "only the Gaussian kernel is implemented"};
  if (!(k->lengthscale > 0.0) || !std::isfinite(k->lengthscale))
    throw Fail{F3M_ERR_INVALID_SPEC, "lengthscale must be > 0 and finite"};
  f3m_config def;
  f3m_default_config(D, &def);
  const f3m_config& cc = c ? *c : def;
  Cfg r;
  r.D = D;
  r.P = cc.nodes_per_dim;
  if (r.P < 2 || r.P > 16) throw Fail{F3M_ERR_INVALID_SPEC, "nodes_per_dim must be in [2, 16]"};
  double m = 1;
  for (int d = 0; d < D; ++d) m *= r.P;
  r.q = cc.sparse_level;
  if (r.q < 0 || r.q > 3) throw Fail{F3M_ERR_INVALID_SPEC, "sparse_level must be in [0, 3]"};
  if (r.q > 0) {  // |H| <= node cap replaces the P^D cap (reading R27)
    if ((double)sparse_grid_size(D, r.q) > (double)cc.node_cap) throw Fail{F3M_ERR_GRID_TOO_LARGE, "sparse grid exceeds node_cap"};
  } else {
    if (m > (double)cc.node_cap) throw Fail{F3M_ERR_GRID_TOO_LARGE, "P^D exceeds node_cap"};
    if (m > 4096) throw Fail{F3M_ERR_GRID_TOO_LARGE, "P^D > 4096 is not supported"};
  }
  r.m = (int64_t)m;
  r.gamma = k->lengthscale;
  r.eta = cc.eta;
  if (!(r.eta > 0.0)) throw Fail{F3M_ERR_INVALID_SPEC, "eta must be > 0"};
  r.rho = cc.rho < 0 ? 2 * r.m : cc.rho;
  r.zeta = cc.zeta < 1 ? r.m : cc.zeta;
  r.max_depth = cc.max_depth;
  r.flags = cc.flags;
  return r;
}

// ---------------------------------------------------------------------------------------
// host tree structures
// ---------------------------------------------------------------------------------------
struct HBox {
  uint64_t key;
  int64_t start, count;  // local sorted interval
  int64_t gcount;        // global count (== count unless sharded)
  int64_t cell[F3M_MAXD];
  int64_t child0, nchild;
};

struct Side {
  const float* X = nullptr;  // device row-major
  const float* b = nullptr;  // device weights (source side) or null
  int64_t n = 0;
  double alpha[F3M_MAXD] = {0};
  float mn[F3M_MAXD] = {0}, mx[F3M_MAXD] = {0};
  // sorted data
  float* xs = nullptr;
  float* bs = nullptr;
  int32_t* perm = nullptr;
  int32_t* sigma = nullptr;
  uint64_t* keys = nullptr;  // sorted keys (multi-pass or debug)
  // counting-sort state (single pass: scatter deferred to the tile-local kernel)
  KeyParams kp{};
  int bits = 0;
  uint32_t* offsets = nullptr;
  uint32_t* scan_tmp = nullptr;
  uint16_t* lrank = nullptr;   // tile-local order of the first pass (single-pass sorts)
  bool lrank_sorted = false;   // true: sorted form (k_s2m_tma), false: rank form (k_local_s2m)
  int64_t tiles = 0;
  bool deferred = false, with_b = false, want_sigma = false, keep_keys = false;
  std::vector<uint64_t> leaf_key;
  std::vector<int64_t> leaf_start, leaf_count, leaf_gcount;
  std::vector<std::vector<HBox>> lev;
  std::map<int, float*> thr_dev;  // exact cell thresholds per depth (device)
  // multi-pass LSD sorts: every pass's scanned counts, tile orders and digit width (the
  // passes are undone in reverse to bring per-point results back to the input order)
  std::vector<uint32_t*> lsd_counts;
  std::vector<uint16_t*> lsd_order;
  std::vector<int> lsd_bits;
};

static void decode_cells(uint64_t prefix, int D, int t, int64_t* cell) {
  for (int d = 0; d < F3M_MAXD; ++d) cell[d] = 0;
  for (int s = 0; s < t; ++s) {  // s = bit position within each cell coordinate
    const uint64_t grp = (prefix >> (D * s)) & ((1ull << D) - 1ull);
    for (int d = 0; d < D; ++d) cell[d] |= (int64_t)((grp >> d) & 1ull) << s;
  }
}

static void keep_empty_levels(Side& S, int D, int T);

static void build_levels(Side& S, int D, int T, bool keep_empty = false) {
  if (keep_empty) {
    build_levels(S, D, T, false);
    keep_empty_levels(S, D, T);
    return;
  }
  S.lev.assign(T + 1, {});
  for (int t = 0; t <= T; ++t) {
    const int sh = D * (T - t);
    std::vector<HBox>& L = S.lev[t];
    for (size_t i = 0; i < S.leaf_key.size(); ++i) {
      const uint64_t pre = sh >= 64 ? 0ull : (S.leaf_key[i] >> sh);
      if (L.empty() || L.back().key != pre) {
        HBox b{};
        b.key = pre;
        b.start = S.leaf_start[i];
        b.count = 0;
        b.gcount = 0;
        decode_cells(pre, D, t, b.cell);
        L.push_back(b);
      }
      L.back().count += S.leaf_count[i];
      L.back().gcount += S.leaf_gcount[i];
    }
  }
  for (int t = 0; t < T; ++t) {
    std::vector<HBox>& Pv = S.lev[t];
    const std::vector<HBox>& Cv = S.lev[t + 1];
    int64_t j = 0;
    for (size_t p = 0; p < Pv.size(); ++p) {
      Pv[p].child0 = j;
      while (j < (int64_t)Cv.size() && (Cv[j].key >> D) == Pv[p].key) ++j;
      Pv[p].nchild = j - Pv[p].child0;
    }
  }
}

// F3M_KEEP_EMPTY (the FFM(GPU) ablation of Tables 5-6; Fig. 5,
// PAPER.md:183-189): no empty-box removal -- every depth holds all 2^{D t} cells in key order
// (empty ones with count 0) and a divided box has all 2^D children.  pi is unchanged; the empty
// boxes only add zero-valued interactions (work and memory, not a different result).
static void keep_empty_levels(Side& S, int D, int T) {
  for (int t = 0; t <= T; ++t) {
    const std::vector<HBox> L0 = S.lev[t];
    const int64_t nb = 1ll << (D * t);
    std::vector<HBox> L(nb);
    size_t j = 0;
    int64_t pos = 0;
    for (int64_t k = 0; k < nb; ++k) {
      HBox& b = L[k];
      b.key = (uint64_t)k;
      if (j < L0.size() && L0[j].key == (uint64_t)k) {
        b.start = L0[j].start;
        b.count = L0[j].count;
        b.gcount = L0[j].gcount;
        pos = b.start + b.count;
        ++j;
      } else {
        b.start = pos;
        b.count = 0;
        b.gcount = 0;
      }
      decode_cells((uint64_t)k, D, t, b.cell);
      b.child0 = k << D;
      b.nchild = t < T ? (1ll << D) : 0;
    }
    S.lev[t].swap(L);
  }
}

struct Pair { int64_t p, q; };

struct FarGroup {
  int t, P;        // P: nodes per dimension (tensor grid) or 2^q + 1 (sparse grid of level q)
  int q = 0;       // sparse-grid level, 0 = tensor grid
  int64_t m;
  std::vector<int64_t> src;       // Y box indices (level t), ascending = W slots
  std::vector<int64_t> tgt;       // X box indices (level t), ascending = U slots
  std::vector<int32_t> ptr;       // CSR over tgt
  std::vector<int32_t> col;       // W slot
  std::vector<uint64_t> off;      // packed per-dimension table index
  double delta0[F3M_MAXD];
  int32_t range[F3M_MAXD];
  // device-built lists (run_alg1 device levels): ptr/col/off live in the workspace instead
  int32_t* d_ptr = nullptr;
  int32_t* d_col = nullptr;
  uint64_t* d_off = nullptr;
  // complete-level group classified by counting (grid_level_shortcut): no pair list, ptr = {0, n};
  // its M2L runs as mode products (grid_m2l_plan), never pairwise
  bool grid_only = false;
};

struct NearGroup {
  int t;
  std::vector<int64_t> tgt;       // X box indices at level t
  std::vector<int32_t> ptr;
  std::vector<int64_t> src;       // Y box indices at level t
};

struct Plan {
  Cfg cfg;
  Workspace* ws = nullptr;
  bool aliased = true;
  double E = 0.0;
  int t_star = 0, T = 0, passes = 0, depth_reached = 0;
  Side X, Y;
  // sharded flow: the near / small field reads its sources from the replicated
  // full source set Yn (every rank's points, sorted with the global cube), not the local slice
  Side Yn;
  bool near_from_full = false;
  std::vector<FarGroup> far;
  std::vector<NearGroup> near;
  f3m_stats stats{};
  bool sharded = false;
};

// level scalars in the operation order of the oracle reading (R3, R5)
static inline double level_edge(double E, int t) { return std::ldexp(E, -t); }
static inline double smooth_bound(int D, double l, double g) { return ((D * l) * l) / ((4.0 * g) * g); }
static inline double adapt_q(double l, double g) { return (l * l) / ((2.0 * g) * g); }

static void level_scalars(Plan& pl) {
  const Cfg& c = pl.cfg;
  const int tcap = 63 / c.D;
  int ts = tcap;
  for (int t = 1; t <= tcap; ++t) {
    if (smooth_bound(c.D, level_edge(pl.E, t), c.gamma) <= c.eta) { ts = t; break; }
  }
  pl.t_star = ts;
  int T = std::min(ts, tcap);
  if (c.max_depth >= 0) T = std::min(T, c.max_depth);
  pl.T = T;
}

// ---------------------------------------------------------------------------------------
// debug / introspection state of the last call (parity tests); guarded by g_dbg_mu
// ---------------------------------------------------------------------------------------
struct DebugCharges {
  int t, P;
  int64_t m = 0;
  int q = 0;
  std::vector<uint64_t> sk, tk;
  std::vector<double> W, U;
};
struct DebugState {
  bool on = false;
  int level = 0;  // 1: everything; 2 (full-size tests): pairs, charges and pi of X as int32
  std::vector<int32_t> perm32;
  std::vector<std::vector<uint64_t>> kp, kq;
  std::vector<std::vector<int32_t>> tag;
  std::vector<int64_t> perm[2];
  std::vector<uint64_t> keys[2];
  std::vector<DebugCharges> charges;
  void reset() {
    kp.assign(F3M_MAX_LEVELS, {});
    kq.assign(F3M_MAX_LEVELS, {});
    tag.assign(F3M_MAX_LEVELS, {});
    perm[0].clear(); perm[1].clear(); keys[0].clear(); keys[1].clear();
    perm32.clear();
    charges.clear();
  }
};
static DebugState g_dbg;
static std::mutex g_dbg_mu;
static inline bool debug_pairs_enabled() { return g_dbg.on; }
static inline void debug_record_pair(int t, uint64_t a, uint64_t b, int tag) {
  g_dbg.kp[t].push_back(a);
  g_dbg.kq[t].push_back(b);
  g_dbg.tag[t].push_back(tag);
}

// Algorithm 1 loop on the host box tables
extern thread_local int64_t g_launches;

// Far-group record of one depth from its pair list (host lists): W slots = source boxes
// ascending, CSR over target boxes, packed per-dimension offset indices (M2L tables).
static void finish_far_group_host(Plan& pl, int t, FarGroup& g, std::vector<Pair>& prs) {
  if (prs.empty()) return;
  const int D = pl.cfg.D;
  const double l = level_edge(pl.E, t);
  const std::vector<HBox>& CX = pl.X.lev[t];
  const std::vector<HBox>& CY = pl.Y.lev[t];
  g.m = 1;
  for (int d = 0; d < D; ++d) g.m *= g.P;
  std::vector<int64_t> qs;
  qs.reserve(prs.size());
  for (const Pair& pr : prs) qs.push_back(pr.q);
  std::sort(qs.begin(), qs.end());
  qs.erase(std::unique(qs.begin(), qs.end()), qs.end());
  g.src = qs;
  int64_t omin[F3M_MAXD], omax[F3M_MAXD];
  for (int d = 0; d < D; ++d) { omin[d] = INT64_MAX; omax[d] = INT64_MIN; }
  for (const Pair& pr : prs)
    for (int d = 0; d < D; ++d) {
      const int64_t o = CX[pr.p].cell[d] - CY[pr.q].cell[d];
      omin[d] = std::min(omin[d], o);
      omax[d] = std::max(omax[d], o);
    }
  for (int d = 0; d < D; ++d) {
    if (omax[d] - omin[d] + 1 > 255) throw Fail{F3M_ERR_INTERNAL, "box offset range exceeds 255"};
    g.range[d] = (int32_t)(omax[d] - omin[d] + 1);
    g.delta0[d] = (pl.X.alpha[d] - pl.Y.alpha[d]) + (double)omin[d] * l;
  }
  size_t i = 0;
  g.ptr.push_back(0);
  while (i < prs.size()) {
    size_t j = i;
    while (j < prs.size() && prs[j].p == prs[i].p) ++j;
    g.tgt.push_back(prs[i].p);
    for (size_t r = i; r < j; ++r) {
      const int64_t slot = std::lower_bound(g.src.begin(), g.src.end(), prs[r].q) - g.src.begin();
      g.col.push_back((int32_t)slot);
      uint64_t pk = 0;
      for (int d = 0; d < D; ++d) pk |= (uint64_t)(CX[prs[r].p].cell[d] - CY[prs[r].q].cell[d] - omin[d]) << (8 * d);
      g.off.push_back(pk);
    }
    g.ptr.push_back((int32_t)g.col.size());
    i = j;
  }
  pl.far.push_back(std::move(g));
}

static void push_near_group(Plan& pl, int t, const std::vector<Pair>& prs) {
  if (prs.empty()) return;
  NearGroup ng;
  ng.t = t;
  ng.ptr.push_back(0);
  size_t i = 0;
  while (i < prs.size()) {
    size_t j = i;
    while (j < prs.size() && prs[j].p == prs[i].p) ++j;
    ng.tgt.push_back(prs[i].p);
    for (size_t r = i; r < j; ++r) ng.src.push_back(prs[r].q);
    ng.ptr.push_back((int32_t)ng.src.size());
    i = j;
  }
  pl.near.push_back(std::move(ng));
}

struct LevelCtx {  // the depth-t scalars of the Alg. 1 loop body
  int t, pfar;
  bool smooth_level, split;
  double l;
  double delta[F3M_MAXD];
};

// Host division + classification of one depth (small trees): the reference order of Fig. 6.
static void level_host(Plan& pl, const LevelCtx& L, const std::vector<Pair>& nearl, std::vector<Pair>& nextnear) {
  const Cfg& c = pl.cfg;
  const int D = c.D, t = L.t;
  f3m_stats& st = pl.stats;
  const std::vector<HBox>& PX = pl.X.lev[t - 1];
  const std::vector<HBox>& PY = pl.Y.lev[t - 1];
  const std::vector<HBox>& CX = pl.X.lev[t];
  const std::vector<HBox>& CY = pl.Y.lev[t];
  FarGroup g0, g1;
  g0.t = g1.t = t;
  g0.P = L.split ? L.pfar : c.P;
  g1.P = c.P;
  std::vector<Pair> fp0, fp1, smallp;
  int64_t M = 0;
  size_t a = 0;
  while (a < nearl.size()) {  // divide I_near, sorted by construction (Fig. 6)
    size_t e = a;
    while (e < nearl.size() && nearl[e].p == nearl[a].p) ++e;
    const HBox& pb = PX[nearl[a].p];
    for (int64_t pc = pb.child0; pc < pb.child0 + pb.nchild; ++pc) {
      const HBox& bp = CX[pc];
      for (size_t r = a; r < e; ++r) {
        const HBox& qb = PY[nearl[r].q];
        for (int64_t qc = qb.child0; qc < qb.child0 + qb.nchild; ++qc) {
          const HBox& bq = CY[qc];
          ++M;
          double dist2 = 0.0, distmax = 0.0;
          for (int d = 0; d < D; ++d) {
            const double o = (double)(bp.cell[d] - bq.cell[d]) + L.delta[d];
            dist2 += o * o;
            distmax = std::max(distmax, std::fabs(o));
          }
          const bool is_far = (c.flags & F3M_ADMISSIBLE_MAXNORM) ? distmax >= 2.0 : dist2 >= 4.0;
          int tag;
          if (is_far) tag = L.pfar > 0 ? 1 : 2;
          else if (L.smooth_level) tag = 3;
          else if (!(c.flags & F3M_NO_SMALL) && bp.gcount + bq.gcount <= c.rho) tag = 4;
          else tag = 0;
          switch (tag) {
            case 1: st.m_far[t]++; fp0.push_back({pc, qc}); break;
            case 2: st.m_far[t]++; st.m_far_dropped[t]++; break;
            case 3: st.m_smooth[t]++; (L.split ? fp1 : fp0).push_back({pc, qc}); break;
            case 4: st.m_small[t]++; smallp.push_back({pc, qc}); break;
            default: st.m_near[t]++; nextnear.push_back({pc, qc}); break;
          }
          if (debug_pairs_enabled()) debug_record_pair(t, bp.key, bq.key, tag);
        }
      }
    }
    a = e;
  }
  st.M[t] = M;
  finish_far_group_host(pl, t, g0, fp0);
  if (L.split) finish_far_group_host(pl, t, g1, fp1);
  push_near_group(pl, t, smallp);
}

// Device tables of one depth for the division kernels (int32 cells, int64 global counts,
// first-child indices into the next depth).
struct DevLevel {
  int32_t* child0 = nullptr;
  int32_t* cell = nullptr;
  int64_t* g = nullptr;
  int64_t n = 0;
};
static DevLevel upload_level(const std::vector<HBox>& L, Workspace& ws, cudaStream_t st, int t) {
  DevLevel d;
  d.n = (int64_t)L.size();
  std::vector<int32_t> c0(L.size()), cell(L.size() * F3M_MAXD, 0);
  std::vector<int64_t> g(L.size());
  for (size_t i = 0; i < L.size(); ++i) {
    c0[i] = (int32_t)L[i].child0;
    for (int k = 0; k < F3M_MAXD; ++k) cell[i * F3M_MAXD + k] = (int32_t)L[i].cell[k];
    g[i] = L[i].gcount;
  }
  d.child0 = ws.upload(c0, "tree children", t);
  d.cell = ws.upload(cell, "tree cells", t);
  d.g = ws.upload(g, "tree counts", t);
  (void)st;
  return d;
}

template <class T>
static std::vector<T> download(const T* d, size_t n, cudaStream_t st) {
  std::vector<T> h(n);
  if (n) CK(cudaMemcpyAsync(h.data(), d, n * sizeof(T), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  return h;
}

// far group from a device pair list (sorted by target): marks and offset ranges on the
// device, O(boxes) bookkeeping on the host, col / off written by a second device pass.
static void finish_far_group_device(Plan& pl, int t, FarGroup& g, int32_t* dP, int32_t* dQ, int64_t n,
                                    const DevLevel& LX, const DevLevel& LY, Workspace& ws, cudaStream_t st) {
  if (n <= 0) return;
  const int D = pl.cfg.D;
  const double l = level_edge(pl.E, t);
  g.m = 1;
  for (int d = 0; d < D; ++d) g.m *= g.P;
  uint32_t* tcount = ws.get<uint32_t>((size_t)LX.n, "far target counts", t);
  uint32_t* smark = ws.get<uint32_t>((size_t)LY.n, "far source marks", t);
  int* om = ws.get<int>(2 * F3M_MAXD, "far offset range", t);
  CK(cudaMemsetAsync(tcount, 0xff, sizeof(uint32_t) * LX.n, st));  // run starts (UINT32_MAX: no pairs)
  CK(cudaMemsetAsync(smark, 0, sizeof(uint32_t) * LY.n, st));
  std::vector<int> init(2 * F3M_MAXD);
  for (int d = 0; d < F3M_MAXD; ++d) { init[d] = INT32_MAX; init[F3M_MAXD + d] = INT32_MIN; }
  CK(cudaMemcpyAsync(om, init.data(), sizeof(int) * init.size(), cudaMemcpyHostToDevice, st));
  launch_far_marks(dP, dQ, n, LX.cell, LY.cell, D, tcount, smark, om, om + F3M_MAXD, st);
  g_launches += 1;
  std::vector<uint32_t> tc = download(tcount, (size_t)LX.n, st);
  std::vector<uint32_t> sm = download(smark, (size_t)LY.n, st);
  std::vector<int> omm = download(om, 2 * F3M_MAXD, st);
  std::vector<uint32_t> sslot(LY.n);
  uint32_t ns = 0;
  for (int64_t q = 0; q < LY.n; ++q) {
    sslot[q] = ns;
    if (sm[q]) { g.src.push_back(q); ++ns; }
  }
  for (int64_t p = 0; p < LX.n; ++p)
    if (tc[p] != UINT32_MAX) {
      g.tgt.push_back(p);
      g.ptr.push_back((int32_t)tc[p]);  // the list is sorted by target: starts ascend with p
    }
  g.ptr.push_back((int32_t)n);
  for (int d = 0; d < D; ++d) {
    if ((int64_t)omm[F3M_MAXD + d] - omm[d] + 1 > 255) throw Fail{F3M_ERR_INTERNAL, "box offset range exceeds 255"};
    g.range[d] = omm[F3M_MAXD + d] - omm[d] + 1;
    g.delta0[d] = (pl.X.alpha[d] - pl.Y.alpha[d]) + (double)omm[d] * l;
  }
  uint32_t* dslot = ws.upload(sslot, "far source slots", t);
  g.d_col = ws.get<int32_t>((size_t)n, "m2l cols", t);
  g.d_off = ws.get<uint64_t>((size_t)n, "m2l offsets", t);
  launch_far_cols(dP, dQ, n, LX.cell, LY.cell, D, dslot, om, g.d_col, g.d_off, st);
  g_launches += 1;
  g.d_ptr = ws.upload(g.ptr, "m2l csr", t);
  pl.far.push_back(std::move(g));
}

// Device division + classification of one depth (large trees).  Same order, tags and
// lists as level_host (tests compare both against the oracle).
static void level_device(Plan& pl, const LevelCtx& L, const std::vector<Pair>& nearl, std::vector<Pair>& nextnear,
                         cudaStream_t st) {
  const Cfg& c = pl.cfg;
  const int D = c.D, t = L.t;
  Workspace& ws = *pl.ws;
  f3m_stats& stt = pl.stats;
  const std::vector<HBox>& PX = pl.X.lev[t - 1];
  const std::vector<HBox>& PY = pl.Y.lev[t - 1];
  // runs of the near list (one per parent target box)
  std::vector<uint64_t> run_base;
  std::vector<int32_t> run_p, run_r0, pair_q;
  std::vector<uint32_t> run_Q, pair_S;
  uint64_t M = 0;
  size_t a = 0;
  while (a < nearl.size()) {
    size_t e = a;
    while (e < nearl.size() && nearl[e].p == nearl[a].p) ++e;
    uint64_t Q = 0;
    for (size_t r = a; r < e; ++r) {
      pair_q.push_back((int32_t)nearl[r].q);
      pair_S.push_back((uint32_t)Q);
      Q += (uint64_t)PY[nearl[r].q].nchild;
    }
    if (Q > UINT32_MAX) throw Fail{F3M_ERR_RESOURCE, "interaction run too large"};
    run_base.push_back(M);
    run_p.push_back((int32_t)nearl[a].p);
    run_r0.push_back((int32_t)a);
    run_Q.push_back((uint32_t)Q);
    M += (uint64_t)PX[nearl[a].p].nchild * Q;
    a = e;
  }
  run_r0.push_back((int32_t)nearl.size());
  stt.M[t] = (int64_t)M;
  if (M == 0) return;
  if (M >= (1ull << 32)) {
    char buf[128];
    snprintf(buf, sizeof buf, "%llu candidate pairs at depth %d exceed 2^32", (unsigned long long)M, t);
    throw Fail{F3M_ERR_RESOURCE, buf};
  }
  DevLevel PXd, PYd, CXd, CYd;
  PXd = upload_level(PX, ws, st, t - 1);
  CXd = upload_level(pl.X.lev[t], ws, st, t);
  if (pl.aliased) { PYd = PXd; CYd = CXd; }
  else { PYd = upload_level(PY, ws, st, t - 1); CYd = upload_level(pl.Y.lev[t], ws, st, t); }
  DivArgs A{};
  A.D = D;
  A.M = M;
  A.nruns = (int)run_p.size();
  A.run_base = ws.upload(run_base, "division runs", t);
  A.run_p = ws.upload(run_p, "division runs", t);
  A.run_Q = ws.upload(run_Q, "division runs", t);
  A.run_r0 = ws.upload(run_r0, "division runs", t);
  A.pair_q = ws.upload(pair_q, "division pairs", t);
  A.pair_S = ws.upload(pair_S, "division pairs", t);
  A.childX0 = PXd.child0;
  A.childY0 = PYd.child0;
  A.cellX = CXd.cell;
  A.cellY = CYd.cell;
  A.gX = CXd.g;
  A.gY = CYd.g;
  for (int d = 0; d < F3M_MAXD; ++d) A.delta[d] = d < D ? L.delta[d] : 0.0;
  A.pfar = L.pfar;
  A.smooth_level = L.smooth_level ? 1 : 0;
  A.no_small = (c.flags & F3M_NO_SMALL) ? 1 : 0;
  A.maxnorm = (c.flags & F3M_ADMISSIBLE_MAXNORM) ? 1 : 0;
  A.rho = c.rho;
  const int64_t nblk = divide_blocks(M);
  A.blockcnt = ws.get<uint32_t>((size_t)nblk * DIV_NCLS, "division counts", t);
  const bool dbg = debug_pairs_enabled();
  if (dbg) {
    A.dbg_pc = ws.get<int32_t>(M, "debug pairs", t);
    A.dbg_qc = ws.get<int32_t>(M, "debug pairs", t);
    A.dbg_tag = ws.get<int8_t>(M, "debug pairs", t);
  }
  launch_divide(A, false, st);
  g_launches += 1;
  std::vector<uint32_t> bc = download(A.blockcnt, (size_t)nblk * DIV_NCLS, st);
  if (dbg) {
    std::vector<int32_t> pc = download(A.dbg_pc, M, st), qc = download(A.dbg_qc, M, st);
    std::vector<int8_t> tg = download(A.dbg_tag, M, st);
    static const int tag_of[DIV_NCLS] = {1, 3, 4, 0, 2};
    for (uint64_t i = 0; i < M; ++i)
      debug_record_pair(t, pl.X.lev[t][pc[i]].key, pl.Y.lev[t][qc[i]].key, tag_of[tg[i]]);
  }
  // lists: 0 = far (and smooth at the same node count), 1 = smooth (split), 2 = small, 3 = near
  int cls_list[DIV_NCLS] = {0, L.split ? 1 : 0, 2, 3, -1};
  int cls_merge[DIV_NCLS] = {L.split ? -1 : DIV_SMOOTH, L.split ? -1 : DIV_FAR, -1, -1, -1};
  std::vector<uint32_t> boff((size_t)nblk * DIV_NCLS);
  uint64_t ltot[4] = {0, 0, 0, 0}, ctot[DIV_NCLS] = {0, 0, 0, 0, 0};
  for (int64_t b = 0; b < nblk; ++b) {
    for (int k = 0; k < DIV_NCLS; ++k) {
      const int li = cls_list[k];
      boff[b * DIV_NCLS + k] = li >= 0 ? (uint32_t)ltot[li] : 0u;
    }
    for (int k = 0; k < DIV_NCLS; ++k) {
      ctot[k] += bc[b * DIV_NCLS + k];
      if (cls_list[k] >= 0) ltot[cls_list[k]] += bc[b * DIV_NCLS + k];
    }
  }
  stt.m_far[t] += (int64_t)(ctot[DIV_FAR] + ctot[DIV_DROP]);
  stt.m_far_dropped[t] += (int64_t)ctot[DIV_DROP];
  stt.m_smooth[t] += (int64_t)ctot[DIV_SMOOTH];
  stt.m_small[t] += (int64_t)ctot[DIV_SMALL];
  stt.m_near[t] += (int64_t)ctot[DIV_NEAR];
  A.blockoff = ws.upload(boff, "division offsets", t);
  for (int k = 0; k < DIV_NCLS; ++k) { A.cls_list[k] = cls_list[k]; A.cls_merge[k] = cls_merge[k]; }
  for (int li = 0; li < 4; ++li) {
    A.outP[li] = ws.get<int32_t>((size_t)ltot[li], "division lists", t);
    A.outQ[li] = ws.get<int32_t>((size_t)ltot[li], "division lists", t);
  }
  A.dbg_pc = nullptr;
  A.dbg_qc = nullptr;
  A.dbg_tag = nullptr;
  launch_divide(A, true, st);
  g_launches += 1;
  FarGroup g0, g1;
  g0.t = g1.t = t;
  g0.P = L.split ? L.pfar : c.P;
  g1.P = c.P;
  finish_far_group_device(pl, t, g0, A.outP[0], A.outQ[0], (int64_t)ltot[0], CXd, CYd, ws, st);
  if (L.split) finish_far_group_device(pl, t, g1, A.outP[1], A.outQ[1], (int64_t)ltot[1], CXd, CYd, ws, st);
  auto host_pairs = [&](int li) {
    std::vector<int32_t> P = download(A.outP[li], (size_t)ltot[li], st), Q = download(A.outQ[li], (size_t)ltot[li], st);
    std::vector<Pair> v(P.size());
    for (size_t i = 0; i < P.size(); ++i) v[i] = {P[i], Q[i]};
    return v;
  };
  push_near_group(pl, t, host_pairs(2));
  nextnear = host_pairs(3);
}

// Sparse grids (reading R27): the groups built with P' in {min(P, 3), P} get the level q (P' =
// P) or the largest level with at most 3^D nodes (P' < P, the adaptive rule's min(r, 3^D))
static void apply_sparse(Plan& pl) {
  const int q = pl.cfg.q;
  if (q <= 0) return;
  for (FarGroup& g : pl.far) {
    g.q = g.P == pl.cfg.P ? q : sparse_level_3d(pl.cfg.D, q);
    g.P = (1 << g.q) + 1;
    g.m = sparse_grid(pl.cfg.D, g.q).m;
  }
}

// ---------------------------------------------------------------------------------------
// Complete levels (reading R29).  On a complete grid with X = Y the near pairs of
// depth t - 1 are exactly the parent offsets o in {-1,0,1}^D with <= 3 non-zero entries
// (Euclidean dist^2 < 4 on integer offsets) or all of {-1,0,1}^D (max norm) -- when every such
// pair is present, which the count decides.
static double admitted_parent_pairs(int D, int t, bool maxnorm) {
  const double Gp = std::ldexp(1.0, t - 1);
  if (maxnorm) return std::pow(3.0 * Gp - 2.0, D);
  double npar = 0.0, binom = 1.0;
  for (int k = 0; k <= std::min(3, D); ++k) {
    npar += binom * std::pow(2.0 * (Gp - 1.0), k) * std::pow(Gp, D - k);
    binom = binom * (D - k) / (k + 1);
  }
  return npar;
}

// the mode-product M2L of a complete level: N = 2^t P per dimension, ndeg degrees; taken when it
// needs fewer FMAs than the pairwise separable M2L of its `pairs` and fits in memory (D >= 4:
// the D = 3 paths keep their pairwise M2L, which is < 1 ms at every BASELINE config)
static bool grid_m2l_worth(int D, int t, int P, double pairs, bool maxnorm, int* N_out, int* ndeg_out,
                           int64_t* total_out, int64_t* fma_out) {
  if (D < 4 || getenv("F3M_NO_GRID_M2L")) return false;
  const int N = (1 << t) * P;
  const int ndeg = maxnorm ? 1 : std::min(3, D) + 1;
  double total = 1.0;
  for (int d = 0; d < D; ++d) total *= N;
  const double fma = (double)D * ndeg * total * 2.0 * N;
  double mP = 1.0;
  for (int d = 0; d <= D; ++d) mP *= P;
  if (2.0 * 8.0 * ndeg * total > 4.0e9 || fma > pairs * D * mP) return false;
  if (N_out) *N_out = N;
  if (ndeg_out) *ndeg_out = ndeg;
  if (total_out) *total_out = (int64_t)total;
  if (fma_out) *fma_out = (int64_t)fma;
  return true;
}

// Alg. 1 at the smooth level t* on a complete grid: every child pair of a near pair is far or
// smooth (adaptive P_far == P, nothing dropped), so the level's pairs form one far group of every
// admitted child pair.  When its M2L will run as mode products the pair list is never needed:
// the counters of Thm. 2 come from counting (far: child offset dist^2 >= 4, resp. max |c| >= 2,
// with c_d = 2 o_d + (b_p - b_q) over the child bits) and the group carries no list.
static bool grid_level_shortcut(Plan& pl, const LevelCtx& L, const std::vector<Pair>& nearl) {
  const Cfg& c = pl.cfg;
  const int D = c.D, t = L.t;
  if (D < 4 || !pl.aliased || c.q > 0 || !L.smooth_level || L.split || L.pfar <= 0 || debug_pairs_enabled())
    return false;
  if (D * t > 24) return false;
  const int64_t nbox = 1ll << (D * t);
  if ((int64_t)pl.X.lev[t].size() != nbox || (int64_t)pl.X.lev[t - 1].size() != (nbox >> D)) return false;
  const bool maxnorm = (c.flags & F3M_ADMISSIBLE_MAXNORM) != 0;
  const double npar = admitted_parent_pairs(D, t, maxnorm);
  if ((double)nearl.size() != npar) return false;
  const double total = npar * std::ldexp(1.0, 2 * D);
  if (total >= 2147483647.0 || !grid_m2l_worth(D, t, c.P, total, maxnorm, nullptr, nullptr, nullptr, nullptr))
    return false;
  // far child pairs: DP over the dimensions of (non-zero parent offsets so far, capped child
  // distance statistic) with the parent-pair multiplicity prod_d (Gp - |o_d|) and the child-bit
  // multiplicity (1, 2, 1 for c_d = 2 o_d - 1, 2 o_d, 2 o_d + 1)
  const int64_t Gp = 1ll << (t - 1);
  const int NZ = maxnorm ? D + 1 : 4, SC = maxnorm ? 3 : 5;  // stat: sum c^2 capped at 4, or max |c| capped at 2
  std::vector<int64_t> cur((size_t)NZ * SC, 0), nxt;
  cur[0] = 1;
  for (int d = 0; d < D; ++d) {
    nxt.assign(cur.size(), 0);
    for (int nz = 0; nz < NZ; ++nz)
      for (int sc = 0; sc < SC; ++sc) {
        const int64_t wgt = cur[(size_t)nz * SC + sc];
        if (!wgt) continue;
        for (int o = -1; o <= 1; ++o) {
          const int64_t pm = Gp - (o < 0 ? -o : o);
          const int nz2 = nz + (o != 0);
          if (pm <= 0 || nz2 >= NZ) continue;
          for (int db = -1; db <= 1; ++db) {
            const int cc = 2 * o + db, cm = db == 0 ? 2 : 1;
            const int sc2 = maxnorm ? std::min(2, std::max(sc, cc < 0 ? -cc : cc)) : std::min(4, sc + cc * cc);
            nxt[(size_t)nz2 * SC + sc2] += wgt * pm * cm;
          }
        }
      }
    cur.swap(nxt);
  }
  int64_t far = 0, all = 0;
  for (int nz = 0; nz < NZ; ++nz)
    for (int sc = 0; sc < SC; ++sc) {
      all += cur[(size_t)nz * SC + sc];
      if (sc >= (maxnorm ? 2 : 4)) far += cur[(size_t)nz * SC + sc];
    }
  if ((double)all != total) return false;
  f3m_stats& st = pl.stats;
  st.M[t] = all;
  st.m_far[t] += far;
  st.m_smooth[t] += all - far;
  FarGroup g;
  g.t = t;
  g.P = c.P;
  g.m = 1;
  for (int d = 0; d < D; ++d) g.m *= c.P;
  g.src.resize(nbox);
  g.tgt.resize(nbox);
  for (int64_t i = 0; i < nbox; ++i) g.src[i] = g.tgt[i] = i;
  g.ptr = {0, (int32_t)all};
  g.grid_only = true;
  pl.far.push_back(std::move(g));
  return true;
}

static void run_alg1(Plan& pl, cudaStream_t st) {
  const Cfg& c = pl.cfg;
  const int D = c.D;
  f3m_stats& stt = pl.stats;
  std::vector<Pair> nearl = {{0, 0}};
  int t = 0;
  auto maxbox = [&](const Side& S, bool xs) {
    int64_t mb = 0;
    for (const Pair& pr : nearl) mb = std::max(mb, S.lev[t][xs ? pr.p : pr.q].gcount);
    return mb;
  };
  // device division for levels with many candidate pairs (F3M_TREE_DEVICE=1 / 0 forces it)
  const char* tdev = getenv("F3M_TREE_DEVICE");
  const int tree_device = tdev ? atoi(tdev) : -1;
  const char* tmin = getenv("F3M_TREE_DEVICE_MIN");  // candidate pairs above which a depth is divided on the device
  const uint64_t tree_device_min = tmin ? (uint64_t)atoll(tmin) : 8192ull;  // measured: C2, EV 12.5 faster, C4 unchanged
  while (!nearl.empty() && maxbox(pl.X, true) > c.zeta && maxbox(pl.Y, false) > c.zeta && t < pl.T) {
    ++t;
    LevelCtx L;
    L.t = t;
    L.l = level_edge(pl.E, t);
    const double sb = smooth_bound(D, L.l, c.gamma);
    const double q = adapt_q(L.l, c.gamma);
    int pfar = q <= 0.01 ? std::min(c.P, 3) : (q <= 5.0 ? c.P : 0);
    if (c.flags & F3M_NO_ADAPTIVE) pfar = c.P;
    if ((c.flags & F3M_NO_DROP) && pfar == 0) pfar = c.P;
    L.pfar = pfar;
    stt.pfar[t] = pfar;
    L.smooth_level = !(c.flags & F3M_NO_SMOOTH) && sb <= c.eta;
    L.split = (pfar > 0 && pfar != c.P);
    for (int d = 0; d < D; ++d) L.delta[d] = pl.aliased ? 0.0 : (pl.X.alpha[d] - pl.Y.alpha[d]) / L.l;
    const std::vector<HBox>& PX = pl.X.lev[t - 1];
    const std::vector<HBox>& PY = pl.Y.lev[t - 1];
    uint64_t Mest = 0;
    {
      std::vector<char> ax(PX.size(), 0), ay(PY.size(), 0);
      for (const Pair& pr : nearl) {
        ax[pr.p] = 1;
        ay[pr.q] = 1;
        Mest += (uint64_t)PX[pr.p].nchild * (uint64_t)PY[pr.q].nchild;
      }
      for (size_t i = 0; i < PX.size(); ++i)
        if (ax[i]) { stt.boxes_x[t] += PX[i].nchild; stt.empty_x[t] += (1ll << D) - PX[i].nchild; }
      for (size_t i = 0; i < PY.size(); ++i)
        if (ay[i]) { stt.boxes_y[t] += PY[i].nchild; stt.empty_y[t] += (1ll << D) - PY[i].nchild; }
    }
    stt.expanded[t] = (int64_t)nearl.size() << (2 * D);
    std::vector<Pair> nextnear;
    // the device tables hold int32 cells and int32 CSR offsets: deeper trees (t > 30, only D = 1 or 2
    // with near-duplicate points) and depths with >= 2^31 candidates divide on the host
    const bool dev_ok = t <= 30 && Mest < (1ull << 31);
    const bool dev = dev_ok && (tree_device == 1 || (tree_device < 0 && Mest >= tree_device_min));
    if (grid_level_shortcut(pl, L, nearl)) {
      // every child pair classified by counting; nothing left near
    } else if (dev) {
      level_device(pl, L, nearl, nextnear, st);
    } else {
      level_host(pl, L, nearl, nextnear);
    }
    nearl.swap(nextnear);
  }
  pl.depth_reached = t;
  stt.n_near_flushed = (int64_t)nearl.size();
  push_near_group(pl, t, nearl);
  stt.depth_reached = t;
  stt.t_star = pl.t_star;
  stt.t_sort = pl.T;
  stt.E = pl.E;
  apply_sparse(pl);
}

}  // namespace f3m

namespace f3m {

thread_local int64_t g_launches = 0;

static NodeConsts node_consts(int P) {
  NodeConsts nc{};
  double s[16];
  const double pi = 3.14159265358979323846;
  for (int k = 0; k < P; ++k) s[k] = std::cos((double)k * pi / (double)(P - 1));
  for (int k = 0; k < P; ++k) {
    double den = 1.0;
    for (int j = 0; j < P; ++j)
      if (j != k) den *= (s[k] - s[j]);
    nc.s[k] = (float)s[k];
    nc.c[k] = (float)(1.0 / den);
  }
  return nc;
}

// ---------------------------------------------------------------------------------------
// phase timing (F3M_TIMING=1 or stats requested with timing): events on the call stream
// ---------------------------------------------------------------------------------------
enum { PH_BBOX = 0, PH_COUNT, PH_SCAN, PH_SCATTER, PH_SORT_MISC, PH_TREE, PH_S2M, PH_M2L, PH_L2T, PH_NEAR, PH_UNPERM,
       PH_TOTAL, PH_N };
static const char* kPhaseNames[PH_N] = {"bbox", "count", "scan", "scatter", "sort_misc", "tree", "s2m",
                                        "m2l", "l2t", "near", "unpermute", "total"};

struct Timer {
  bool on = false;
  cudaStream_t st = nullptr;
  cudaEvent_t ev[2 * PH_N] = {};
  bool used[PH_N] = {};
  float acc[PH_N] = {};
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> spans[PH_N];
  std::vector<cudaEvent_t> pool;
  void begin(int ph, cudaEvent_t& a) {
    if (!on) return;
    a = make();
    cudaEventRecord(a, st);
  }
  void end(int ph, cudaEvent_t a) {
    if (!on) return;
    cudaEvent_t b = make();
    cudaEventRecord(b, st);
    spans[ph].push_back({a, b});
  }
  cudaEvent_t make() {
    cudaEvent_t e;
    cudaEventCreate(&e);
    pool.push_back(e);
    return e;
  }
  void collect(float* out) {
    if (!on) return;
    cudaStreamSynchronize(st);
    for (int p = 0; p < PH_N; ++p) {
      float s = 0.f;
      for (auto& pr : spans[p]) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, pr.first, pr.second);
        s += ms;
      }
      out[p] = s;
    }
  }
  ~Timer() {
    for (cudaEvent_t e : pool) cudaEventDestroy(e);
  }
};

struct Span {
  Timer& tm;
  int ph;
  cudaEvent_t a = nullptr;
  Span(Timer& t, int p) : tm(t), ph(p) { tm.begin(ph, a); }
  ~Span() { tm.end(ph, a); }
};

// ---------------------------------------------------------------------------------------
// a1: enclosing cube
// ---------------------------------------------------------------------------------------
static void bbox(Side& S, int D, Workspace& ws, cudaStream_t st) {
  const int nb = bbox_blocks(S.n);
  float* part = ws.get<float>((size_t)nb * (2 * F3M_MAXD + 1), "bbox partials");
  float* out = ws.get<float>(2 * F3M_MAXD + 1, "bbox");
  launch_bbox(S.X, S.n, D, part, nb, st);
  launch_bbox_final(part, nb, D, out, st);
  g_launches += 2;
  float h[2 * F3M_MAXD + 1];
  CK(cudaMemcpyAsync(h, out, sizeof(float) * (2 * D + 1), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (h[2 * D] != 0.f) throw Fail{F3M_ERR_INVALID_INPUT, "non-finite coordinate in the input points"};
  for (int d = 0; d < D; ++d) {
    S.mn[d] = h[d];
    S.mx[d] = h[D + d];
    S.alpha[d] = (double)h[d];
  }
}

// E = max over d of max(maxX_d - minX_d, maxY_d - minY_d), fp64
static double enclosing_edge(const Side& X, const Side& Y, int D) {
  double E = 0.0;
  for (int d = 0; d < D; ++d) {
    const double rx = (double)X.mx[d] - (double)X.mn[d];
    const double ry = (double)Y.mx[d] - (double)Y.mn[d];
    E = std::max(E, std::max(rx, ry));
  }
  return E;
}

// ---------------------------------------------------------------------------------------
// a2-a4: keys, LSD passes of <= 8-bit digits, leaf table
// ---------------------------------------------------------------------------------------
// ---- exact cell thresholds (reading R12): cell(x) = min(floor(RN(RN(x - alpha)/E) 2^T), 2^T - 1)
// is monotone in x, so theta_j = the smallest fp32 with cell >= j gives cell(x) = #{theta_j <= x}
static inline uint32_t fkey(float f) {
  uint32_t b;
  std::memcpy(&b, &f, 4);
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
static inline float funkey(uint32_t u) {
  const uint32_t b = (u & 0x80000000u) ? (u & 0x7fffffffu) : ~u;
  float f;
  std::memcpy(&f, &b, 4);
  return f;
}
static inline uint64_t cell_exact(float x, double alpha, double E, int T) {
  const double u = ((double)x - alpha) / E;
  const double f = std::floor(std::ldexp(u, T));
  if (!(f > 0.0)) return 0;
  const uint64_t cmax = (1ull << T) - 1ull;
  if (f >= (double)cmax) return cmax;  // (also avoids the undefined huge double -> uint64 cast)
  return (uint64_t)f;
}
static std::vector<float> cell_thresholds(const double* alpha, int D, double E, int T) {
  const int NT = (1 << T) - 1;
  std::vector<float> th((size_t)D * NT);
  for (int d = 0; d < D; ++d) {
    for (int j = 1; j <= NT; ++j) {
      uint32_t lo = fkey((float)alpha[d]), hi = fkey(3.4028234663852886e38f);
      if (cell_exact(funkey(hi), alpha[d], E, T) < (uint64_t)j) { th[(size_t)d * NT + j - 1] = INFINITY; continue; }
      while (lo < hi) {
        const uint32_t mid = lo + (hi - lo) / 2;
        if (cell_exact(funkey(mid), alpha[d], E, T) >= (uint64_t)j) hi = mid;
        else lo = mid + 1;
      }
      th[(size_t)d * NT + j - 1] = funkey(lo);
    }
  }
  return th;
}

static KeyParams make_kp(const Side& S, int D, double E, int T) {
  KeyParams kp{};
  kp.D = D;
  kp.T = T;
  for (int d = 0; d < D; ++d) {
    kp.alpha[d] = S.alpha[d];
    kp.alpha_f[d] = S.mn[d];
  }
  kp.E = E;
  kp.twoT = std::ldexp(1.0, T);
  kp.scale_f = (float)(kp.twoT / E);
  kp.margin = std::ldexp(1.0f, T - 22);
  return kp;
}

// Single-pass keys (D*T <= 8) with defer = true: count over 4096-point tiles + scan + leaf
// table only; the stable scatter runs later inside the tile-local kernel (fused with S2M).
// Otherwise: the full LSD counting sort over 8192-point tiles.
static void sort_side(Plan& pl, Side& S, bool with_b, bool want_sigma, bool keep_keys, Workspace& ws, cudaStream_t st,
                      Timer& tm, bool defer) {
  const int D = pl.cfg.D, T = pl.T;
  const int64_t n = S.n;
  const KeyParams kp = make_kp(S, D, pl.E, T);
  const int bits = D * T;
  const int passes = (bits + MAX_DIGIT_BITS - 1) / MAX_DIGIT_BITS;
  pl.passes = passes;
  int w[16];
  for (int p = 0; p < passes; ++p) w[p] = bits / passes + (p < bits % passes ? 1 : 0);
  const bool deferred = defer && passes == 1;
  // multi-pass sorts: LSD passes with stored tile orders (coalesced scatter), 4096-point tiles
  const bool lsd = !deferred;
  const int tile = (deferred || lsd) ? LT_TILE_PTS : SORT_TILE;
  const int64_t tiles = (n + tile - 1) / tile;
  const int nbmax = 1 << w[0];
  uint32_t* counts = ws.get<uint32_t>((size_t)nbmax * tiles + 1, "sort counts");
  uint32_t* tmp = ws.get<uint32_t>((size_t)scan_tmp_words((int64_t)nbmax * tiles), "scan tmp");
  S.kp = kp;
  S.bits = bits;
  S.offsets = counts;
  S.scan_tmp = tmp;
  S.tiles = tiles;
  S.deferred = deferred;
  S.with_b = with_b;
  S.want_sigma = want_sigma;
  S.keep_keys = keep_keys;
  if (deferred) return;  // counts come from the first tile-local pass (first_pass)
  if (lsd) {
    struct Buf { float* xs; float* bs; int32_t* perm; uint64_t* keys; } A{}, B{};
    const bool need_keys = passes > 1 || keep_keys;
    A.xs = ws.get<float>((size_t)D * n, "sorted coords");
    A.bs = with_b ? ws.get<float>(n, "sorted weights") : nullptr;
    A.perm = ws.get<int32_t>(n, "permutation");
    A.keys = need_keys ? ws.get<uint64_t>(n, "sorted keys") : nullptr;
    if (passes > 1) {
      B.xs = ws.get<float>((size_t)D * n, "sorted coords (ping-pong)");
      B.bs = with_b ? ws.get<float>(n, "sorted weights (ping-pong)") : nullptr;
      B.perm = ws.get<int32_t>(n, "permutation (ping-pong)");
      B.keys = ws.get<uint64_t>(n, "sorted keys (ping-pong)");
    }
    Buf* cur = nullptr;
    Buf* out = &A;
    int shift = 0;
    S.lsd_counts.clear();
    S.lsd_order.clear();
    S.lsd_bits.clear();
    for (int p = 0; p < passes; ++p) {
      if (p > 0) counts = ws.get<uint32_t>((size_t)nbmax * tiles + 1, "sort counts");
      uint16_t* order = ws.get<uint16_t>((size_t)n, "tile orders");
      S.lsd_counts.push_back(counts);
      S.lsd_order.push_back(order);
      S.lsd_bits.push_back(w[p]);
      S.offsets = counts;
      {
        Span sp(tm, p == 0 ? PH_COUNT : PH_SORT_MISC);
        launch_lsd_rank(p == 0, S.X, p == 0 ? nullptr : cur->keys, n, D, kp, shift, w[p], (int)tiles, counts, order, st);
        launch_scan_u32(counts, (int64_t)(1 << w[p]) * tiles, tmp, st);
      }
      ScatterIO io{};
      if (p == 0) {
        io.X = S.X;
        io.b = with_b ? S.b : nullptr;
      } else {
        io.keys_in = cur->keys;
        io.perm_in = cur->perm;
        io.xs_in = cur->xs;
        io.bs_in = cur->bs;
      }
      io.keys_out = out->keys;
      io.perm_out = out->perm;
      io.xs_out = out->xs;
      io.bs_out = out->bs;
      {
        Span sp(tm, p == 0 ? PH_SCATTER : PH_SORT_MISC);
        launch_lsd_scatter(p == 0, io, n, D, kp, w[p], (int)tiles, counts, order, st);
      }
      g_launches += 5;
      shift += w[p];
      cur = out;
      out = (out == &A) ? &B : &A;
    }
    // no sigma: every far level of a multi-pass tree runs on the sorted copies, and the
    // output is un-permuted with pi (one random write per point instead of building sigma by a
    // random scatter and then gathering through it)
    S.sigma = nullptr;
    S.xs = cur->xs;
    S.bs = cur->bs;
    S.perm = cur->perm;
    S.keys = cur->keys;
  }

  // leaf table (non-empty leaf boxes in key order)
  Span sp_misc(tm, PH_SORT_MISC);
  S.leaf_key.clear();
  S.leaf_start.clear();
  S.leaf_count.clear();
  if (passes == 1) {
    const int nb = 1 << w[0];
    std::vector<uint32_t> starts(nb + 1);
    CK(cudaMemcpy2DAsync(starts.data(), sizeof(uint32_t), counts, sizeof(uint32_t) * tiles, sizeof(uint32_t), nb,
                         cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    starts[nb] = (uint32_t)n;
    for (int b = 0; b < nb; ++b) {
      const int64_t c = (int64_t)starts[b + 1] - (int64_t)starts[b];
      if (c > 0) {
        S.leaf_key.push_back((uint64_t)b);
        S.leaf_start.push_back(starts[b]);
        S.leaf_count.push_back(c);
      }
    }
  } else {
    uint32_t* flags = ws.get<uint32_t>(n + 1, "run heads");
    uint32_t* tmp2 = ws.get<uint32_t>((size_t)scan_tmp_words(n + 1), "scan tmp");
    launch_key_heads(S.keys, n, flags, st);
    launch_scan_u32(flags, n + 1, tmp2, st);
    uint32_t nboxes = 0;
    CK(cudaMemcpyAsync(&nboxes, flags + n, sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    uint64_t* bk = ws.get<uint64_t>(nboxes, "leaf keys");
    int64_t* bst = ws.get<int64_t>(nboxes, "leaf starts");
    launch_compact_heads(S.keys, flags, n, bk, bst, st);
    g_launches += 5;
    S.leaf_key.resize(nboxes);
    S.leaf_start.resize(nboxes);
    CK(cudaMemcpyAsync(S.leaf_key.data(), bk, sizeof(uint64_t) * nboxes, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(S.leaf_start.data(), bst, sizeof(int64_t) * nboxes, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    S.leaf_count.resize(nboxes);
    for (uint32_t i = 0; i < nboxes; ++i)
      S.leaf_count[i] = (i + 1 < nboxes ? S.leaf_start[i + 1] : n) - S.leaf_start[i];
  }
  S.leaf_gcount = S.leaf_count;
}

// single-pass leaf table from the scanned [bin][tile] counts (column 0 = bin starts)
static void leaf_table_from_scan(Side& S, int nb, Workspace& ws, cudaStream_t st) {
  (void)ws;
  const int64_t n = S.n;
  std::vector<uint32_t> starts(nb + 1);
  CK(cudaMemcpy2DAsync(starts.data(), sizeof(uint32_t), S.offsets, sizeof(uint32_t) * S.tiles, sizeof(uint32_t), nb,
                       cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  starts[nb] = (uint32_t)n;
  S.leaf_key.clear();
  S.leaf_start.clear();
  S.leaf_count.clear();
  for (int b = 0; b < nb; ++b) {
    const int64_t c = (int64_t)starts[b + 1] - (int64_t)starts[b];
    if (c > 0) {
      S.leaf_key.push_back((uint64_t)b);
      S.leaf_start.push_back(starts[b]);
      S.leaf_count.push_back(c);
    }
  }
  S.leaf_gcount = S.leaf_count;
}

struct Spec {               // speculative S2M of the first pass (leaf depth, P nodes)
  bool ok = false;
  float* Wpart = nullptr;
  int grid = 0, nbox = 0;
};

static LocalS2MArgs local_args(const Plan& pl, const Side& S, const float* b, int t, int P);

// First tile-local pass of a deferred (single-pass) side: the per-tile key histogram of the
// counting sort, fused (source side) with a speculative S2M of every leaf box at P nodes --
// at the leaf depth D*T <= 8 this is exactly the far field of the deepest level whenever the
// tree needs it (config C4: depth 2).  Then the scan and the leaf table.
static void first_pass(Plan& pl, Side& S, bool source, Spec& spec, Workspace& ws, cudaStream_t st, Timer& tm) {
  if (!S.deferred) return;
  const int D = pl.cfg.D, T = pl.T, P = pl.cfg.P;
  const int nbox = 1 << (D * T);
  const bool s2m = source && local_supported(D, P, nbox) && !getenv("F3M_NO_LOCAL");
  LocalS2MArgs a = local_args(pl, S, source ? S.b : S.X, T, s2m ? P : 2);
  a.counts = S.offsets;
  S.lrank = ws.get<uint16_t>(S.n, "tile-local ranks");
  a.lrank = S.lrank;
  a.do_s2m = s2m ? 1 : 0;
  const bool use_tma = tma_supported(D, s2m ? P : 2, nbox, s2m ? nbox : 1, s2m);
  const int grid = use_tma ? tma_grid(a.num_tiles) : local_grid(a.num_tiles);
  if (s2m) {
    a.Wpart = ws.get<float>((size_t)grid * nbox * (int64_t)std::pow((double)P, D), "speculative s2m partials");
    spec.ok = true;
    spec.Wpart = a.Wpart;
    spec.grid = grid;
    spec.nbox = nbox;
  } else {
    a.nbox = 1;
    a.shift = a.bits;
  }
  S.lrank_sorted = use_tma;
  const bool use_ws = use_tma && s2m && a.kp.thr && a.shift == 0 && s2m_ws_supported(D, P, T, nbox);
  {
    Span sp(tm, s2m ? PH_S2M : PH_COUNT);
    if (use_ws) launch_s2m_ws(D, P, T, a, grid, st);
    else if (use_tma) launch_s2m_tma(D, s2m ? P : 2, a, grid, st);
    else launch_local_s2m(D, s2m ? P : 2, a, grid, st);
  }
  {
    Span sp(tm, PH_SCAN);
    launch_scan_u32(S.offsets, (int64_t)nbox * S.tiles, S.scan_tmp, st);
  }
  g_launches += 4;
  Span sp(tm, PH_SORT_MISC);
  leaf_table_from_scan(S, nbox, ws, st);
}

// the deferred single-pass scatter: outputs of a tile-local kernel launch
static void scatter_outputs(Plan& pl, Side& S, bool need_sorted, Workspace& ws, LocalS2MArgs& a) {
  const int D = pl.cfg.D;
  const int64_t n = S.n;
  S.perm = ws.get<int32_t>(n, "permutation");
  a.offsets = S.offsets;
  a.sort_tiles = (int)S.tiles;
  a.perm = S.perm;
  if (need_sorted) {
    S.xs = ws.get<float>((size_t)D * n, "sorted coords");
    S.bs = ws.get<float>(n, "sorted weights");  // also staged for a target-only side (harmless)
    a.xs = S.xs;
    a.bs = S.bs;
    if (S.want_sigma) {
      S.sigma = ws.get<int32_t>(n, "sigma");
      a.sigma = S.sigma;
    }
  }
  if (S.keep_keys) {
    S.keys = ws.get<uint64_t>(n, "sorted keys");
    a.keys = S.keys;
  }
  S.deferred = false;
}

static LocalS2MArgs local_args(const Plan& pl, const Side& S, const float* b, int t, int P) {
  const int D = pl.cfg.D;
  LocalS2MArgs a{};
  const bool leaf0 = (D * pl.T <= MAX_DIGIT_BITS);
  const int Tk = leaf0 ? pl.T : t;
  // exact thresholds of this side at depth Tk (uploaded once per side and depth)
  Side& Sm = const_cast<Side&>(S);
  if (D * Tk <= MAX_DIGIT_BITS && pl.ws) {
    auto it = Sm.thr_dev.find(Tk);
    if (it == Sm.thr_dev.end()) {
      const std::vector<float> th = cell_thresholds(S.alpha, D, pl.E, Tk);
      it = Sm.thr_dev.emplace(Tk, pl.ws->upload(th, "cell thresholds")).first;
    }
    a.kp.thr = it->second;
  }
  a.X = S.X;
  a.b = b;
  a.n = S.n;
  // single-pass keys: rank by the whole leaf key, level-t box = prefix; otherwise rank by
  // the level-t key itself (its cells are the prefixes of the leaf cells, reading R12)
  const bool leaf = (D * pl.T <= MAX_DIGIT_BITS);
  const float* thr_keep = a.kp.thr;
  a.kp = make_kp(S, D, pl.E, leaf ? pl.T : t);
  a.kp.thr = thr_keep;
  a.bits = D * a.kp.T;
  a.shift = D * (a.kp.T - t);
  a.nbox = 1 << (D * t);
  for (int d = 0; d < D; ++d) a.alpha[d] = S.alpha[d];
  a.l = level_edge(pl.E, t);
  a.nc = node_consts(P);
  a.num_tiles = (int)((S.n + LT_TILE_PTS - 1) / LT_TILE_PTS);
  return a;
}

// ---------------------------------------------------------------------------------------
// a6-a8: far field for every (depth, node count) group
// ---------------------------------------------------------------------------------------
static void box_jobs(const Side& S, const std::vector<HBox>& L, const std::vector<int64_t>& boxes, double l, int D,
                     std::vector<BoxGeom>& geo, std::vector<Chunk>& chunks, std::vector<int32_t>& cptr) {
  geo.clear();
  chunks.clear();
  cptr.clear();
  for (size_t slot = 0; slot < boxes.size(); ++slot) {
    const HBox& b = L[boxes[slot]];
    BoxGeom g{};
    for (int d = 0; d < D; ++d) {
      const double lo = S.alpha[d] + (double)b.cell[d] * l;
      g.lo_hi[d] = (float)lo;
      g.lo_lo[d] = (float)(lo - (double)g.lo_hi[d]);
    }
    g.scale = (float)(2.0 / l);
    g.start = b.start;
    g.count = b.count;
    geo.push_back(g);
    cptr.push_back((int32_t)chunks.size());
    for (int64_t s = 0; s < b.count; s += FAR_CHUNK)
      chunks.push_back({(int32_t)slot, (int32_t)std::min<int64_t>(FAR_CHUNK, b.count - s), b.start + s});
  }
  cptr.push_back((int32_t)chunks.size());
}

struct FarBuffers {
  std::vector<int64_t> w_off;  // per group offset into the charge buffer (doubles)
  int64_t w_total = 0;
  double* W = nullptr;
  std::vector<double*> U;
  // multi-level sorted far field (exact M2M / L2L): one S2M at the deepest level, one L2T
  bool ml = false;
  int tmin = 0, tmax = 0, P = 0;
  int64_t m = 0;
};

// tile-local kernels apply to a far level whose boxes fit one <= 8-bit digit
static bool group_is_local(const Plan& pl, const FarGroup& g) {
  const int D = pl.cfg.D;
  if (g.q > 0) return false;  // sparse grids run on the globally sorted points
  if (D * g.t > MAX_DIGIT_BITS) return false;
  // a multi-pass sort already produced the sorted copies: every level uses them (the
  // tile-local kernels would re-rank each tile and gather the sorted levels' results)
  if (pl.passes > 1) return false;
  if (getenv("F3M_NO_LOCAL")) return false;
  return local_supported(D, g.P, 1 << (D * g.t));
}

static void count_groups(Plan& pl) {
  pl.stats.far_groups_local = pl.stats.far_groups_sorted = 0;
  for (const FarGroup& g : pl.far) {
    if (group_is_local(pl, g)) pl.stats.far_groups_local++;
    else pl.stats.far_groups_sorted++;
  }
}

static bool needs_sorted(const Plan& pl) {
  if (!pl.near.empty()) return true;
  for (const FarGroup& g : pl.far)
    if (!group_is_local(pl, g)) return true;
  return false;
}

// S2M of every group.  Local groups reuse the speculative first-pass charges when they
// match (leaf depth, P); otherwise a tile-local S2M pass runs.  The deferred scatter of
// sorted copies (pi, sigma, SoA coordinates, weights) runs only when the sorted-order
// kernels need them; otherwise pi is written by the first tile-local L2T pass.
// The sorted (global-order) far groups qualify for the exact multi-level form when they span
// at least two depths with one common node count (M2M / L2L are exact only between equal P).
static bool multilevel_ok(const Plan& pl, FarBuffers& fb) {
  int P = -1, tmin = 1 << 30, tmax = -1;
  for (const FarGroup& g : pl.far) {
    if (group_is_local(pl, g)) continue;
    if (g.q > 0) return false;  // no exact M2M / L2L between sparse grids here
    if (P >= 0 && g.P != P) return false;
    P = g.P;
    tmin = std::min(tmin, g.t);
    tmax = std::max(tmax, g.t);
  }
  if (P < 0 || tmax <= tmin || !(far_supported(pl.cfg.D, P) || blk_supported(pl.cfg.D, P))) return false;
  fb.ml = true;
  fb.P = P;
  fb.tmin = tmin;
  fb.tmax = tmax;
  fb.m = 1;
  for (int d = 0; d < pl.cfg.D; ++d) fb.m *= P;
  return true;
}

struct LevelLinks {  // device tables of one depth for the translations
  int32_t* child0 = nullptr;
  int32_t* nchild = nullptr;
  int32_t* bits = nullptr;    // child position: bit d = parity of the cell along d
  int32_t* parent = nullptr;  // index of the parent box at depth t - 1
};
static LevelLinks level_links(const std::vector<HBox>& L, const std::vector<HBox>* parent_level, int D, Workspace& ws,
                              int t) {
  LevelLinks k;
  std::vector<int32_t> c0(L.size()), nc(L.size()), bt(L.size()), par(L.size(), 0);
  for (size_t i = 0; i < L.size(); ++i) {
    c0[i] = (int32_t)L[i].child0;
    nc[i] = (int32_t)L[i].nchild;
    int b = 0;
    for (int d = 0; d < D; ++d) b |= (int)(L[i].cell[d] & 1) << d;
    bt[i] = b;
  }
  if (parent_level)
    for (size_t p = 0; p < parent_level->size(); ++p)
      for (int64_t c = (*parent_level)[p].child0; c < (*parent_level)[p].child0 + (*parent_level)[p].nchild; ++c)
        par[c] = (int32_t)p;
  k.child0 = ws.upload(c0, "level links", t);
  k.nchild = ws.upload(nc, "level links", t);
  k.bits = ws.upload(bt, "level links", t);
  k.parent = ws.upload(par, "level links", t);
  return k;
}

// multi-level S2M: charges of every box at the deepest depth from the points, M2M upwards,
// then each sorted group's W rows gathered from its depth
static void multilevel_s2m(Plan& pl, FarBuffers& fb, Workspace& ws, cudaStream_t st) {
  const int D = pl.cfg.D;
  Side& Ys = pl.Y;
  const int P = fb.P;
  const int64_t m = fb.m;
  std::vector<double*> Wl(fb.tmax + 1, nullptr);
  {
    const int t = fb.tmax;
    const double l = level_edge(pl.E, t);
    std::vector<int64_t> all(Ys.lev[t].size());
    for (size_t i = 0; i < all.size(); ++i) all[i] = (int64_t)i;
    std::vector<BoxGeom> geo;
    std::vector<Chunk> chunks;
    std::vector<int32_t> cptr;
    box_jobs(Ys, Ys.lev[t], all, l, D, geo, chunks, cptr);
    for (const BoxGeom& bg : geo) pl.stats.s2m_points += bg.count;
    BoxGeom* dgeo = ws.upload(geo, "s2m boxes", t);
    Chunk* dch = ws.upload(chunks, "s2m chunks", t);
    int32_t* dcp = ws.upload(cptr, "s2m chunk ptr", t);
    float* part = ws.get<float>(std::max<size_t>(1, chunks.size()) * m, "s2m partials", t);
    Wl[t] = ws.get<double>(all.size() * m, "level charges", t);
    if (blk_supported(D, P)) {  // register-blocked Lagrange-basis S2M: nodal charges directly
      launch_s2m_blk(D, P, Ys.xs, Ys.bs, Ys.n, dgeo, dch, (int64_t)chunks.size(), node_consts(P), part, st);
      launch_chunk_reduce(part, dcp, (int32_t)all.size(), (int)m, Wl[t], st);
      g_launches += 2;
    } else {
      launch_s2m(D, P, Ys.xs, Ys.bs, Ys.n, dgeo, dch, (int64_t)chunks.size(), node_consts(P), part, st);
      launch_chunk_reduce(part, dcp, (int32_t)all.size(), (int)m, Wl[t], st);
      launch_cheb_transform(Wl[t], (int)all.size(), D, P, 0, st);  // Chebyshev moments -> nodal charges
      g_launches += 3;
    }
  }
  for (int t = fb.tmax - 1; t >= fb.tmin; --t) {
    const LevelLinks lk = level_links(Ys.lev[t], nullptr, D, ws, t);
    const LevelLinks lc = level_links(Ys.lev[t + 1], &Ys.lev[t], D, ws, t + 1);
    Wl[t] = ws.get<double>(Ys.lev[t].size() * m, "level charges", t);
    double* scr = ws.get<double>((size_t)Ys.lev[t].size() * m2m_split(D, (int)Ys.lev[t].size()) * m, "m2m partials", t);
    launch_m2m(D, P, (int)m, (int)Ys.lev[t].size(), lk.child0, lk.nchild, lc.bits, Wl[t + 1], Wl[t], scr, st);
    g_launches += 1;
  }
  for (size_t gi = 0; gi < pl.far.size(); ++gi) {
    const FarGroup& g = pl.far[gi];
    if (group_is_local(pl, g)) continue;
    std::vector<int32_t> idx(g.src.begin(), g.src.end());
    launch_rows(Wl[g.t], ws.upload(idx, "group rows", g.t), (int64_t)idx.size(), (int)m, fb.W + fb.w_off[gi], false, st);
    g_launches += 1;
  }
}

// multi-level L2T: groups' locals scattered into per-depth arrays, L2L downwards, one L2T at
// the deepest depth over every box
static void multilevel_l2t(Plan& pl, FarBuffers& fb, float* vs, Workspace& ws, cudaStream_t st) {
  const int D = pl.cfg.D;
  Side& Xs = pl.X;
  const int P = fb.P;
  const int64_t m = fb.m;
  std::vector<double*> Ul(fb.tmax + 1, nullptr);
  for (int t = fb.tmin; t <= fb.tmax; ++t) {
    Ul[t] = ws.get<double>(Xs.lev[t].size() * m, "level locals", t);
    CK(cudaMemsetAsync(Ul[t], 0, sizeof(double) * Xs.lev[t].size() * m, st));
  }
  for (size_t gi = 0; gi < pl.far.size(); ++gi) {
    const FarGroup& g = pl.far[gi];
    if (group_is_local(pl, g)) continue;
    std::vector<int32_t> idx(g.tgt.begin(), g.tgt.end());
    launch_rows(fb.U[gi], ws.upload(idx, "group rows", g.t), (int64_t)idx.size(), (int)m, Ul[g.t], true, st);
    g_launches += 1;
  }
  for (int t = fb.tmin; t < fb.tmax; ++t) {
    const LevelLinks lc = level_links(Xs.lev[t + 1], &Xs.lev[t], D, ws, t + 1);
    launch_l2l(D, P, (int)m, (int)Xs.lev[t + 1].size(), lc.parent, lc.bits, Ul[t], Ul[t + 1], st);
    g_launches += 1;
  }
  const int t = fb.tmax;
  const double l = level_edge(pl.E, t);
  std::vector<int64_t> all(Xs.lev[t].size());
  for (size_t i = 0; i < all.size(); ++i) all[i] = (int64_t)i;
  std::vector<BoxGeom> geo;
  std::vector<Chunk> chunks;
  std::vector<int32_t> cptr;
  box_jobs(Xs, Xs.lev[t], all, l, D, geo, chunks, cptr);
  for (const BoxGeom& bg : geo) pl.stats.l2t_points += bg.count;
  BoxGeom* dgeo = ws.upload(geo, "l2t boxes", t);
  Chunk* dch = ws.upload(chunks, "l2t chunks", t);
  if (blk_supported(D, P))
    launch_l2t_blk(D, P, Xs.xs, Xs.n, dgeo, dch, (int64_t)chunks.size(), node_consts(P), Ul[t], vs, st);
  else
    launch_l2t(D, P, Xs.xs, Xs.n, dgeo, dch, (int64_t)chunks.size(), node_consts(P), Ul[t], vs, st);
  g_launches += 1;
}

static void far_s2m(Plan& pl, FarBuffers& fb, const Spec& spec, Workspace& ws, cudaStream_t st, Timer& tm) {
  const int D = pl.cfg.D;
  count_groups(pl);
  const bool need_sorted = needs_sorted(pl);
  fb.w_off.clear();
  fb.w_total = 0;
  for (const FarGroup& g : pl.far) {
    fb.w_off.push_back(fb.w_total);
    fb.w_total += (int64_t)g.src.size() * g.m;
  }
  fb.W = ws.get<double>(fb.w_total, "charges");
  Side& Ys = pl.Y;
  for (size_t gi = 0; gi < pl.far.size(); ++gi) {
    const FarGroup& g = pl.far[gi];
    if (!group_is_local(pl, g)) continue;
    Span sp(tm, PH_S2M);
    const float* Wpart;
    int grid, nbox;
    if (spec.ok && g.t == pl.T && g.P == pl.cfg.P) {
      Wpart = spec.Wpart;
      grid = spec.grid;
      nbox = spec.nbox;
    } else {
      LocalS2MArgs a = local_args(pl, Ys, Ys.b, g.t, g.P);
      grid = local_grid(a.num_tiles);
      nbox = a.nbox;
      a.do_s2m = 1;
      float* wp = ws.get<float>((size_t)grid * a.nbox * g.m, "local s2m partials", g.t);
      a.Wpart = wp;
      launch_local_s2m(D, g.P, a, grid, st);
      g_launches += 1;
      Wpart = wp;
    }
    std::vector<int32_t> slot_box;
    for (int64_t q : g.src) slot_box.push_back((int32_t)Ys.lev[g.t][q].key);
    for (int64_t q : g.src) pl.stats.s2m_points += Ys.lev[g.t][q].count;
    int32_t* dsb = ws.upload(slot_box, "local slot boxes", g.t);
    launch_local_reduce(Wpart, grid, nbox, (int)g.m, dsb, (int)g.src.size(), fb.W + fb.w_off[gi], st);
    launch_cheb_transform(fb.W + fb.w_off[gi], (int)g.src.size(), D, g.P, 0, st);  // moments -> nodal
    g_launches += 2;
  }
  // deferred scatters: sorted copies when needed; pi of a side no tile-local L2T will write
  const bool local_l2t = pl.stats.far_groups_local > 0;
  auto plain_scatter = [&](Side& S, bool target) {
    if (!S.deferred) return;
    if (!need_sorted && target && local_l2t) return;  // pi from the first local L2T pass
    Span sp(tm, PH_SCATTER);
    LocalS2MArgs a = local_args(pl, S, S.with_b ? S.b : S.X, pl.T, 2);
    a.nbox = 1;
    a.shift = a.bits;
    scatter_outputs(pl, S, need_sorted, ws, a);
    a.do_s2m = 0;
    if (S.lrank && S.lrank_sorted) {  // from the first pass's tile orders
      a.lrank = S.lrank;
      launch_scatter_ord(D, a, st);
    } else {
      launch_local_s2m(D, 2, a, local_grid(a.num_tiles), st);
    }
    g_launches += 1;
  };
  if (pl.aliased) {
    plain_scatter(Ys, true);
    pl.X.deferred = Ys.deferred;
    pl.X.perm = Ys.perm; pl.X.xs = Ys.xs; pl.X.bs = Ys.bs; pl.X.sigma = Ys.sigma; pl.X.keys = Ys.keys;
  } else {
    plain_scatter(Ys, false);
    plain_scatter(pl.X, true);
  }
  if (multilevel_ok(pl, fb)) {
    Span sp(tm, PH_S2M);
    multilevel_s2m(pl, fb, ws, st);
    return;
  }
  for (size_t gi = 0; gi < pl.far.size(); ++gi) {
    const FarGroup& g = pl.far[gi];
    if (group_is_local(pl, g)) continue;
    Span sp(tm, PH_S2M);
    if (g.q > 0) {  // sparse grid: Chebyshev moments over K_q, then W = A M (nodal charges)
      const SparseGrid& sg = sparse_grid(D, g.q);
      const double l = level_edge(pl.E, g.t);
      std::vector<BoxGeom> geo;
      std::vector<Chunk> chunks;
      std::vector<int32_t> cptr;
      box_jobs(Ys, Ys.lev[g.t], g.src, l, D, geo, chunks, cptr);
      for (const BoxGeom& bg : geo) pl.stats.s2m_points += bg.count;
      BoxGeom* dgeo = ws.upload(geo, "s2m boxes", g.t);
      Chunk* dch = ws.upload(chunks, "s2m chunks", g.t);
      int32_t* dcp = ws.upload(cptr, "s2m chunk ptr", g.t);
      float* part = ws.get<float>(std::max<size_t>(1, chunks.size()) * g.m, "s2m partials", g.t);
      double* mom = ws.get<double>((size_t)g.src.size() * g.m, "sparse moments", g.t);
      launch_s2m_sparse(D, sg.n1, (int)g.m, Ys.xs, Ys.bs, Ys.n, dgeo, dch, (int64_t)chunks.size(), sg.d_fac, part, st);
      launch_chunk_reduce(part, dcp, (int32_t)g.src.size(), (int)g.m, mom, st);
      launch_dense_rows(mom, (int64_t)g.src.size(), (int)g.m, sg.d_Vinv, fb.W + fb.w_off[gi], st);
      g_launches += (chunks.empty() ? 0 : 1) + 2;
      continue;
    }
    const bool gen = !far_supported(D, g.P);
    if (gen && !gen_supported(D, g.P))
      throw Fail{F3M_ERR_GRID_TOO_LARGE, "no far-field kernel instantiation for this (D, P)"};
    const double l = level_edge(pl.E, g.t);
    std::vector<BoxGeom> geo;
    std::vector<Chunk> chunks;
    std::vector<int32_t> cptr;
    box_jobs(Ys, Ys.lev[g.t], g.src, l, D, geo, chunks, cptr);
    for (const BoxGeom& bg : geo) pl.stats.s2m_points += bg.count;
    const NodeConsts nc = node_consts(g.P);
    BoxGeom* dgeo = ws.upload(geo, "s2m boxes", g.t);
    Chunk* dch = ws.upload(chunks, "s2m chunks", g.t);
    int32_t* dcp = ws.upload(cptr, "s2m chunk ptr", g.t);
    float* part = ws.get<float>(std::max<size_t>(1, chunks.size()) * g.m, "s2m partials", g.t);
    const bool blk = blk_supported(D, g.P);  // register-blocked, nodal charges directly
    if (blk)
      launch_s2m_blk(D, g.P, Ys.xs, Ys.bs, Ys.n, dgeo, dch, (int64_t)chunks.size(), nc, part, st);
    else if (gen)
      launch_s2m_gen(D, g.P, Ys.xs, Ys.bs, Ys.n, dgeo, dch, (int64_t)chunks.size(), nc, part, st);
    else
      launch_s2m(D, g.P, Ys.xs, Ys.bs, Ys.n, dgeo, dch, (int64_t)chunks.size(), nc, part, st);
    launch_chunk_reduce(part, dcp, (int32_t)g.src.size(), (int)g.m, fb.W + fb.w_off[gi], st);
    const bool cheb = !gen && !blk;  // k_s2m accumulates Chebyshev moments
    if (cheb) launch_cheb_transform(fb.W + fb.w_off[gi], (int)g.src.size(), D, g.P, 0, st);  // moments -> nodal
    g_launches += (chunks.empty() ? 0 : 1) + 1 + (cheb ? 1 : 0);
  }
}

// M2L of a far group over a complete level as Kronecker mode products (kernels_grid.cu,
// DESIGN.md reading R29).  Applies when X = Y, level t holds all 2^{Dt} boxes on both sides, and
// the group's pairs are exactly the children of every near pair of depth t - 1: with integer
// parent offsets o, the near rule admits o in {-1,0,1}^D with <= 3 non-zero entries (Euclidean)
// or every o in {-1,0,1}^D (max norm).  Every child pair of such a parent pair is in the group
// by construction of Alg. 1 (it is far or smooth and not split), so comparing the group's pair
// count with the count of all admitted child pairs proves the set equality.  Used only where
// the mode products are cheaper than the pairwise separable M2L and fit in memory.
struct GridM2L {
  int N = 0, ndeg = 0;
  std::vector<double> B0, B1;      // [D][N][N]
  std::vector<int64_t> sbase, tbase;
  int64_t total = 0, fma = 0;
};
static bool grid_m2l_plan(const Plan& pl, const FarGroup& g, GridM2L& G) {
  const int D = pl.cfg.D, t = g.t, P = g.P;
  if (!pl.aliased || g.q > 0 || t < 1 || D * t > 24) return false;
  const int64_t nbox = 1ll << (D * t);
  const std::vector<HBox>& L = pl.X.lev[t];
  if ((int64_t)L.size() != nbox || (int64_t)g.src.size() != nbox || (int64_t)g.tgt.size() != nbox) return false;
  const bool maxnorm = (pl.cfg.flags & F3M_ADMISSIBLE_MAXNORM) != 0;
  // admitted parent pairs on the complete depth-(t-1) grid, times 4^D children pairs
  const double want = admitted_parent_pairs(D, t, maxnorm) * std::pow(4.0, D);
  const int64_t have = g.ptr.empty() ? 0 : (int64_t)g.ptr.back();
  if (want != (double)have) return false;
  if (!grid_m2l_worth(D, t, P, (double)have, maxnorm, &G.N, &G.ndeg, &G.total, &G.fma)) return false;
  // per-dimension factors: K_d between node (cell c, node k) and (cell c', node j), split by
  // the parent offset (c >> 1) - (c' >> 1)
  const double l = level_edge(pl.E, t), gamma = pl.cfg.gamma, pi = 3.14159265358979323846;
  std::vector<double> s(P);
  for (int k = 0; k < P; ++k) s[k] = std::cos((double)k * pi / (double)(P - 1));
  const int N = G.N;
  G.B0.assign((size_t)D * N * N, 0.0);
  G.B1.assign((size_t)D * N * N, 0.0);
  for (int d = 0; d < D; ++d)
    for (int i = 0; i < N; ++i)
      for (int j = 0; j < N; ++j) {
        const int ci = i / P, k = i % P, cj = j / P, jn = j % P;
        const int po = (ci >> 1) - (cj >> 1);
        if (po < -1 || po > 1) continue;
        const double diff = (double)(ci - cj) * l + (l / 2.0) * (s[k] - s[jn]);
        const double kv = std::exp(-(diff * diff) / (2.0 * gamma * gamma));
        ((po == 0 || maxnorm) ? G.B0 : G.B1)[((size_t)d * N + i) * N + j] = kv;
      }
  auto bases = [&](const std::vector<int64_t>& boxes, std::vector<int64_t>& out) {
    out.resize(boxes.size());
    for (size_t q = 0; q < boxes.size(); ++q) {
      int64_t b = 0, stride = 1;
      for (int d = 0; d < D; ++d) {
        b += L[boxes[q]].cell[d] * P * stride;
        stride *= N;
      }
      out[q] = b;
    }
  };
  bases(g.src, G.sbase);
  bases(g.tgt, G.tbase);
  return true;
}

// M2L for every group; L2T for the global-sorted groups into vs (sorted order).
// Returns true if vs holds contributions (global groups evaluated).
static bool far_eval(Plan& pl, FarBuffers& fb, float* vs, Workspace& ws, cudaStream_t st, Timer& tm) {
  const int D = pl.cfg.D;
  fb.U.clear();
  {
    Span sp(tm, PH_M2L);
    for (size_t gi = 0; gi < pl.far.size(); ++gi) {
      const FarGroup& g = pl.far[gi];
      GridM2L G;
      if (grid_m2l_plan(pl, g, G)) {
        double* U = ws.get<double>(g.tgt.size() * g.m, "locals", g.t);
        double* Za = ws.get<double>((size_t)G.ndeg * G.total, "grid m2l tensor", g.t);
        double* Zb = ws.get<double>((size_t)G.ndeg * G.total, "grid m2l tensor", g.t);
        launch_grid_m2l(D, g.P, G.N, G.ndeg, ws.upload(G.B0, "grid m2l factors", g.t), ws.upload(G.B1, "grid m2l factors", g.t),
                        fb.W + fb.w_off[gi], ws.upload(G.sbase, "grid m2l bases", g.t), (int)g.src.size(),
                        ws.upload(G.tbase, "grid m2l bases", g.t), (int)g.tgt.size(), Za, Zb, U, st);
        g_launches += 3 + D;
        pl.stats.m2l_grid_groups += 1;
        pl.stats.m2l_grid_fma += G.fma;
        pl.stats.m2l_grid_pairs += g.ptr.back();
        fb.U.push_back(U);
        continue;
      }
      if (g.grid_only) throw Fail{F3M_ERR_INTERNAL, "complete-level group without its mode-product M2L"};
      const double l = level_edge(pl.E, g.t);
      int maxr = 1;
      for (int d = 0; d < D; ++d) maxr = std::max(maxr, g.range[d]);
      const int stride = maxr * g.P * g.P;
      float* tables = ws.get<float>((size_t)D * stride, "m2l tables", g.t);
      const NodeConsts nc = node_consts(g.P);
      launch_m2l_tables(D, g.P, g.delta0, l, g.range, pl.cfg.gamma, nc, tables, stride, st);
      int32_t* dptr = g.d_ptr ? g.d_ptr : ws.upload(g.ptr, "m2l csr", g.t);
      int32_t* dcol = g.d_col ? g.d_col : ws.upload(g.col, "m2l cols", g.t);
      uint64_t* doff = g.d_off ? g.d_off : ws.upload(g.off, "m2l offsets", g.t);
      double* U = ws.get<double>(g.tgt.size() * g.m, "locals", g.t);
      float* W32 = ws.get<float>(g.src.size() * g.m, "charges fp32", g.t);
      launch_to_f32(fb.W + fb.w_off[gi], (int64_t)(g.src.size() * g.m), W32, st);
      if (g.q > 0)  // node-pair kernels evaluated on the fly over the sparse nodes
        launch_m2l_sparse(D, g.P, (int)g.m, (int32_t)g.tgt.size(), dptr, dcol, doff, tables, stride, W32,
                          sparse_grid(D, g.q).d_nodes, U, st);
      else
        launch_m2l(D, g.P, (int32_t)g.tgt.size(), dptr, dcol, doff, tables, stride, W32, U, st);
      g_launches += 3;
      fb.U.push_back(U);
    }
  }
  bool any = false;
  if (fb.ml) {
    Span sp(tm, PH_L2T);
    multilevel_l2t(pl, fb, vs, ws, st);
    any = true;
  } else {
    Span sp(tm, PH_L2T);
    for (size_t gi = 0; gi < pl.far.size(); ++gi) {
      const FarGroup& g = pl.far[gi];
      if (group_is_local(pl, g)) continue;
      const double l = level_edge(pl.E, g.t);
      std::vector<BoxGeom> geo;
      std::vector<Chunk> chunks;
      std::vector<int32_t> cptr;
      box_jobs(pl.X, pl.X.lev[g.t], g.tgt, l, D, geo, chunks, cptr);
      for (const BoxGeom& bg : geo) pl.stats.l2t_points += bg.count;
      BoxGeom* dgeo = ws.upload(geo, "l2t boxes", g.t);
      Chunk* dch = ws.upload(chunks, "l2t chunks", g.t);
      if (g.q > 0) {  // Ut = A^T U (Chebyshev coefficients of the local expansion), then L2T
        const SparseGrid& sg = sparse_grid(D, g.q);
        double* Ut = ws.get<double>(g.tgt.size() * g.m, "sparse chebyshev locals", g.t);
        launch_dense_rows(fb.U[gi], (int64_t)g.tgt.size(), (int)g.m, sg.d_VinvT, Ut, st);
        launch_l2t_sparse(D, sg.n1, (int)g.m, pl.X.xs, pl.X.n, dgeo, dch, (int64_t)chunks.size(), sg.d_fac, Ut, vs, st);
        g_launches += 1 + (chunks.empty() ? 0 : 1);
        any = true;
        continue;
      }
      if (blk_supported(D, g.P)) {
        launch_l2t_blk(D, g.P, pl.X.xs, pl.X.n, dgeo, dch, (int64_t)chunks.size(), node_consts(g.P), fb.U[gi], vs, st);
      } else if (far_supported(D, g.P)) {
        launch_l2t(D, g.P, pl.X.xs, pl.X.n, dgeo, dch, (int64_t)chunks.size(), node_consts(g.P), fb.U[gi], vs, st);
      } else {
        launch_l2t_gen(D, g.P, pl.X.xs, pl.X.n, dgeo, dch, (int64_t)chunks.size(), node_consts(g.P), fb.U[gi], vs, st);
      }
      if (!chunks.empty()) g_launches += 1;
      any = true;
    }
  }
  if (g_dbg.on) {
    CK(cudaStreamSynchronize(st));
    for (size_t gi = 0; gi < pl.far.size(); ++gi) {
      const FarGroup& g = pl.far[gi];
      DebugCharges dc;
      dc.t = g.t;
      dc.P = g.P;
      dc.m = g.m;
      dc.q = g.q;
      for (int64_t q : g.src) dc.sk.push_back(pl.Y.lev[g.t][q].key);
      for (int64_t p : g.tgt) dc.tk.push_back(pl.X.lev[g.t][p].key);
      dc.W.resize(g.src.size() * g.m);
      dc.U.resize(g.tgt.size() * g.m);
      CK(cudaMemcpy(dc.W.data(), fb.W + fb.w_off[gi], sizeof(double) * dc.W.size(), cudaMemcpyDeviceToHost));
      CK(cudaMemcpy(dc.U.data(), fb.U[gi], sizeof(double) * dc.U.size(), cudaMemcpyDeviceToHost));
      g_dbg.charges.push_back(std::move(dc));
    }
  }
  return any;
}

// final output in the original order: tile-local L2T of the local groups (plus the
// sorted-order contributions vs[sigma[i]]), or the plain un-permutation
static void finish_output(Plan& pl, FarBuffers& fb, const float* vs, bool vs_used, float* v, Workspace& ws,
                          cudaStream_t st, Timer& tm) {
  const int D = pl.cfg.D;
  bool first = true;
  for (size_t gi = 0; gi < pl.far.size(); ++gi) {
    const FarGroup& g = pl.far[gi];
    if (!group_is_local(pl, g)) continue;
    Span sp(tm, PH_L2T);
    const LocalS2MArgs s = local_args(pl, pl.X, nullptr, g.t, g.P);
    LocalL2TArgs a{};
    a.X = pl.X.X;
    a.n = pl.X.n;
    a.kp = s.kp;
    a.bits = s.bits;
    a.shift = s.shift;
    a.nbox = s.nbox;
    for (int d = 0; d < D; ++d) a.alpha[d] = s.alpha[d];
    a.l = s.l;
    a.nc = s.nc;
    a.num_tiles = s.num_tiles;
    double* Ut = ws.get<double>(g.tgt.size() * g.m, "chebyshev locals", g.t);
    CK(cudaMemcpyAsync(Ut, fb.U[gi], sizeof(double) * g.tgt.size() * g.m, cudaMemcpyDeviceToDevice, st));
    launch_cheb_transform(Ut, (int)g.tgt.size(), D, g.P, 1, st);  // nodal -> Chebyshev coefficients
    g_launches += 1;
    a.U = Ut;
    std::vector<int32_t> box_slot(a.nbox, -1);
    for (size_t p = 0; p < g.tgt.size(); ++p) box_slot[pl.X.lev[g.t][g.tgt[p]].key] = (int32_t)p;
    for (int64_t p : g.tgt) pl.stats.l2t_points += pl.X.lev[g.t][p].count;
    a.box_slot = ws.upload(box_slot, "local box slots", g.t);
    a.v = v;
    a.accumulate = first ? 0 : 1;
    a.vs = (first && vs_used) ? vs : nullptr;
    a.sigma = (first && vs_used) ? pl.X.sigma : nullptr;
    if (first && pl.X.deferred) {  // the counting-sort permutation of the target side
      pl.X.perm = ws.get<int32_t>(pl.X.n, "permutation");
      a.offsets = pl.X.offsets;
      a.sort_tiles = (int)pl.X.tiles;
      a.perm = pl.X.perm;
      a.lrank = pl.X.lrank;
      if (pl.X.keep_keys) {
        pl.X.keys = ws.get<uint64_t>(pl.X.n, "sorted keys");
        a.keys = pl.X.keys;
      }
      pl.X.deferred = false;
      if (pl.aliased) { pl.Y.perm = pl.X.perm; pl.Y.keys = pl.X.keys; pl.Y.deferred = false; }
    } else if (pl.X.lrank && s.kp.T == pl.T) {  // leaf-digit ranking of the first pass is valid here
      a.lrank = pl.X.lrank;
      a.offsets = pl.X.offsets;
      a.sort_tiles = (int)pl.X.tiles;
    }
    const bool tma_l2t = a.lrank && tma_supported(D, g.P, 1 << a.bits, a.nbox, false);
    if (a.lrank && tma_l2t != pl.X.lrank_sorted) {  // the other form of the tile order
      uint16_t* inv = ws.get<uint16_t>(pl.X.n, "tile order (inverse form)", g.t);
      launch_tile_invert(a.lrank, pl.X.n, inv, st);
      g_launches += 1;
      a.lrank = inv;
    }
    if (tma_l2t) {
      if (l2t_fix_supported(D, g.P, 1 << a.bits, a.nbox, a.shift)) launch_l2t_fix(D, g.P, a, tma_grid(a.num_tiles), st);
      else launch_l2t_tma(D, g.P, a, tma_grid(a.num_tiles), st);
      g_launches += 1;
      first = false;
      continue;
    }
    launch_local_l2t(D, g.P, a, local_grid(a.num_tiles), st);
    g_launches += 1;
    first = false;
  }
  if (first) {
    Span sp(tm, PH_UNPERM);
    if (vs_used && pl.X.sigma) {
      launch_unpermute(vs, pl.X.sigma, pl.X.n, v, st);
    } else if (vs_used && !pl.X.lsd_order.empty()) {
      // undo the LSD passes in reverse (coalesced per-bin runs; no random scatter)
      const int np = (int)pl.X.lsd_order.size();
      const float* cur = vs;
      float* tmp = np > 1 ? ws.get<float>((size_t)pl.X.n, "unpermute tmp") : nullptr;
      float* tmp2 = np > 2 ? ws.get<float>((size_t)pl.X.n, "unpermute tmp") : nullptr;
      for (int p = np - 1; p >= 0; --p) {
        float* dst = p == 0 ? v : ((np - 1 - p) % 2 == 0 ? tmp : tmp2);
        launch_lsd_unscatter(cur, dst, pl.X.n, pl.X.lsd_bits[p], (int)pl.X.tiles, pl.X.lsd_counts[p],
                             pl.X.lsd_order[p], st);
        g_launches += 1;
        cur = dst;
      }
    } else if (vs_used) {
      launch_unpermute_perm(vs, pl.X.perm, pl.X.n, v, st);
    }
    else CK(cudaMemsetAsync(v, 0, sizeof(float) * pl.X.n, st));
    g_launches += 1;
  }
}

// ---------------------------------------------------------------------------------------
// a9: near / small field
// ---------------------------------------------------------------------------------------
static void near_eval(Plan& pl, float* vs, Workspace& ws, cudaStream_t st) {
  const int D = pl.cfg.D;
  const Side& SY = pl.near_from_full ? pl.Yn : pl.Y;
  for (const NearGroup& ng : pl.near) {
    std::vector<NearJob> jobs;
    std::vector<int64_t> ss, sc;
    for (size_t i = 0; i < ng.tgt.size(); ++i) {
      const HBox& b = pl.X.lev[ng.t][ng.tgt[i]];
      for (int64_t s = 0; s < b.count; s += NEAR_TILE)
        jobs.push_back({b.start + s, (int32_t)std::min<int64_t>(NEAR_TILE, b.count - s), (int32_t)i, 0});
    }
    for (int64_t q : ng.src) {
      ss.push_back(SY.lev[ng.t][q].start);
      sc.push_back(SY.lev[ng.t][q].count);
    }
    for (size_t i = 0; i < ng.tgt.size(); ++i)
      for (int32_t r = ng.ptr[i]; r < ng.ptr[i + 1]; ++r)
        pl.stats.near_pairs += pl.X.lev[ng.t][ng.tgt[i]].count * sc[r];
    if (jobs.empty()) continue;
    NearJob* dj = ws.upload(jobs, "near jobs", ng.t);
    int32_t* dp = ws.upload(ng.ptr, "near csr", ng.t);
    int64_t* dss = ws.upload(ss, "near src starts", ng.t);
    int64_t* dsc = ws.upload(sc, "near src counts", ng.t);
    launch_near(D, pl.X.xs, pl.X.n, SY.xs, SY.bs, SY.n, dj, (int64_t)jobs.size(), dp, dss, dsc, pl.cfg.gamma,
                vs, st);
    g_launches += 1;
  }
}

// exact direct sum in the original order: v = k(X, Y) b  (fp32 eval, fp64 tile accumulation)
static void direct_into(const float* X, int64_t nx, const float* Y, int64_t ny, int D, const float* b, float* v,
                        double gamma, Workspace& ws, cudaStream_t st) {
  float* xs = ws.get<float>((size_t)D * nx, "soa X");
  launch_to_soa(X, nx, D, xs, st);
  const float* ys = xs;
  if (Y != X || ny != nx) {
    float* y2 = ws.get<float>((size_t)D * ny, "soa Y");
    launch_to_soa(Y, ny, D, y2, st);
    ys = y2;
    g_launches += 1;
  }
  // split the sources so that small target sets still fill the 148 SMs; fixed-order reduce
  const int64_t tiles = (nx + NEAR_TILE - 1) / NEAR_TILE;
  int splits = 1;
  while (tiles * splits < 148 * 8 && splits < 1024 && (ny / (splits * 2)) >= 4 * NEAR_TILE) splits *= 2;
  std::vector<NearJob> jobs;
  std::vector<int32_t> ptr = {0};
  std::vector<int64_t> ss, sc;
  const int64_t per = (ny + splits - 1) / splits;
  for (int sp = 0; sp < splits; ++sp) {
    const int64_t s0 = sp * per, s1 = std::min(ny, s0 + per);
    ss.push_back(s0);
    sc.push_back(std::max<int64_t>(0, s1 - s0));
    ptr.push_back(sp + 1);
    for (int64_t s = 0; s < nx; s += NEAR_TILE)
      jobs.push_back({s, (int32_t)std::min<int64_t>(NEAR_TILE, nx - s), sp, (int64_t)sp * nx});
  }
  NearJob* dj = ws.upload(jobs, "direct jobs");
  int32_t* dp = ws.upload(ptr, "direct csr");
  int64_t* dss = ws.upload(ss, "direct src");
  int64_t* dsc = ws.upload(sc, "direct cnt");
  float* out = v;
  if (splits > 1) out = ws.get<float>((size_t)splits * nx, "direct partials");
  CK(cudaMemsetAsync(out, 0, sizeof(float) * nx * splits, st));
  launch_near(D, xs, nx, ys, b, ny, dj, (int64_t)jobs.size(), dp, dss, dsc, gamma, out, st);
  g_launches += 2;
  if (splits > 1) {
    launch_reduce_splits_f32(out, splits, nx, v, st);
    g_launches += 1;
  }
}

static bool is_host_ptr(const void* p) {
  if (!p) return false;
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return true;
  }
  return a.type == cudaMemoryTypeHost || a.type == cudaMemoryTypeUnregistered;
}

// ---------------------------------------------------------------------------------------
// the whole call
// ---------------------------------------------------------------------------------------
// ---------------------------------------------------------------------------------------
// Two-digit (MSD) path for deep D = 3 trees (T_sort = 3 or 4, e.g. C4 with EV = 10): the
// leaf key splits into a top digit (depth T-2) and a two-level low digit (6 bits).  Instead
// of an LSD counting sort of the whole key into globally sorted SoA copies, one counting-sort
// scatter groups the points by top digit into buckets padded to whole tiles, and each bucket is
// then processed exactly like the single-pass headline path: a warp-specialised tile-local
// S2M ranks the bucket's tiles by the low digit (its 64 leaves) and accumulates their moments,
// and L2T runs tile-locally from the stored tile orders.  The leaf charges feed the exact
// multi-level form (M2M up, M2L per depth, L2L down; SURVEY 8(a) note 1), and the bucket-order
// result goes back to the input order by undoing the one scatter.  Same tree, same charges
// (per box) as the LSD path up to the fp32 summation order; used when the tree has no near or
// small field and every far group shares P with the deepest far depth at the leaf depth
// (otherwise, and in debug runs that inspect pi and the sorted keys, the LSD path runs).
// ---------------------------------------------------------------------------------------
static bool msd_applicable(const Plan& pl) {
  const Cfg& c = pl.cfg;
  if (c.D != 3 || !pl.aliased || c.q > 0 || (c.flags & (F3M_KEEP_EMPTY | F3M_EXACT))) return false;
  if (pl.T != 3 && pl.T != 4) return false;
  if (g_dbg.on || getenv("F3M_NO_LOCAL")) return false;
  if (!s2m_ws_supported(3, c.P, 2, 64) || !l2t_fix_supported(3, c.P, 64, 64, 0)) return false;
  return pl.X.n >= 16 * (int64_t)LT_TILE_PTS;
}

// returns false (nothing written to v) when the tree needs the globally sorted path
static bool msd_matvec(Plan& pl, float* v, Workspace& ws, cudaStream_t st, Timer& tm) {
  const int D = 3, T = pl.T, Th = T - 2, bitsA = D * Th, nbA = 1 << bitsA, P = pl.cfg.P;
  const int64_t m = (int64_t)P * P * P;
  Side& S = pl.X;
  const int64_t n = S.n;
  const int64_t tiles = (n + LT_TILE_PTS - 1) / LT_TILE_PTS;
  // ---- top digit: tile-local stable ranks (sorted-form tile orders) + per-tile counts
  uint32_t* countsA = ws.get<uint32_t>((size_t)nbA * tiles + 1, "msd counts A");
  uint16_t* orderA = ws.get<uint16_t>((size_t)n, "msd tile orders A");
  {
    Span sp(tm, PH_COUNT);
    LocalS2MArgs a{};
    a.X = S.X;
    a.b = S.b;
    a.n = n;
    a.kp = make_kp(S, D, pl.E, Th);
    a.kp.thr = ws.upload(cell_thresholds(S.alpha, D, pl.E, Th), "msd thresholds A");
    a.bits = bitsA;
    a.shift = bitsA;
    a.nbox = 1;
    for (int d = 0; d < D; ++d) a.alpha[d] = S.alpha[d];
    a.l = level_edge(pl.E, Th);
    a.nc = node_consts(2);
    a.num_tiles = (int)tiles;
    a.do_s2m = 0;
    a.counts = countsA;
    a.lrank = orderA;
    if (Th == 2 && s2m_ws_supported(D, 4, 2, 64)) {  // ranking-only warp-specialised pass
      a.shift = 0;
      a.nbox = 64;
      launch_s2m_ws(D, 4, 2, a, tma_grid((int)tiles), st);
    } else {
      launch_s2m_tma(D, 2, a, tma_grid((int)tiles), st);
    }
    uint32_t* tmp = ws.get<uint32_t>((size_t)scan_tmp_words((int64_t)nbA * tiles), "scan tmp");
    launch_scan_u32(countsA, (int64_t)nbA * tiles, tmp, st);
    g_launches += 4;
  }
  pl.passes = 2;  // (restart marker for the caller if the path declines)
  std::vector<uint32_t> startA(nbA + 1);
  CK(cudaMemcpy2DAsync(startA.data(), sizeof(uint32_t), countsA, sizeof(uint32_t) * tiles, sizeof(uint32_t), nbA,
                       cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  startA[nbA] = (uint32_t)n;
  std::vector<int64_t> nB(nbA), PB(nbA), tilesB(nbA), cboff(nbA);
  std::vector<int32_t> tile0B(nbA + 1);
  std::vector<uint32_t> pad(nbA);
  int64_t Np = 0, ctot = 0;
  for (int b = 0; b < nbA; ++b) {
    nB[b] = (int64_t)startA[b + 1] - startA[b];
    PB[b] = Np;
    tile0B[b] = (int32_t)(Np / LT_TILE_PTS);
    pad[b] = (uint32_t)(Np - startA[b]);
    tilesB[b] = (nB[b] + LT_TILE_PTS - 1) / LT_TILE_PTS;
    Np += tilesB[b] * LT_TILE_PTS;
    cboff[b] = ctot;
    ctot += 64 * tilesB[b];
  }
  tile0B[nbA] = (int32_t)(Np / LT_TILE_PTS);
  // a bucket that is empty or holds few points per leaf means small / near pairs (sparse or
  // clustered data): the sorted LSD path handles those, decline before the expensive passes
  for (int b = 0; b < nbA; ++b)
    if (nB[b] < 64 * 2 * std::max<int64_t>(pl.cfg.rho, 1)) return false;
  // unbalanced buckets mean unbalanced leaves inside them (clustered data): one 4-lane group
  // per leaf then carries most of a tile (C3-shaped clustered data at 1e8: 19.5 ms here vs 9.2 ms
  // on the LSD path), so decline when the largest bucket holds > 1.5x the mean
  {
    int64_t mx = 0;
    for (int b = 0; b < nbA; ++b) mx = std::max(mx, nB[b]);
    if ((double)mx * nbA > 1.5 * (double)n) return false;
  }
  const int tilesP = (int)(Np / LT_TILE_PTS);
  const int gridP = tma_grid(std::max(1, tilesP));
  float* xp = ws.get<float>((size_t)Np * D, "msd bucket coords");
  float* bp = ws.get<float>((size_t)Np, "msd bucket weights");
  uint32_t* pad_dev = ws.upload(pad, "msd bucket pads");
  {
    Span sp(tm, PH_SCATTER);
    launch_scatter_msd(D, S.X, S.b, n, bitsA, (int)tiles, countsA, pad_dev, orderA, xp, bp, st);
    g_launches += 1;
  }
  // ---- low digit per bucket: rank + leaf moments (warp-specialised S2M)
  const std::vector<float> thrT = cell_thresholds(S.alpha, D, pl.E, T);
  const int NT = (1 << T) - 1;
  std::vector<float> thrB((size_t)nbA * D * 3);
  std::vector<std::array<int, 3>> cb(nbA);
  std::vector<int32_t> cellB((size_t)nbA * D);
  for (int b = 0; b < nbA; ++b)
    for (int d = 0; d < D; ++d) {
      int c = 0;
      for (int sb = 0; sb < Th; ++sb) c |= ((b >> (D * sb + d)) & 1) << sb;
      cb[b][d] = 4 * c;
      cellB[(size_t)b * D + d] = 4 * c;
      for (int j = 0; j < 3; ++j) thrB[((size_t)b * D + d) * 3 + j] = thrT[(size_t)d * NT + 4 * c + j];
    }
  float* thrB_dev = ws.upload(thrB, "msd thresholds B");
  uint32_t* countsB = ws.get<uint32_t>((size_t)ctot + 1, "msd counts B");
  CK(cudaMemsetAsync(countsB + ctot, 0, sizeof(uint32_t), st));
  uint16_t* orderB = ws.get<uint16_t>((size_t)Np, "msd tile orders B");
  // one launch over every bucket: Wpart[bucket][CTA][leaf][m], written by the CTAs whose tile
  // range meets the bucket (only those slices are reduced)
  const size_t wcount = (size_t)nbA * gridP * 64 * m;
  float* wpart = ws.get<float>(wcount, "msd s2m partials");
  const int tpbP = (tilesP + gridP - 1) / gridP;  // the kernel's tiles per CTA
  const double lT = level_edge(pl.E, T);
  {
    Span sp(tm, PH_S2M);
    LocalS2MArgs a{};
    a.X = xp;
    a.b = bp;
    a.n = Np;
    a.kp.D = D;
    a.kp.T = 2;
    a.kp.thr = thrB_dev;
    a.bits = 6;
    a.shift = 0;
    a.nbox = 64;
    for (int d = 0; d < D; ++d) a.alpha[d] = S.alpha[d];
    a.l = lT;
    a.nc = node_consts(P);
    a.num_tiles = tilesP;
    a.do_s2m = 1;
    a.Wpart = wpart;
    a.counts = countsB;
    a.lrank = orderB;
    a.nbuckets = nbA;
    a.bk_tile0 = ws.upload(tile0B, "msd bucket tiles");
    a.bk_n = ws.upload(nB, "msd bucket sizes");
    int2* tinfo = ws.get<int2>((size_t)std::max(1, tilesP), "msd tile table");
    launch_bucket_tiles(a.bk_tile0, a.bk_n, nbA, tilesP, tinfo, st);
    a.bk_tile = tinfo;
    a.bk_thr = thrB_dev;
    a.bk_cell = ws.upload(cellB, "msd bucket cells");
    a.bk_coff = ws.upload(cboff, "msd bucket count offsets");
    launch_s2m_ws(D, P, 2, a, gridP, st);
    g_launches += 1;
  }
  // ---- leaf table from the global scan of the per-bucket [leaf][tile] counts
  {
    Span sp(tm, PH_SCAN);
    uint32_t* tmp = ws.get<uint32_t>((size_t)scan_tmp_words(ctot + 1), "scan tmp");
    launch_scan_u32(countsB, ctot + 1, tmp, st);
    g_launches += 3;
  }
  std::vector<int64_t> gidx;
  std::vector<uint64_t> gkey;
  for (int b = 0; b < nbA; ++b)
    if (nB[b] > 0)
      for (int sub = 0; sub < 64; ++sub) {
        gidx.push_back(cboff[b] + (int64_t)sub * tilesB[b]);
        gkey.push_back(((uint64_t)b << 6) | (uint64_t)sub);
      }
  gidx.push_back(ctot);
  uint32_t* gst = ws.get<uint32_t>(gidx.size(), "msd leaf starts");
  launch_gather_u32(countsB, ws.upload(gidx, "msd leaf index"), (int64_t)gidx.size(), gst, st);
  g_launches += 1;
  std::vector<uint32_t> lst(gidx.size());
  CK(cudaMemcpyAsync(lst.data(), gst, sizeof(uint32_t) * lst.size(), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  S.leaf_key.clear();
  S.leaf_start.clear();
  S.leaf_count.clear();
  std::vector<int> leaf_bucket;
  for (size_t i = 0; i + 1 < lst.size(); ++i) {
    const int64_t c = (int64_t)lst[i + 1] - (int64_t)lst[i];
    if (c > 0) {
      S.leaf_key.push_back(gkey[i]);
      S.leaf_start.push_back(lst[i]);
      S.leaf_count.push_back(c);
      leaf_bucket.push_back((int)(gkey[i] >> 6));
    }
  }
  S.leaf_gcount = S.leaf_count;
  {
    Span sp(tm, PH_TREE);
    build_levels(S, D, T, false);
    pl.Y = pl.X;
    run_alg1(pl, st);
  }
  pl.passes = 2;
  pl.stats.far_groups_local = (int32_t)pl.far.size();  // every far group runs tile-locally here
  int tmin = T + 1, tmax = -1;
  for (const FarGroup& g : pl.far) {
    if (g.P != P || g.q > 0) return false;
    tmin = std::min(tmin, g.t);
    tmax = std::max(tmax, g.t);
  }
  if (!pl.near.empty() || pl.far.empty() || tmax != T) return false;
  // ---- leaf charges (moments -> nodal), M2M up, group rows
  const int64_t nleaf = (int64_t)S.lev[T].size();
  std::vector<double*> Wl(T + 1, nullptr);
  Wl[T] = ws.get<double>((size_t)nleaf * m, "level charges", T);
  FarBuffers fb;
  {
    Span sp(tm, PH_S2M);
    std::vector<int64_t> first(nbA + 1, 0);
    for (int64_t i = 0; i < nleaf; ++i) first[leaf_bucket[i] + 1]++;
    for (int b = 0; b < nbA; ++b) first[b + 1] += first[b];
    std::vector<int32_t> sbox(nleaf);
    for (int64_t i = 0; i < nleaf; ++i) sbox[i] = (int32_t)(S.leaf_key[i] & 63u);
    int32_t* sbox_dev = ws.upload(sbox, "msd leaf sub-boxes");
    for (int b = 0; b < nbA; ++b) {
      const int64_t ns = first[b + 1] - first[b];
      if (ns == 0) continue;
      const int c_lo = tile0B[b] / tpbP, c_hi = (tile0B[b + 1] - 1) / tpbP;  // CTAs meeting bucket b
      launch_local_reduce(wpart + ((size_t)b * gridP + c_lo) * 64 * m, c_hi - c_lo + 1, 64, (int)m,
                          sbox_dev + first[b], (int)ns, Wl[T] + first[b] * m, st);
      g_launches += 1;
    }
    launch_cheb_transform(Wl[T], (int)nleaf, D, P, 0, st);  // moments -> nodal charges
    for (int t = T - 1; t >= tmin; --t) {
      const LevelLinks lk = level_links(S.lev[t], nullptr, D, ws, t);
      const LevelLinks lc = level_links(S.lev[t + 1], &S.lev[t], D, ws, t + 1);
      Wl[t] = ws.get<double>(S.lev[t].size() * m, "level charges", t);
      double* scr = ws.get<double>((size_t)S.lev[t].size() * m2m_split(D, (int)S.lev[t].size()) * m, "m2m partials", t);
      launch_m2m(D, P, (int)m, (int)S.lev[t].size(), lk.child0, lk.nchild, lc.bits, Wl[t + 1], Wl[t], scr, st);
      g_launches += 1;
    }
    for (const FarGroup& g : pl.far) {
      fb.w_off.push_back(fb.w_total);
      fb.w_total += (int64_t)g.src.size() * g.m;
    }
    fb.W = ws.get<double>(fb.w_total, "charges");
    for (size_t gi = 0; gi < pl.far.size(); ++gi) {
      const FarGroup& g = pl.far[gi];
      std::vector<int32_t> idx(g.src.begin(), g.src.end());
      launch_rows(Wl[g.t], ws.upload(idx, "group rows", g.t), (int64_t)idx.size(), (int)m, fb.W + fb.w_off[gi], false, st);
      g_launches += 1;
    }
    for (const FarGroup& g : pl.far)
      for (int64_t q : g.src) pl.stats.s2m_points += S.lev[g.t][q].count;
  }
  // ---- M2L per group
  {
    Span sp(tm, PH_M2L);
    for (size_t gi = 0; gi < pl.far.size(); ++gi) {
      const FarGroup& g = pl.far[gi];
      const double l = level_edge(pl.E, g.t);
      int maxr = 1;
      for (int d = 0; d < D; ++d) maxr = std::max(maxr, g.range[d]);
      const int stride = maxr * g.P * g.P;
      float* tables = ws.get<float>((size_t)D * stride, "m2l tables", g.t);
      launch_m2l_tables(D, g.P, g.delta0, l, g.range, pl.cfg.gamma, node_consts(g.P), tables, stride, st);
      int32_t* dptr = g.d_ptr ? g.d_ptr : ws.upload(g.ptr, "m2l csr", g.t);
      int32_t* dcol = g.d_col ? g.d_col : ws.upload(g.col, "m2l cols", g.t);
      uint64_t* doff = g.d_off ? g.d_off : ws.upload(g.off, "m2l offsets", g.t);
      double* U = ws.get<double>(g.tgt.size() * g.m, "locals", g.t);
      float* W32 = ws.get<float>(g.src.size() * g.m, "charges fp32", g.t);
      launch_to_f32(fb.W + fb.w_off[gi], (int64_t)(g.src.size() * g.m), W32, st);
      launch_m2l(D, g.P, (int32_t)g.tgt.size(), dptr, dcol, doff, tables, stride, W32, U, st);
      g_launches += 3;
      fb.U.push_back(U);
    }
  }
  // ---- L2L down to the leaves, then tile-local L2T per bucket (bucket order)
  float* vb = ws.get<float>((size_t)Np, "msd bucket output");
  {
    Span sp(tm, PH_L2T);
    std::vector<double*> Ul(T + 1, nullptr);
    for (int t = tmin; t <= T; ++t) {
      Ul[t] = ws.get<double>(S.lev[t].size() * m, "level locals", t);
      CK(cudaMemsetAsync(Ul[t], 0, sizeof(double) * S.lev[t].size() * m, st));
    }
    for (size_t gi = 0; gi < pl.far.size(); ++gi) {
      const FarGroup& g = pl.far[gi];
      std::vector<int32_t> idx(g.tgt.begin(), g.tgt.end());
      launch_rows(fb.U[gi], ws.upload(idx, "group rows", g.t), (int64_t)idx.size(), (int)m, Ul[g.t], true, st);
      g_launches += 1;
    }
    for (int t = tmin; t < T; ++t) {
      const LevelLinks lc = level_links(S.lev[t + 1], &S.lev[t], D, ws, t + 1);
      launch_l2l(D, P, (int)m, (int)S.lev[t + 1].size(), lc.parent, lc.bits, Ul[t], Ul[t + 1], st);
      g_launches += 1;
    }
    launch_cheb_transform(Ul[T], (int)nleaf, D, P, 1, st);  // nodal -> Chebyshev coefficients
    g_launches += 1;
    std::vector<int32_t> slot((size_t)nbA * 64, -1);
    std::vector<int64_t> first(nbA, -1);
    for (int64_t i = 0; i < nleaf; ++i) {
      const int b = leaf_bucket[i];
      if (first[b] < 0) first[b] = i;
      slot[(size_t)b * 64 + (S.leaf_key[i] & 63u)] = (int32_t)(i - first[b]);
    }
    int32_t* slot_dev = ws.upload(slot, "msd leaf slots");
    for (int b = 0; b < nbA; ++b) {
      if (nB[b] == 0) continue;
      LocalL2TArgs a{};
      a.X = xp + PB[b] * D;
      a.n = nB[b];
      a.kp.D = D;
      a.kp.T = 2;
      a.bits = 6;
      a.shift = 0;
      a.nbox = 64;
      for (int d = 0; d < D; ++d) {
        a.alpha[d] = S.alpha[d];
        a.cell_base[d] = cb[b][d];
      }
      a.l = lT;
      a.nc = node_consts(P);
      a.num_tiles = (int)tilesB[b];
      a.U = Ul[T] + (first[b] < 0 ? 0 : first[b]) * m;
      a.box_slot = slot_dev + (size_t)b * 64;
      a.v = vb + PB[b];
      a.accumulate = 0;
      a.offsets = countsB + cboff[b];
      a.sort_tiles = (int)tilesB[b];
      a.offsets_tail = 1;
      a.lrank = orderB + PB[b];
      launch_l2t_fix(D, P, a, tma_grid((int)tilesB[b]), st);
      g_launches += 1;
    }
    pl.stats.l2t_points += n;
  }
  {
    Span sp(tm, PH_UNPERM);
    launch_lsd_unscatter(vb, v, n, bitsA, (int)tiles, countsA, orderA, st, pad_dev);
    g_launches += 1;
  }
  return true;
}

static void matvec(const float* X, int64_t nx, const float* Y, int64_t ny, int D, const float* b, float* v,
                   const f3m_kernel* k, const f3m_config* cfgp, const f3m_allocator* alloc, cudaStream_t st,
                   f3m_stats* stats) {
  Plan pl;
  pl.cfg = resolve(D, k, cfgp);
  if (nx < 1) throw Fail{F3M_ERR_INVALID_INPUT, "nx must be >= 1"};
  if (!X || !b || !v) throw Fail{F3M_ERR_INVALID_INPUT, "NULL X, b or v"};
  pl.aliased = (Y == nullptr);
  if (pl.aliased) ny = nx;
  if (ny < 1) throw Fail{F3M_ERR_INVALID_INPUT, "ny must be >= 1"};
  if (nx >= (1ll << 31) || ny >= (1ll << 31)) throw Fail{F3M_ERR_INVALID_INPUT, "n >= 2^31 per call"};
  g_launches = 0;
  Timer tm;
  tm.st = st;
  const char* te = getenv("F3M_TIMING");
  tm.on = (te && te[0] == '1');
  Workspace ws(st, alloc);
  pl.ws = &ws;
  cudaEvent_t t_all = nullptr;
  tm.begin(PH_TOTAL, t_all);

  // host staging (the e2e path): inputs copied to the device on the call stream
  const bool hX = is_host_ptr(X), hY = Y && is_host_ptr(Y), hb = is_host_ptr(b), hv = is_host_ptr(v);
  if (hX) {
    float* d = ws.get<float>((size_t)nx * D, "X staging");
    CK(cudaMemcpyAsync(d, X, sizeof(float) * nx * D, cudaMemcpyHostToDevice, st));
    X = d;
  }
  if (hY) {
    float* d = ws.get<float>((size_t)ny * D, "Y staging");
    CK(cudaMemcpyAsync(d, Y, sizeof(float) * ny * D, cudaMemcpyHostToDevice, st));
    Y = d;
  }
  if (hb) {
    float* d = ws.get<float>((size_t)ny, "b staging");
    CK(cudaMemcpyAsync(d, b, sizeof(float) * ny, cudaMemcpyHostToDevice, st));
    b = d;
  }
  float* vhost = nullptr;
  if (hv) {
    vhost = v;
    v = ws.get<float>((size_t)nx, "v staging");
  }

  pl.X.X = X;
  pl.X.n = nx;
  pl.X.b = pl.aliased ? b : nullptr;
  pl.Y.X = pl.aliased ? X : Y;
  pl.Y.n = ny;
  pl.Y.b = b;
  {
    Span sp(tm, PH_BBOX);
    bbox(pl.X, D, ws, st);
    if (pl.aliased) pl.Y = pl.X, pl.Y.b = b;
    else bbox(pl.Y, D, ws, st);
  }
  pl.E = enclosing_edge(pl.X, pl.Y, D);
  bool direct_only = (pl.E == 0.0) || (pl.cfg.flags & F3M_EXACT);
  if (!direct_only) {
    level_scalars(pl);
    if (pl.T < 1) direct_only = true;
  }
  if (!direct_only && (pl.cfg.flags & F3M_KEEP_EMPTY) && (int64_t)D * pl.T > 24)
    throw Fail{F3M_ERR_RESOURCE, "F3M_KEEP_EMPTY (no empty-box removal) needs D * T_sort <= 24"};
  if (g_dbg.on) g_dbg.reset();
  if (direct_only) {
    Span sp(tm, PH_NEAR);
    direct_into(X, nx, pl.Y.X, ny, D, b, v, pl.cfg.gamma, ws, st);
  } else if (msd_applicable(pl) && msd_matvec(pl, v, ws, st, tm)) {
    // two-digit path done (v written)
  } else {
    if (pl.passes == 2) {  // the two-digit path declined after its tree: restart from the sort
      pl.far.clear();
      pl.near.clear();
      pl.stats = f3m_stats{};
    }
    {
      sort_side(pl, pl.X, pl.aliased, true, g_dbg.on && g_dbg.level == 1, ws, st, tm, true);
      if (pl.aliased) pl.Y = pl.X;
      else sort_side(pl, pl.Y, true, false, g_dbg.on && g_dbg.level == 1, ws, st, tm, true);
    }
    Spec spec;
    if (pl.aliased) {
      first_pass(pl, pl.X, true, spec, ws, st, tm);
      pl.Y = pl.X;
    } else {
      first_pass(pl, pl.Y, true, spec, ws, st, tm);
      Spec none;
      first_pass(pl, pl.X, false, none, ws, st, tm);
    }
    {
      Span sp(tm, PH_TREE);
      build_levels(pl.X, D, pl.T, pl.cfg.flags & F3M_KEEP_EMPTY);
      if (pl.aliased) pl.Y.lev = pl.X.lev;
      else build_levels(pl.Y, D, pl.T, pl.cfg.flags & F3M_KEEP_EMPTY);
      run_alg1(pl, st);
    }
    FarBuffers fb;
    far_s2m(pl, fb, spec, ws, st, tm);
    float* vs = nullptr;
    const bool sorted_parts = needs_sorted(pl);
    if (sorted_parts) {
      vs = ws.get<float>((size_t)nx, "sorted output");
      CK(cudaMemsetAsync(vs, 0, sizeof(float) * nx, st));
    }
    bool vs_used = far_eval(pl, fb, vs, ws, st, tm);
    if (!pl.near.empty()) {
      Span sp(tm, PH_NEAR);
      near_eval(pl, vs, ws, st);
      vs_used = true;
    }
    finish_output(pl, fb, vs, vs_used, v, ws, st, tm);
    if (g_dbg.on && g_dbg.level == 2) {
      CK(cudaStreamSynchronize(st));
      g_dbg.perm32.resize(pl.X.n);
      CK(cudaMemcpy(g_dbg.perm32.data(), pl.X.perm, sizeof(int32_t) * pl.X.n, cudaMemcpyDeviceToHost));
    } else if (g_dbg.on) {
      CK(cudaStreamSynchronize(st));
      for (int side = 0; side < 2; ++side) {
        const Side& S = side == 0 ? pl.X : pl.Y;
        std::vector<int32_t> p32(S.n);
        CK(cudaMemcpy(p32.data(), S.perm, sizeof(int32_t) * S.n, cudaMemcpyDeviceToHost));
        g_dbg.perm[side].assign(p32.begin(), p32.end());
        g_dbg.keys[side].resize(S.n);
        if (S.keys) CK(cudaMemcpy(g_dbg.keys[side].data(), S.keys, sizeof(uint64_t) * S.n, cudaMemcpyDeviceToHost));
      }
    }
  }
  if (hv) CK(cudaMemcpyAsync(vhost, v, sizeof(float) * nx, cudaMemcpyDeviceToHost, st));
  tm.end(PH_TOTAL, t_all);
  CK(cudaGetLastError());
  ws.release();
  CK(cudaStreamSynchronize(st));
  if (stats) {
    *stats = pl.stats;
    stats->num_sort_passes = pl.passes;
    stats->t_star = pl.t_star;
    stats->t_sort = pl.T;
    stats->E = pl.E;
    stats->kernel_launches = (int32_t)g_launches;
    tm.collect(stats->ms_phase);
  }
}

static void direct_call(const float* X, int64_t nx, const float* Y, int64_t ny, int D, const float* b, void* v,
                        int fp64, const f3m_kernel* k, cudaStream_t st) {
  if (D < 1 || D > 7) throw Fail{F3M_ERR_INVALID_INPUT, "D must be in [1, 7]"};
  if (!k || !(k->lengthscale > 0.0)) throw Fail{F3M_ERR_INVALID_SPEC, "lengthscale must be > 0"};
  if (nx < 1 || (Y && ny < 1)) throw Fail{F3M_ERR_INVALID_INPUT, "nx, ny must be >= 1"};
  if (!X || !b || !v) throw Fail{F3M_ERR_INVALID_INPUT, "X, b and v must be non-NULL device pointers"};
  if (is_host_ptr(X) || is_host_ptr(b) || is_host_ptr(v) || (Y && is_host_ptr(Y)))
    throw Fail{F3M_ERR_INVALID_INPUT, "f3m_direct takes device pointers only (X, Y, b, v)"};
  if (!Y) { Y = X; ny = nx; }
  Workspace ws(st, nullptr);
  g_launches = 0;
  if (fp64) {
    float* xs = ws.get<float>((size_t)D * nx, "soa X");
    float* ys = ws.get<float>((size_t)D * ny, "soa Y");
    launch_to_soa(X, nx, D, xs, st);
    launch_to_soa(Y, ny, D, ys, st);
    const int64_t tiles = (nx + NEAR_TILE - 1) / NEAR_TILE;
    int splits = 1;
    while (tiles * splits < 148 * 8 && splits < 4096 && (ny / (splits * 2)) >= 4 * NEAR_TILE) splits *= 2;
    double* part = ws.get<double>((size_t)splits * nx, "direct partials");
    launch_direct_f64(D, xs, nx, ys, b, ny, k->lengthscale, splits, part, st);
    launch_reduce_splits_f64(part, splits, nx, static_cast<double*>(v), st);
    g_launches += 4;
  } else {
    direct_into(X, nx, Y, ny, D, b, static_cast<float*>(v), k->lengthscale, ws, st);
  }
  CK(cudaGetLastError());
  ws.release();
  CK(cudaStreamSynchronize(st));
}

}  // namespace f3m

// =======================================================================================
// C ABI
// =======================================================================================
using namespace f3m;

#define F3M_TRY(...)                           \
  try {                                        \
    __VA_ARGS__;                               \
    return F3M_OK;                             \
  } catch (const Fail& f) {                    \
    g_err = f.msg;                             \
    return f.st;                               \
  } catch (const std::bad_alloc&) {            \
    g_err = "host out of memory";              \
    return F3M_ERR_RESOURCE;                   \
  } catch (const std::exception& e) {          \
    g_err = e.what();                          \
    return F3M_ERR_INTERNAL;                   \
  }

extern "C" {

const char* f3m_last_error(void) { return g_err.c_str(); }
const char* f3m_version(void) { return "f3m-b200 0.2 (sm_100a)"; }
const char* f3m_phase_name(int32_t i) { return (i >= 0 && i < PH_N) ? kPhaseNames[i] : ""; }

f3m_status f3m_default_config(int32_t D, f3m_config* out) {
  if (!out) return F3M_ERR_INVALID_INPUT;
  if (D < 1 || D > 7) return F3M_ERR_INVALID_INPUT;
  out->nodes_per_dim = 4;
  out->node_cap = 2048;
  out->eta = 0.5;
  int64_t m = 1;
  for (int d = 0; d < D; ++d) m *= 4;
  out->rho = 2 * m;
  out->zeta = m;
  out->max_depth = 63 / D;
  out->flags = 0;
  out->sparse_level = 0;
  return F3M_OK;
}

f3m_status f3m_matvec(const float* X, int64_t nx, const float* Y, int64_t ny, int32_t D, const float* b, float* v,
                      const f3m_kernel* k, const f3m_config* cfg, const f3m_allocator* alloc, void* cuda_stream,
                      f3m_stats* stats) {
  std::unique_lock<std::mutex> lk(g_dbg_mu, std::defer_lock);
  if (g_dbg.on) lk.lock();
  F3M_TRY(matvec(X, nx, Y, ny, D, b, v, k, cfg, alloc, static_cast<cudaStream_t>(cuda_stream), stats));
}

f3m_status f3m_direct(const float* X, int64_t nx, const float* Y, int64_t ny, int32_t D, const float* b, void* v,
                      int32_t fp64, const f3m_kernel* k, void* cuda_stream) {
  F3M_TRY(direct_call(X, nx, Y, ny, D, b, v, fp64, k, static_cast<cudaStream_t>(cuda_stream)));
}

void f3m_debug_enable(int32_t on) {
  std::lock_guard<std::mutex> lk(g_dbg_mu);
  g_dbg.on = on != 0;
  g_dbg.level = on;
  g_dbg.reset();
}

f3m_status f3m_debug_last_perm32(int32_t* perm_host, int64_t n) {
  if ((int64_t)g_dbg.perm32.size() != n) return F3M_ERR_INVALID_INPUT;
  std::memcpy(perm_host, g_dbg.perm32.data(), sizeof(int32_t) * n);
  return F3M_OK;
}

f3m_status f3m_debug_last_perm(int32_t side, int64_t* perm_host, int64_t n) {
  if (side < 0 || side > 1 || (int64_t)g_dbg.perm[side].size() != n) return F3M_ERR_INVALID_INPUT;
  std::memcpy(perm_host, g_dbg.perm[side].data(), sizeof(int64_t) * n);
  return F3M_OK;
}

f3m_status f3m_debug_last_keys(int32_t side, uint64_t* keys_host, int64_t n) {
  if (side < 0 || side > 1 || (int64_t)g_dbg.keys[side].size() != n) return F3M_ERR_INVALID_INPUT;
  std::memcpy(keys_host, g_dbg.keys[side].data(), sizeof(uint64_t) * n);
  return F3M_OK;
}

int64_t f3m_debug_num_pairs(int32_t t) {
  if (t < 0 || t >= (int32_t)g_dbg.tag.size()) return 0;
  return (int64_t)g_dbg.tag[t].size();
}

f3m_status f3m_debug_pairs(int32_t t, uint64_t* kp, uint64_t* kq, int32_t* tag) {
  if (t < 0 || t >= (int32_t)g_dbg.tag.size()) return F3M_ERR_INVALID_INPUT;
  for (size_t i = 0; i < g_dbg.tag[t].size(); ++i) {
    kp[i] = g_dbg.kp[t][i];
    kq[i] = g_dbg.kq[t][i];
    tag[i] = g_dbg.tag[t][i];
  }
  return F3M_OK;
}

int32_t f3m_debug_num_charge_sets(void) { return (int32_t)g_dbg.charges.size(); }

f3m_status f3m_debug_charge_info(int32_t i, int64_t* info) {
  if (i < 0 || i >= (int32_t)g_dbg.charges.size()) return F3M_ERR_INVALID_INPUT;
  const DebugCharges& c = g_dbg.charges[i];
  info[0] = c.t;
  info[1] = c.P;
  info[2] = (int64_t)c.sk.size();
  info[3] = (int64_t)c.tk.size();
  info[4] = c.m;
  info[5] = c.q;
  return F3M_OK;
}

f3m_status f3m_debug_charges(int32_t i, uint64_t* src_key, double* W, uint64_t* tgt_key, double* U) {
  if (i < 0 || i >= (int32_t)g_dbg.charges.size()) return F3M_ERR_INVALID_INPUT;
  const DebugCharges& c = g_dbg.charges[i];
  std::memcpy(src_key, c.sk.data(), sizeof(uint64_t) * c.sk.size());
  std::memcpy(W, c.W.data(), sizeof(double) * c.W.size());
  std::memcpy(tgt_key, c.tk.data(), sizeof(uint64_t) * c.tk.size());
  std::memcpy(U, c.U.data(), sizeof(double) * c.U.size());
  return F3M_OK;
}

}  // extern "C"

// =======================================================================================
// Plan API (sharded targets): the caller all-reduces between the stages
// =======================================================================================
struct f3m_plan {
  f3m::Plan pl;
  cudaStream_t st = nullptr;
  f3m::Workspace* ws = nullptr;
  int stage = 0;
  uint64_t* keys_dev = nullptr;   // local non-empty leaves (key ascending) and their counts
  int64_t* counts_dev = nullptr;
  std::vector<uint64_t> local_key;
  std::vector<int64_t> local_count;
  const float* Yfull = nullptr;   // replicated sources for the near / small field (may be NULL)
  const float* bfull = nullptr;
  int64_t ny = 0;
  f3m_allocator alloc{};          // the caller's allocator (copied: it must not outlive the call)
  f3m::FarBuffers fb;
  f3m::Spec spec;
  f3m::Timer tm;  // per-phase CUDA events across the stages (F3M_TIMING=1)
  ~f3m_plan() { delete ws; }
};

namespace f3m {

// Stage 2: the global cube -> keys, the local counting sort (fused with the speculative S2M of
// the first tile-local pass), and this rank's non-empty leaves as a sparse (key, count) list.
static void plan_leaves(f3m_plan* P, const double* mm, uint64_t** keys_dev, int64_t** counts_dev, int64_t* len) {
  Plan& pl = P->pl;
  const int D = pl.cfg.D;
  if (P->stage != 1) throw Fail{F3M_ERR_INVALID_INPUT, "f3m_plan_leaves must follow f3m_plan_bbox"};
  double E = 0.0;
  for (int d = 0; d < D; ++d) {
    pl.X.alpha[d] = mm[d];
    pl.X.mn[d] = (float)mm[d];
    if ((double)pl.X.mn[d] != mm[d]) throw Fail{F3M_ERR_INVALID_INPUT, "global minima must be fp32 values"};
    E = std::max(E, mm[D + d] - mm[d]);
  }
  pl.E = E;
  if (E == 0.0 || (pl.cfg.flags & F3M_EXACT)) throw Fail{F3M_ERR_INVALID_INPUT, "degenerate cube / exact mode is not sharded"};
  level_scalars(pl);
  if (pl.T < 1) throw Fail{F3M_ERR_INVALID_INPUT, "sharded mode needs T_sort >= 1"};
  Timer& tm = P->tm;
  sort_side(pl, pl.X, true, true, false, *P->ws, P->st, tm, true);
  first_pass(pl, pl.X, true, P->spec, *P->ws, P->st, tm);
  P->local_key = pl.X.leaf_key;
  P->local_count = pl.X.leaf_count;
  const int64_t nl = (int64_t)P->local_key.size();
  P->keys_dev = nl ? P->ws->upload(P->local_key, "local leaf keys") : nullptr;
  P->counts_dev = nl ? P->ws->upload(P->local_count, "local leaf counts") : nullptr;
  *keys_dev = P->keys_dev;
  *counts_dev = P->counts_dev;
  *len = nl;
  P->stage = 2;
}

// Stage 3: the concatenation of every rank's (key, count) lists (any order; equal keys are
// summed) -> the global leaf table; every rank then builds the identical tree (Alg. 1).
static void plan_set_leaves(f3m_plan* P, const uint64_t* keys, const int64_t* counts, int64_t len) {
  Plan& pl = P->pl;
  if (P->stage != 2) throw Fail{F3M_ERR_INVALID_INPUT, "f3m_plan_set_leaves must follow f3m_plan_leaves"};
  if (len < 0 || (len > 0 && (!keys || !counts))) throw Fail{F3M_ERR_INVALID_INPUT, "bad leaf list"};
  std::vector<uint64_t> k(len);
  std::vector<int64_t> c(len);
  const bool host = len > 0 && is_host_ptr(keys);
  if (len > 0) {
    if (host) {
      std::memcpy(k.data(), keys, sizeof(uint64_t) * len);
      std::memcpy(c.data(), counts, sizeof(int64_t) * len);
    } else {
      CK(cudaMemcpyAsync(k.data(), keys, sizeof(uint64_t) * len, cudaMemcpyDeviceToHost, P->st));
      CK(cudaMemcpyAsync(c.data(), counts, sizeof(int64_t) * len, cudaMemcpyDeviceToHost, P->st));
      CK(cudaStreamSynchronize(P->st));
    }
  }
  const int D = pl.cfg.D;
  const uint64_t kmax = D * pl.T >= 64 ? ~0ull : (1ull << (D * pl.T)) - 1ull;
  std::vector<int64_t> idx(len);
  for (int64_t i = 0; i < len; ++i) {
    if (k[i] > kmax || c[i] < 0) throw Fail{F3M_ERR_INVALID_INPUT, "leaf key out of range or negative count"};
    idx[i] = i;
  }
  std::sort(idx.begin(), idx.end(), [&](int64_t a, int64_t b) { return k[a] < k[b]; });
  Side& S = pl.X;
  S.leaf_key.clear();
  S.leaf_start.clear();
  S.leaf_count.clear();
  S.leaf_gcount.clear();
  size_t li = 0;  // walk the local list alongside
  int64_t run = 0;
  for (int64_t i = 0; i < len;) {
    const uint64_t key = k[idx[i]];
    int64_t g = 0;
    for (; i < len && k[idx[i]] == key; ++i) g += c[idx[i]];
    if (g == 0) continue;
    int64_t loc = 0;
    while (li < P->local_key.size() && P->local_key[li] < key)
      throw Fail{F3M_ERR_INVALID_INPUT, "a local leaf is missing from the global list"};
    if (li < P->local_key.size() && P->local_key[li] == key) loc = P->local_count[li++];
    if (g < loc) throw Fail{F3M_ERR_INVALID_INPUT, "global counts smaller than local counts"};
    S.leaf_key.push_back(key);
    S.leaf_start.push_back(run);
    S.leaf_count.push_back(loc);
    S.leaf_gcount.push_back(g);
    run += loc;
  }
  if (li != P->local_key.size()) throw Fail{F3M_ERR_INVALID_INPUT, "a local leaf is missing from the global list"};
  {
    Span sp(P->tm, PH_TREE);
    build_levels(S, D, pl.T, pl.cfg.flags & F3M_KEEP_EMPTY);
    pl.Y = pl.X;
    run_alg1(pl, P->st);
  }
  P->stage = 3;
}

// The near / small field needs the sources of every rank: sort the replicated Yfull with the
// global cube (one counting sort; skipped when the tree has no near / small pairs, e.g. C4).
static void plan_near_sources(f3m_plan* P) {
  Plan& pl = P->pl;
  if (pl.near.empty()) return;
  if (!P->Yfull || !P->bfull)
    throw Fail{F3M_ERR_INVALID_INPUT,
               "the tree has near/small pairs: the sharded flow needs the replicated sources (Yfull, bfull)"};
  const int D = pl.cfg.D;
  Side& Yn = pl.Yn;
  Yn = Side{};
  Yn.X = P->Yfull;
  Yn.b = P->bfull;
  Yn.n = P->ny;
  for (int d = 0; d < D; ++d) {
    Yn.alpha[d] = pl.X.alpha[d];
    Yn.mn[d] = pl.X.mn[d];
  }
  Timer& tm = P->tm;
  sort_side(pl, Yn, true, false, false, *P->ws, P->st, tm, false);
  // its leaves must be exactly the global leaf table (the ranks' slices partition Yfull)
  if (Yn.leaf_key != pl.X.leaf_key || Yn.leaf_count != pl.X.leaf_gcount)
    throw Fail{F3M_ERR_INVALID_INPUT, "Yfull does not match the union of the ranks' shards (global leaf counts differ)"};
  Yn.leaf_gcount = Yn.leaf_count;
  build_levels(Yn, D, pl.T, pl.cfg.flags & F3M_KEEP_EMPTY);
  pl.near_from_full = true;
}

static void plan_s2m(f3m_plan* P, double** charges, int64_t* len) {
  Plan& pl = P->pl;
  if (P->stage != 3) throw Fail{F3M_ERR_INVALID_INPUT, "f3m_plan_s2m must follow f3m_plan_set_leaves"};
  plan_near_sources(P);
  Timer& tm = P->tm;
  far_s2m(pl, P->fb, P->spec, *P->ws, P->st, tm);
  *charges = P->fb.W;
  *len = P->fb.w_total;
  P->stage = 4;
}

static void plan_evaluate(f3m_plan* P, float* v, f3m_stats* stats) {
  Plan& pl = P->pl;
  if (P->stage != 4) throw Fail{F3M_ERR_INVALID_INPUT, "f3m_plan_evaluate must follow f3m_plan_s2m"};
  Timer& tm = P->tm;
  float* vs = nullptr;
  if (needs_sorted(pl)) {
    vs = P->ws->get<float>((size_t)pl.X.n, "sorted output");
    CK(cudaMemsetAsync(vs, 0, sizeof(float) * pl.X.n, P->st));
  }
  bool vs_used = far_eval(pl, P->fb, vs, *P->ws, P->st, tm);
  if (!pl.near.empty()) {
    near_eval(pl, vs, *P->ws, P->st);
    vs_used = true;
  }
  finish_output(pl, P->fb, vs, vs_used, v, *P->ws, P->st, tm);
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(P->st));
  if (stats) {
    *stats = pl.stats;
    stats->num_sort_passes = pl.passes;
    stats->t_star = pl.t_star;
    stats->t_sort = pl.T;
    stats->E = pl.E;
    stats->kernel_launches = (int32_t)g_launches;
    tm.collect(stats->ms_phase);
  }
  P->stage = 5;
}

}  // namespace f3m

extern "C" {

f3m_status f3m_plan_create(const float* Xlocal, int64_t nx_local, const float* Ylocal, int64_t ny_local,
                           const float* blocal, const float* Yfull, const float* bfull, int64_t ny, int32_t D,
                           const f3m_kernel* k, const f3m_config* cfg, const f3m_allocator* alloc, void* cuda_stream,
                           f3m_plan** out) {
  F3M_TRY({
    if (!out) throw Fail{F3M_ERR_INVALID_INPUT, "out is NULL"};
    *out = nullptr;
    if (!Xlocal || !blocal || nx_local < 1 || nx_local >= (1ll << 31)) throw Fail{F3M_ERR_INVALID_INPUT, "bad local shard"};
    if (Ylocal && (Ylocal != Xlocal || ny_local != nx_local))
      throw Fail{F3M_ERR_INVALID_INPUT, "the sharded flow is the k(X, X) case: Ylocal must be NULL or Xlocal"};
    if ((Yfull != nullptr) != (bfull != nullptr)) throw Fail{F3M_ERR_INVALID_INPUT, "Yfull and bfull go together"};
    if (Yfull && (ny < nx_local || ny >= (1ll << 31))) throw Fail{F3M_ERR_INVALID_INPUT, "bad ny for Yfull"};
    for (const void* p : {(const void*)Xlocal, (const void*)blocal, (const void*)Yfull, (const void*)bfull})
      if (p && is_host_ptr(p)) throw Fail{F3M_ERR_INVALID_INPUT, "the plan API takes device pointers"};
    f3m_plan* P = new f3m_plan();
    P->pl.cfg = resolve(D, k, cfg);
    P->pl.aliased = true;
    P->pl.sharded = true;
    P->st = static_cast<cudaStream_t>(cuda_stream);
    if (alloc) P->alloc = *alloc;
    P->ws = new Workspace(P->st, alloc ? &P->alloc : nullptr);
    P->pl.ws = P->ws;
    P->pl.X.X = Xlocal;
    P->pl.X.b = blocal;
    P->pl.X.n = nx_local;
    P->Yfull = Yfull;
    P->bfull = bfull;
    P->ny = Yfull ? ny : 0;
    P->tm.st = P->st;
    const char* te = getenv("F3M_TIMING");
    P->tm.on = (te && te[0] == '1');
    g_launches = 0;
    *out = P;
  });
}

f3m_status f3m_plan_bbox(f3m_plan* P, double* minmax_host) {
  F3M_TRY({
    if (!P || P->stage != 0) throw Fail{F3M_ERR_INVALID_INPUT, "bad plan state"};
    {
      Span sp(P->tm, PH_BBOX);
      bbox(P->pl.X, P->pl.cfg.D, *P->ws, P->st);
    }
    const int D = P->pl.cfg.D;
    for (int d = 0; d < D; ++d) {
      minmax_host[d] = (double)P->pl.X.mn[d];
      minmax_host[D + d] = (double)P->pl.X.mx[d];
    }
    P->stage = 1;
  });
}

f3m_status f3m_plan_leaves(f3m_plan* P, const double* mm, uint64_t** keys_dev, int64_t** counts_dev, int64_t* len) {
  F3M_TRY({
    if (!P || !mm || !keys_dev || !counts_dev || !len) throw Fail{F3M_ERR_INVALID_INPUT, "NULL argument"};
    plan_leaves(P, mm, keys_dev, counts_dev, len);
  });
}

f3m_status f3m_plan_set_leaves(f3m_plan* P, const uint64_t* keys, const int64_t* counts, int64_t len) {
  F3M_TRY({
    if (!P) throw Fail{F3M_ERR_INVALID_INPUT, "NULL plan"};
    plan_set_leaves(P, keys, counts, len);
  });
}

f3m_status f3m_plan_s2m(f3m_plan* P, double** charges_dev, int64_t* len) {
  F3M_TRY({
    if (!P) throw Fail{F3M_ERR_INVALID_INPUT, "NULL plan"};
    plan_s2m(P, charges_dev, len);
  });
}

f3m_status f3m_plan_evaluate(f3m_plan* P, float* v, f3m_stats* stats) {
  F3M_TRY({
    if (!P || !v) throw Fail{F3M_ERR_INVALID_INPUT, "NULL plan or output"};
    plan_evaluate(P, v, stats);
  });
}

void f3m_plan_destroy(f3m_plan* P) {
  if (!P) return;
  if (P->ws) {
    P->ws->release();
    cudaStreamSynchronize(P->st);
  }
  delete P;
}

}  // extern "C"

// =======================================================================================
// Operator API (plan reuse across right-hand sides).  Everything that does
// not depend on b -- cube, keys, the counting sort's histogram and tile orders, box tables,
// interaction lists -- is built once by f3m_op_create.  f3m_op_apply then runs only the
// b-dependent work: S2M from the stored tile orders (k_s2m_ord: no ranking), M2L, L2T.
// Multi-pass (LSD) trees -- every far level on the globally sorted copies, near field allowed,
// e.g. the C5 D = 5 / 7 and the deep D = 3 configurations -- keep the sorted coordinates, pi,
// the LSD tile orders, the tree and the lists; an apply gathers b into the sorted order and
// runs S2M, M2L, near field, L2T and the LSD un-scatter.  Single-pass trees with a near field
// and k(X, Y) keep no state: every apply runs the whole method (f3m_matvec).
// =======================================================================================
struct f3m_op {
  f3m::Plan pl;
  cudaStream_t st = nullptr;
  f3m::Workspace* ws = nullptr;  // persistent: the b-independent state
  bool reuse = false;
  bool sorted = false;           // multi-pass sorted-path reuse (op_create_sorted)
  const float* X = nullptr;
  const float* Y = nullptr;
  int64_t nx = 0, ny = 0;
  int D = 0;
  f3m_kernel k{};
  f3m_config cfg{};
  f3m_stats base{};
  ~f3m_op() { delete ws; }
};

namespace f3m {

static void op_create(f3m_op* O) {
  Plan& pl = O->pl;
  const int D = O->D;
  cudaStream_t st = O->st;
  pl.cfg = resolve(D, &O->k, &O->cfg);
  if (O->nx < 1) throw Fail{F3M_ERR_INVALID_INPUT, "nx must be >= 1"};
  if (!O->X) throw Fail{F3M_ERR_INVALID_INPUT, "NULL X"};
  if (O->nx >= (1ll << 31) || O->ny >= (1ll << 31)) throw Fail{F3M_ERR_INVALID_INPUT, "n >= 2^31 per call"};
  if (is_host_ptr(O->X) || (O->Y && is_host_ptr(O->Y))) throw Fail{F3M_ERR_INVALID_INPUT, "f3m_op needs device pointers"};
  pl.aliased = (O->Y == nullptr);
  if (!pl.aliased) return;  // k(X, Y): no reuse state (every apply runs f3m_matvec)
  O->ws = new Workspace(st, nullptr);
  Workspace& ws = *O->ws;
  pl.ws = O->ws;
  g_launches = 0;
  Timer tm;
  tm.st = st;
  pl.X.X = O->X;
  pl.X.n = O->nx;
  pl.X.b = nullptr;
  bbox(pl.X, D, ws, st);
  pl.Y = pl.X;
  pl.E = enclosing_edge(pl.X, pl.Y, D);
  if (pl.E == 0.0 || (pl.cfg.flags & F3M_EXACT)) return;
  level_scalars(pl);
  if (pl.T < 1) return;
  if (D * pl.T > MAX_DIGIT_BITS) {  // multi-pass LSD sort: every level on the sorted copies
    sort_side(pl, pl.X, false, false, false, ws, st, tm, true);
    pl.Y = pl.X;
    build_levels(pl.X, D, pl.T, pl.cfg.flags & F3M_KEEP_EMPTY);
    pl.Y.lev = pl.X.lev;
    run_alg1(pl, st);
    for (const FarGroup& g : pl.far)
      if (group_is_local(pl, g)) return;
    count_groups(pl);
    O->sorted = true;
    O->reuse = true;
    O->base = pl.stats;
    CK(cudaStreamSynchronize(st));
    return;
  }
  sort_side(pl, pl.X, true, true, false, ws, st, tm, true);
  if (!pl.X.deferred) return;
  Spec none;
  first_pass(pl, pl.X, false, none, ws, st, tm);  // histogram + tile orders, no moments
  pl.Y = pl.X;
  build_levels(pl.X, D, pl.T, pl.cfg.flags & F3M_KEEP_EMPTY);
  pl.Y.lev = pl.X.lev;
  run_alg1(pl, st);
  if (!pl.near.empty() || needs_sorted(pl) || !pl.X.lrank || !pl.X.lrank_sorted) return;
  for (const FarGroup& g : pl.far) {
    if (!group_is_local(pl, g)) return;
    if (!s2m_ord_supported(D, g.P, 1 << (D * pl.T), 1 << (D * g.t))) return;
    if (!tma_supported(D, g.P, 1 << (D * pl.T), 1 << (D * g.t), false)) return;
  }
  count_groups(pl);
  O->reuse = true;
  O->base = pl.stats;
  CK(cudaStreamSynchronize(st));
}

static void op_apply(f3m_op* O, const float* b, float* v, cudaStream_t st, f3m_stats* stats) {
  Plan& pl = O->pl;
  const int D = O->D;
  g_launches = 0;
  Timer tm;
  tm.st = st;
  const char* te = getenv("F3M_TIMING");
  tm.on = (te && te[0] == '1');
  cudaEvent_t t_all = nullptr;
  tm.begin(PH_TOTAL, t_all);
  Workspace ws(st, nullptr);
  pl.stats = O->base;
  pl.X.b = b;
  pl.Y.b = b;
  if (O->sorted) {
    // b in the sorted order (bs[p] = b[pi[p]]) by replaying the LSD passes on b (coalesced
    // per-bin runs, as the un-scatter), then the b-dependent stages of matvec
    float* bs = ws.get<float>((size_t)pl.X.n, "sorted weights");
    {
      Span sp(tm, PH_SCATTER);
      const int np = (int)pl.X.lsd_order.size();
      float* tmp = np > 1 ? ws.get<float>((size_t)pl.X.n, "sorted weights (ping-pong)") : nullptr;
      const float* cur = b;
      for (int p = 0; p < np; ++p) {
        float* dst = ((np - 1 - p) % 2 == 0) ? bs : tmp;
        launch_lsd_rescatter(cur, dst, pl.X.n, pl.X.lsd_bits[p], (int)pl.X.tiles, pl.X.lsd_counts[p],
                             pl.X.lsd_order[p], st);
        cur = dst;
      }
      g_launches += np;
    }
    pl.X.bs = bs;
    pl.Y.bs = bs;
    FarBuffers fb;
    Spec none;
    far_s2m(pl, fb, none, ws, st, tm);
    float* vs = ws.get<float>((size_t)pl.X.n, "sorted output");
    CK(cudaMemsetAsync(vs, 0, sizeof(float) * pl.X.n, st));
    bool vs_used = far_eval(pl, fb, vs, ws, st, tm);
    if (!pl.near.empty()) {
      Span sp(tm, PH_NEAR);
      near_eval(pl, vs, ws, st);
      vs_used = true;
    }
    finish_output(pl, fb, vs, vs_used, v, ws, st, tm);
    pl.X.bs = pl.Y.bs = nullptr;
    tm.end(PH_TOTAL, t_all);
    CK(cudaGetLastError());
    ws.release();
    CK(cudaStreamSynchronize(st));
    if (stats) {
      *stats = pl.stats;
      stats->num_sort_passes = pl.passes;
      stats->t_star = pl.t_star;
      stats->t_sort = pl.T;
      stats->E = pl.E;
      stats->kernel_launches = (int32_t)g_launches;
      tm.collect(stats->ms_phase);
    }
    return;
  }
  // S2M from the stored tile orders
  FarBuffers fb;
  fb.w_total = 0;
  for (const FarGroup& g : pl.far) {
    fb.w_off.push_back(fb.w_total);
    fb.w_total += (int64_t)g.src.size() * g.m;
  }
  fb.W = ws.get<double>(fb.w_total, "charges");
  for (size_t gi = 0; gi < pl.far.size(); ++gi) {
    const FarGroup& g = pl.far[gi];
    Span sp(tm, PH_S2M);
    LocalS2MArgs a = local_args(pl, pl.Y, b, g.t, g.P);
    a.lrank = pl.X.lrank;
    a.offsets = pl.X.offsets;
    a.sort_tiles = (int)pl.X.tiles;
    a.do_s2m = 1;
    const int grid = tma_grid(a.num_tiles);
    a.Wpart = ws.get<float>((size_t)grid * a.nbox * g.m, "s2m partials", g.t);
    launch_s2m_ord(D, g.P, a, grid, st);
    std::vector<int32_t> slot_box;
    for (int64_t q : g.src) slot_box.push_back((int32_t)pl.Y.lev[g.t][q].key);
    for (int64_t q : g.src) pl.stats.s2m_points += pl.Y.lev[g.t][q].count;
    int32_t* dsb = ws.upload(slot_box, "local slot boxes", g.t);
    launch_local_reduce(a.Wpart, grid, a.nbox, (int)g.m, dsb, (int)g.src.size(), fb.W + fb.w_off[gi], st);
    launch_cheb_transform(fb.W + fb.w_off[gi], (int)g.src.size(), D, g.P, 0, st);  // moments -> nodal
    g_launches += 3;
  }
  far_eval(pl, fb, nullptr, ws, st, tm);
  finish_output(pl, fb, nullptr, false, v, ws, st, tm);
  pl.X.perm = nullptr;  // the first apply's pi lived in its own workspace
  pl.Y.perm = nullptr;
  tm.end(PH_TOTAL, t_all);
  CK(cudaGetLastError());
  ws.release();
  CK(cudaStreamSynchronize(st));
  if (stats) {
    *stats = pl.stats;
    stats->num_sort_passes = pl.passes;
    stats->t_star = pl.t_star;
    stats->t_sort = pl.T;
    stats->E = pl.E;
    stats->kernel_launches = (int32_t)g_launches;
    tm.collect(stats->ms_phase);
  }
}

}  // namespace f3m

extern "C" {

f3m_status f3m_op_create(const float* X, int64_t nx, const float* Y, int64_t ny, int32_t D, const f3m_kernel* k,
                         const f3m_config* cfg, void* cuda_stream, f3m_op** out) {
  using namespace f3m;
  if (!out) {
    g_err = "NULL output handle";
    return F3M_ERR_INVALID_INPUT;
  }
  *out = nullptr;
  f3m_op* O = new f3m_op();
  O->st = static_cast<cudaStream_t>(cuda_stream);
  O->X = X;
  O->Y = Y;
  O->nx = nx;
  O->ny = Y ? ny : nx;
  O->D = D;
  if (k) O->k = *k;
  if (cfg) O->cfg = *cfg;
  else f3m_default_config(D, &O->cfg);
  const f3m_status s = [&]() -> f3m_status { F3M_TRY(op_create(O)); }();
  if (s != F3M_OK) {
    if (O->ws) { O->ws->release(); cudaStreamSynchronize(O->st); }
    delete O;
    return s;
  }
  *out = O;
  return F3M_OK;
}

f3m_status f3m_op_apply(f3m_op* O, const float* b, float* v, void* cuda_stream, f3m_stats* stats) {
  using namespace f3m;
  F3M_TRY({
    if (!O || !b || !v) throw Fail{F3M_ERR_INVALID_INPUT, "NULL operator, b or v"};
    cudaStream_t st = cuda_stream ? static_cast<cudaStream_t>(cuda_stream) : O->st;
    if (!O->reuse) {
      matvec(O->X, O->nx, O->Y, O->ny, O->D, b, v, &O->k, &O->cfg, nullptr, st, stats);
    } else {
      if (is_host_ptr(b) || is_host_ptr(v)) throw Fail{F3M_ERR_INVALID_INPUT, "f3m_op_apply needs device b and v"};
      op_apply(O, b, v, st, stats);
    }
  });
}

f3m_status f3m_op_apply_batch(f3m_op* O, const float* B, int64_t ldb, int32_t nrhs, float* V, int64_t ldv,
                              void* cuda_stream, f3m_stats* stats) {
  using namespace f3m;
  F3M_TRY({
    if (!O || !B || !V || nrhs < 0) throw Fail{F3M_ERR_INVALID_INPUT, "NULL operator, B or V, or nrhs < 0"};
    if (ldb < O->ny || ldv < O->nx) throw Fail{F3M_ERR_INVALID_INPUT, "leading dimensions smaller than ny / nx"};
    cudaStream_t st = cuda_stream ? static_cast<cudaStream_t>(cuda_stream) : O->st;
    for (int32_t r = 0; r < nrhs; ++r) {
      const float* b = B + (int64_t)r * ldb;
      float* v = V + (int64_t)r * ldv;
      if (!O->reuse) matvec(O->X, O->nx, O->Y, O->ny, O->D, b, v, &O->k, &O->cfg, nullptr, st, stats);
      else op_apply(O, b, v, st, stats);
    }
  });
}

int32_t f3m_op_reuses_plan(const f3m_op* O) { return O && O->reuse ? 1 : 0; }

void f3m_op_destroy(f3m_op* O) {
  if (!O) return;
  if (O->ws) {
    O->ws->release();
    cudaStreamSynchronize(O->st);
  }
  delete O;
}

}  // extern "C"
