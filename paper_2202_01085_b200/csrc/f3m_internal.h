// Internal declarations shared by the sm_100a kernels and the host engine of libf3m.so.
// Not part of the ABI (include/f3m.h is).  Paper: arXiv 2202.01085.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#define F3M_MAXD 7

namespace f3m {

// ---------------------------------------------------------------------------------------
// Binning (Sec. 4.1-4.2).  Integer cell of one coordinate at depth T, reading R12:
//   c = min(floor(RN64(RN64(x - alpha) / E) * 2^T), 2^T - 1)
// evaluated with an fp32 fast path whose error bound decides when the exact fp64 path
// must run.
struct KeyParams {
  int D, T;
  double alpha[F3M_MAXD];
  double E;
  double twoT;                // 2^T
  float alpha_f[F3M_MAXD];    // alpha (exactly representable: a min over fp32 values)
  float scale_f;              // RN32(2^T / E)
  float margin;               // 2^(T-22): fp32 fast-path error bound on q = (x-alpha) 2^T / E
  // optional (D*T <= 8): per-dimension cell thresholds [D][2^T - 1] (device), theta_j = the
  // smallest fp32 x whose exact cell is >= j, so cell(x) = #{j : theta_j <= x} bit-exactly
  const float* thr;
};

// sort configuration
constexpr int SORT_THREADS = 512;
constexpr int SORT_ITEMS = 16;
constexpr int SORT_TILE = SORT_THREADS * SORT_ITEMS;  // 8192 points per tile
constexpr int SORT_WARPS = SORT_THREADS / 32;
constexpr int MAX_DIGIT_BITS = 8;

// ---------------------------------------------------------------------------------------
// Far field (Sec. 3 "Interpolating k(x,y)", Fig. 4; Sec. 4.3).  A "box job" is one box of a
// level with its geometry; chunks split boxes into <= FAR_CHUNK points for load balance.
struct BoxGeom {
  float lo_hi[F3M_MAXD];  // fp32 head of the box's lower corner alpha + i l
  float lo_lo[F3M_MAXD];  // fp32 tail (lo - lo_hi)
  float scale;            // 2 / l : tau = (x - lo) * scale - 1
  int64_t start, count;   // interval in the sorted order
};
struct Chunk {
  int32_t box;            // box-job slot
  int32_t len;
  int64_t start;
};
constexpr int FAR_CHUNK = 8192;
constexpr int FAR_THREADS = 256;

// node constants for P nodes (fp32): s_k and c_k = 1/prod_{j != k}(s_k - s_j)
struct NodeConsts {
  float s[16];
  float c[16];
};

// ---------------------------------------------------------------------------------------
// kernel launchers (kernels_*.cu).  All enqueue on `st`; none synchronise.
// binning / sort
void launch_bbox(const float* X, int64_t n, int D, float* partials, int nblocks, cudaStream_t st);
int bbox_blocks(int64_t n);
void launch_bbox_final(const float* partials, int nblocks, int D, float* out /*2D+1*/, cudaStream_t st);

// tile = SORT_TILE (8192, multi-pass scatter) or SORT_TILE/2 (4096, single-pass tile-local path)
// exclusive scan of a uint32 array in place (tmp >= scan_tmp_words(len) words)
int64_t scan_tmp_words(int64_t len);
void launch_scan_u32(uint32_t* data, int64_t len, uint32_t* tmp, cudaStream_t st);

struct ScatterIO {
  // first pass input: row-major points + optional weights
  const float* X;
  const float* b;
  // later-pass inputs (SoA)
  const uint64_t* keys_in;
  const int32_t* perm_in;
  const float* xs_in;      // [D][n]
  const float* bs_in;      // [n] or null
  // outputs
  uint64_t* keys_out;      // may be null (single pass)
  int32_t* perm_out;
  float* xs_out;           // [D][n]
  float* bs_out;           // [n] or null
  int32_t* sigma;          // first pass of a single-pass sort: orig -> sorted pos (or null)
};
// LSD pass with stored tile orders (4096-point tiles): rank (counts [bin][tile] + order), scatter
int lsd_tile();
void launch_lsd_unscatter(const float* in, float* out, int64_t n, int bits, int num_tiles, const uint32_t* offsets,
                          const uint16_t* order, cudaStream_t st, const uint32_t* pad = nullptr);
// the LSD pass applied to a float payload (original / previous-pass order -> the pass's order)
void launch_lsd_rescatter(const float* in, float* out, int64_t n, int bits, int num_tiles, const uint32_t* offsets,
                          const uint16_t* order, cudaStream_t st);
void launch_lsd_rank(bool first, const float* X, const uint64_t* keys, int64_t n, int D, const KeyParams& kp, int shift,
                     int bits, int num_tiles, uint32_t* counts, uint16_t* order, cudaStream_t st);
void launch_lsd_scatter(bool first, const ScatterIO& io, int64_t n, int D, const KeyParams& kp, int bits, int num_tiles,
                        const uint32_t* offsets, const uint16_t* order, cudaStream_t st);
void launch_unpermute_perm(const float* vs, const int32_t* perm, int64_t n, float* v, cudaStream_t st);
// run-length heads of sorted keys -> flags (uint32 0/1)
void launch_key_heads(const uint64_t* keys, int64_t n, uint32_t* flags, cudaStream_t st);
void launch_compact_heads(const uint64_t* keys, const uint32_t* flags_scanned, int64_t n,
                          uint64_t* box_key, int64_t* box_start, cudaStream_t st);
// v[i] = vs[sigma[i]]
void launch_unpermute(const float* vs, const int32_t* sigma, int64_t n, float* v, cudaStream_t st);
// SoA transpose for the direct path: xs[d*n+i] = X[i*D+d]
void launch_to_soa(const float* X, int64_t n, int D, float* xs, cudaStream_t st);

// far field
bool far_supported(int D, int P);  // register-tiled instantiation exists
void launch_s2m(int D, int P, const float* xs, const float* bs, int64_t n, const BoxGeom* boxes,
                const Chunk* chunks, int64_t nchunks, const NodeConsts& nc, float* partials,
                cudaStream_t st);
void launch_chunk_reduce(const float* partials, const int32_t* chunk_ptr, int32_t nboxes, int m,
                         double* W, cudaStream_t st);
void launch_m2l_tables(int D, int P, const double* delta0 /*[D] Delta for idx 0*/, double l,
                       const int32_t* range /*[D]*/, double gamma, const NodeConsts& nc,
                       float* tables, int table_stride, cudaStream_t st);
void launch_m2l(int D, int P, int32_t ntgt, const int32_t* csr_ptr, const int32_t* src, const uint64_t* offs,
                const float* tables, int table_stride, const float* W32, double* U, cudaStream_t st);
void launch_to_f32(const double* a, int64_t n, float* b, cudaStream_t st);
// exact level translations (Lagrange basis, fp64): M2M up, L2L down, row gather / scatter-add
// scratch: nparents * m2m_split(D, nparents) * m doubles (NULL: one block per parent)
int m2m_split(int D, int nparents);
void launch_m2m(int D, int P, int m, int nparents, const int32_t* child0, const int32_t* nchild,
                const int32_t* child_bits, const double* Wc, double* Wp, double* scratch, cudaStream_t st);
void launch_l2l(int D, int P, int m, int nchildren, const int32_t* parent, const int32_t* child_bits,
                const double* Up, double* Uc, cudaStream_t st);
void launch_rows(const double* src, const int32_t* idx, int64_t rows, int m, double* dst, bool scatter_add,
                 cudaStream_t st);
void launch_l2t(int D, int P, const float* xs, int64_t n, const BoxGeom* boxes, const Chunk* chunks,
                int64_t nchunks, const NodeConsts& nc, const double* U, float* vs, cudaStream_t st);
// large grids (128 < P^D <= 4096): node-parallel S2M, point-parallel L2T (kernels_far_gen.cu)
bool gen_supported(int D, int P);
void launch_s2m_gen(int D, int P, const float* xs, const float* bs, int64_t n, const BoxGeom* boxes,
                    const Chunk* chunks, int64_t nchunks, const NodeConsts& nc, float* partials, cudaStream_t st);
void launch_l2t_gen(int D, int P, const float* xs, int64_t n, const BoxGeom* boxes, const Chunk* chunks,
                    int64_t nchunks, const NodeConsts& nc, const double* U, float* vs, cudaStream_t st);

// D = 5, P = 4 (m = 1024): register-blocked S2M / L2T in the Lagrange basis (nodal charges /
// locals, kernels_far_blk.cu)
bool blk_supported(int D, int P);
void launch_s2m_blk(int D, int P, const float* xs, const float* bs, int64_t n, const BoxGeom* boxes,
                    const Chunk* chunks, int64_t nchunks, const NodeConsts& nc, float* partials, cudaStream_t st);
void launch_l2t_blk(int D, int P, const float* xs, int64_t n, const BoxGeom* boxes, const Chunk* chunks,
                    int64_t nchunks, const NodeConsts& nc, const double* U, float* vs, cudaStream_t st);

// M2L over a complete level as Kronecker mode products (kernels_grid.cu; reading R29): B0 / B1
// [D][N][N] per-dimension factors (parent offset 0 / +-1), ndeg = 4 (Euclidean near rule) or 1
// (max norm: B0 holds every admitted offset); *_base[slot] = flattened index of the box's node 0
void launch_grid_m2l(int D, int P, int N, int ndeg, const double* B0, const double* B1, const double* W,
                     const int64_t* src_base, int nsrc, const int64_t* tgt_base, int ntgt, double* Za, double* Zb,
                     double* U, cudaStream_t st);

// Smolyak sparse grids (kernels_sparse.cu; reading R27): S2M moments over K_q, fp64 row
// transforms, M2L over the sparse nodes, L2T from Chebyshev coefficients
bool sparse_supported(int D, int q, int64_t m);
void launch_s2m_sparse(int D, int n1, int m, const float* xs, const float* bs, int64_t n, const BoxGeom* boxes,
                       const Chunk* chunks, int64_t nchunks, const uint2* fac, float* partials, cudaStream_t st);
void launch_dense_rows(const double* in, int64_t R, int m, const double* matT, double* out, cudaStream_t st);
void launch_m2l_sparse(int D, int n1, int m, int32_t ntgt, const int32_t* csr_ptr, const int32_t* src,
                       const uint64_t* offs, const float* tables, int table_stride, const float* W32,
                       const uint8_t* nodes, double* U, cudaStream_t st);
void launch_l2t_sparse(int D, int n1, int m, const float* xs, int64_t n, const BoxGeom* boxes, const Chunk* chunks,
                       int64_t nchunks, const uint2* fac, const double* Ut, float* vs, cudaStream_t st);

// near field / direct (Sec. 3 Eq. (1); KeOps-style map-reduce)
struct NearJob {        // one CTA: up to NEAR_TILE targets of one target box
  int64_t tstart;
  int32_t tlen;
  int32_t list;         // index into the source-list CSR
  int64_t out_off;      // output offset (split-source partial buffers; 0 otherwise)
};
constexpr int NEAR_TILE = 128;
void launch_near(int D, const float* xs_t, int64_t nt, const float* xs_s, const float* bs, int64_t ns,
                 const NearJob* jobs, int64_t njobs, const int32_t* list_ptr, const int64_t* src_start,
                 const int64_t* src_count, double gamma, float* vs, cudaStream_t st);
// fp64 exact sum: sources split into `splits` ranges (grid y), partial sums [splits][nt]
void launch_direct_f64(int D, const float* xs_t, int64_t nt, const float* xs_s, const float* bs,
                       int64_t ns, double gamma, int splits, double* partial, cudaStream_t st);
// out[i] = sum_s partial[s][i] (fixed order)
void launch_reduce_splits_f64(const double* partial, int splits, int64_t nt, double* out, cudaStream_t st);
void launch_reduce_splits_f32(const float* partial, int splits, int64_t nt, float* out, cudaStream_t st);

// ---------------------------------------------------------------------------------------
// tile-local far field (kernels_local.cu)
struct LocalS2MArgs {
  const float* X;
  const float* b;
  int64_t n;
  KeyParams kp;           // keys at depth kp.T (the local sort digit = whole key, <= 8 bits)
  int bits;               // D * kp.T
  int shift;              // level-t box = digit >> shift, shift = D * (kp.T - t)
  int nbox;               // 2^{D t}
  double alpha[F3M_MAXD];
  double l;               // level-t edge
  NodeConsts nc;
  int num_tiles;          // tiles of LT_TILE points
  int do_s2m;             // 0: scatter only
  float* Wpart;           // [grid][nbox][m] per-CTA charges
  // counting-sort scatter (may be null): global offsets = scanned [bin][tile] counts of
  // the single-pass sort over tiles of SORT_TILE points (tile sizes must then match)
  const uint32_t* offsets;
  int sort_tiles;
  int32_t* perm;
  int32_t* sigma;
  float* xs;              // [D][n]
  float* bs;
  uint64_t* keys;
  uint32_t* counts;       // optional: per-tile digit counts [bin][tile] (the counting-sort histogram)
  uint16_t* lrank;        // optional: the tile's stable order (rank form for k_local_s2m, sorted
                          // form for k_s2m_tma; see launch_tile_invert)
  int cell_base[F3M_MAXD];  // level-t cell of local box 0 (two-digit path: the bucket's first cell)
  // two-digit path, one launch over every bucket (k_s2m_ws only): tiles of the padded bucket
  // layout; bucket k spans tiles [bk_tile0[k], bk_tile0[k+1]) and holds bk_n[k] points; its
  // exact low-digit thresholds bk_thr[k][D][3], cell base bk_cell[k][D], counts at
  // counts + bk_coff[k] ([leaf][tile of the bucket]); Wpart = [bucket][CTA][nbox][m]
  int nbuckets;
  const int2* bk_tile;            // per tile of the layout: {bucket | valid points << 8, tile of the bucket}
  const int32_t* bk_tile0;
  const int64_t* bk_n;
  const float* bk_thr;
  const int32_t* bk_cell;
  const int64_t* bk_coff;
};
struct LocalL2TArgs {
  const float* X;
  int64_t n;
  KeyParams kp;
  int bits, shift, nbox;
  double alpha[F3M_MAXD];
  double l;
  NodeConsts nc;
  int num_tiles;
  const double* U;          // [nslots][m]
  const int32_t* box_slot;  // [nbox] -> U slot or -1
  float* v;                 // output, original order
  int accumulate;           // v += (1) or v = (0)
  const float* vs;          // optional: v += vs[sigma[i]] (global-sorted contributions)
  const int32_t* sigma;
  // optional counting-sort scatter of the permutation (kp at the leaf depth, shift as above)
  const uint32_t* offsets;  // scanned [bin][tile] counts
  int sort_tiles;
  int32_t* perm;
  uint64_t* keys;
  const uint16_t* lrank;    // optional: tile-local ranks of the first pass (skips re-ranking;
                            // requires offsets: bin counts and starts come from the scan)
  int cell_base[F3M_MAXD];  // level-t cell of local box 0 (two-digit path: the bucket's first cell)
  int offsets_tail;         // 1: offsets continue past this array's [bin][tile] block (global scan)
};
constexpr int LT_TILE_PTS = 4096;
bool local_supported(int D, int P, int nbox);
int local_grid(int num_tiles);
void launch_local_s2m(int D, int P, const LocalS2MArgs& a, int grid, cudaStream_t st);
void launch_local_reduce(const float* Wpart, int nctas, int nbox, int m, const int32_t* slot_box, int nslots,
                         double* W, cudaStream_t st);
void launch_local_l2t(int D, int P, const LocalL2TArgs& a, int grid, cudaStream_t st);
// TMA-pipelined tile-local kernels (kernels_tma.cu): 512-thread persistent CTAs
bool tma_supported(int D, int P, int nb, int nbox, bool s2m_owned);
int tma_grid(int num_tiles);
void launch_s2m_tma(int D, int P, const LocalS2MArgs& a, int grid, cudaStream_t st);
void launch_l2t_tma(int D, int P, const LocalL2TArgs& a, int grid, cudaStream_t st);
// L2T with register-resident coefficients: one leaf bin per box, <= 128 boxes, D <= 3, m <= 64
bool l2t_fix_supported(int D, int P, int nb, int nbox, int shift);
void launch_l2t_fix(int D, int P, const LocalL2TArgs& a, int grid, cudaStream_t st);
// two-digit (MSD) path: scatter into top-digit buckets padded to whole tiles (AoS coordinates,
// weights), destination = scanned offset + pad[bin]
void launch_scatter_msd(int D, const float* X, const float* b, int64_t n, int bits, int num_tiles,
                        const uint32_t* offsets, const uint32_t* pad, const uint16_t* order, float* xp, float* bp,
                        cudaStream_t st);
void launch_gather_u32(const uint32_t* in, const int64_t* idx, int64_t n, uint32_t* out, cudaStream_t st);
void launch_bucket_tiles(const int32_t* tile0, const int64_t* nb_pts, int nbuckets, int ntiles, int2* out,
                         cudaStream_t st);
// ---------------------------------------------------------------------------------------
// Interaction division + classification of one depth on the device (kernels_tree.cu)
enum { DIV_FAR = 0, DIV_SMOOTH = 1, DIV_SMALL = 2, DIV_NEAR = 3, DIV_DROP = 4, DIV_NCLS = 5 };
struct DivArgs {
  int D;
  uint64_t M;                       // candidate pairs of this depth
  int nruns;
  const uint64_t* run_base;         // [nruns] first candidate of each run
  const int32_t* run_p;             // [nruns] parent target box (depth t-1)
  const uint32_t* run_Q;            // [nruns] sum of the partners' child counts
  const int32_t* run_r0;            // [nruns + 1] first near pair of each run
  const int32_t* pair_q;            // [L] parent source box of near pair r
  const uint32_t* pair_S;           // [L] exclusive prefix of child counts inside the run
  const int32_t* childX0;           // depth t-1 X boxes: first child (depth-t index)
  const int32_t* childY0;
  const int32_t* cellX;             // depth t boxes: integer cells [box][F3M_MAXD]
  const int32_t* cellY;
  const int64_t* gX;                // depth t boxes: global point counts
  const int64_t* gY;
  double delta[F3M_MAXD];           // (alpha_X - alpha_Y) / l (0 when Y = X)
  int pfar;                         // adaptive far-field node count (0: drop)
  int smooth_level;
  int no_small;
  int maxnorm;                      // F3M_ADMISSIBLE_MAXNORM
  int64_t rho;
  // scatter pass
  const uint32_t* blockoff;         // [blocks][DIV_NCLS] list offset of each class's block run
  int cls_list[DIV_NCLS];           // output list of each class (-1: not stored)
  int cls_merge[DIV_NCLS];          // class sharing the same list (-1: none)
  int32_t* outP[4];
  int32_t* outQ[4];
  // count pass
  uint32_t* blockcnt;               // [blocks][DIV_NCLS]
  int32_t* dbg_pc;                  // optional (debug): every candidate in canonical order
  int32_t* dbg_qc;
  int8_t* dbg_tag;
};
void launch_divide(const DivArgs& a, bool scatter, cudaStream_t st);
int64_t divide_blocks(uint64_t M);
void launch_far_marks(const int32_t* P, const int32_t* Q, int64_t n, const int32_t* cellX, const int32_t* cellY, int D,
                      uint32_t* tcount, uint32_t* smark, int* omin, int* omax, cudaStream_t st);
void launch_far_cols(const int32_t* P, const int32_t* Q, int64_t n, const int32_t* cellX, const int32_t* cellY, int D,
                     const uint32_t* sslot, const int* omin, int32_t* col, uint64_t* off, cudaStream_t st);

// k_s2m_tma stores each tile's stable order as sorted position -> original local index
// ("sorted" form, what k_l2t_tma reads); k_local_s2m stores per-point ranks ("rank" form,
// what k_local_l2t reads).  The two forms are inverse permutations per tile.
// S2M of a new right-hand side with the tile order stored by a previous pass (sorted form)
bool s2m_ord_supported(int D, int P, int nb, int nbox);
void launch_s2m_ord(int D, int P, const LocalS2MArgs& a, int grid, cudaStream_t st);
// warp-specialised S2M (rank group + moment group, mbarrier ring) for small leaf grids
bool s2m_ws_supported(int D, int P, int T, int nbox);
void launch_s2m_ws(int D, int P, int T, const LocalS2MArgs& a, int grid, cudaStream_t st);
// deferred counting-sort scatter (pi, sorted SoA coords / weights, sigma, keys) from the
// stored tile orders (sorted form), coalesced per-bin runs
void launch_scatter_ord(int D, const LocalS2MArgs& a, cudaStream_t st);
void launch_tile_invert(const uint16_t* in, int64_t n, uint16_t* out, cudaStream_t st);
// tile-local kernels work in the Chebyshev basis: moments -> nodal (0) / nodal -> Chebyshev (1)
void launch_cheb_transform(double* V, int nslots, int D, int P, int transpose, cudaStream_t st);

}  // namespace f3m
