/*
 * fpvs.h — C ABI of libfpvs.so, the B200 (sm_100a) NeuralPVS hot path.
 *
 * The reference (pkg/src/froxelpvs) is pure Python/numpy and has no FFI of
 * its own; its boundary is the Python API of froxelpvs.interleave and
 * froxelpvs.neural.  Each entry point below states the
 * reference function it replaces.  The Python package
 * paper_2509_24677_b200 binds these through ctypes and re-exposes the
 * reference names; INTEGRATION.md shows the binding.
 *
 * Conventions
 *  - every pointer argument is a DEVICE pointer unless named host_*;
 *  - every call takes a cudaStream_t passed as void* and is stream-ordered,
 *    never synchronises and never allocates (graph-capturable);
 *  - row counts produced on the device (active cells) are passed back as
 *    device int32 pointers ("n_*_dev"), so kernels size their work from
 *    device memory and a whole frame runs with no host round trip; buffers
 *    are sized by a host-known capacity ("cap_*");
 *  - return 0 on success, FPVS_EINVAL (1) on bad arguments, FPVS_ESHAPE (2)
 *    on shape mismatch, FPVS_ECUDA (3) on a CUDA launch error;
 *    fpvs_last_error() returns a thread-local message.  The Python layer maps
 *    1/2 to ValueError, as the reference raises ValueError
 *    (interleave.py:58-59, 78-79; neural.py:203-205, 518-522).
 *
 * Layouts (HBM)
 *  - packed grid: B x (Nz, Ny, Nx/8) bytes, x-fastest LSB-first, the FPVS
 *    payload of froxel.py:3-4 / 96-104, one grid after another;
 *  - dense grid: (B, Nx, Ny, Nz) C-order, as the reference's ndarray;
 *  - cells: (B, X, Y, Z, d^3) channels-last, channel k = lx + d*(ly + d*lz)
 *    (interleave.py:54-65);
 *  - sparse features: rows of active cells in C-order of (b, x, y, z),
 *    row stride ld (elements) so concatenation is a column offset;
 *  - coords: int32 [cap][4] = (b, x, y, z);
 *  - neighbour tables: int32 [cap][K] row index or -1; subm K = 27 with
 *    offset j = 9a + 3b + c <-> (a-1, b-1, c-1) (neural.py:187-199),
 *    down K = 8 with child = 2*parent + (a, b, c), j = 4a + 2b + c,
 *    up K = 8 with only the fine cell's own parity slot set;
 *  - weights (reference layout): f32 (K*Cin, Cout), row = j*Cin + ci
 *    (neural.py:163-166); the tensor-core path takes them pre-packed by
 *    fpvs_pack_weights_tc.
 */
#ifndef FPVS_H_
#define FPVS_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { FPVS_OK = 0, FPVS_EINVAL = 1, FPVS_ESHAPE = 2, FPVS_ECUDA = 3 };
enum { FPVS_IN_PACKED = 0, FPVS_IN_U8 = 1, FPVS_IN_F32 = 2, FPVS_IN_F64 = 3 };
enum { FPVS_F32 = 0, FPVS_BF16 = 1, FPVS_F64 = 2 };
enum { FPVS_ACT_NONE = 0, FPVS_ACT_RELU = 1, FPVS_ACT_SIGMOID = 2, FPVS_ACT_MASK = 3 };
/* OR into fpvs_spconv_halo's act when the neighbour / halo tables and tile
 * masks were written two or more launches earlier on the stream: the conv then
 * decodes its work units before its programmatic-launch wait (overlapping the
 * previous kernel's tail).  Without it the decode waits (safe directly after a
 * table build). */
#define FPVS_TABLES_SETTLED 0x100

const char* fpvs_last_error(void);
int fpvs_abi_version(void);

/* ---- (1) interleave / deinterleave ------------------------------------ */

/* Replaces interleave(grid, d) (interleave.py:54-65) for B grids at once.
 * in: packed bits, u8, f32 or f64 dense; out: (B, Nx/d, Ny/d, Nz/d, d^3)
 * f32/bf16 (the cast fused), or f64 for f64 input (an exact permutation, as
 * the reference keeps an ndarray's dtype, interleave.py:45-51);
 * cell_active (nullable): u8 (B, X, Y, Z), 1 iff the block holds a nonzero.
 * d in {1, 2, 4, 8}: shared-memory tiled transpose with 16-byte loads and
 * stores (HBM-bound); other d: a generic kernel. */
int fpvs_interleave(const void* in, int in_fmt, int B, int Nx, int Ny, int Nz, int d,
                    void* out, int out_dtype, uint8_t* cell_active, void* stream);

/* Replaces deinterleave(t, d, threshold) (interleave.py:68-85).
 * in: (B, X, Y, Z, d^3) f32/bf16/f64.  If tau is NaN, out is dense
 * (B, X*d, Y*d, Z*d): f64 for f64 cells (exact inverse), else f32; otherwise
 * out is packed bits of [value >= tau], compared in the cells' precision
 * (float64 for f64, float32 otherwise: numpy's comparison under NEP 50). */
int fpvs_deinterleave(const void* in, int in_dtype, int B, int X, int Y, int Z, int d,
                      double tau, void* out, void* stream);

/* ---- (2) kernel maps --------------------------------------------------- */

/* Scratch bytes for fpvs_kmap_compact over a (B, X, Y, Z) cell grid. */
size_t fpvs_kmap_workspace_size(int B, int X, int Y, int Z);

/* Active cells straight from packed bits (fused interleave): cell_active[c] =
 * any bit of the d^3 block is set. */
int fpvs_cell_active_from_bits(const uint8_t* bits, int B, int Nx, int Ny, int Nz, int d,
                               uint8_t* cell_active, void* stream);

/* Stream compaction of cell_active in C-order: coords[rank] = (b,x,y,z),
 * index_vol[cell] = rank or -1, *n_active_dev = count (clamped to cap). */
int fpvs_kmap_compact(const uint8_t* cell_active, int B, int X, int Y, int Z,
                      int32_t* coords, int32_t* index_vol, int32_t* n_active_dev, int cap,
                      void* workspace, size_t workspace_bytes, void* stream);

/* Submanifold 3x3x3 neighbour table: nbr[i][j] = index_vol[coords[i] + o_j]. */
int fpvs_kmap_subm(const int32_t* coords, const int32_t* n_active_dev, int cap,
                   const int32_t* index_vol, int B, int X, int Y, int Z,
                   int32_t* nbr, void* stream);

/* Submanifold map for any odd kernel size k (K = k^3 taps; k = 3 gives the
 * fpvs_kmap_subm table): nbr[i][(a*k + b)*k + c] = row of
 * coords[i] + (a - k/2, b - k/2, c - k/2) or -1 (neural.py:187-199 im2col
 * order; ModelConfig accepts any odd kernel, neural.py:49-51). */
int fpvs_kmap_subm_k(const int32_t* coords, const int32_t* n_active_dev, int cap,
                     const int32_t* index_vol, int B, int X, int Y, int Z, int k,
                     int32_t* nbr, void* stream);

/* Parent flags of a k2s2 down-conv: coarse_active[b, x>>1, y>>1, z>>1] = 1.
 * coarse_active must be zeroed first (fine dims X, Y, Z must be even). */
int fpvs_kmap_coarsen(const int32_t* coords, const int32_t* n_active_dev, int cap,
                      int B, int X, int Y, int Z, uint8_t* coarse_active, void* stream);

/* down[p][j] = fine row of child 2*coarse[p] + (a,b,c) or -1. */
int fpvs_kmap_down(const int32_t* coarse_coords, const int32_t* n_coarse_dev, int cap_coarse,
                   const int32_t* fine_index_vol, int B, int X, int Y, int Z,
                   int32_t* down, void* stream);

/* up[i][j] = parent row if j == parity(fine[i]) else -1 (fine dims X, Y, Z). */
int fpvs_kmap_up(const int32_t* fine_coords, const int32_t* n_fine_dev, int cap_fine,
                 const int32_t* coarse_index_vol, int B, int X, int Y, int Z,
                 int32_t* up, void* stream);

/* Per-offset pair lists of a neighbour table (SURVEY.md §8(a) row KM): for
 * offset j the pairs (in = table[i][j], out = i) with in >= 0, sorted by
 * out, stored at [pair_off[j], pair_off[j+1]) of pair_in / pair_out;
 * pair_off: int64 [K+1] (device), exclusive prefix of the list lengths.
 * At most cap_pairs pairs are stored (pair_off[K] is the full count).
 * Deterministic; workspace fpvs_kmap_pairs_workspace_size(K, cap). */
size_t fpvs_kmap_pairs_workspace_size(int K, int cap);
int fpvs_kmap_pairs(const int32_t* table, int K, const int32_t* n_dev, int cap, int32_t* pair_in,
                    int32_t* pair_out, int64_t* pair_off, long long cap_pairs, void* workspace,
                    size_t workspace_bytes, void* stream);

/* Per 128-row tile of a neighbour table: bit j set iff some live row of the
 * tile has table[row][j] >= 0.  masks: uint32 [ceil(cap/128)].  The
 * tensor-core conv skips K-chunks of offsets absent from a whole tile. */
int fpvs_kmap_tile_masks(const int32_t* table, int K, const int32_t* n_dev, int cap,
                         uint32_t* masks, void* stream);

/* One frame's whole map hierarchy in three launches (levels.cu): level-0
 * active cells from packed bits (cell = d^3 block), levels l > 0 = parents
 * of level l-1 (k2s2), each compacted in C-order, plus every table below
 * that is non-NULL.  Produces exactly what fpvs_cell_active_from_bits ->
 * fpvs_kmap_compact -> fpvs_kmap_subm / coarsen / down / up / tile_masks
 * produce step by step (the reference builds the same maps implicitly in
 * neural.py:187-199 im2col and unet.py:26-64).
 * Per level (device pointers, caps on the host):
 *   coords [cap][4], index_vol [B*X*Y*Z], n (int32, device);
 *   nbr [cap][27] + nbr_masks (NULL = skip);
 *   level > 0: down [cap][8] rows of l -> children in l-1, down_masks;
 *              up [cap(l-1)][8] rows of l-1 -> parent in l, up_masks.
 * Optional: feat = level-0 features (fpvs_gather_cells_bits), clear_bits =
 * clear_bytes to zero (the output grid of the fused head).
 * workspace: fpvs_levels_workspace_size bytes, ZEROED once before first use
 * (every call leaves it zeroed again).  d in {1, 2, 4, 8}, nlev <= 4. */
typedef struct fpvs_level {
  int32_t* coords;
  int32_t* index_vol;
  int32_t* n;
  int cap;
  int32_t* nbr;
  uint32_t* nbr_masks;
  int32_t* down;
  uint32_t* down_masks;
  int32_t* up;
  uint32_t* up_masks;
  /* nullable: the halo-cached conv's per-tile tables of this level's 3^3 map
   * (as fpvs_kmap_halo writes them), built in the same launch as the map */
  int32_t* halo_rows;
  int32_t* halo_n;
  int16_t* halo_lnbr;
} fpvs_level;

size_t fpvs_levels_workspace_size(int B, int Nx, int Ny, int Nz, int d, int nlev);
int fpvs_levels_from_bits(const uint8_t* bits, int B, int Nx, int Ny, int Nz, int d, int nlev,
                          const fpvs_level* levels, void* workspace, size_t workspace_bytes,
                          void* feat, int feat_dtype, int ldf, uint8_t* clear_bits, size_t clear_bytes,
                          void* stream);

/* Open-addressing GPU hash alternative to index_vol (general, unbounded
 * grids): capacity slots of (key int64, value int32); key = linear cell id. */
int fpvs_hash_build(const int32_t* coords, const int32_t* n_active_dev, int cap,
                    int B, int X, int Y, int Z, int64_t* keys, int32_t* vals,
                    int hash_capacity, void* stream);
int fpvs_kmap_subm_hash(const int32_t* coords, const int32_t* n_active_dev, int cap,
                        const int64_t* keys, const int32_t* vals, int hash_capacity,
                        int B, int X, int Y, int Z, int32_t* nbr, void* stream);

/* Features of active cells from packed bits (the sparse interleave):
 * x[i][k] = bit of (b, x*d + lx, y*d + ly, z*d + lz), k = lx + d*(ly + d*lz). */
int fpvs_gather_cells_bits(const uint8_t* bits, int B, int Nx, int Ny, int Nz, int d,
                           const int32_t* coords, const int32_t* n_active_dev, int cap,
                           void* x, int ldx, int dtype, void* stream);

/* ---- (3) sparse convolution ------------------------------------------- */

/* Implicit gather-GEMM: y[i][col_off + c] = act(bias[c] + sum_j x[nbr[i][j]] . W_j[:, c]).
 * nbr may be NULL with K == 1 (identity gather, 1x1x1 conv).
 * SIMT FFMA path (fp32 mode, correctness anchor): w f32 (K*Cin, Cout). */
int fpvs_spconv_simt(const void* x, int ldx, int in_dtype, const int32_t* nbr, int K,
                     const int32_t* n_out_dev, int cap_out, const float* w, const float* bias,
                     int cin, int cout, int act, void* y, int ldy, int col_off, int out_dtype,
                     void* stream);

/* Bytes of the packed tensor-core weight image for (K, Cin, Cout) cut into
 * BN-wide output-column blocks (bn = 0 picks the smallest of 32/64/128/256
 * that covers Cout; smaller bn splits N across CTAs for layers with few rows). */
size_t fpvs_pack_weights_tc_size(int K, int cin, int cout, int bn);
/* Pack f32 (K*Cin, Cout) weights into the bf16 SW128 K-major smem image,
 * layout [Cout/bn][ceil(K*Cin/64)][bn][128 B]. */
int fpvs_pack_weights_tc(const float* w, int K, int cin, int cout, int bn, void* packed, void* stream);

/* tcgen05 path: bf16 in, fp32 TMEM accumulate, fused bias + act, bf16 out.
 * x has x_rows rows of stride ldx; rows of x are gathered by TMA
 * with cp.async; tile_masks (from fpvs_kmap_tile_masks on nbr) is required
 * when nbr is given.  w_packed must have been packed with the same bn. */
int fpvs_spconv_tc(const void* x, int ldx, int x_rows, const int32_t* nbr, int K,
                   const uint32_t* tile_masks, const int32_t* n_out_dev, int cap_out,
                   const void* w_packed, int bn,
                   const float* bias, int cin, int cout, int act,
                   void* y, int ldy, int col_off, void* stream);

/* k2s2 up-conv rows grouped by parity (upsort.cu).  In an up table every fine
 * row has one valid tap (its parity); the rows are stably sorted by that
 * class, each class padded to a multiple of 128 rows, so each 128-row tile of
 * the up conv uses one weight slice instead of eight.  Outputs, for
 * cap_pad = fpvs_up_sort_cap(cap_fine) rows: sorted_table int32 [cap_pad][8]
 * (the up table in sorted order, -1 rows for padding), perm int32 [cap_pad]
 * (sorted position -> fine row, -1 for padding), masks uint32 [cap_pad/128]
 * (1 << class per tile), n_pad_dev (padded row count, device).  Pass them to
 * fpvs_spconv_tc_scatter with K = 8. */
typedef struct fpvs_up_sort_job {
  const int32_t* up;
  const int32_t* n_fine_dev;
  int cap_fine;
  int32_t* sorted_table;
  int32_t* perm;
  uint32_t* masks;
  int32_t* n_pad_dev;
  void* workspace;
  size_t workspace_bytes;
} fpvs_up_sort_job;
int fpvs_up_sort_cap(int cap_fine);
size_t fpvs_up_sort_workspace_size(int cap_fine);
int fpvs_up_sort(const int32_t* up, const int32_t* n_fine_dev, int cap_fine, int32_t* sorted_table,
                 int32_t* perm, uint32_t* masks, int32_t* n_pad_dev, void* workspace,
                 size_t workspace_bytes, void* stream);
int fpvs_up_sort_multi(const fpvs_up_sort_job* jobs, int njobs, void* stream);

/* fpvs_spconv_tc as the consumer of tile-level dataflow (see
 * fpvs_spconv_halo_flow): x is the output of the launch immediately before,
 * which publishes tile_done_in[t] = 4 per 128-row tile of its level
 * (done_n_dev: that level's row count); each output tile waits only for the
 * producer tiles its gathered rows lie in.  The weights must be packed before
 * the producer launched and y must be disjoint from the producer's buffers. */
int fpvs_spconv_tc_flow(const void* x, int ldx, int x_rows, const int32_t* nbr, int K,
                        const uint32_t* tile_masks, const int32_t* n_out_dev, int cap_out, const void* w_packed,
                        int bn, const float* bias, int cin, int cout, int act, void* y, int ldy, int col_off,
                        const int32_t* tile_done_in, const int32_t* done_n_dev, void* stream);

/* fpvs_spconv_tc with an output-row map: tile row i is written to row
 * out_rows[i] of y (skipped when -1).  Used with the parity-sorted up conv. */
int fpvs_spconv_tc_scatter(const void* x, int ldx, int x_rows, const int32_t* nbr, int K,
                           const uint32_t* tile_masks, const int32_t* n_out_dev, int cap_out,
                           const int32_t* out_rows, const void* w_packed, int bn,
                           const float* bias, int cin, int cout, int act,
                           void* y, int ldy, int col_off, void* stream);

/* The k2s2 transposed (up) conv as ONE dense GEMM over the coarse rows
 * (the config-2 U-Net's up21 / up10, oracle/sparse.py:196 up_conv; weight rows
 * k = j Cin + ci as neural.py:163-166):
 * Y = act(X_coarse W' + b') with W'[ci][j Cout + co] = W[j Cin + ci][co]
 * (w_packed: fpvs_pack_weights_tc of W' as a K = 1, Cin -> 8 Cout conv;
 * bias8 = b tiled 8 times), and column block j of coarse row r is written to
 * fine row child_rows[8 r + j] of y (the coarse level's down table: its child
 * in parity class j = 4(x&1) + 2(y&1) + (z&1); -1 = no child, skipped).  Each
 * fine row has exactly one parent, so every active fine row is written once.
 * Bit-identical to the gathered up conv (same operands, same K order). */
int fpvs_spconv_tc_upblocks(const void* x, int ldx, int x_rows, const int32_t* n_coarse_dev, int cap_coarse,
                            const void* w_packed, int bn, const float* bias8, int cin, int cout, int act,
                            const int32_t* child_rows, void* y, int ldy, int col_off, void* stream);

/* Halo-cached submanifold conv (spconv_halo.cu), same math as
 * fpvs_spconv_tc with K = 27 (neural.py:187-219 on the active set), for
 * Cin and Cout multiples of 64.  Each 128-row tile's distinct neighbour rows
 * (its halo) are staged once per 64-channel chunk in shared memory and the
 * per-offset A operand is assembled in tensor memory.
 * fpvs_kmap_halo builds, per tile of a K = 27 table: halo_rows
 * int32 [tiles][FPVS_HALO_MAX] (sorted distinct rows), halo_n int32 [tiles],
 * lnbr int16 [tiles][128][27] (slot in halo_rows, -1 = none, -2 = not
 * cached: read directly; every row of a tile whose neighbours span more than
 * 16384 rows is read directly); tiles = ceil(cap / 128).  fpvs_kmap_halo_size is
 * the total bytes of the three arrays (each 256-byte aligned, in that order).
 * fpvs_spconv_halo: bn in {0 (auto), 64, 128, 256}; split >= 1 cuts each
 * tile's K range across CTAs (fp32 partials in ws, reduced in a fixed order by
 * the last CTA: deterministic); split = -S keeps whole waves of tiles whole
 * and cuts only the last partial wave's tiles into up to S K ranges (load
 * balance; the workspace then covers one grid of items, not the capacity).
 * Calls with different (cap, Cout, bn, split) must not share a workspace.  ws = fpvs_spconv_halo_workspace_size bytes,
 * ZEROED before its first use (the kernel leaves its counters at zero). */
#define FPVS_HALO_MAX 512
size_t fpvs_kmap_halo_size(int cap);
int fpvs_kmap_halo(const int32_t* nbr, const int32_t* n_dev, int cap, int32_t* halo_rows,
                   int32_t* halo_n, int16_t* lnbr, void* stream);
/* The same tables for up to 4 levels in one launch. */
typedef struct fpvs_halo_job {
  const int32_t* nbr;
  const int32_t* n_dev;
  int cap;
  int32_t* halo_rows;
  int32_t* halo_n;
  int16_t* lnbr;
} fpvs_halo_job;
int fpvs_kmap_halo_multi(const fpvs_halo_job* jobs, int njobs, void* stream);
size_t fpvs_spconv_halo_workspace_size(int cap, int cout, int bn, int split);
int fpvs_spconv_halo(const void* x, int ldx, int x_rows, const int32_t* nbr, const int16_t* lnbr,
                     const int32_t* halo_rows, const int32_t* halo_n, const uint32_t* tile_masks,
                     const int32_t* n_dev, int cap, const void* w_packed, int bn, int split,
                     const float* bias, int cin, int cout, int act, void* y, int ldy, int col_off,
                     void* ws, size_t ws_bytes, void* stream);

/* fpvs_spconv_halo with tile-level dataflow between two convs of ONE level
 * (same tables; the consumer reads the producer's output):
 * tile_done_out (int32 [tiles], nullable): the producer's per-tile flags — the
 * CTA owning tile t zeroes it at its start and it reaches 4 once the tile's
 * output rows are stored (one release add per epilogue warp; split must be 1,
 * bn = Cout).  tile_done_in
 * (nullable): the producer's flags; the consumer, launched right after it
 * with programmatic dependent launch, then skips the grid-wide wait and each
 * CTA waits only for the producer tiles holding its tile's halo rows (all of
 * them when the halo was capped), so its first tiles start on the SMs the
 * producer's last wave leaves idle.  Requires FPVS_TABLES_SETTLED in act, a
 * weight image packed before the producer launched, and a y the producer
 * does not read or write.  With both NULL this is fpvs_spconv_halo. */
int fpvs_spconv_halo_flow(const void* x, int ldx, int x_rows, const int32_t* nbr, const int16_t* lnbr,
                          const int32_t* halo_rows, const int32_t* halo_n, const uint32_t* tile_masks,
                          const int32_t* n_dev, int cap, const void* w_packed, int bn, int split,
                          const float* bias, int cin, int cout, int act, void* y, int ldy, int col_off,
                          void* ws, size_t ws_bytes, int32_t* tile_done_out, const int32_t* tile_done_in,
                          void* stream);

/* Submanifold 3x3x3 conv over DENSE BRICKS of 1 x 16 x 8 cells of a level
 * (B x X x Y x Z cells, C order; index_vol[cell] = the cell's row of x or -1),
 * for well-filled levels: every brick is an M = 128 tile whose 27 tap
 * operands are shifted views of one dense halo brick in shared memory
 * (tcgen05 SS MMAs, no gather builders).  Computes the same rows as
 * fpvs_spconv_halo (reference Conv3d.forward, neural.py:187-219, on the
 * active set): y[row] for every active cell; inactive cells read as zero and
 * are not written.  w_packed: fpvs_pack_weights_tc image (K = 27, bn).
 * split (dividing Cin / 64) cuts the channel chunks over CTAs with fp32
 * partials in ws (fpvs_spconv_brick_workspace_size bytes, zeroed once; the
 * kernel leaves its counters zero); split = 1 needs no workspace.  act may
 * carry FPVS_TABLES_SETTLED (index_vol written two or more launches back:
 * its lookups start before the programmatic-launch wait). */
size_t fpvs_spconv_brick_workspace_size(int B, int X, int Y, int Z, int cout, int bn, int split);
int fpvs_spconv_brick(const void* x, int ldx, int x_rows, const int32_t* index_vol, int B, int X, int Y, int Z,
                      const void* w_packed, int bn, int split, const float* bias, int cin, int cout, int act,
                      void* y, int ldy, int col_off, void* ws, size_t ws_bytes, void* stream);

/* The U-Net's last level-0 conv (Cout = 64, relu) with the 1x1x1 head fused
 * into its epilogue (d = 4): each tile's bf16 activations become the A
 * operand of the head's tcgen05 MMAs in tensor memory, and active row r's
 * 64 thresholded outputs [sigmoid(z) >= tau] go to row_bits[r] (bit k =
 * channel k = lx + 4 ly + 16 lz); the conv's own output never goes to HBM.
 * Same conv arguments as fpvs_spconv_halo with bn = 64, split = 1 (flags:
 * FPVS_TABLES_SETTLED or 0, as fpvs_spconv_halo's act flag; tile_done_in:
 * as fpvs_spconv_halo_flow's consumer side, nullable);
 * head_w_packed: the head's fpvs_pack_weights_tc image (K = 1, bn = 64).
 * With fpvs_rowbits_to_grid this replaces the final Conv3d + sigmoid +
 * deinterleave(tau) of the reference (neural.py:513-526, interleave.py:68-80). */
int fpvs_spconv_halo_head(const void* x, int ldx, int x_rows, const int32_t* nbr, const int16_t* lnbr,
                          const int32_t* halo_rows, const int32_t* halo_n, const uint32_t* tile_masks,
                          const int32_t* n_dev, int cap, const void* w_packed, const float* bias, int cin,
                          void* ws, size_t ws_bytes, const void* head_w_packed, const float* head_bias,
                          float tau, uint64_t* row_bits, int flags, const int32_t* tile_done_in,
                          void* stream);

/* fpvs_spconv_halo_head that also publishes tile_done_out[t] = 4 once the
 * row masks of 128-row tile t are stored (as fpvs_spconv_halo_flow's
 * producer side; zeroed by the launch itself), for
 * fpvs_rowbits_to_grid_flow. */
int fpvs_spconv_halo_head_flow(const void* x, int ldx, int x_rows, const int32_t* nbr, const int16_t* lnbr,
                               const int32_t* halo_rows, const int32_t* halo_n, const uint32_t* tile_masks,
                               const int32_t* n_dev, int cap, const void* w_packed, const float* bias, int cin,
                               void* ws, size_t ws_bytes, const void* head_w_packed, const float* head_bias,
                               float tau, uint64_t* row_bits, int flags, const int32_t* tile_done_in,
                               int32_t* tile_done_out, void* stream);

/* Per-row 64-bit cell masks (fpvs_spconv_halo_head) -> the packed froxel grid
 * B x Nx x Ny x Nz (FPVS bit order, d = 4, N_x % 32 == 0): every 32-bit word
 * of out_bits is written exactly once (no clear needed); cells whose
 * level-0 index_vol entry is -1 are 0. */
int fpvs_rowbits_to_grid(const uint64_t* row_bits, const int32_t* index_vol, int B, int Nx, int Ny, int Nz, int d,
                         uint8_t* out_bits, void* stream);
/* The same grid as a dataflow consumer of fpvs_spconv_halo_head_flow launched
 * immediately before: each block (an 8-cell x octet of one cell row) waits
 * only for the done flags of the tiles holding its cells' rows (N_z <= 1024).
 * index_vol must be two or more launches old. */
int fpvs_rowbits_to_grid_flow(const uint64_t* row_bits, const int32_t* index_vol, int B, int Nx, int Ny, int Nz,
                              int d, uint8_t* out_bits, const int32_t* tile_done_in, void* stream);

/* Fused head (replaces the final Conv3d + sigmoid + deinterleave(tau),
 * neural.py:513-526): 1x1x1 conv Cin -> d^3, sigmoid, [p >= tau], packed-bit
 * scatter into out_bits (zeroed first; u32-aligned).  probs (nullable):
 * f32 [cap][d^3] per-active-cell probabilities; logits likewise. */
int fpvs_head_simt(const void* x, int ldx, int in_dtype, const int32_t* coords,
                   const int32_t* n_dev, int cap, const float* w, const float* bias,
                   int cin, int d, int B, int Nx, int Ny, int Nz, float tau,
                   uint8_t* out_bits, float* probs, float* logits, void* stream);
int fpvs_head_tc(const void* x, int ldx, int x_rows, const int32_t* coords, const int32_t* n_dev,
                 int cap, const void* w_packed, const float* bias, int cin, int d,
                 int B, int Nx, int Ny, int Nz, float tau,
                 uint8_t* out_bits, float* probs, float* logits, void* stream);

/* ---- (4) training ------------------------------------------------------ */

/* Per-sample soft counts over active-cell probabilities (ConfusionCounts,
 * neural.py:130-144): sums[3b..3b+2] = (sum p*g, sum p, sum g) in f64, sum g
 * over the whole label grid.  p: f32 [cap][C]; gt_bits: packed label grids.
 * sums must hold fpvs_loss_sums_size(B, cap) bytes (results, then per-row
 * scratch); reductions run in a fixed order (deterministic). */
size_t fpvs_loss_sums_size(int B, int cap);
int fpvs_loss_counts(const float* probs, int C, const int32_t* coords, const int32_t* n_dev,
                     int cap, const uint8_t* gt_bits, int d, int B, int Nx, int Ny, int Nz,
                     double* sums, void* stream);
/* dL/dlogit for combined_loss (neural.py:353-399) averaged over the batch,
 * written as f32 [cap][C]; loss_out[0] = batch-mean loss (f64). */
int fpvs_loss_grad(const float* probs, int C, const int32_t* coords, const int32_t* n_dev,
                   int cap, const uint8_t* gt_bits, int d, int B, int Nx, int Ny, int Nz,
                   const double* sums, double alpha, double lam, float* dlogits,
                   double* loss_out, void* stream);

/* Head epilogue over logits rows f32 [cap][ld] (a head layer with kernel
 * k > 1, run first as a conv with no activation): sigmoid, [p >= tau],
 * packed-bit scatter into out_bits (nullable), probs f32 [cap][d^3] (nullable). */
int fpvs_head_rows(const float* logits, int ld, const int32_t* coords, const int32_t* n_dev, int cap,
                   int d, int B, int Nx, int Ny, int Nz, float tau, uint8_t* out_bits, float* probs,
                   void* stream);
/* dz = dy * act'(y) on active rows from the layer's kept output y
 * (relu: y > 0 <=> z > 0, neural.py:227-228; sigmoid: y (1 - y), :229-230). */
int fpvs_act_backward(const float* dy, int lddy, const void* y, int y_dtype, int ldy,
                      const int32_t* n_dev, int cap, int C, int act, float* dz, int lddz, void* stream);

/* dgrad: dx[n] += dz[i] . W_j^T over pairs n = nbr[i][j] (mirrored gather:
 * dx[n] = sum_j dz[nbr[n][K-1-j]] . W_j^T for the symmetric subm map), then
 * optionally times (ymask[n] > 0) (relu' with z > 0, neural.py:227-228). */
int fpvs_spconv_dgrad_simt(const float* dz, int lddz, const int32_t* nbr, int K,
                           const int32_t* n_dev, int cap, const float* w, int cin, int cout,
                           const void* ymask, int mask_dtype, int ldm, float* dx, int lddx, void* stream);
/* wgrad: dw[j*Cin + ci][co] = sum_i x[nbr[i][j]][ci] * dz[i][co]; db = sum_i dz.
 * Deterministic (fixed split + fixed-order reduction, no float atomics). */
size_t fpvs_wgrad_workspace_size(int K, int cin, int cout, int cap);
int fpvs_spconv_wgrad_simt(const void* x, int ldx, int x_dtype, const float* dz, int lddz,
                           const int32_t* nbr, int K, const int32_t* n_dev, int cap,
                           int cin, int cout, float* dw, float* db,
                           void* workspace, size_t workspace_bytes, void* stream);

/* Tensor-core backward (bf16 operands, fp32 accumulate), BASELINE config 5.
 * dgrad: dx = conv over the same table with mirrored offsets and per-offset
 * transposed weights (nbr[i][j] = k <=> nbr[k][K-1-j] = i for submanifold
 * tables), packed by fpvs_pack_weights_tc_dgrad from the reference-layout
 * W (K*Cin, Cout); the epilogue multiplies by relu'(z) = [mask > 0] taken from
 * the kept bf16 output of the layer below (neural.py:227-228) and writes bf16.
 * wgrad: dW[j*Cin + ci][co] = sum_i x[nbr[i][j]][ci] * dz[i][co] and
 * db = sum_i dz[i] on tcgen05 with both operands MN-major (gathered x, dz),
 * fixed-order reduction of per-CTA partials (deterministic). */
int fpvs_pack_weights_tc_dgrad(const float* w, int K, int cin, int cout, int bn, void* packed, void* stream);

/* Several weight images in ONE launch (the training step re-packs every
 * layer's forward and dgrad image after each optimizer update): job i is
 * fpvs_pack_weights_tc (dgrad = 0) or fpvs_pack_weights_tc_dgrad (dgrad = 1)
 * of (w, K, cin, cout, bn) into packed, byte-identical to the single calls. */
typedef struct fpvs_pack_job {
  const float* w;
  int K, cin, cout, bn, dgrad;
  void* packed;
} fpvs_pack_job;
int fpvs_pack_weights_tc_multi(const fpvs_pack_job* jobs, int njobs, void* stream);
int fpvs_spconv_tc_dgrad(const void* dz, int lddz, int dz_rows, const int32_t* nbr, int K,
                         const uint32_t* tile_masks, const int32_t* n_dev, int cap,
                         const void* w_packed_dgrad, int bn, int cin, int cout, const void* mask, int ldm,
                         void* dx, int lddx, void* stream);
size_t fpvs_wgrad_tc_workspace_size(int K, int cin, int cout, int cap);
int fpvs_spconv_wgrad_tc(const void* x, int ldx, const void* dz, int lddz, const int32_t* nbr, int K,
                         const int32_t* n_dev, int cap, int cin, int cout, float* dw, float* db,
                         void* workspace, size_t workspace_bytes, void* stream);
/* f32 -> bf16 (round to nearest even), n elements. */
int fpvs_cast_bf16(const float* src, long long n, void* dst, void* stream);
/* The first min(*n_dev, cap) rows of an fp32 [cap][cols] matrix to bf16
 * (rows past the device count are left untouched). */
int fpvs_cast_bf16_rows(const float* src, int cols, const int32_t* n_dev, int cap, void* dst, void* stream);

/* Optimizer steps over ONE flat fp32 parameter buffer (all layers' weights
 * and biases back to back; the data-parallel gradient is one all-reduce of
 * the matching flat gradient).  SGD replaces PvsNet.sgd_step
 * (neural.py:293-297) with lr = lr0 * (1 - decay)^step (neural.py:481);
 * AdamW (BASELINE config 5, fp32 master weights): m, v zero-initialised,
 * step counts from 1, decoupled weight decay. */
int fpvs_sgd_step(float* params, const float* grads, size_t n, float lr, void* stream);

/* Data-parallel exchange (one all-reduce per step): flat = [gradient n f32 |
 * FPVS_EXCHANGE_TAIL f32].  fpvs_exchange_pack scales the local mean gradient
 * by weight = B_local / B_global (the sum over ranks is the batch mean of
 * neural.py:472-477) and writes the tail: batch-mean loss x B_local, B_local,
 * and the summed TP/FP/FN/GTP of counts[4B] as exact 12-bit f32 digits.
 * After the all-reduce fpvs_exchange_accumulate adds the tail into the epoch
 * accumulator acc f64[8] = {loss x samples, samples, TP, FP, FN, GTP,
 * first non-finite batch index (init -1), its loss} on the device, so the
 * training loop needs no host round trip per step (TrainingDiverged is raised
 * from acc[6] at the end of the epoch). */
#define FPVS_EXCHANGE_TAIL 10
int fpvs_exchange_pack(float* flat, size_t n, float weight, const double* loss, const int64_t* counts,
                       int B, void* stream);
int fpvs_exchange_accumulate(const float* tail, double* acc, int batch_index, void* stream);
int fpvs_adamw_step(float* params, const float* grads, float* m, float* v, size_t n, float lr,
                    float beta1, float beta2, float eps, float weight_decay, int step, void* stream);

/* Hard confusion counts of thresholded predictions against labels, both as
 * packed grids (replaces the hard-count loops of neural.py:423-439 and
 * 485-490): counts[4b..4b+3] = (TP, FP, FN, GTP) as int64 for sample b. */
size_t fpvs_bits_confusion_workspace_size(int B);
int fpvs_bits_confusion(const uint8_t* pred_bits, const uint8_t* gt_bits, int B, long long grid_bytes,
                        long long* counts, void* workspace, size_t workspace_bytes, void* stream);

/* Synthetic PVS labels (row LBL): first occupied froxel of any column within
 * +-radius in x/y; packed in, packed out. */
int fpvs_first_hit_labels(const uint8_t* bits, int B, int Nx, int Ny, int Nz, int radius,
                          uint8_t* out_bits, int32_t* zfirst_ws, void* stream);

/* Halo-cached weight gradient of a 27-tap conv with Cin = 32 (wgrad_halo.cu):
 * the same dW / db as fpvs_spconv_wgrad_tc (K = 27), reading each 128-row
 * tile's neighbour rows once from the halo tables of fpvs_kmap_halo
 * (halo_rows, halo_n, lnbr) instead of gathering 27 pieces per row.
 * Cout in {8, 16, 24, 32}; workspace fpvs_wgrad_halo_workspace_size(cap). */
size_t fpvs_wgrad_halo_workspace_size(int cap);
int fpvs_spconv_wgrad_halo(const void* x, int ldx, const void* dz, int lddz, const int32_t* nbr,
                           const int32_t* n_dev, int cap, const int32_t* halo_rows, const int32_t* halo_n,
                           const int16_t* lnbr, int cin, int cout, float* dw, float* db, void* workspace,
                           size_t workspace_bytes, void* stream);

/* ---- (§8(f) #1) perspective froxelization ------------------------------ */
/* Frustum of pkg/src/froxelpvs/core.py:297-325 as the rasterizer reads it:
 * origin (_o), basis rows (right, up, forward) (_basis), half_extent =
 * tan(fov/2), near, far. */
typedef struct {
  double origin[3];
  double basis[9];
  double half_extent, near_z, far_z;
} fpvs_frustum;

enum { FPVS_DEPTH_LINEAR = 0, FPVS_DEPTH_LOG = 1 };

/* Rasterize a triangle scene into a packed geometry grid; replaces
 * froxel.py:387-394 froxelize() in mode "perspective" (froxel.py:328-348,
 * 292-325, 229-285, 203-219).  verts: float64 [nverts][3] world positions;
 * tris: int64 [ntris][3] vertex indices (TriScene.triangles, after its
 * degenerate-triangle drop); frustum: HOST pointer; dims (Nx % 8 == 0),
 * supersample >= 1, depth_mode FPVS_DEPTH_*.  out_bits (Nz, Ny, Nx/8) is
 * overwritten.  Triangle indices outside [0, nverts) are skipped.  Results
 * equal the reference bit-for-bit in linear depth mode (the arithmetic is
 * the reference's float64 expression sequence, unfused). */
size_t fpvs_froxelize_workspace_size(long long ntris, int Nx, int Ny, int Nz, int supersample);
int fpvs_froxelize(const double* verts, long long nverts, const int64_t* tris, long long ntris,
                   const fpvs_frustum* frustum, int Nx, int Ny, int Nz, int supersample, int depth_mode,
                   uint8_t* out_bits, void* workspace, size_t workspace_bytes, void* stream);
/* Orthographic three-view froxelization; replaces froxel.py:351-376
 * froxelize_orthographic() (FroxelizeConfig(mode="ortho"), the dataset
 * generator's default).  Three axis-aligned passes over the frustum's world
 * AABB at spacing max(extent) / (supersample * max(N)); every covered sample
 * point is reconstructed in world space, projected into the frustum and its
 * froxel bit set.  Same arguments and output as fpvs_froxelize; bit-exact
 * with the reference in both depth modes. */
size_t fpvs_froxelize_ortho_workspace_size(long long ntris, int Nx, int Ny, int Nz, int supersample);
int fpvs_froxelize_ortho(const double* verts, long long nverts, const int64_t* tris, long long ntris,
                         const fpvs_frustum* frustum, int Nx, int Ny, int Nz, int supersample, int depth_mode,
                         uint8_t* out_bits, void* workspace, size_t workspace_bytes, void* stream);
/* Ground-truth PVS by dense viewpoint sampling; replaces oracle.py:141-172
 * compute_gt_pvs() (render_depth oracle.py:107-138 per camera, then
 * reprojection core.py:380-452 into the viewcell frustum).  cams: DEVICE
 * array of ncams cameras in fpvs_frustum form (origin = camera position,
 * basis rows right/up/forward, half_extent, near, far); frustum: HOST
 * pointer (build_viewcell_frustum).  res_w x res_h is the depth-buffer
 * resolution (OracleConfig.resolution_for: default 4 Nx x 4 Ny).  prim_ids
 * (int64 per triangle) is only needed when some id is negative: exact depth
 * ties then resolve to the smallest id and pixels won by a negative id are
 * not fragments; NULL means ids 0..T-1.  gt_bits is cleared unless
 * accumulate != 0 (several camera batches into one grid); geometry_bits
 * (nullable) gets every GT bit OR-ed in too.  Grids must be 4-byte aligned
 * with Nx*Ny*Nz/8 % 4 == 0.  Linear depth is bit-exact with the reference. */
size_t fpvs_gt_pvs_workspace_size(long long ntris, int ncams, int res_w, int res_h, int with_prim_ids);
int fpvs_gt_pvs(const double* verts, long long nverts, const int64_t* tris, long long ntris,
                const int64_t* prim_ids, const fpvs_frustum* cams, int ncams, int res_w, int res_h,
                const fpvs_frustum* frustum, int Nx, int Ny, int Nz, int depth_mode, int accumulate,
                uint8_t* gt_bits, uint8_t* geometry_bits, void* workspace, size_t workspace_bytes,
                void* stream);

/* Culling from a froxel PVS: kept[t] = 1 iff scene
 * triangle t has a perspective fragment (the froxelize() stream with the
 * same frustum / dims / supersample / depth mode) in a froxel whose pvs bit
 * is set — i.e. evalrt.py:62-68 cull() over froxel_id_map() (froxel.py:
 * 397-417) without materialising the map.  kept: uint8 [ntris], zeroed by
 * the call; pvs_bits 4-byte aligned, Nx*Ny*Nz/8 % 4 == 0.  Workspace:
 * fpvs_froxelize_workspace_size. */
int fpvs_froxel_cull(const double* verts, long long nverts, const int64_t* tris, long long ntris,
                     const fpvs_frustum* frustum, int Nx, int Ny, int Nz, int supersample, int depth_mode,
                     const uint8_t* pvs_bits, uint8_t* kept, void* workspace, size_t workspace_bytes, void* stream);

/* The fragment pairs behind froxel_id_map() (froxel.py:397-417): one int64
 * key = (x + Nx*(y + Ny*z)) * ntris + triangle per fragment, duplicates
 * within a warp dropped (callers unique the keys).  At most cap keys are
 * written; *npairs_dev (device) receives the number produced, which may
 * exceed cap (then call again with a larger buffer; cap = the candidate
 * sample count from fpvs_froxelize_samples always suffices). */
int fpvs_froxel_pairs(const double* verts, long long nverts, const int64_t* tris, long long ntris,
                      const fpvs_frustum* frustum, int Nx, int Ny, int Nz, int supersample, int depth_mode,
                      long long* pairs, long long cap, unsigned long long* npairs_dev, void* workspace,
                      size_t workspace_bytes, void* stream);

/* The same two consumers over the orthographic fragment stream
 * (froxel.py:351-376, 397-417 with FroxelizeConfig(mode="ortho"), as the
 * reference's CLI infer/metrics path uses it, cli.py:297-300).  Arguments as
 * above; workspace: fpvs_froxelize_ortho_workspace_size; cap = the candidate
 * sample count from fpvs_froxelize_samples after fpvs_froxelize_ortho. */
int fpvs_froxel_cull_ortho(const double* verts, long long nverts, const int64_t* tris, long long ntris,
                           const fpvs_frustum* frustum, int Nx, int Ny, int Nz, int supersample, int depth_mode,
                           const uint8_t* pvs_bits, uint8_t* kept, void* workspace, size_t workspace_bytes,
                           void* stream);
int fpvs_froxel_pairs_ortho(const double* verts, long long nverts, const int64_t* tris, long long ntris,
                            const fpvs_frustum* frustum, int Nx, int Ny, int Nz, int supersample, int depth_mode,
                            long long* pairs, long long cap, unsigned long long* npairs_dev, void* workspace,
                            size_t workspace_bytes, void* stream);

/* Depth + primitive-id buffers of oracle.py:107-138 render_depth() for
 * ncams cameras (DEVICE array, fpvs_frustum form) at res_w x res_h:
 * depth_out float64 [ncams][res_h][res_w] (+inf where empty, nullable),
 * prim_out int64 (-1 where empty; exact depth ties -> smallest id).
 * prim_ids NULL = triangle index.  Workspace:
 * fpvs_gt_pvs_workspace_size(ntris, ncams, res_w, res_h, 1). */
int fpvs_render_depth(const double* verts, long long nverts, const int64_t* tris, long long ntris,
                      const int64_t* prim_ids, const fpvs_frustum* cams, int ncams, int res_w, int res_h,
                      double* depth_out, int64_t* prim_out, void* workspace, size_t workspace_bytes, void* stream);

/* Debug/measurement: number of candidate samples (sum of clipped bounding
 * boxes) of the last fpvs_froxelize / fpvs_gt_pvs on this workspace, read back to host
 * (synchronises the stream). */
long long fpvs_froxelize_samples(const void* workspace, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* FPVS_H_ */
