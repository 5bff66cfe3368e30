// Symbolic structure of the smoothed stiffness for the own node range [n_lo, n_lo + nloc)
// (S5; DESIGN.md §5 "symmetric block storage").
//
// K is symmetric (Eq. 9: K = sum_k V_k B_k^T c B_k with c symmetric), so each own node row i
// stores only the 3x3 blocks K_ij with j >= i, plus the blocks whose column node j is below the
// rank's range (j < n_lo, a "halo" block no local row stores).  The remaining blocks of row i
// (n_lo <= j < i) are read transposed from row j: K_ij = K_ji^T.  Values are block-contiguous:
// entry (a, c) of stored block b is vals[9*b + 3*a + c].  Arrays the SpMV streams with bulk
// copies (sptr, tptr, snbr, tlist, vals) carry >= 16 B of slack after their last element.
#pragma once
#include <vector>
#include "common.cuh"

namespace fsfem {

// SpMV streaming chunk (pcg.cu): own nodes [n0, n1), their stored blocks [Ps0, Ps1) and
// transposed entries [Pt0, Pt1).  Chunks hold <= kChunkNodes nodes and <= kCapBlocks of each.
#ifndef FSFEM_CHUNK_NODES
#define FSFEM_CHUNK_NODES 32
#endif
#ifndef FSFEM_CAP_BLOCKS
#define FSFEM_CAP_BLOCKS 512
#endif
constexpr int kChunkNodes = FSFEM_CHUNK_NODES;
constexpr int kCapBlocks = FSFEM_CAP_BLOCKS;
#ifndef FSFEM_MAX_DEPS
#define FSFEM_MAX_DEPS 48
#endif
constexpr int kMaxDeps = FSFEM_MAX_DEPS;
struct SpmvChunk {
  int32_t n0, n1, Ps0, Ps1, Pt0, Pt1, pad0, pad1;
};

struct Pattern {
  int64_t n_lo = 0, nloc = 0;
  int64_t nblk = 0;  // blocks of the full node graph (public CSR nnz = 9 * nblk)
  int64_t nsb = 0;   // stored blocks
  int64_t ntb = 0;   // transposed (gathered) blocks
  int64_t nfi = 0;   // node-face incidences (sum over own nodes of |F(i)|)
  DevBuf<int64_t> node_ptr;  // [nloc+1] full neighbour list offsets
  DevBuf<int32_t> nbr;       // [nblk] sorted neighbour node ids of every own node
  DevBuf<int64_t> sptr;      // [nloc+1] stored block offsets
  DevBuf<int32_t> snbr;      // [nsb] column node of each stored block (ascending per row)
  DevBuf<int32_t> sdiag;     // [nloc] slot of the diagonal block inside the stored row
  DevBuf<int32_t> diag_full; // [nloc] slot of the diagonal inside the full neighbour list
  DevBuf<int64_t> tptr;      // [nloc+1] transposed block offsets
  DevBuf<int2> tlist;        // [ntb] (stored block index of K_ji, node j), ascending j
  int64_t nchunks = 0;
  DevBuf<SpmvChunk> chunks;  // [nchunks] SpMV streaming chunks
  // Dataflow push SpMV (pcg.cu k_spmv_df): the transposed product K_ij^T x_i of stored block
  // b = (i, j) is written by row i to tbuf[tpos[b]] (the slot of K_ji in row j's transposed list),
  // and row j sums its contiguous slots once every chunk holding a producer row has finished.
  DevBuf<int32_t> tpos;      // [nsb + 4] slot in the transposed list, or -1 (diagonal, halo, beyond range)
  DevBuf<double> tbuf;       // [3 ntb + 2] pushed transposed products
  DevBuf<int32_t> deps;      // [nchunks * kMaxDeps] distinct earlier chunks holding producer rows
  DevBuf<int32_t> ndeps;     // [nchunks] their number, or -1 (more than kMaxDeps: no dataflow SpMV)
  DevBuf<uint32_t> cflags;   // [nchunks] epoch at which the chunk became ready for phase 2
  DevBuf<uint32_t> sync;     // [2] epoch, last-CTA ticket
  // chunk d needs ndeps[d] + 1 finished phase-1 chunks (its producers and itself);
  // dep_ptr/dep_list = for each chunk c the chunks d that need it (c itself first), with that count.
  bool df_ok = false;        // every chunk's producer list fits kMaxDeps
  DevBuf<int32_t> dep_ptr;   // [nchunks + 1]
  DevBuf<int2> dep_list;     // [dep_ptr[nchunks]] (chunk d, need[d])
  DevBuf<int2> dep_tmp;      // [nchunks * (kMaxDeps + 1)] unsorted lists (symbolic scratch)
  // split SpMV (halo overlap): the chunks reordered interior first, nch_int of them interior
  bool have_ov = false;
  int64_t nch_int = 0;
  DevBuf<SpmvChunk> chunks_ov;
  DevBuf<uint32_t> cnt;      // [nchunks] arrival counters, wrapping at need (atomicInc: 0 .. need-1)
  DevBuf<double> dotc;       // [nchunks] per-chunk p.q partials
  // halo of the rank (halo.cu, row partitions only): columns of the own rows outside the range
  int64_t nhalo = 0;
  DevBuf<int32_t> halo;      // [nhalo] global node ids, ascending (grouped by owner rank)
  DevBuf<int64_t> nf_ptr;    // [nloc+1]
  DevBuf<int32_t> nf_idx;    // [nfi] faces whose field holds node i, ascending
  // Assembly tiles (assemble.cu, built once per pattern): the own nodes in Morton order cut into
  // tiles of <= kTileRows rows; per tile one contiguous blob (TileHdr + rows, vertices, field
  // positions, tasks, program entries), tile t at tile_blob + t * kBlobCap, tile_bytes[t] long.
  int64_t ntiles = 0;
  int64_t tile_blob_max = 0;    // largest tile blob (bytes)
  int64_t tile_blob_bytes = 0;  // sum of the blob sizes (read once per numeric assembly)
  DevBuf<int64_t> tile_bytes;   // [ntiles]
  DevBuf<int32_t> tile_order, tile_tmp, tile_redo;  // builder scratch (kept: no cudaFree per mesh)
  DevBuf<int2> tile_range;                           // [ntiles] own-row range of tile t in tile_order
  DevBuf<unsigned char> tile_blob;
};

}  // namespace fsfem
