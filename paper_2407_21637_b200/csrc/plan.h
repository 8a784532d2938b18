// Packed device layout of a (possibly sharded) HODLR matrix.
//
// Index model.  With leaves numbered 0..2^l-1, node j of level k (1 <= k <= l)
// covers leaves [j*2^(l-k), (j+1)*2^(l-k)).  The reference stores, per sibling
// pair i of level k (hodlr.py:55-60, 111-123), an upper block (rows node 2i,
// cols node 2i+1) and a lower block (rows 2i+1, cols 2i).  We re-key the two
// factors of every block by the node whose ROWS they span:
//     U_{k,j}  = the U of the block whose row range is node j
//     V'_{k,j} = the V of the block whose column range is node j
// so that Alg. 3 becomes, per level,
//     t_{k,j} = V'_{k,j}^T x[I_j]            (phase A, a reduction over rows)
//     b[I_j] += U_{k,j} t_{k,sib(j)}          (phase B, disjoint rows, no atomics)
// and every row of the matrix touches exactly one U and one V' per level.
//
// Storage: "precision-segregated, level-batched, rank-major".  Each factor is a
// set of rank columns; a column is the node's rows, contiguous, zero-padded to a
// 16-byte multiple, in its block's storage format.  Columns of one format are
// packed level by level in one segment of the arena, so a warp streaming a
// column slab issues 16-byte coalesced loads whatever the format (16 q52 / 8
// bf16|fp16 / 4 fp32 / 2 fp64 values per load).  Leaves are row-major m x ld in
// the leaf (working) format, ld padded to 16 bytes.
#pragma once
#include <cstdint>

namespace hodlr {

struct NodeDesc {
    int64_t u_off, v_off;   // byte offsets of column 0 in the arena
    int32_t u_ld, v_ld;     // column stride in elements
    int32_t ru, rv;         // rank of U_{k,j} (= rank of V'_{k,sib j}) and of V'_{k,j}
    int32_t u_fmt, v_fmt;   // hodlr_format of the two factors
    int32_t row0, nrows;    // local rows spanned (a slice of the node for external levels)
    int32_t chunk0, nchunk; // chunks (row tiles) inside this node
    int64_t part_off;       // partials of V'^T x: [rv][s][nchunk] at part_off*s
    int64_t t_off;          // t_{k,j} (rv x s) at t_off*s in the coefficient buffer
    int64_t tsrc_off;       // coefficients U_{k,j} consumes (ru x s) at tsrc_off*s
    int32_t ext_slot;       // >= 0: external level, this rank's partial goes to send[ext_slot*s]
    int32_t level;          // 1-based tree level
};

struct ChunkDesc {
    int32_t row0, nrows;    // local rows of the tile (inside one leaf)
    int32_t leaf;           // local leaf index
    int32_t pad;
};

struct LeafDesc {
    int64_t off;            // byte offset of the leaf in the arena
    int32_t row0, m;        // local first row and size
    int32_t ld, fmt;        // row stride (elements), storage format
};

// External-level reduction after the all-gather: t = sum over ranks [g0, g1)
// of recv[g*count + slot*s + c*s + q], c < rank, written to tbuf[tdst*s].
struct ExtDesc {
    int32_t slot, rank;     // slot offset (per unit s) and coefficient count
    int32_t g0, g1;         // contributing ranks (sibling subtree), fixed order
    int64_t tdst;           // destination in the coefficient buffer (per unit s)
};

// Everything a kernel needs; passed by value.
struct PlanView {
    const uint8_t* arena;
    const NodeDesc* nodes;
    const ChunkDesc* chunks;
    const int32_t* chunk_nodes;  // [nchunks][nlev]: node id at each level
    const LeafDesc* leaves;
    const ExtDesc* ext;
    int32_t nnodes, nchunks, nlev, nleaves, next;
    int32_t n_local;
    int64_t part_count;          // per unit s
    int64_t t_count;             // per unit s
    int64_t ext_count;           // per unit s: one rank's send size
};

}  // namespace hodlr
