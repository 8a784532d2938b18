// Tensor-core (tcgen05 kind::tf32) phase B for fp32 working precision and s > 1:
//     b[leaf rows] = [D | U_1 .. U_l] [X_leaf ; T_1 .. T_l]
// as one contraction per leaf (K = 256 + sum_k round8(ru_k)), the 256 leaf rows
// as two M = 128 tiles, N = up to 64 right-hand sides per pass.
//
// "Item slab" layout (built at create time from the arena, pure byte moves):
// per leaf, the sequence of K-blocks ("items") the kernel consumes -- 8 items of
// 32 leaf columns, then each level's U columns (rounded up to 8) in items of at
// most 32 -- each item stored as [kc = column/4][row 0..255][4 values] in its
// storage format, so
//   * one cp.async.bulk moves an item (<= 32 KB) into the shared-memory ring;
//   * a converter thread (one leaf row) reads its 4 values of a column quad with
//     ONE 16/8/4-byte load, and a warp's load is 512/256/128 contiguous bytes
//     (no bank conflicts);
// the converters split each value into tf32 hi/lo in registers and store them
// to tensor memory (A operand of tcgen05.mma, TS form); narrow formats are exact
// in tf32 and skip the lo part.  See kernels_tc.cu.
#pragma once
#include <cstdint>

namespace hodlr {

constexpr int kTcMaxItems = 160;
constexpr int kTcItemCols = 32;   // K columns per item (max)
constexpr int kTcRows = 256;      // leaf rows (two M = 128 tiles)
constexpr int kTcN = 64;          // right-hand sides per pass (N of the MMA)

struct TcItem {
    int32_t off;       // byte offset inside the leaf's region
    int32_t bytes;     // 256 * ncols * bytes(fmt)
    int16_t fmt;       // storage format
    int16_t ncols;     // multiple of 8, <= 32
    int16_t lv;        // -1: leaf (D) item, else 0-based level of the U factor
    int16_t col0;      // first column (leaf column, or U column inside the level)
};

struct TcView {
    int32_t nitems;
    int32_t nlev;
    int32_t finite;         // every stored value finite: converters use the fast hi/lo split
    int64_t leaf_bytes;     // bytes of one leaf region
    const uint8_t* slab;    // [chunk][leaf_bytes]
    TcItem item[kTcMaxItems];
};

// Phase A on the tensor cores: t = V'^T X per node as, per 256-row chunk,
//     D (M x N) = [V'_1 ; V'_2 ; ... ; V'_l]^T[chunk rows] (M x 256) * X[chunk rows] (256 x N)
// with the levels' (padded) ranks stacked along M (<= 4 tiles of 128), K = the
// chunk's rows in 16 items of 16.  Item layout (A slab, per chunk and item):
// for each level, [kc 0..3][c 0..r8-1][4 values] in the level's format.
constexpr int kTcAMaxTiles = 4;
constexpr int kTcAItemRows = 16;
struct TcALevel {
    int32_t mbase;     // first stacked M row of the level
    int32_t r8;        // rows of the level in the stack (= rv_max, no padding)
    int32_t fmt;       // V' storage format
    int32_t seg;       // byte offset of the level's segment inside an item
};
struct TcAView {
    int32_t nlev, mtot, nmt;
    int32_t finite;           // every stored value finite (fast split)
    int32_t item_bytes;       // bytes of one item (16 rows, all levels)
    int64_t chunk_bytes;      // 16 items
    uint32_t tile_full;       // bit t: tile t holds an fp32 level (needs the A_lo pass)
    const uint8_t* slab;
    TcALevel lev[31];
};

}  // namespace hodlr
