/* hodlr_b200.h -- C ABI of the B200-native mixed-precision HODLR matvec.
 *
 * This is the drop-in boundary for the reference's HODLR matrix-vector product.
 * The reference (arXiv 2407.21637, package `hodlrmp`) has no FFI: its hot-path
 * operator is the Python function
 *
 *     linops.matvec(H: HodlrMatrix, x, working: PrecisionFormat) -> vector
 *         /root/reference/SPEC.md:334-342  (Algorithm 3)
 *
 * operating on the object model of /root/reference/pkg/src/hodlrmp/hodlr.py:
 *     HodlrMatrix.offdiag_blocks()   hodlr.py:111-123  -> hodlr_desc.factors order
 *     HodlrMatrix.leaves()           hodlr.py:125-135  -> hodlr_desc.leaves
 *     LowRankFactor(U, V, fmt)       lowrank.py:30-67  -> hodlr_factor_in
 *     PrecisionFormat / named fmts   fpsim.py:48-116   -> hodlr_format
 *     store_factor -> round_matrix   lowrank.py:117-119, fpsim.py:160-185
 *                                                      -> hodlr_quantize (K0)
 * The Python host layer (paper_2407_21637_b200.linops.matvec) keeps that
 * signature and calls the entry points below through ctypes; INTEGRATION.md
 * shows the binding.  Plain C types only: no torch, no C++ in the signatures.
 *
 * Error convention (mirrors the reference's ValueError convention,
 * hodlr.py:164-170): every entry point returns a hodlr_status;
 * hodlr_last_error() returns a thread-local message for the last failure.
 *   HODLR_ERR_INVALID      -> ValueError          (shape / length / layout)
 *   HODLR_ERR_UNSUPPORTED  -> NotImplementedError (custom formats, ...)
 *   HODLR_ERR_CUDA         -> RuntimeError        (CUDA or allocation failure)
 */
#ifndef HODLR_B200_H
#define HODLR_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HODLR_B200_ABI_VERSION 3

typedef enum {
    HODLR_OK = 0,
    HODLR_ERR_INVALID = 1,
    HODLR_ERR_UNSUPPORTED = 2,
    HODLR_ERR_CUDA = 3
} hodlr_status;

/* The five named formats of fpsim.py:110-114 (q52 = fp8 E5M2). */
typedef enum {
    HODLR_FMT_Q52 = 0,  /* t=3,  e in [-14,15],     8 bits  */
    HODLR_FMT_BF16 = 1, /* t=8,  e in [-126,127],   16 bits */
    HODLR_FMT_FP16 = 2, /* t=11, e in [-14,15],     16 bits */
    HODLR_FMT_FP32 = 3, /* t=24, e in [-126,127],   32 bits */
    HODLR_FMT_FP64 = 4  /* t=53, e in [-1022,1023], 64 bits */
} hodlr_format;

/* One LowRankFactor (lowrank.py:30-67): block = U V^T, U rows x rank,
 * V cols x rank, given as binary64 with arbitrary element strides (so numpy
 * C-order U and F-order V are passed without copies).  Values need not be
 * pre-rounded: hodlr_create rounds them into `fmt` bit-exactly (store_factor). */
typedef struct {
    int32_t fmt;            /* hodlr_format of the block (PrecisionPlan level format) */
    int32_t rank;
    int64_t rows, cols;     /* U is rows x rank, V is cols x rank */
    const double* U;        /* U[i,c] = U[i*u_rs + c*u_cs]  (void* of the fmt encoding
                               when hodlr_desc.payload_encoded = 1; same for V, leaves) */
    int64_t u_rs, u_cs;
    const double* V;        /* V[j,c] = V[j*v_rs + c*v_cs] */
    int64_t v_rs, v_cs;
} hodlr_factor_in;

/* A whole HodlrMatrix (hodlr.py:95-135) in host memory. */
typedef struct {
    int64_t n;
    int32_t depth;            /* l >= 0 */
    int32_t leaf_fmt;         /* H.working_format: format of the dense leaves */
    const int64_t* leaf_bounds; /* 2^depth + 1 boundaries of the leaf intervals */
    const double* const* leaves;/* 2^depth pointers: leaf i is m_i x m_i */
    const int64_t* leaf_ld;   /* row stride (elements) of each leaf, >= m_i */
    const hodlr_factor_in* factors; /* 2*(2^depth - 1) entries, offdiag_blocks()
                                      order: level-major, pair-major, [upper, lower] */
    int32_t payload_encoded;  /* 0: every payload is binary64 (the reference's in-memory
                                 model and container v1, hodlr.py:297-363).
                                 1: narrow payloads (container v2): leaf i points at its
                                 leaf_fmt encoding and each factor's U / V at their `fmt`
                                 encoding (q52: 1 byte, bf16 / fp16: 2, fp32: 4, fp64: 8
                                 per element; strides still in elements), so a stored
                                 matrix reaches the device without a binary64 copy */
} hodlr_desc;

typedef struct hodlr_handle hodlr_handle;

/* Row-range shard of the tree: with nranks = 2^L ranks the
 * rank `rank` owns level-L node `rank`; levels 1..L become "external" levels
 * whose coefficients are exchanged between ranks.  nranks = 1 is the whole
 * matrix. */
typedef struct {
    int32_t rank;
    int32_t nranks;
} hodlr_shard;

/* Pack + quantise H onto `device`.  The handle owns all device memory. */
hodlr_status hodlr_create(const hodlr_desc* d, int32_t device, hodlr_handle** out);
hodlr_status hodlr_create_sharded(const hodlr_desc* d, int32_t device, hodlr_shard shard,
                                  hodlr_handle** out);
hodlr_status hodlr_destroy(hodlr_handle* h);

/* Workspace bytes for a matvec with s right-hand sides. */
hodlr_status hodlr_workspace_size(const hodlr_handle* h, int64_t s, size_t* bytes);

/* b = H x  (Algorithm 3) on `stream`.  x, b: device, row-major n_local x s
 * with leading dimensions ldx, ldb (elements), element type = working format
 * (HODLR_FMT_FP64 -> double, HODLR_FMT_FP32 -> float).  Stream-ordered: no host
 * synchronisation, no allocation once warm.  ws may be NULL: the handle keeps
 * one workspace per CUDA stream (allocated on the first call on that stream and
 * zeroed with cudaMemsetAsync on it), so calls on different streams may overlap
 * and calls on one stream are ordered by it; or ws is a caller buffer of
 * hodlr_workspace_size bytes, zero-filled once before its first use and not
 * modified by the caller afterwards (the fused kernel keeps its per-call
 * synchronisation state there); concurrent calls with distinct ws are safe
 * (SPEC.md:403-404).  Sharded handles: see hodlr_matvec_shard_* below.
 * Narrow working formats (HODLR_FMT_Q52 / BF16 / FP16, the paper's bf16-working
 * experiment): x and b are binary64 carrying working-format
 * values (the reference's own representation); x is rounded to `working` on
 * entry and the call runs the strict-order kernels (see hodlr_matvec_strict);
 * a caller workspace must then have hodlr_workspace_size_for bytes. */
hodlr_status hodlr_matvec(hodlr_handle* h, int32_t working, const void* x, int64_t ldx,
                          void* b, int64_t ldb, int64_t s, void* ws, size_t ws_bytes,
                          void* stream);

/* Strict-order matvec: Algorithm 3 evaluated exactly as the reference's
 * Arithmetic(working) does (arithmetic.py:14-67: every product and partial sum
 * rounded to `working`, contractions strictly left to right, level-major
 * accumulation, leaves last) -- bit-identical to the reference arithmetic for
 * any of the five named working formats (fp64: sequential binary64, which
 * differs from the reference's BLAS order in the last bits).  x, b: device
 * binary64, row-major n x s.  One thread per output chain: the fidelity path of
 * the sweep harness, not the throughput path.  Unsharded handles only. */
hodlr_status hodlr_matvec_strict(hodlr_handle* h, int32_t working, const double* x, int64_t ldx,
                                 double* b, int64_t ldb, int64_t s, void* ws, size_t ws_bytes,
                                 void* stream);
/* Workspace bytes of a call in `working` (strict != 0: hodlr_matvec_strict). */
hodlr_status hodlr_workspace_size_for(const hodlr_handle* h, int32_t working, int32_t strict,
                                      int64_t s, size_t* bytes);

/* End-to-end call with HOST buffers (the reference-facing drop-in): x_host and
 * b_host are binary64, n x s row-major.  Copies x in, rounds it to `working`,
 * runs the matvec, widens b to binary64 and copies it out; returns after the
 * result is in b_host.  Not valid on sharded handles.  When b_host is
 * page-locked (cudaHostAlloc / torch pin_memory) the kernel that stores each b
 * element once (the widening kernel, or the fused s = 1 kernel for binary64
 * working) writes it through the mapped address instead of a D2H copy
 * (HODLR_B200_NO_ZEROCOPY=1 disables this).  Multi-RHS calls with a large result
 * (binary64 working, fragment-slab path, >= 8 MB) run phase B over row ranges and
 * copy each finished range out on a second stream while the next ranges are
 * computed (HODLR_B200_NO_E2E_PIPELINE=1 disables this).
 * Safe to call from several host threads on one handle: the
 * handle keeps two staging contexts, so two calls on different streams overlap
 * (one call's device-to-host copy runs under the other's host-to-device copy:
 * PCIe is full duplex) and further callers wait for a free context. */
hodlr_status hodlr_matvec_host(hodlr_handle* h, int32_t working, const double* x_host,
                               double* b_host, int64_t s, void* stream);

/* Sharded matvec: three stream-ordered steps around one all-gather.
 *   1. shard_begin: this rank's partial V'^T x coefficients of every external
 *      level (1..log2 nranks), over its own rows -> `send` (device,
 *      hodlr_shard_exchange_count(h, s) elements of the working type);
 *   2. the caller starts an all-gather of `send` from every rank, in rank
 *      order, into `recv` (nranks * count elements), e.g. ncclAllGather over
 *      NVLink, and meanwhile calls
 *      shard_local: b_local = D x + sum_{k > L} U_k t_k, the communication-free
 *      subtree part (the single-vector fused kernel when it applies), which
 *      overlaps the exchange;
 *   3. once `recv` is complete on `stream`, shard_end: fixed-order (rank order)
 *      reduction of the gathered coefficients of the sibling subtrees, then
 *      b_local += sum_{k <= L} U_k t_k.
 * shard_local must precede shard_end on the same b_local.  The three calls
 * share the handle's workspace (or `ws`) and must not interleave with another
 * matvec on the same workspace. */
hodlr_status hodlr_shard_exchange_count(const hodlr_handle* h, int64_t s, int64_t* count);
hodlr_status hodlr_matvec_shard_begin(hodlr_handle* h, int32_t working, const void* x_local,
                                      int64_t ldx, int64_t s, void* send, void* ws,
                                      size_t ws_bytes, void* stream);
hodlr_status hodlr_matvec_shard_local(hodlr_handle* h, int32_t working, const void* x_local,
                                      int64_t ldx, void* b_local, int64_t ldb, int64_t s,
                                      void* ws, size_t ws_bytes, void* stream);
hodlr_status hodlr_matvec_shard_end(hodlr_handle* h, int32_t working, const void* x_local,
                                    int64_t ldx, const void* recv, void* b_local, int64_t ldb,
                                    int64_t s, void* ws, size_t ws_bytes, void* stream);

/* K0: bit-exact RNE quantisation of binary64 into `fmt` (round_matrix,
 * fpsim.py:160-185): dst holds the narrow encoding (1/2/2/4/8 bytes each).
 * device pointers, stream-ordered. */
hodlr_status hodlr_quantize(int32_t fmt, const double* src, void* dst, int64_t count,
                            void* stream);
/* Exact widening of a narrow encoding back to binary64. */
hodlr_status hodlr_dequantize(int32_t fmt, const void* src, double* dst, int64_t count,
                              void* stream);
/* The same conversions compiled for the host (same source, same rounding). */
hodlr_status hodlr_quantize_host(int32_t fmt, const double* src, void* dst, int64_t count);
hodlr_status hodlr_dequantize_host(int32_t fmt, const void* src, double* dst, int64_t count);

/* Pack round-trip: copy factor `index` (offdiag_blocks order, [upper, lower])
 * back to the host as binary64, U (rows x rank, C-order) and V (cols x rank,
 * C-order).  Leaf i likewise (m_i x m_i, C-order).  Synchronous. */
hodlr_status hodlr_unpack_factor(const hodlr_handle* h, int64_t index, double* U, double* V);
hodlr_status hodlr_unpack_leaf(const hodlr_handle* h, int64_t leaf, double* D);

/* Accounting: algorithmic bytes of the stored matrix (storage_bits/8,
 * hodlr.py:279-287) of this handle's rows, rows owned, kernel launches per
 * matvec, device bytes held. */
typedef struct {
    int64_t n_local;
    int64_t row0;
    int64_t matrix_bytes;     /* storage_bits(H)/8 restricted to this handle */
    int64_t device_bytes;     /* packed layout incl. alignment padding */
    int32_t depth;
    int32_t leaf_fmt;
    int32_t launches_per_matvec;
    int32_t num_levels_external;
} hodlr_info_t;
hodlr_status hodlr_info(const hodlr_handle* h, hodlr_info_t* info);

/* Which kernels a matvec with `s` right-hand sides in `working` precision
 * runs on this handle (for a sharded handle: shard_local), and how many
 * kernel launches that is.  *path: 0 generic (three launches, any layout),
 * 1 fused single-vector kernel, 2 multi-RHS tensor-core kernels over the
 * level-batched arena, 3 multi-RHS tensor-core kernels over the fragment
 * slabs (uniform 256-row leaves, bulk-copy streamed), 4 the same with phase B
 * on the tcgen05 tensor cores (fp32 working, kind::tf32, item slabs). */
typedef enum {
    HODLR_PATH_GENERIC = 0,
    HODLR_PATH_FUSED_SV = 1,
    HODLR_PATH_MRHS = 2,
    HODLR_PATH_MRHS_SLAB = 3,
    HODLR_PATH_MRHS_TC = 4,
    HODLR_PATH_STRICT = 5   /* strict-order kernels (narrow working formats) */
} hodlr_path;
hodlr_status hodlr_matvec_path(const hodlr_handle* h, int32_t working, int64_t s, int32_t* path,
                               int32_t* launches);

const char* hodlr_last_error(void);
int32_t hodlr_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* HODLR_B200_H */
