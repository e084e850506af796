/*
 * fmb200.h -- C ABI of libfmb200.so, the B200 (sm_100a) fused-expression
 * backend.  Every entry point is `extern "C"`, takes plain pointers and
 * 64-bit sizes, and returns an int status (0 = ok; otherwise the message is
 * available from fm_last_error()).  Device pointers are ordinary CUDA device
 * pointers; `stream` is a cudaStream_t passed as void* (NULL = legacy stream).
 *
 * Each entry point names the reference interface it replaces.  Reference
 * paths are relative to /root/reference/pkg/src/fusemat/.
 *
 *   reference Backend contract      (backend.py:53-89)      -> this ABI
 *   -----------------------------------------------------------------------
 *   alloc(etype, n_elem)            (backend.py:203-207)    -> fm_alloc (zero-filled)
 *   free(handle)                    (backend.py:218-223)    -> fm_free
 *   upload(host, handle)            (backend.py:227-232)    -> fm_memcpy_h2d
 *   download(handle)                (backend.py:234-235)    -> fm_memcpy_d2h
 *   synchronize()                   (backend.py:237-239)    -> fm_stream_sync
 *   compile(KernelSource)           (cjit.py:113-120)       -> fm_kernel_lookup
 *   launch(kernel, args, geometry)  (cjit.py:132-154)       -> fm_launch_copy
 *     reduce_accu skeleton          (codegen.py:94-114)     -> fm_launch_accu
 *     (new) sum/mean/max/index_max along a dim              -> fm_launch_reduce_dim
 *   matmul(out,left,right,m,k,n,t)  (cjit.py:171-182)       -> fm_gemm
 *   rng.uniform_fill / randi        (rng.py:54-72)          -> fm_randu / fm_randi
 *   measure_copy_bandwidth          (cjit.py:186-208)       -> fm_copy
 */
#ifndef FMB200_H
#define FMB200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FMB200_ABI_VERSION 3

/* element types (exprtree.ElemType.code) */
enum {
  FM_F32 = 0,
  FM_F64 = 1,
  FM_U32 = 2,
  FM_I32 = 3,
  FM_BF16 = 4
};

/* leaf index maps (expr.py:118-204: Leaf / Subview / Diag) */
enum { FM_MAP_DENSE = 0, FM_MAP_SUBVIEW = 1, FM_MAP_DIAG = 2 };

/*
 * Fused program: a postfix (Sethi-Ullman ordered) instruction list evaluated
 * per output element on a register stack.  `key` = (opcode << 3) | depth,
 * where depth is the stack slot the instruction writes (binary ops read
 * depth and depth+1).  This is the B200 replacement for the reference's
 * generated access text (codegen.py:172-227): the same per-node semantics,
 * executed by ahead-of-time compiled kernels instead of a C compiler.
 */
#define FM_MAX_DEPTH 8
#define FM_MAX_INSTR 128
#define FM_MAX_SLOTS 40
#define FM_MAX_SCALARS 32
#define FM_MAX_REDUCE_OUT 6

/* The *_S opcodes are binary ops whose second operand is slot `arg` (a PUSH
 * and the op in one dispatch, one stack register less). */
enum fm_opcode {
  FM_OP_PUSH32 = 0, FM_OP_PUSH64,
  FM_OP_ADD_F, FM_OP_SUB_F, FM_OP_RSUB_F, FM_OP_MUL_F, FM_OP_DIV_F, FM_OP_RDIV_F,
  FM_OP_ADD_D, FM_OP_SUB_D, FM_OP_RSUB_D, FM_OP_MUL_D, FM_OP_DIV_D, FM_OP_RDIV_D,
  FM_OP_ADD_I, FM_OP_SUB_I, FM_OP_RSUB_I, FM_OP_MUL_I,
  FM_OP_SADD_F, FM_OP_SMUL_F, FM_OP_SDIV_F, FM_OP_GTS_F,
  FM_OP_SADD_D, FM_OP_SMUL_D, FM_OP_SDIV_D, FM_OP_GTS_D,
  FM_OP_SADD_I, FM_OP_SMUL_I, FM_OP_GTS_I32, FM_OP_GTS_U32,
  FM_OP_NEG_F, FM_OP_NEG_D, FM_OP_NEG_I, FM_OP_ABS_F, FM_OP_ABS_D, FM_OP_ABS_I32,
  FM_OP_EXP_F, FM_OP_LOG_F, FM_OP_SQRT_F, FM_OP_TANH_F,
  FM_OP_EXP_D, FM_OP_LOG_D, FM_OP_SQRT_D, FM_OP_TANH_D,
  FM_OP_POW_F, FM_OP_POW_D, FM_OP_POW_I,
  FM_OP_ONE_F, FM_OP_ONE_D, FM_OP_ONE_I,
  FM_OP_CVT_F_D, FM_OP_CVT_D_F, FM_OP_CVT_F_I, FM_OP_CVT_D_I,
  FM_OP_CVT_I32_F, FM_OP_CVT_U32_F, FM_OP_CVT_I32_D, FM_OP_CVT_U32_D,
  FM_OP_RND_BF_F, FM_OP_CVT_D_BF,
  FM_OP_ADD_F_S, FM_OP_SUB_F_S, FM_OP_RSUB_F_S, FM_OP_MUL_F_S, FM_OP_DIV_F_S, FM_OP_RDIV_F_S,
  FM_OP_ADD_D_S, FM_OP_SUB_D_S, FM_OP_RSUB_D_S, FM_OP_MUL_D_S, FM_OP_DIV_D_S, FM_OP_RDIV_D_S,
  FM_OP_ADD_I_S, FM_OP_SUB_I_S, FM_OP_RSUB_I_S, FM_OP_MUL_I_S,
  FM_OP_COUNT
};

typedef struct {
  uint16_t key;   /* (opcode << 3) | depth */
  uint16_t arg;   /* slot / scalar index / exponent */
} fm_instr;

typedef struct {
  const void *ptr;   /* parent buffer (column-major) */
  int64_t ld;        /* parent n_rows */
  int64_t row_off;   /* view offsets (subview / diag), 0 for dense */
  int64_t col_off;
  int32_t etype;     /* FM_F32 .. FM_BF16 */
  int32_t map;       /* FM_MAP_* */
  int32_t transposed;/* read parent at (col,row) */
  int32_t reserved;
} fm_slot;

typedef struct {
  int32_t n_instr;
  int32_t n_slots;
  int32_t n_scalars;
  int32_t result_etype;  /* element type of the expression root */
  int32_t flat;          /* 1: every slot is dense, untransposed, same shape as the domain */
  int32_t depth;         /* stack depth used (<= FM_MAX_DEPTH) */
  int32_t wide;          /* 1: some value is 64-bit (f64) */
  int32_t reserved;
  uint64_t scalars[FM_MAX_SCALARS];  /* bit patterns in the slot's compute type */
  fm_instr code[FM_MAX_INSTR];
  fm_slot slots[FM_MAX_SLOTS];
} fm_program;

/* reduction kinds for fm_launch_reduce_dim (exprtree.ReduceKind order) */
enum { FM_RED_SUM = 0, FM_RED_MEAN, FM_RED_MAX, FM_RED_MIN, FM_RED_IMAX, FM_RED_IMIN };

typedef struct {
  int32_t kind;    /* FM_RED_* */
  int32_t etype;   /* output element type */
  void *out;       /* 1 x n_cols (dim 0) or n_rows x 1 (dim 1) */
} fm_reduce_out;

/* accu finalisers */
enum { FM_FINAL_NONE = 0, FM_FINAL_SQRT = 1 };

/* GEMM arguments, all column-major:
 *   T   = round_out(alpha * op(A) @ op(B))
 *   C   = T                                              (c_in == NULL)
 *   C   = round_out(round_out(alpha2 * T) + round_out(beta * C_in))   (epilogue)
 * The epilogue is the elementwise step the reference plans as a separate
 * fused launch after its MatMulStep (e.g. `2*(A@B) + C`, plan.py:171-205),
 * with the same per-operation rounding; C_in may alias C (read then written
 * by the same thread). */
typedef struct {
  const void *a;  int64_t lda;  int32_t trans_a;
  const void *b;  int64_t ldb;  int32_t trans_b;
  void *c;        int64_t ldc;
  int64_t m, n, k;
  double alpha;
  int32_t in_etype;    /* FM_BF16, FM_F32, FM_F64 */
  int32_t out_etype;   /* FM_F32 (bf16/f32 inputs) or FM_F64 */
  int32_t precision;   /* FM_GEMM_* */
  int32_t reserved;
  const void *c_in;    /* epilogue addend (out_etype), or NULL */
  int64_t ld_c_in;
  double alpha2;       /* epilogue scale of the rounded product (1 = none) */
  double beta;         /* epilogue scale of c_in */
} fm_gemm_args;

enum {
  FM_GEMM_AUTO = 0,     /* bf16 -> tensor core; f32 -> split-bf16 tensor core when m*n*k >= 2^28,
                           else SIMT exact; f64 -> SIMT */
  FM_GEMM_TENSOR = 1,   /* force tcgen05 path (bf16, f32 via 3-way bf16 split) */
  FM_GEMM_EXACT = 2     /* SIMT, f64 accumulation (reference cjit.py:33-51 numerics) */
};

/* ---- errors / device ---------------------------------------------------- */
const char *fm_last_error(void);
int fm_abi_version(void);
int fm_device_count(int *count);
int fm_set_device(int device);
int fm_get_device(int *device);
int fm_device_info(int device, int *sm_count, int *cc_major, int *cc_minor,
                   int64_t *l2_bytes, int64_t *hbm_bytes);
/* "0000:1b:00.0"-style id: identifies a GPU across processes whatever their
 * CUDA_VISIBLE_DEVICES numbering (transport choice of the sharded path) */
int fm_device_pci_bus_id(int device, char *buf, int len);

/* ---- memory (backend.py:192-239) ---------------------------------------- */
int fm_alloc(void **ptr, size_t bytes, void *stream);          /* zero-filled */
int fm_free(void *ptr, void *stream);
int fm_host_alloc(void **ptr, size_t bytes);                   /* pinned */
int fm_host_free(void *ptr);
int fm_memcpy_h2d(void *dst, const void *src, size_t bytes, void *stream);
int fm_memcpy_d2h(void *dst, const void *src, size_t bytes, void *stream);
int fm_memcpy_d2d(void *dst, const void *src, size_t bytes, void *stream);
int fm_memset(void *dst, int value, size_t bytes, void *stream);

/* ---- streams / events ----------------------------------------------------- */
int fm_stream_create(void **stream);
int fm_stream_destroy(void *stream);
int fm_stream_sync(void *stream);
int fm_event_create(void **event);
int fm_event_destroy(void *event);
int fm_event_record(void *event, void *stream);
int fm_event_elapsed_ms(void *start, void *stop, float *ms);   /* synchronises `stop` */

/* ---- kernels ---------------------------------------------------------------- */
/* Ahead-of-time template registry: qualified signature -> kernel id (>= 0),
 * or -1 when only the generic fused kernel (the register VM) can run it. */
int fm_kernel_lookup(const char *qualified_signature, int *kernel_id);
int fm_kernel_count(int *count);
int fm_kernel_signature(int kernel_id, const char **signature);

/* copy skeleton: out[r + c*n_rows] = EXPR(r, c) */
int fm_launch_copy(int kernel_id, const fm_program *prog, void *out,
                   int64_t n_rows, int64_t n_cols, void *stream);
/* reduce_accu skeleton: *out = finalize(sum EXPR) in f64 (floats) or wrapping int */
int fm_launch_accu(int kernel_id, const fm_program *prog, void *out,
                   int64_t n_rows, int64_t n_cols, int32_t finalize, void *stream);
/* dim reductions of EXPR; several outputs share one pass */
int fm_launch_reduce_dim(int kernel_id, const fm_program *prog, int32_t dim,
                         int64_t n_rows, int64_t n_cols,
                         const fm_reduce_out *outs, int32_t n_outs, void *stream);

int fm_gemm(const fm_gemm_args *args, void *stream);
/* GEMM whose operand A and/or B is an elementwise expression (a MatMul-free
 * fused program over the operand's stored shape, rows = lda) instead of a
 * buffer -- the operand prologue.  The reference materialises such operands
 * into temps first (plan.py:125-151); on the f32 tensor path the program is
 * evaluated straight into the GEMM's bf16 operand planes.  NULL programs
 * read args->a / args->b as fm_gemm does. */
int fm_gemm_prologue(const fm_gemm_args *args, const fm_program *a_prog, const fm_program *b_prog,
                     void *stream);
/* which kernel fm_gemm would run for these arguments, without launching:
 * FM_GEMM_PATH_EXACT (SIMT, f64 accumulation) or FM_GEMM_PATH_TCGEN05 */
enum { FM_GEMM_PATH_EXACT = 0, FM_GEMM_PATH_TCGEN05 = 1 };
int fm_gemm_plan(const fm_gemm_args *args, int *path);

/* splitmix64 counter stream (rng.py:35-72); element k of the stream is
 * written to out[k - offset] for k in [offset, offset + n). */
int fm_randu(void *out, int32_t etype, int64_t n, uint64_t seed, int64_t offset, void *stream);
int fm_randi(void *out, int32_t etype, int64_t n, uint32_t high, uint64_t seed,
             int64_t offset, void *stream);
int fm_fill(void *out, int32_t etype, int64_t n, uint64_t value_bits, void *stream);

/* plain device copy kernel, for the copy-bandwidth roofline probe */
int fm_copy(void *dst, const void *src, size_t bytes, void *stream);
/* write `bytes` of scratch to evict L2 between timed trials */
int fm_flush_l2(void *scratch, size_t bytes, void *stream);

/* CUDA graphs: capture the launches enqueued on `stream` between begin and
 * end into a replayable graph (per-step host work -> one graph launch) */
int fm_graph_begin(void *stream);
int fm_graph_end(void *stream, void **graph, int64_t *kernels);
int fm_graph_launch(void *graph, void *stream);
int fm_graph_destroy(void *graph);
/* Buffers allocated or freed while a thread captures (between fm_graph_begin
 * and fm_graph_end) are owned by the graph: plain allocations, released only
 * once every graph that captured them is destroyed and the owner freed them.
 * Returns how many such buffers are currently alive (tests). */
int64_t fm_graph_owned_count(void);

/* ---- collectives of the column-sharded path (csrc/comm.cu) -----------------
 * New API: the reference has no multi-device code.  A
 * communicator joins one rank per process (per GPU).  Every collective
 * gathers the ranks' contributions and combines them IN RANK ORDER, so all
 * ranks get bit-identical results whatever the transport:
 *   FM_COMM_PEER -- one kernel per collective over CUDA-IPC peer memory
 *                   (NVLink between GPUs; also works for ranks sharing a GPU)
 *   FM_COMM_NCCL -- ncclAllGather (libnccl dlopen'ed) + a combine kernel
 * All calls are stream-ordered and may be captured into CUDA graphs.       */
enum { FM_COMM_NCCL = 1, FM_COMM_PEER = 2 };
enum { FM_COMBINE_SUM = 0, FM_COMBINE_MAX = 1, FM_COMBINE_MIN = 2 };

int fm_comm_nccl_load(const char *path);            /* NULL: "libnccl.so.2" */
int fm_comm_nccl_version(int *version);
int fm_comm_nccl_unique_id(uint8_t *id128);         /* rank 0 makes it, the others receive it */
int fm_comm_init_nccl(void **comm, int nranks, int rank, const uint8_t *id128);
/* peer transport: each rank allocates its exchange block (header + 2 data
 * parities of `slot_bytes`) and shares the 64-byte IPC handle; then every
 * rank opens the others' blocks with all nranks handles (rank order) */
int fm_comm_peer_block(void **block, size_t slot_bytes, uint8_t *ipc_handle64);
int fm_comm_init_peer(void **comm, int nranks, int rank, void *block, const uint8_t *handles,
                      size_t slot_bytes);
int fm_comm_destroy(void *comm);
int fm_comm_info(void *comm, int *nranks, int *rank, int *transport);
int fm_comm_status(void *comm, int64_t *error);      /* peer: nonzero if a wait timed out (30 s) */
/* in place: buf = combine over ranks (rank order) of every rank's buf;
 * FM_F32 / FM_F64 / FM_U32 / FM_I32; SUM (ints wrap), MAX / MIN (NaN
 * propagates); divisor > 0 divides the combined value (mean of f64 sums) */
int fm_allreduce(void *comm, void *buf, int64_t count, int32_t etype, int32_t op, double divisor,
                 void *stream);
/* in place arg-select: per element the (value, index) pair of the extreme
 * over ranks -- first index wins ties, NaN wins (numpy argmax / argmin);
 * `idx_offset` is added to this rank's indices first (local -> global) */
int fm_allreduce_arg(void *comm, void *vals, uint32_t *idx, int64_t count, int32_t etype,
                     uint32_t idx_offset, int32_t maximize, void *stream);
/* dst[q * bytes .. (q+1) * bytes) = rank q's src, on every rank */
int fm_allgather(void *comm, const void *src, size_t bytes, void *dst, void *stream);

/* number of kernels this library launched since load (for bench gpu_launches) */
int64_t fm_launch_counter(void);

#ifdef __cplusplus
}
#endif
#endif /* FMB200_H */
