/*
 * dfx.h -- C ABI of the B200 data-flow fixpoint engine (libdfx.so).
 *
 * Drop-in boundary for the hot path of the OMPDart host/device data-flow
 * analysis (reference package `dartomp` 0.1.0, pure Python).  Each entry point
 * below replaces one reference interface; the Python shim in
 * `paper_2406_13881_b200/` (ctypes) keeps the reference signatures:
 *
 *   dfx_replay_batch   <- dartomp.dataflow.analyze_function
 *                         (pkg/src/dartomp/dataflow.py:737-740), batched over
 *                         functions (pipeline.plan_transform calls it once per
 *                         function, pipeline.py:85-96).
 *   dfx_summaries      <- dartomp.interproc.summarize_all
 *                         (pkg/src/dartomp/interproc.py:90-144).
 *   dfx_mfp_csr        <- the north-star CSR fixpoint (kernel a) plus the
 *                         per-edge transfer-requirement kernel (kernel b); the
 *                         gen/kill core of dataflow.py:299-378 with the AND meet
 *                         of dataflow.py:130-134 on an explicit CSR graph.
 *
 * Conventions: plain pointers and sizes, no torch types.  Host-pointer entry
 * points copy in and out themselves; `_dev` variants take device pointers
 * that the caller owns.  All calls return 0 on success and a negative status
 * otherwise; dfx_last_error() returns the message for the calling thread.
 * A handle is bound to one CUDA device and is not thread-safe.
 */
#ifndef DFX_H
#define DFX_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DFX_ABI_VERSION 1

#define DFX_OK 0
#define DFX_E_ARG (-1)
#define DFX_E_CUDA (-2)
#define DFX_E_NOSPC (-3)     /* output capacity too small; required size reported */
#define DFX_E_LIMIT (-4)     /* program exceeds an engine limit */

typedef struct dfx_handle dfx_handle;

int dfx_abi_version(void);
const char *dfx_last_error(void);
int dfx_open(int device, dfx_handle **out);
int dfx_close(dfx_handle *h);

/* ------------------------------------------------------------------------ */
/* E1: exact schedule replay of `_Analyzer` (dataflow.py:194-734)            */
/* ------------------------------------------------------------------------ */

/* opcodes: low 8 bits of op word 0; flags above (see lower.py).
 * Words 2-3 of BR_BEGIN / LOOP_BEGIN and word 3 of BR_END / LOOP_END are
 * reserved: the library fills them in its device copy of the program with
 * the region table (chunk mask, extent, dynamic length) that lets a warp
 * skip a region none of its variables is accessed in. */
enum {
  DFX_OP_END = 0, DFX_OP_HR = 1, DFX_OP_HW = 2, DFX_OP_DR = 3, DFX_OP_DW = 4,
  DFX_OP_BR_BEGIN = 5, DFX_OP_ARM_FORK = 6, DFX_OP_ARM_CLOSE = 7,
  DFX_OP_ARM_PASSIVE = 8, DFX_OP_BR_END = 9, DFX_OP_LOOP_BEGIN = 10,
  DFX_OP_LOOP_END = 11, DFX_OP_ERR = 12
};
#define DFX_F_AFTER_REGION (1 << 8)
#define DFX_F_OVR (1 << 9)
#define DFX_F_FP (1 << 10)
#define DFX_F_CAPTURE (1 << 11)
#define DFX_F_MAY_SKIP (1 << 12)

/* per-variable flags (low 16 bits) | name rank << 16 */
#define DFX_V_SCALAR 1
#define DFX_V_ALLOW_STALE 2
#define DFX_V_DECL_LATE 4
#define DFX_V_NONLOCAL 8

/* anchor codes in hoist tables */
#define DFX_AC_NODE_MASK ((1 << 20) - 1)
#define DFX_AC_ERR (1 << 20)
#define DFX_AC_QUAL (1 << 21)
#define DFX_AC_CLEAN (1 << 22)

/* arm anchor kinds */
enum { DFX_ARM_BEFORE = 0, DFX_ARM_AFTER = 1, DFX_ARM_ERR_ARM = 2, DFX_ARM_ERR_LOOP = 3 };

/* plan positions (dataflow.py:47-52) */
enum { DFX_POS_BEFORE = 0, DFX_POS_AFTER = 1, DFX_POS_BODY_END = 2, DFX_POS_KERNEL = 3 };

/* event kinds */
enum {
  DFX_EV_UPDATE_FROM = 1, DFX_EV_UPDATE_TO = 2, DFX_EV_FIRSTPRIVATE = 3,
  DFX_EV_SUPPRESS = 4,
  DFX_EV_ERR_DATAMAP = 16,     /* PreconditionError, dataflow.py:459-463 */
  DFX_EV_ERR_BRACES_LOOP = 17, /* PreconditionError, dataflow.py:291-294 */
  DFX_EV_ERR_BRACES_ARM = 18,  /* PreconditionError, dataflow.py:554-557 */
  DFX_EV_ERR_DECL = 19,        /* DeclPlacementError, dataflow.py:250-255 */
  DFX_EV_ERR_ENGINE = 20       /* engine resource limit hit (slots) */
};

/* per-variable output bits */
#define DFX_OUT_PRESENCE 1
#define DFX_OUT_TO 2
#define DFX_OUT_FROM 4
#define DFX_OUT_H 8
#define DFX_OUT_D 16

typedef struct {
  int32_t op_off, n_ops;       /* into ops (units of 4 int32) */
  int32_t var_off, n_vars;     /* into var_flags / var_out */
  int32_t stmt_off, n_stmts;   /* into stmt_span (units of 2 int32) */
  int32_t site_off, arm_off;   /* into sites (int32) / arms (units of 2) */
  int32_t region_begin_start;  /* -1: function has no kernels */
  int32_t n_slots, max_loop_depth, max_br_depth, max_arms;
  int32_t flags;               /* DFX_FN_* (0: none) */
  int32_t reserved[2];
} dfx_fn_desc;

/* dfx_fn_desc.flags.  DFX_FN_NO_ERR_SITES: no hoist-table entry and no arm
 * anchor of the function can raise a braces error (the lowering knows this
 * statically).  It lets the replay drop, per variable, the dry round of a
 * loop that never writes the variable (exact: see replay.cu "dry-round lane
 * skip"); without it every dry round is replayed in full. */
#define DFX_FN_NO_ERR_SITES 1

typedef struct {
  int32_t n_funcs;
  const dfx_fn_desc *fns;
  const int32_t *ops;
  const int32_t *var_flags;
  const int32_t *stmt_span;
  const int32_t *sites;
  const int32_t *arms;
  int64_t n_ops, n_vars, n_stmts, n_sites, n_arms; /* array lengths, in units */
} dfx_replay_in;

typedef struct {
  uint64_t key;     /* visit order: seq << 24 | name_rank << 8 | arm */
  int32_t fn;
  int32_t var;      /* function-local variable index */
  int32_t node;     /* function-local statement id (anchor / error site) */
  uint8_t kind;
  uint8_t pos;
  uint16_t pad;
} dfx_event;

typedef struct {
  dfx_event *events;   /* capacity event_cap */
  int64_t event_cap;
  int64_t n_events;    /* out: events produced (may exceed cap -> DFX_E_NOSPC) */
  uint8_t *var_out;    /* [n_vars] DFX_OUT_* bits */
  float kernel_ms;     /* out: device time of the replay kernel */
} dfx_replay_out;

/* Host buffers in, host buffers out (H2D + kernel + D2H). */
int dfx_replay_batch(dfx_handle *h, const dfx_replay_in *in, dfx_replay_out *out);

/* dfx_replay_batch with the ops packed into 8 bytes each (half the host->
 * device bytes of the ops): in->ops points at n_ops pairs of uint32
 *   word 0: opcode (bits 0-3) | flags >> 8 (bits 4-8) | c (bits 9-31)
 *   word 1: a (bits 0-15) | b (bits 16-31)
 * where, by opcode, the op words 1-3 of the 16-byte form are
 *   HR, DR: (a, b, c)   HW, DW: (a, b, 0)   BR_END: (c, b, 0)
 *   LOOP_BEGIN: (a, 0, 0)   LOOP_END: (c, 0, 0)   ERR: (a, b, 0)   others: 0.
 * The device unpacks each function range as it lands, before its region
 * table; a batch whose fields do not fit (variables or statements beyond
 * 65535, offsets beyond 2^23) must use dfx_replay_batch. */
int dfx_replay_batch_packed(dfx_handle *h, const dfx_replay_in *in, dfx_replay_out *out);

/* Device-resident batch (configuration C4 timing): upload once, replay many
 * times; dfx_replay_run leaves events/bits on the device and reports counts. */
typedef struct dfx_replay dfx_replay;
int dfx_replay_create(dfx_handle *h, const dfx_replay_in *in, int64_t event_cap, dfx_replay **out);
int dfx_replay_run(dfx_handle *h, dfx_replay *r, int64_t *n_events, float *kernel_ms);
int dfx_replay_fetch(dfx_handle *h, dfx_replay *r, dfx_replay_out *out);
int dfx_replay_destroy(dfx_handle *h, dfx_replay *r);

/* Configuration C4 generator: synthetic structured functions emitted
 * directly as replay programs (csrc/c4gen.cpp).  dfx_gen_c4 takes the
 * function ids to generate; call it with NULL arrays first to get the sizes
 * (ops, vars, stmts, sites, arms). */
int dfx_gen_c4_shapes(uint64_t seed, int32_t n, int32_t n_min, int32_t n_max,
                      const int32_t *var_choices, int32_t n_choices, int32_t *N, int32_t *V);
int dfx_gen_c4(uint64_t seed, const int32_t *fids, int32_t n, int32_t n_min, int32_t n_max,
               const int32_t *var_choices, int32_t n_choices, dfx_fn_desc *fns, int32_t *ops,
               int32_t *var_flags, int32_t *stmt_span, int32_t *sites, int32_t *arms,
               int64_t *sizes, int64_t *facts_out);
/* Dynamic op visits per function (loops: dry + planning round; branches
 * once): the final value of E1's visit counter, for roofline accounting. */
int dfx_program_visits(const dfx_fn_desc *fns, int32_t n_funcs, const int32_t *ops,
                       int64_t *visits);

/* ------------------------------------------------------------------------ */
/* Kernels (a)+(b): CSR fixpoint and transfer requirements (north star)      */
/* ------------------------------------------------------------------------ */
/* The gen/kill core of dataflow.py:299-378 with the AND meet of
 * dataflow.py:130-134 on an explicit predecessor CSR.  Bitplanes are
 * node-major: plane[node * words + w], bit b of word w = variable 32*w + b.
 *   host node  : H' = H | A        D' = D & ~B            (A = R|W, B = W)
 *   kernel node: H' = H & ~B       D' = D | (A & ~(F & H_in)), F = A & ~B & S
 * IN = AND over predecessors; nodes without predecessors take (H=1, D=0). */
typedef struct dfx_csr dfx_csr;            /* device-resident problem */

typedef struct {
  int64_t n_nodes;
  int32_t words;                /* V/32: multiple of 4, at most 512 */
  int64_t nnz;
  const int32_t *row_ptr;       /* [n_nodes+1] */
  const int32_t *col;           /* [nnz] predecessor ids */
  const uint8_t *node_kind;     /* [n_nodes] 0 host, 1 kernel */
  const uint32_t *R;            /* [n_nodes*words] reads */
  const uint32_t *W;            /* [n_nodes*words] writes */
  const uint32_t *S;            /* [words] scalar-variable mask */
} dfx_csr_in;

typedef struct {                /* configuration C3 generator */
  uint64_t seed;
  int64_t n_nodes;
  int32_t words;                /* word columns generated ... */
  int32_t w0;                   /* ... starting at global word w0 */
  int32_t n_scalar;             /* variables [0, n_scalar) are scalars */
} dfx_c3_spec;

/* Kernel (b) output: order-preserving compaction of the requirement planes
 * into sparse word-rows.  For node n, occ[n*occ_words .. +occ_words) holds
 * two bitmaps of ceil(words/32) uint32 each: which requirement words and
 * which firstprivate words are nonzero.  masks[row_off[n] .. row_off[n+1])
 * lists the nonzero 32-variable masks: requirement words ascending, then
 * firstprivate words ascending.  Requirement kind is implied by the node:
 * host node -> update-from (host read of a stale host copy), kernel node ->
 * update-to (device read of a stale device copy); firstprivate words mark
 * scalars captured by value. */
typedef struct {
  int64_t *row_off;             /* [n_nodes+1] (NULL: not copied) */
  uint32_t *occ;                /* [n_nodes*occ_words] (NULL: not copied) */
  uint32_t *masks;              /* [cap] (NULL: count only) */
  int64_t cap;
  int64_t n_masks;              /* out */
  int32_t occ_words;            /* out: 2*ceil(words/32) */
} dfx_req_out;

typedef struct {
  int32_t rounds_h, rounds_d;   /* relaxation rounds per phase (incl. the last, unchanged one) */
  int64_t evaluated;            /* node-row evaluations (both phases) */
  int64_t rows_read, rows_written; /* 512-B-per-4096-var row transfers counted by the kernel */
  float solve_ms;               /* device time of kernel (a), all rounds, incl. the
                                   host round-trip that checks convergence */
  float kernel_ms;              /* sum of the round-kernel durations alone */
  float req_ms;                 /* device time of kernel (b) incl. compaction */
  int64_t n_masks;              /* kernel (b): nonzero 32-variable masks */
} dfx_csr_stats;

int dfx_set_stream(dfx_handle *h, void *cuda_stream);   /* NULL: the handle's own */
int dfx_csr_create(dfx_handle *h, const dfx_csr_in *in, dfx_csr **out);   /* H2D */
int dfx_csr_generate_c3(dfx_handle *h, const dfx_c3_spec *spec, dfx_csr **out);
int dfx_csr_destroy(dfx_handle *h, dfx_csr *p);
/* kernel (a); chunk_nodes <= 0 picks the default */
int dfx_csr_solve(dfx_handle *h, dfx_csr *p, int32_t chunk_nodes, dfx_csr_stats *stats);
/* kernel (a) enqueued on the handle's stream without host synchronisation
 * (convergence is decided on the device); back-to-back solves of a resident
 * problem pipeline on the GPU */
int dfx_csr_solve_async(dfx_handle *h, dfx_csr *p, int32_t chunk_nodes);
/* kernel (b): requirement planes + order-preserving compaction (D2H of the
 * parts of `out` that are non-NULL) */
int dfx_csr_requirements(dfx_handle *h, dfx_csr *p, dfx_req_out *out, dfx_csr_stats *stats);
/* D2H of the fixpoint OUT planes and the dense requirement plane (any NULL
 * pointer is skipped) */
int dfx_csr_download(dfx_handle *h, dfx_csr *p, uint32_t *out_h, uint32_t *out_d, uint32_t *req);
/* D2H of the problem's inputs (row_ptr [n+1], col [nnz], node_kind [n],
 * R, W [n*words]); any NULL pointer is skipped */
int dfx_csr_export(dfx_handle *h, dfx_csr *p, int32_t *row_ptr, int32_t *col, uint8_t *node_kind,
                   uint32_t *R, uint32_t *W);
int64_t dfx_csr_nnz(dfx_csr *p);
/* all-in-one host-buffer call: H2D, kernel (a), kernel (b), D2H of `out` */
int dfx_mfp_csr(dfx_handle *h, const dfx_csr_in *in, dfx_req_out *out, dfx_csr_stats *stats);

/* List forms of the same problem (csrc/acc.cu).  The reference describes each
 * statement by its list of memory accesses (access.py:58-86 `MemoryAccess`,
 * kind READ/WRITE/READWRITE) and answers with per-statement directive plans
 * naming variables (dataflow.py:37-95).  Entries are uint16:
 *   access      : var | kind << 14, kind 1 = read, 2 = write, 3 = read+write
 *   requirement : var, | DFX_REQ_FIRSTPRIVATE for a firstprivate capture
 * so the boundary moves accesses and planned transfers, not nodes x vars.
 * V = 32 * words <= 16384. */
#define DFX_ACC_READ 1
#define DFX_ACC_WRITE 2
#define DFX_REQ_FIRSTPRIVATE 0x8000

typedef struct {
  int64_t n_nodes;
  int32_t words;                /* V/32: multiple of 4, at most 512 */
  int64_t nnz;
  int64_t n_acc;
  const int32_t *row_ptr;       /* [n_nodes+1] */
  const int32_t *col;           /* [nnz] predecessor ids */
  const uint8_t *node_kind;     /* [n_nodes] 0 host, 1 kernel */
  const int64_t *acc_off;       /* [n_nodes+1] node n's accesses: acc[acc_off[n] .. acc_off[n+1]) */
  const uint16_t *acc;          /* [n_acc] any order; duplicates OR together */
  const uint32_t *S;            /* [words] scalar-variable mask */
} dfx_acc_in;

/* Kernel (b) as per-node variable lists: node n's entries are
 * vars[row_off[n] .. row_off[n+1]): transfer requirements ascending (update
 * from at host nodes, update to at kernel nodes), then firstprivate captures
 * ascending (DFX_REQ_FIRSTPRIVATE set). */
typedef struct {
  int64_t *row_off;             /* [n_nodes+1] (NULL: not copied) */
  uint16_t *vars;               /* [cap] (NULL: count only) */
  int64_t cap;
  int64_t n_out;                /* out: total entries */
} dfx_req_list;

int dfx_csr_create_acc(dfx_handle *h, const dfx_acc_in *in, dfx_csr **out);   /* H2D + expand */
int dfx_csr_requirements_list(dfx_handle *h, dfx_csr *p, dfx_req_list *out, dfx_csr_stats *stats);
/* D2H of the problem's accesses as lists; acc == NULL: only *n_acc and acc_off */
int dfx_csr_export_acc(dfx_handle *h, dfx_csr *p, int64_t *acc_off, uint16_t *acc, int64_t cap,
                       int64_t *n_acc);
/* all-in-one host-buffer call on lists: H2D, expand, kernel (a), kernel (b),
 * D2H of the requirement lists */
int dfx_mfp_acc(dfx_handle *h, const dfx_acc_in *in, dfx_req_list *out, dfx_csr_stats *stats);

/* Byte-coded lists (B8): the same entries in about 1.2 bytes each instead of
 * 2, for the host<->device link that bounds the host-buffer call.  Per node,
 * entries ascend by variable; an entry is one or more bytes
 *   b = kind << 6 | d:  d == 63 adds 63 and continues, d < 63 ends the entry,
 * and its variable is prev + 1 + (the sum of its d fields), with prev = -1 at
 * the start of the node (and, in the output, again where the firstprivate
 * entries begin).  Input kind: DFX_ACC_READ / DFX_ACC_WRITE / both.  Output
 * kind: DFX_B8_REQ for a transfer requirement, DFX_B8_FP for a firstprivate
 * capture (after the node's requirements).  Offsets are int32 (a list of at
 * most 2^31 - 1 bytes). */
#define DFX_B8_REQ 1
#define DFX_B8_FP 2

typedef struct {
  int64_t n_nodes;
  int32_t words;                /* V/32: multiple of 4, at most 512 */
  int64_t nnz;
  int64_t n_bytes;
  const int32_t *row_ptr;       /* [n_nodes+1] */
  const int32_t *col;           /* [nnz] predecessor ids */
  const uint8_t *node_kind;     /* [n_nodes] 0 host, 1 kernel */
  const int32_t *byte_off;      /* [n_nodes+1] node n's entries: bytes[byte_off[n] .. byte_off[n+1]) */
  const uint8_t *bytes;         /* [n_bytes] */
  const uint32_t *S;            /* [words] scalar-variable mask */
} dfx_acc8_in;

typedef struct {
  int32_t *row_off;             /* [n_nodes+1] */
  uint8_t *bytes;               /* [cap] */
  int64_t cap;
  int64_t n_out;                /* out: total bytes (> cap -> DFX_E_NOSPC) */
} dfx_req8_list;

/* all-in-one host-buffer call on byte-coded lists (same kernels as dfx_mfp_acc) */
int dfx_mfp_acc8(dfx_handle *h, const dfx_acc8_in *in, dfx_req8_list *out, dfx_csr_stats *stats);

/* ------------------------------------------------------------------------ */
/* Kernel (c): interprocedural summaries (interproc.py:90-156)              */
/* ------------------------------------------------------------------------ */
/* One byte per (function, slot): bit0 R, bit1 W, bit2 HOST, bit3 DEVICE.
 * Slots: [0, n_params) pointer parameters, [n_params, n_slots) globals.
 * The engine replays the reference's Gauss-Seidel passes exactly (dict
 * order, interproc.py:105-143): each pass rebuilds every function from its
 * sources in order -- a static slot list (its own accesses, calls to
 * external or undefined functions) or a call to a defined function (callee
 * parameter i bound to a caller slot, callee globals copied, spaces forced
 * to DEVICE for calls inside kernels) -- and tracks each summary's insertion
 * order (the order of the reference's dicts).  Sources: int32 x4 rows
 * (kind | dev << 8, a, b, c): STATIC: a = offset into slist, b = length;
 * CALL: a = callee, b = offset into bind, c = number of bindings.
 * Functions of one wave read no same-pass result of another, so a wave runs
 * in parallel; waves run in order; passes repeat until no set changes. */
typedef struct {
  int32_t n_funcs, n_slots, n_params, n_waves, max_passes;
  const uint8_t *init_bits;    /* [n_funcs * n_slots] pass-0 summaries */
  const int16_t *init_list;    /* [n_funcs * n_slots] pass-0 insertion order */
  const int32_t *init_len;     /* [n_funcs] */
  const uint8_t *direct;       /* [n_funcs * n_slots] static-source bits */
  const int32_t *src_off;      /* [n_funcs+1] */
  const int32_t *src;          /* [n_src*4] */
  const int16_t *slist;        /* [n_slist] */
  const int32_t *bind;         /* [n_bind*2] (callee param, caller slot) */
  const int32_t *wave_off;     /* [n_waves+1] */
  const int32_t *wave_fns;     /* [n_funcs] */
  int64_t n_src, n_slist, n_bind;
} dfx_cg_in;

typedef struct {
  uint8_t *bits;               /* [n_funcs * n_slots] final summaries (host) */
  int16_t *list;               /* [n_funcs * n_slots] insertion order (host) */
  int32_t *len;                /* [n_funcs] */
  int32_t passes;              /* passes run, as the reference counts them */
  int32_t launches;            /* wave kernel launches */
  float kernel_ms;
} dfx_cg_out;

/* replaces dartomp.interproc.summarize_all: host buffers in and out */
int dfx_summaries(dfx_handle *h, const dfx_cg_in *in, dfx_cg_out *out);

/* NCCL on the handle (SURVEY §8 b): one communicator per handle, for the
 * multi-GPU summaries solve.  dfx_comm_unique_id fills DFX_COMM_ID_BYTES
 * bytes on one rank; every rank passes them to dfx_comm_init (e.g. after a
 * broadcast).  NCCL is loaded at run time (libnccl.so.2). */
#define DFX_COMM_ID_BYTES 128
int dfx_comm_unique_id(void *id_out);
int dfx_comm_init(dfx_handle *h, const void *unique_id, int32_t nranks, int32_t rank);
int dfx_comm_destroy(dfx_handle *h);

/* summarize_all across the communicator's ranks, sharded by call-graph
 * component (replaces interproc.py:90-144 like dfx_summaries): owner[f] is
 * the rank that rebuilds function f, and a function and its callees must
 * share an owner.  Per pass: one cooperative launch over the rank's own
 * waves, then ONE ncclAllReduce(MAX) of the pass's changed flag (the
 * reference's global termination test); after the last pass ONE
 * ncclAllGather of the owned rows.  Every rank receives every summary;
 * *n_collectives = passes + 1 (+0 at one rank). */
int dfx_summaries_sharded(dfx_handle *h, const dfx_cg_in *in, const int32_t *owner,
                          dfx_cg_out *out, int32_t *n_collectives);

/* Sharded building blocks (multi-GPU: one process per GPU; the caller
 * all-gathers the rows each shard computed after every wave).  Tables are
 * caller-owned DEVICE memory: bits [n_funcs * nsp] uint8, list
 * [n_funcs * nsp] int16, len [n_funcs] int32, nsp = dfx_cg_nsp(). */
typedef struct dfx_cg dfx_cg;
typedef struct { uint8_t *bits; int16_t *list; int32_t *len; } dfx_cg_tables;
int dfx_cg_create(dfx_handle *h, const dfx_cg_in *in, dfx_cg **out);
int dfx_cg_destroy(dfx_handle *h, dfx_cg *cg);
int32_t dfx_cg_nsp(dfx_cg *cg);
/* rebuild the functions of `wave` at positions p (p % nshards == shard) into
 * `cur`, reading callees from `cur` (earlier in dict order) or `prev`;
 * *changed = 1 if any rebuilt bit set differs from `prev` */
int dfx_cg_wave(dfx_handle *h, dfx_cg *cg, const dfx_cg_tables *prev, dfx_cg_tables *cur,
                int32_t wave, int32_t shard, int32_t nshards, int32_t *changed);

/* Fused multi-GPU kernel (c) over peer memory (NVLink P2P via CUDA IPC).
 * One process per GPU, one dfx_cgp per process.  A wave's functions are
 * split round-robin over the ranks; the kernel that rebuilds a function's
 * summary row also stores it into every peer's tables, and a wave ends when
 * every rank has released its arrival on every peer (system-scope atomics).
 * This replaces the NCCL path's all-gather after each wave.  Protocol:
 *   dfx_cgp_create on every rank  ->  exchange the DFX_IPC_HANDLE_BYTES
 *   handles (e.g. an all-gather of bytes)  ->  dfx_cgp_connect(handles of
 *   ranks 0..nranks-1)  ->  dfx_cgp_solve on every rank (same number of
 *   solves on every rank; no rank may start solve k+1 before every rank
 *   returned from solve k).  out receives the same summaries on every rank.
 * A peer that never arrives makes dfx_cgp_solve fail with DFX_E_CUDA after
 * a bounded wait instead of hanging. */
#define DFX_IPC_HANDLE_BYTES 64
typedef struct dfx_cgp dfx_cgp;
int dfx_cgp_create(dfx_handle *h, const dfx_cg_in *in, int32_t nranks, int32_t rank, dfx_cgp **out);
int dfx_cgp_handle(dfx_cgp *p, void *ipc_handle);
int dfx_cgp_connect(dfx_handle *h, dfx_cgp *p, const void *ipc_handles);
int dfx_cgp_solve(dfx_handle *h, dfx_cgp *p, dfx_cg_out *out);
int dfx_cgp_destroy(dfx_handle *h, dfx_cgp *p);

/* ------------------------------------------------------------------------ */
/* Transfer simulator: batched replacement of                 */
/* dartomp.simulator.simulate (simulator.py:180-708)                         */
/* ------------------------------------------------------------------------ */
/* A program is the simulator's walk of one translation unit with its
 * control (concrete scalar values, if decisions, trip counts, returns, call
 * inlining and aliases) resolved by the host lowering
 * (paper_2406_13881_b200/simlower.py), leaving the per-variable state
 * machine (ref count, host-valid, device-valid) to the device: one warp per
 * (program, 32-variable chunk), one lane per resolved variable.  Ops are
 * int32 x4 (code | flags << 8, var, a, b) plus one int64 argument each
 * (bytes per transfer, loop trip count):
 *   READ var space site | WRITE var space | ENTER var maptype [bytes] |
 *   EXIT var maptype warn [bytes] | UPDATE var dir warn [bytes] |
 *   SHIELD_SAVE / SHIELD_SET / UNSHIELD var |
 *   CHECK_BEGIN extent chunkmask | CHECK_END (untaken if-arm: its stale
 *   reads count, its state and transfers roll back) |
 *   LOOP extent chunkmask nvariants [trip] { VAR_BEGIN extent (F_RET)
 *   ... VAR_END back } x nvariants (round r runs variant min(r, n)) | END
 * Loops iterate per variable until that variable's state repeats under the
 * steady variant; the rest of the trip count is then accounted by one more
 * round counted trip - r times (simulator.py:528-550, `_scale_tail`). */
enum {
  DFX_SIM_END = 0, DFX_SIM_READ = 1, DFX_SIM_WRITE = 2, DFX_SIM_ENTER = 3,
  DFX_SIM_EXIT = 4, DFX_SIM_UPDATE = 5, DFX_SIM_SHIELD_SAVE = 6, DFX_SIM_SHIELD_SET = 7,
  DFX_SIM_UNSHIELD = 8, DFX_SIM_CHECK_BEGIN = 9, DFX_SIM_CHECK_END = 10, DFX_SIM_LOOP = 11,
  DFX_SIM_VAR_BEGIN = 12, DFX_SIM_VAR_END = 13,
  DFX_SIM_WARN = 14             /* control warning (call depth, unknown clause
                                   variable): host-side text, no device effect */
};
#define DFX_SIM_F_RET (1 << 8)
#define DFX_SIM_MAX_NEST 16          /* loops + untaken arms nested */
#define DFX_SIM_MAX_ROUNDS 10000     /* simulator.py _MAX_CONCRETE_ROUNDS */

typedef struct {
  int32_t op_off, n_ops;        /* into ops (units of 4 int32) and arg64 */
  int32_t var_off, n_vars;      /* into the per-variable outputs */
} dfx_sim_prog;

typedef struct {
  int32_t n_progs;
  const dfx_sim_prog *progs;
  const int32_t *ops;           /* [n_ops * 4] */
  const int64_t *arg64;         /* [n_ops] */
  int64_t n_ops, n_vars;
} dfx_sim_in;

/* per-variable result: transfer totals, stale reads, final state */
typedef struct {
  uint64_t htod_calls, htod_bytes, dtoh_calls, dtoh_bytes, stale;
  int64_t ref;
  uint8_t host_valid, device_valid, flags, pad[5];
} dfx_sim_var;
#define DFX_SIM_VF_OVERFLOW 1        /* a count exceeded 64 bits */
#define DFX_SIM_VF_FAULT 2           /* shield stack / malformed program */

/* records: stale reads (id = site, count), warnings (id = warn id) */
enum { DFX_SIM_REC_STALE = 0, DFX_SIM_REC_WARN = 1, DFX_SIM_REC_NOSETTLE = 2 };
typedef struct {
  int32_t prog, var, id, kind;
  uint64_t count;
} dfx_sim_rec;

typedef struct {
  dfx_sim_var *vars;            /* [n_vars] */
  dfx_sim_rec *recs;            /* capacity rec_cap */
  int64_t rec_cap;
  int64_t n_recs;               /* out (may exceed rec_cap -> DFX_E_NOSPC) */
  float kernel_ms;
} dfx_sim_out;

/* host buffers in and out */
int dfx_sim_batch(dfx_handle *h, const dfx_sim_in *in, dfx_sim_out *out);

/* ------------------------------------------------------------------------ */
/* Batched emission: rewriter.apply_plans (rewriter.py:255)  */
/* and report.plan_lines (report.py:13) for many translation units          */
/* ------------------------------------------------------------------------ */
/* Host code, no device.  Text is UTF-32 (code point offsets = the
 * reference's string indices).  Plans: int32 x6 (function, class 0 update /
 * 1 kernel clause, kind, position DFX_POS_*, kernel group, 0) and int64 x3
 * (anchor start, anchor end, loop-body closing brace or -1).  Update kinds
 * DFX_EMIT_TO / DFX_EMIT_FROM; kernel-clause kinds 0 map(to) 1 map(tofrom)
 * 2 map(from) 3 map(alloc) 4 firstprivate.  Strings (names, clause texts,
 * function names) are ids into one string pool. */
#define DFX_EMIT_TO 0
#define DFX_EMIT_FROM 1
#define DFX_EMIT_REPORT 1        /* flags: also produce the report lines */
#define DFX_EMIT_AFTER_LINES 2   /* flags: report AFTER updates ("after line N")
                                    instead of failing like report.py:35 */
enum { DFX_EMIT_ERR_BRACES = 1, DFX_EMIT_ERR_CLASH = 2, DFX_EMIT_ERR_POSITION = 3 };

typedef struct {
  int32_t n_units;
  const uint32_t *text; const int64_t *text_off;          /* [n_units+1] */
  const int32_t *unit_len;                                 /* indent unit length, -1: detect */
  const uint32_t *unit_text; const int64_t *unit_off;
  int32_t n_fns;
  const int32_t *fn_unit;                                  /* [n_fns] */
  const int64_t *fn_region;                                /* [n_fns*2] begin start, end end; -1 */
  const int32_t *fn_clause;                                /* [n_fns] region clause text (string id) */
  const int32_t *fn_name;                                  /* [n_fns] function name (string id) */
  const int64_t *fn_supp_off; const int32_t *supp_idx;     /* suppressed names */
  int32_t n_plans;
  const int32_t *plan;                                     /* [n_plans*6] */
  const int64_t *plan_pos;                                 /* [n_plans*3] */
  const int64_t *plan_names_off; const int32_t *name_idx;  /* names (string ids) */
  const int64_t *str_off; const uint32_t *strpool;         /* string pool */
  int32_t flags;
} dfx_emit_in;

typedef struct {
  uint32_t *text; int64_t text_cap; int64_t *text_off;     /* rewritten texts [n_units+1] */
  int64_t *ins; int64_t ins_cap; int64_t *ins_off;         /* placed (start, length) pairs */
  uint32_t *report; int64_t report_cap; int64_t *report_off;   /* report lines, '\n'-ended */
  int32_t *err_kind; int64_t *err_offset;                  /* [n_units] rewriter errors */
  int32_t *report_err;                                     /* [n_units] 1: AFTER update (KeyError) */
  int64_t text_need, ins_need, report_need;                /* out: sizes (DFX_E_NOSPC) */
} dfx_emit_out;

int dfx_emit_batch(const dfx_emit_in *in, dfx_emit_out *out);

#ifdef __cplusplus
}
#endif
#endif /* DFX_H */
