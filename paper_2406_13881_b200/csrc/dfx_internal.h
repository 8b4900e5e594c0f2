// dfx_internal.h -- shared declarations between the C-ABI layer and kernels.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/dfx.h"

namespace dfx {

struct ReplayDev {
  const dfx_fn_desc* fns;
  const int32_t* ops;
  const int32_t* var_flags;
  const int32_t* stmt_span;
  const int32_t* sites;
  const int32_t* arms;
  const int32_t* item_fn;
  const int32_t* item_chunk;
  int n_items;
  int fn_lo, fn_hi;   // functions of this launch (region_kernel)
  int max_slots;
  dfx_event* events;
  int64_t event_cap;
  unsigned long long* event_count;
  uint8_t* var_out;
  unsigned* next;     // work-queue counter of this launch (cleared by replay_launch)
  // functions beyond the narrow replay's limits (api.cu fn_class): their
  // items run in a second, wide launch (replay.cu Wide traits)
  const int32_t* wide_item_fn = nullptr;
  const int32_t* wide_item_chunk = nullptr;
  int n_wide_items = 0;
  int wide_max_slots = 0;
  unsigned* wide_next = nullptr;
};

// Range gating of the host-buffer pipeline (replay.cu replay_kernel)
struct GateDev {
  int K;
  const int* fn_cut;                 // [K+1] function bounds of the ranges
  const int* ready;                  // [K]
  const long long* ev_off;           // [K] region offsets into events
  const long long* ev_cap;           // [K]
  const unsigned* range_items;       // [K] items per range
  unsigned* items_done;              // [K]
  unsigned long long* host_done;     // [K] mapped host memory: count + 1 when done
  unsigned* timed_out;
  unsigned long long timeout_ns;     // a range not ready by then fails the wait ($DFX_GATE_TIMEOUT_MS)
};

// region tables of functions [fn_lo, fn_hi) (replay.cu region_kernel)
int region_launch(const ReplayDev& r, int fn_lo, int fn_hi, cudaStream_t stream);
// packed ops (dfx_replay_batch_packed): device unpack of [lo, hi), host unpack of n
int unpack_ops_launch(const uint32_t* packed, int32_t* ops, int64_t lo, int64_t hi, cudaStream_t st);
void unpack_ops_host(const uint32_t* packed, int32_t* ops, int64_t n);
// replay (persistent grid); with `gate`, items wait for their range's ready
// flag and the region tables are the caller's (region_launch per range)
// (without a gate, the wide items follow in a second launch on the stream)
int replay_launch(const ReplayDev& r, cudaStream_t stream, const GateDev* gate = nullptr);
// the wide items only (no region pass): after a gated launch
int replay_launch_wide(const ReplayDev& r, cudaStream_t stream);
// gated only: a second launch into the block slots the gated launch leaves to
// the region kernels, on a stream where every range is already open; it
// shares the item queue (`next` is not reset)
int replay_launch_backfill(const ReplayDev& r, cudaStream_t stream, const GateDev* gate);

// replay class of a function: 0 narrow, 1 wide, 2 beyond the wide limits
int fn_class(const dfx_fn_desc& d);

}  // namespace dfx

namespace dfx {

struct CsrDev {
  int64_t n_nodes;
  int32_t words;
  int64_t nnz;
  int32_t* row_ptr;
  int32_t* col;
  uint8_t* kind;
  uint32_t* A;      // R | W
  uint32_t* B;      // W
  uint32_t* USE;    // R
  uint32_t* S;      // [words]
  uint32_t* OH;
  uint32_t* OD;
  uint32_t* REQ;
  uint32_t* FPQ;    // [n_nodes][n_fp_slots] uint4
  int32_t* fp_slot; // [words/4] quad -> slot or -1
  int32_t n_fp_slots;
  int32_t* stamp;
  int32_t* popc;    // per-node population count of the current OUT row
  int32_t s_quads_low;  // every nonzero scalar quad has index < 8
  int32_t* desc;        // [n_nodes][8] node descriptors (rs, deg|kind<<30, p0..p3)
  int32_t* seen;        // [nnz] per-edge seen round, edges >= 4 of a node (kernel a frontier)
  int32_t* succ_ptr;    // [n_nodes+1] successor (reverse) CSR: candidate flags of kernel (a)
  int32_t* succ;        // [nnz]
  int32_t* seen4;       // [n_nodes][4] seen rounds of a node's first 4 edges
  int32_t* chunk_done;  // [n_nodes] per-chunk round completed (kernel a frontier)
};

struct SolveStats {
  int rounds[2];
  int64_t evaluated, rows_read, rows_written;
  float kernel_ms;
};


int c3_generate(CsrDev& p, uint64_t seed, int w0, cudaStream_t st, void* scratch, size_t scratch_bytes);
int or_planes(const CsrDev& p, cudaStream_t st);
// CSR validation (acc.cu): bit 2 of *bad on a malformed row_ptr / col
int check_csr(const CsrDev& p, int* bad, cudaStream_t st);
int build_desc(const CsrDev& p, cudaStream_t st);
int build_succ(const CsrDev& p, void* scratch, size_t scratch_bytes, int32_t* tmp, cudaStream_t st);
int vpl_for(int words);
int mfp_solve(const CsrDev& p, void* ctl_mem, uint8_t* flags, cudaStream_t st, int chunk_nodes,
              SolveStats* stats, bool collect = true);
int requirements(const CsrDev& p, int32_t* counts, int64_t* offsets, void* scratch,
                 size_t scratch_bytes, uint32_t* occ, uint32_t* masks, int64_t cap,
                 int64_t* n_out, cudaStream_t st);
int requirements_scan(const CsrDev& p, int32_t* counts, int64_t* offsets, void* scratch,
                      size_t scratch_bytes, int count_bits, int64_t* n_out, cudaStream_t st);
int scan_counts(int64_t n, const int32_t* counts, int64_t* offsets, void* scratch,
                size_t scratch_bytes, int64_t* n_out, cudaStream_t st);
// access lists (acc.cu)
int expand_acc(const CsrDev& p, const int64_t* off, const uint16_t* acc, int* bad, int64_t n_lo,
               int64_t n_hi, cudaStream_t st);
int count_acc(const CsrDev& p, int32_t* counts, cudaStream_t st);
int expand_b8(const CsrDev& p, const int32_t* off, const uint8_t* bytes, int* bad, int64_t n_lo,
              int64_t n_hi, cudaStream_t st);
int count_b8(const CsrDev& p, int32_t* counts, int64_t n_lo, int64_t n_hi, cudaStream_t st);
int compact_b8(const CsrDev& p, const int64_t* offsets, uint8_t* out, int64_t cap, int64_t n_lo,
               int64_t n_hi, cudaStream_t st);
int export_acc(const CsrDev& p, const int64_t* off, uint16_t* acc, cudaStream_t st);
int compact_list(const CsrDev& p, const int64_t* offsets, uint16_t* vars, int64_t cap,
                 int64_t n_lo, int64_t n_hi, cudaStream_t st);
int requirements_range(const CsrDev& p, int32_t* counts, int64_t* offsets, void* scratch,
                       size_t scratch_bytes, int n_lo, int n_hi, cudaStream_t st, bool b8 = false);
size_t scan_scratch_bytes(int64_t n);
size_t round_ctl_bytes();

}  // namespace dfx

namespace dfx {

struct CgDev {
  int32_t n_funcs, n_slots, nsp, n_params, n_waves;
  int32_t many;              // some function has more than kCgManySources sources (summ.cu)
  const uint8_t* direct;     // [n_funcs * nsp]
  const int32_t* src_off;
  const int32_t* src;        // int32 x4 rows
  const int16_t* slist;
  const int32_t* bind;
  const int32_t* wave_fns;
  const int32_t* h_wave_off; // host copy
};

// whether a call graph needs kernel (c)'s many-sources path (and its shared memory)
bool cg_many_sources(const int32_t* src_off_host, int n_funcs);
int cg_wave(const CgDev& g, uint8_t* pbits, int16_t* plist, int32_t* plen, uint8_t* cbits,
            int16_t* clist, int32_t* clen, int wave, int shard, int nshards, int* d_changed,
            cudaStream_t st);
int repitch(const void* src, size_t sp, void* dst, size_t dp, size_t width, size_t rows,
            cudaStream_t st);

// fused multi-GPU kernel (c) over peer memory (summ.cu, dfx_cgp_*)
constexpr int kMaxPeers = 8;
struct PeerTables {                 // every rank's exchange block, mapped here
  uint8_t* bits[kMaxPeers][2];
  int16_t* list[kMaxPeers][2];
  int32_t* len[kMaxPeers][2];
  unsigned long long* arrive[kMaxPeers];   // waves finished, summed over ranks
  int* changed[kMaxPeers];                 // [max_passes + 1] per-pass flags (= generation if changed)
};
int cg_peer_wave(const CgDev& g, const PeerTables& tab, int cur, int wave, int rank, int nranks,
                 int pass, int gen, unsigned int* blocks_done, cudaStream_t st);
int cg_peer_wait(const unsigned long long* arrive, unsigned long long expect, long long spins,
                 int* err, cudaStream_t st);
int cg_solve(const CgDev& g, uint8_t* b0, int16_t* l0, int32_t* n0, uint8_t* b1, int16_t* l1,
             int32_t* n1, const int32_t* d_wave_off, int max_passes, int* d_changed,
             int* d_passes, cudaStream_t st, int first_pass = 1);
// pack (unpack=false) the listed functions' rows of a table into `out`
// (rowb = 3*nsp + 4 bytes per row), or scatter them back (unpack=true)
int cg_pack(uint8_t* b, int16_t* l, int32_t* n, int nsp, const int32_t* fns, int count,
            uint8_t* out, int rowb, bool unpack, cudaStream_t st);

}  // namespace dfx

namespace dfx {

// transfer simulator (sim.cu): one persistent launch over (program, chunk) items
struct SimDev {
  const dfx_sim_prog* progs;
  const int32_t* ops;
  const int64_t* arg64;
  const int32_t* item_prog;
  const int32_t* item_chunk;
  int n_items;
  dfx_sim_var* vars;
  dfx_sim_rec* recs;
  int64_t rec_cap;
  unsigned long long* rec_count;
  unsigned* next;
};
int sim_launch(const SimDev& s, cudaStream_t stream);

}  // namespace dfx
