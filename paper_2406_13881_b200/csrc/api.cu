// api.cu -- C ABI of libdfx.so (include/dfx.h): handles, buffers, entry points.
#include <algorithm>
#include <chrono>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include "../../include/dfx.h"
#include "dfx_internal.h"
#include "c3gen.cuh"

struct dfx_csr;
namespace { int csr_destroy_impl(dfx_csr* c); }

struct dfx_handle {
  static constexpr int kPipe = 8;      // node ranges of the pipelined CSR calls
  static constexpr int kPipeMax = 32;  // function ranges of dfx_replay_batch
  static constexpr int kComp = 3;     // compute streams of dfx_replay_batch
  cudaStream_t s_copy = nullptr, s_d2h = nullptr;
  cudaStream_t s_comp[kComp] = {};    // [0] unused: the call's own stream
  cudaEvent_t jev[kComp] = {};        // joins of the compute streams
  cudaEvent_t pev[1 + 2 * kPipeMax] = {};
  unsigned long long* pin_cnt = nullptr;   // pinned, kPipeMax counters
  unsigned long long* host_done = nullptr; // mapped pinned: E1 range k complete (count + 1)
  unsigned long long* host_done_dev = nullptr;
  int* pin_one = nullptr;                  // pinned 1s: E1 range-ready flags (H2D)
  cudaError_t pipeline_init() {
    if (s_copy) return cudaSuccess;
    cudaError_t e = cudaStreamCreateWithFlags(&s_copy, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&s_d2h, cudaStreamNonBlocking);
    for (int i = 1; i < kComp; i++)
      if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&s_comp[i], cudaStreamNonBlocking);
    for (auto& ev : jev)
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
    for (auto& ev : pev)
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaHostAlloc((void**)&pin_cnt, sizeof(unsigned long long) * kPipeMax, cudaHostAllocDefault);
    if (e == cudaSuccess)
      e = cudaHostAlloc((void**)&host_done, sizeof(unsigned long long) * kPipeMax, cudaHostAllocMapped);
    if (e == cudaSuccess) e = cudaHostGetDevicePointer((void**)&host_done_dev, host_done, 0);
    if (e == cudaSuccess) e = cudaHostAlloc((void**)&pin_one, sizeof(int) * kPipeMax, cudaHostAllocDefault);
    if (e == cudaSuccess)
      for (int i = 0; i < kPipeMax; i++) pin_one[i] = 1;
    return e;
  }
  int device = 0;
  cudaStream_t stream = nullptr;      // the handle's own stream
  cudaStream_t ext_stream = nullptr;  // caller's stream (dfx_set_stream)
  cudaStream_t st() const { return ext_stream ? ext_stream : stream; }
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  // DFX_TRACE=1: per-range timeline of the pipelined calls on stderr
  // (H2D done, replay start / end, relative to the call's first event)
  bool trace = false;
  cudaEvent_t tev[3 * kPipeMax + 1] = {};
  struct dfx_csr* csr_cache = nullptr;   // reused by dfx_mfp_csr across calls
  ncclComm_t comm = nullptr;             // dfx_comm_init: the handle's NCCL communicator
  int comm_rank = 0, comm_size = 1;
  std::unordered_map<std::string, std::pair<void*, size_t>> bufs;
};

namespace {

thread_local std::string g_err;

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

#define CK(expr)                                                                  \
  do {                                                                            \
    cudaError_t e_ = (expr);                                                      \
    if (e_ != cudaSuccess)                                                        \
      return fail(DFX_E_CUDA, "%s: %s (%s:%d)", #expr, cudaGetErrorString(e_),   \
                  __FILE__, __LINE__);                                            \
  } while (0)

// grow-only named device buffer
void* dbuf(dfx_handle* h, const char* name, size_t bytes) {
  auto& b = h->bufs[name];
  if (b.second < bytes) {
    if (b.first) cudaFree(b.first);
    size_t want = bytes + bytes / 4 + 256;
    if (cudaMalloc(&b.first, want) != cudaSuccess) {
      b.first = nullptr;
      b.second = 0;
      return nullptr;
    }
    b.second = want;
  }
  return b.first;
}

}  // namespace

extern "C" {

int dfx_abi_version(void) { return DFX_ABI_VERSION; }

const char* dfx_last_error(void) { return g_err.c_str(); }

int dfx_open(int device, dfx_handle** out) {
  if (!out) return fail(DFX_E_ARG, "dfx_open: null out");
  int n = 0;
  CK(cudaGetDeviceCount(&n));
  if (device < 0 || device >= n) return fail(DFX_E_ARG, "dfx_open: device %d of %d", device, n);
  CK(cudaSetDevice(device));
  auto* h = new dfx_handle();
  h->device = device;
  CK(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
  CK(cudaEventCreate(&h->ev0));
  CK(cudaEventCreate(&h->ev1));
  if (const char* t = getenv("DFX_TRACE")) h->trace = t[0] == '1';
  if (h->trace)
    for (auto& e : h->tev) CK(cudaEventCreate(&e));
  *out = h;
  return DFX_OK;
}

int dfx_close(dfx_handle* h) {
  if (!h) return DFX_OK;
  cudaSetDevice(h->device);
  for (auto& kv : h->bufs)
    if (kv.second.first) cudaFree(kv.second.first);
  if (h->ev0) cudaEventDestroy(h->ev0);
  if (h->ev1) cudaEventDestroy(h->ev1);
  for (auto& e : h->tev)
    if (e) cudaEventDestroy(e);
  if (h->csr_cache) csr_destroy_impl(h->csr_cache);
  dfx_comm_destroy(h);
  for (auto& ev : h->pev)
    if (ev) cudaEventDestroy(ev);
  if (h->pin_cnt) cudaFreeHost(h->pin_cnt);
  if (h->host_done) cudaFreeHost(h->host_done);
  if (h->pin_one) cudaFreeHost(h->pin_one);
  if (h->s_copy) cudaStreamDestroy(h->s_copy);
  if (h->s_d2h) cudaStreamDestroy(h->s_d2h);
  for (auto& cs : h->s_comp)
    if (cs) cudaStreamDestroy(cs);
  for (auto& ev : h->jev)
    if (ev) cudaEventDestroy(ev);
  if (h->stream) cudaStreamDestroy(h->stream);
  delete h;
  return DFX_OK;
}

int dfx_set_stream(dfx_handle* h, void* stream) {
  if (!h) return fail(DFX_E_ARG, "dfx_set_stream: null handle");
  h->ext_stream = (cudaStream_t)stream;
  return DFX_OK;
}

// ---------------------------------------------------------------------------
// E1: device-resident replay batches
// ---------------------------------------------------------------------------
}  // extern "C"

struct dfx_replay {
  std::vector<void*> allocs;
  dfx::ReplayDev r{};
  int64_t n_vars = 0;
  int32_t n_funcs = 0;
  std::vector<dfx_event> host_events;   // functions beyond the wide limits (fn_class 2)
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  ~dfx_replay() {
    for (void* p : allocs) cudaFree(p);
    if (e0) cudaEventDestroy(e0);
    if (e1) cudaEventDestroy(e1);
  }
};

namespace {
// Work items of functions [f0, f1): one per (function, 32-variable chunk), at
// least one per function so statically known errors surface without
// variables.  Functions go longest program first (counting sort on n_ops), so
// the long warps start in the first waves and a launch does not end on a
// tail of them; chunks of one function stay adjacent (similar cost in a block).
void append_items(const dfx_fn_desc* fns, int f0, int f1, std::vector<int32_t>& item_fn,
                  std::vector<int32_t>& item_chunk, const std::vector<uint8_t>& cls, int want) {
  constexpr int kBins = 4096;
  auto bin = [&](int f) {
    const int b = fns[f].n_ops >> 4;
    return kBins - 1 - (b < kBins - 1 ? b : kBins - 1);
  };
  std::vector<int32_t> start(kBins + 1, 0), order((size_t)(f1 - f0));
  for (int f = f0; f < f1; f++) start[bin(f) + 1]++;
  for (int b = 0; b < kBins; b++) start[b + 1] += start[b];
  for (int f = f0; f < f1; f++) order[start[bin(f)]++] = f;
  for (int f : order) {
    if (cls[f] != want) continue;
    int chunks = (fns[f].n_vars + 31) / 32;
    if (chunks == 0) chunks = 1;
    for (int c = 0; c < chunks; c++) {
      item_fn.push_back(f);
      item_chunk.push_back(c);
    }
  }
}
// A function beyond the wide replay's limits gets one engine-error event
// (visit key 0): the host raises for that function only.
dfx_event engine_error_event(int f) {
  dfx_event e{};
  e.key = 0; e.fn = f; e.var = -1; e.node = 0;
  e.kind = (uint8_t)DFX_EV_ERR_ENGINE; e.pos = 0; e.pad = 0;
  return e;
}

// Classify every function (dfx::fn_class) and fold the per-class slot maxima.
void classify(const dfx_replay_in* in, std::vector<uint8_t>& cls, int& max_slots,
              int& wide_slots, std::vector<dfx_event>& host_events) {
  const int nf = in->n_funcs;
  cls.assign((size_t)nf, 0);
  max_slots = wide_slots = 2;
  for (int f = 0; f < nf; f++) {
    const dfx_fn_desc& d = in->fns[f];
    cls[f] = (uint8_t)dfx::fn_class(d);
    if (cls[f] == 0 && d.n_slots > max_slots) max_slots = d.n_slots;
    if (cls[f] == 1 && d.n_slots > wide_slots) wide_slots = d.n_slots;
    if (cls[f] == 2) host_events.push_back(engine_error_event(f));
  }
}
}  // namespace

namespace dfx {
// Narrow replay limits (replay.cu Narrow): 64 slots, loop depth 24, branch
// depth 48, 192 open arms, statement ids < 0xFFFF (16-bit provenance).  Wide:
// 256 / 64 / 256 / 1024, ids < 2^20 - 1 (the hoist table's node field).
int fn_class(const dfx_fn_desc& d) {
  if (d.n_slots <= 64 && d.max_loop_depth <= 24 && d.max_br_depth <= 48 && d.max_arms <= 192 &&
      d.n_stmts < 0xFFFF)
    return 0;
  if (d.n_slots <= 256 && d.max_loop_depth <= 64 && d.max_br_depth <= 256 && d.max_arms <= 1024 &&
      d.n_stmts < DFX_AC_NODE_MASK)
    return 1;
  return 2;
}
}  // namespace dfx

extern "C" {

int dfx_replay_create(dfx_handle* h, const dfx_replay_in* in, int64_t event_cap, dfx_replay** out) {
  if (!h || !in || !out) return fail(DFX_E_ARG, "dfx_replay_create: null argument");
  CK(cudaSetDevice(h->device));
  const int nf = in->n_funcs;
  std::vector<int32_t> item_fn, item_chunk, wide_fn, wide_chunk;
  std::vector<uint8_t> cls;
  std::vector<dfx_event> host_events;
  int max_slots = 2, wide_slots = 2;
  classify(in, cls, max_slots, wide_slots, host_events);
  append_items(in->fns, 0, nf, item_fn, item_chunk, cls, 0);
  append_items(in->fns, 0, nf, wide_fn, wide_chunk, cls, 1);
  auto* rp = new dfx_replay();
  rp->host_events = std::move(host_events);
  cudaStream_t st = h->st();
  auto up = [&](const void* src, size_t bytes) -> void* {
    void* p = nullptr;
    if (cudaMalloc(&p, bytes + 16) != cudaSuccess) return nullptr;
    rp->allocs.push_back(p);
    if (src && bytes) cudaMemcpyAsync(p, src, bytes, cudaMemcpyHostToDevice, st);
    return p;
  };
  dfx::ReplayDev& r = rp->r;
  r.fns = (const dfx_fn_desc*)up(in->fns, sizeof(dfx_fn_desc) * (size_t)nf);
  r.ops = (const int32_t*)up(in->ops, sizeof(int32_t) * 4 * (size_t)in->n_ops);
  r.var_flags = (const int32_t*)up(in->var_flags, sizeof(int32_t) * (size_t)in->n_vars);
  r.stmt_span = (const int32_t*)up(in->stmt_span, sizeof(int32_t) * 2 * (size_t)in->n_stmts);
  r.sites = (const int32_t*)up(in->sites, sizeof(int32_t) * (size_t)in->n_sites);
  r.arms = (const int32_t*)up(in->arms, sizeof(int32_t) * 2 * (size_t)in->n_arms);
  r.item_fn = (const int32_t*)up(item_fn.data(), sizeof(int32_t) * item_fn.size());
  r.item_chunk = (const int32_t*)up(item_chunk.data(), sizeof(int32_t) * item_chunk.size());
  r.n_items = (int)item_fn.size();
  r.fn_lo = 0;
  r.fn_hi = nf;
  r.max_slots = max_slots;
  r.event_cap = event_cap > 0 ? event_cap : 1;
  r.events = (dfx_event*)up(nullptr, sizeof(dfx_event) * (size_t)r.event_cap);
  r.event_count = (unsigned long long*)up(nullptr, sizeof(unsigned long long));
  r.var_out = (uint8_t*)up(nullptr, (size_t)in->n_vars + 1);
  r.next = (unsigned*)up(nullptr, sizeof(unsigned));
  r.wide_item_fn = (const int32_t*)up(wide_fn.data(), sizeof(int32_t) * wide_fn.size());
  r.wide_item_chunk = (const int32_t*)up(wide_chunk.data(), sizeof(int32_t) * wide_chunk.size());
  r.n_wide_items = (int)wide_fn.size();
  r.wide_max_slots = wide_slots;
  r.wide_next = (unsigned*)up(nullptr, sizeof(unsigned));
  for (void* p : rp->allocs)
    if (!p) { delete rp; return fail(DFX_E_CUDA, "dfx_replay_create: allocation failed"); }
  if (rp->allocs.size() != 15) { delete rp; return fail(DFX_E_CUDA, "dfx_replay_create: allocation failed"); }
  rp->n_vars = in->n_vars;
  rp->n_funcs = nf;
  CK(cudaEventCreate(&rp->e0));
  CK(cudaEventCreate(&rp->e1));
  CK(cudaStreamSynchronize(st));
  *out = rp;
  return DFX_OK;
}

int dfx_replay_run(dfx_handle* h, dfx_replay* rp, int64_t* n_events, float* kernel_ms) {
  if (!h || !rp) return fail(DFX_E_ARG, "dfx_replay_run: null argument");
  CK(cudaSetDevice(h->device));
  cudaStream_t st = h->st();
  CK(cudaMemsetAsync(rp->r.event_count, 0, sizeof(unsigned long long), st));
  CK(cudaEventRecord(rp->e0, st));
  int rc = dfx::replay_launch(rp->r, st);
  if (rc != DFX_OK) return fail(rc, "replay launch failed: %s", cudaGetErrorString(cudaGetLastError()));
  CK(cudaEventRecord(rp->e1, st));
  unsigned long long count = 0;
  CK(cudaMemcpyAsync(&count, rp->r.event_count, sizeof count, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  float ms = 0.f;
  CK(cudaEventElapsedTime(&ms, rp->e0, rp->e1));
  if (n_events) *n_events = (int64_t)count + (int64_t)rp->host_events.size();
  if (kernel_ms) *kernel_ms = ms;
  if ((int64_t)count > rp->r.event_cap)
    return fail(DFX_E_NOSPC, "event capacity %lld < %llu", (long long)rp->r.event_cap, count);
  return DFX_OK;
}

int dfx_replay_fetch(dfx_handle* h, dfx_replay* rp, dfx_replay_out* out) {
  if (!h || !rp || !out) return fail(DFX_E_ARG, "dfx_replay_fetch: null argument");
  CK(cudaSetDevice(h->device));
  cudaStream_t st = h->st();
  unsigned long long count = 0;
  CK(cudaMemcpyAsync(&count, rp->r.event_count, sizeof count, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  int64_t n = (int64_t)count < out->event_cap ? (int64_t)count : out->event_cap;
  if (n > rp->r.event_cap) n = rp->r.event_cap;
  if (n) CK(cudaMemcpyAsync(out->events, rp->r.events, sizeof(dfx_event) * (size_t)n, cudaMemcpyDeviceToHost, st));
  if (rp->n_vars) CK(cudaMemcpyAsync(out->var_out, rp->r.var_out, (size_t)rp->n_vars, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  const int64_t total = (int64_t)count + (int64_t)rp->host_events.size();
  for (size_t i = 0; i < rp->host_events.size(); i++)
    if (n + (int64_t)i < out->event_cap) out->events[n + i] = rp->host_events[i];
  out->n_events = total;
  return total > out->event_cap ? DFX_E_NOSPC : DFX_OK;
}

int dfx_replay_destroy(dfx_handle* h, dfx_replay* rp) {
  if (h) cudaSetDevice(h->device);
  delete rp;
  return DFX_OK;
}

// ---------------------------------------------------------------------------
// E1: dfx_replay_batch  (replaces dartomp.dataflow.analyze_function,
// pkg/src/dartomp/dataflow.py:737-740, batched over functions)
// ---------------------------------------------------------------------------
static int replay_batch_impl(dfx_handle* h, const dfx_replay_in* in, dfx_replay_out* out, bool packed);

int dfx_replay_batch(dfx_handle* h, const dfx_replay_in* in, dfx_replay_out* out) {
  return replay_batch_impl(h, in, out, false);
}

int dfx_replay_batch_packed(dfx_handle* h, const dfx_replay_in* in, dfx_replay_out* out) {
  return replay_batch_impl(h, in, out, true);
}

static int replay_batch_impl(dfx_handle* h, const dfx_replay_in* in, dfx_replay_out* out, bool packed) {
  if (!h || !in || !out) return fail(DFX_E_ARG, "dfx_replay_batch: null argument");
  CK(cudaSetDevice(h->device));
  const int nf = in->n_funcs;
  std::vector<int32_t> item_fn, item_chunk, wide_fn, wide_chunk;
  std::vector<uint8_t> cls;
  std::vector<dfx_event> host_events;
  int max_slots = 2, wide_slots = 2;
  classify(in, cls, max_slots, wide_slots, host_events);
  bool ordered = true;   // per-function array ranges ascending and contiguous
  for (int f = 0; f < nf; f++) {
    const dfx_fn_desc& d = in->fns[f];
    if (f > 0) {
      const dfx_fn_desc& e = in->fns[f - 1];
      ordered &= d.op_off >= e.op_off + e.n_ops && d.var_off >= e.var_off + e.n_vars &&
                 d.stmt_off >= e.stmt_off + e.n_stmts && d.site_off >= e.site_off &&
                 d.arm_off >= e.arm_off;
    }
  }
  // Pipeline: the programs go H2D in K function ranges (copy stream); a
  // region stream builds each range's region table as it lands and then
  // opens the range (ready[k] = 1); ONE persistent replay launch takes the
  // work items in range order, each waiting only for its own range
  // (GateDev), so the replay runs while the H2D of later ranges is still in
  // flight; range k's events go home (D2H stream) as soon as its last item
  // is done, which the kernel publishes in mapped host memory.  Functions
  // are independent (SURVEY F3 / SPEC), so ranges change nothing but the
  // order of events in the buffer.  32 ranges of equal ops (C4 sweep: 8 /
  // 16 / 32 / 64 ranges 216 / 191 / 188 / 198 ms; ramped sizes were no
  // better).  Ranges start at functions whose ops begin on a 128-B line: no
  // L1 line read by one range holds another range's region table before it
  // is written.
  int K = ordered && nf >= 256 ? dfx_handle::kPipeMax : 1;
  std::vector<int> cut(K + 1, nf);
  cut[0] = 0;
  if (K > 1) {
    int f = 0;
    for (int k = 1; k < K; k++) {
      const double target = (double)k / K * (double)in->n_ops;
      while (f < nf && (double)in->fns[f].op_off < target) f++;
      while (f < nf && (in->fns[f].op_off & 7) != 0) f++;   // line-aligned start
      cut[k] = f;
    }
    if (in->fns[0].op_off & 7) K = 1;        // the first range must start aligned too
  }
  if (K == 1) { cut.assign(2, nf); cut[0] = 0; }
  std::vector<int32_t> range_item0(K + 1, 0), range_items(K, 0);
  for (int k = 0; k < K; k++) {
    append_items(in->fns, cut[k], cut[k + 1], item_fn, item_chunk, cls, 0);
    range_item0[k + 1] = (int32_t)item_fn.size();
    range_items[k] = range_item0[k + 1] - range_item0[k];
  }
  const size_t n_items = item_fn.size();
  // functions beyond the narrow limits: one wide launch after the gated one
  append_items(in->fns, 0, nf, wide_fn, wide_chunk, cls, 1);
  const size_t n_wide = wide_fn.size();
  cudaStream_t st = h->st();
  void* d_fns = dbuf(h, "fns", sizeof(dfx_fn_desc) * (size_t)nf + 16);
  void* d_ops = dbuf(h, "ops", sizeof(int32_t) * 4 * (size_t)in->n_ops + 16);
  void* d_pk = packed ? dbuf(h, "ops_packed", sizeof(uint32_t) * 2 * (size_t)in->n_ops + 16) : d_ops;
  void* d_vf = dbuf(h, "vf", sizeof(int32_t) * (size_t)in->n_vars + 16);
  void* d_span = dbuf(h, "span", sizeof(int32_t) * 2 * (size_t)in->n_stmts + 16);
  void* d_sites = dbuf(h, "sites", sizeof(int32_t) * (size_t)in->n_sites + 16);
  void* d_arms = dbuf(h, "arms", sizeof(int32_t) * 2 * (size_t)in->n_arms + 16);
  void* d_ifn = dbuf(h, "ifn", sizeof(int32_t) * n_items + 16);
  void* d_ich = dbuf(h, "ich", sizeof(int32_t) * n_items + 16);
  void* d_iwf = dbuf(h, "iwf", sizeof(int32_t) * n_wide + 16);
  void* d_iwc = dbuf(h, "iwc", sizeof(int32_t) * n_wide + 16);
  const int64_t cap = out->event_cap;
  // per-range event regions, sized from the caller's capacity by ops share;
  // a range that overflows its region is replayed again into an exact-size
  // one (rare) unless the total already exceeds the caller's capacity
  std::vector<long long> ev_off(K + 1, 0), ev_cap(K, 0);
  for (int k = 0; k < K; k++) {
    const int f0 = cut[k], f1 = cut[k + 1];
    int64_t ops_k = 0;
    if (K == 1) ops_k = in->n_ops;
    else if (f0 < f1) ops_k = (f1 < nf ? (int64_t)in->fns[f1].op_off : in->n_ops) - in->fns[f0].op_off;
    const double share = in->n_ops > 0 ? (double)ops_k / (double)in->n_ops : 1.0;
    ev_cap[k] = (long long)(1.25 * (double)(cap > 0 ? cap : 0) * share) + 4096;
    ev_off[k + 1] = ev_off[k] + ev_cap[k];
  }
  auto* d_ev = (dfx_event*)dbuf(h, "events", sizeof(dfx_event) * (size_t)ev_off[K]);
  auto* d_cnt = (unsigned long long*)dbuf(h, "evcount", sizeof(unsigned long long) * (K + 2));
  auto* d_vout = (uint8_t*)dbuf(h, "vout", (size_t)in->n_vars + 1);
  // gate block: fn_cut[K+1] ready[K] range_items[K] items_done[K] next[3]
  // timed_out[1] (ints), then ev_off[K] ev_cap[K] (long long)
  const size_t gate_ints = (size_t)(K + 1) + 3 * (size_t)K + 4;
  auto* d_gate = (int*)dbuf(h, "gate", sizeof(int) * gate_ints + 16 + 2 * sizeof(long long) * K);
  if (!d_fns || !d_ops || !d_pk || !d_vf || !d_span || !d_sites || !d_arms || !d_ifn || !d_ich || !d_ev ||
      !d_cnt || !d_vout || !d_gate || !d_iwf || !d_iwc)
    return fail(DFX_E_CUDA, "dfx_replay_batch: device allocation failed");
  int* g_cut = d_gate;
  int* g_ready = g_cut + K + 1;
  int* g_items = g_ready + K;
  int* g_done = g_items + K;
  int* g_next = g_done + K;          // [0] the launch, [1] a redo, [2] the wide launch
  int* g_timeout = g_next + 3;
  auto* g_evoff = reinterpret_cast<long long*>(
      reinterpret_cast<uintptr_t>(d_gate + gate_ints + 1) & ~(uintptr_t)7) + 1;
  long long* g_evcap = g_evoff + K;
  CK(h->pipeline_init());
  for (int k = 0; k < K; k++) h->host_done[k] = 0ull;
  // small arrays first, on the call's stream
  std::vector<int> gate_host(gate_ints, 0);
  for (int k = 0; k <= K; k++) gate_host[k] = cut[k];
  for (int k = 0; k < K; k++) gate_host[2 * K + 1 + k] = range_items[k];
  CK(cudaMemcpyAsync(d_fns, in->fns, sizeof(dfx_fn_desc) * (size_t)nf, cudaMemcpyHostToDevice, st));
  if (n_items) {
    CK(cudaMemcpyAsync(d_ifn, item_fn.data(), sizeof(int32_t) * n_items, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(d_ich, item_chunk.data(), sizeof(int32_t) * n_items, cudaMemcpyHostToDevice, st));
  }
  if (n_wide) {
    CK(cudaMemcpyAsync(d_iwf, wide_fn.data(), sizeof(int32_t) * n_wide, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(d_iwc, wide_chunk.data(), sizeof(int32_t) * n_wide, cudaMemcpyHostToDevice, st));
  }
  CK(cudaMemcpyAsync(d_gate, gate_host.data(), sizeof(int) * gate_ints, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(g_evoff, ev_off.data(), sizeof(long long) * K, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(g_evcap, ev_cap.data(), sizeof(long long) * K, cudaMemcpyHostToDevice, st));
  CK(cudaMemsetAsync(d_cnt, 0, sizeof(unsigned long long) * (K + 2), st));
  dfx::ReplayDev r{};
  r.fns = (const dfx_fn_desc*)d_fns;
  r.ops = (const int32_t*)d_ops;
  r.var_flags = (const int32_t*)d_vf;
  r.stmt_span = (const int32_t*)d_span;
  r.sites = (const int32_t*)d_sites;
  r.arms = (const int32_t*)d_arms;
  r.item_fn = (const int32_t*)d_ifn;
  r.item_chunk = (const int32_t*)d_ich;
  r.n_items = (int)n_items;
  r.fn_lo = 0;
  r.fn_hi = nf;
  r.max_slots = max_slots;
  r.events = d_ev;
  r.event_cap = cap;
  r.event_count = d_cnt;
  r.var_out = d_vout;
  r.next = reinterpret_cast<unsigned*>(g_next);
  r.wide_item_fn = (const int32_t*)d_iwf;
  r.wide_item_chunk = (const int32_t*)d_iwc;
  r.n_wide_items = (int)n_wide;
  r.wide_max_slots = wide_slots;
  r.wide_next = reinterpret_cast<unsigned*>(g_next + 2);
  dfx::GateDev gate{};
  gate.K = K;
  gate.fn_cut = g_cut;
  gate.ready = g_ready;
  gate.ev_off = g_evoff;
  gate.ev_cap = g_evcap;
  gate.range_items = reinterpret_cast<const unsigned*>(g_items);
  gate.items_done = reinterpret_cast<unsigned*>(g_done);
  gate.host_done = h->host_done_dev;
  gate.timed_out = reinterpret_cast<unsigned*>(g_timeout);
  gate.timeout_ns = 20000000000ull;                 // 20 s, then the ungated replay
  if (const char* e = getenv("DFX_GATE_TIMEOUT_MS")) gate.timeout_ns = 1000000ull * strtoull(e, nullptr, 10);
  auto lo = [&](int f, int32_t dfx_fn_desc::*off) -> int64_t { return f < nf ? in->fns[f].*off : -1; };
  // region tables on two streams, alternating by range: a region kernel
  // shares the SMs with the running replay, so consecutive ranges' tables
  // are built side by side rather than one after the other
  cudaStream_t s_regs[2] = {h->s_comp[1], h->s_comp[2]};
  CK(cudaEventRecord(h->pev[0], st));   // uploads done, gate state cleared
  if (h->trace) CK(cudaEventRecord(h->tev[3 * dfx_handle::kPipeMax], st));
  CK(cudaStreamWaitEvent(h->s_copy, h->pev[0], 0));
  for (cudaStream_t sr : s_regs) CK(cudaStreamWaitEvent(sr, h->pev[0], 0));
  // every copy and region launch is enqueued before the replay launch (a
  // failed enqueue must not leave the kernel waiting for a range)
  for (int k = 0; k < K; k++) {
    const int f0 = cut[k], f1 = cut[k + 1];
    if (f0 < f1) {
      struct Rng { const int32_t* src; void* dst; int64_t a, b, n; int unit; };
      const int64_t ops_a = K == 1 ? 0 : lo(f0, &dfx_fn_desc::op_off);
      const int64_t ops_b = K == 1 || f1 == nf ? in->n_ops : lo(f1, &dfx_fn_desc::op_off);
      const int64_t vf_a = K == 1 ? 0 : lo(f0, &dfx_fn_desc::var_off);
      const int64_t vf_b = K == 1 || f1 == nf ? in->n_vars : lo(f1, &dfx_fn_desc::var_off);
      const int64_t sp_a = K == 1 ? 0 : lo(f0, &dfx_fn_desc::stmt_off);
      const int64_t sp_b = K == 1 || f1 == nf ? in->n_stmts : lo(f1, &dfx_fn_desc::stmt_off);
      const int64_t si_a = K == 1 ? 0 : lo(f0, &dfx_fn_desc::site_off);
      const int64_t si_b = K == 1 || f1 == nf ? in->n_sites : lo(f1, &dfx_fn_desc::site_off);
      const int64_t ar_a = K == 1 ? 0 : lo(f0, &dfx_fn_desc::arm_off);
      const int64_t ar_b = K == 1 || f1 == nf ? in->n_arms : lo(f1, &dfx_fn_desc::arm_off);
      // each copy runs 128 B into the next range's data, so no L1 line a
      // range's warps read holds bytes not yet copied (the next copy writes
      // the same bytes again)
      // packed ops: exactly the range (unpacked on the device below; a range's
      // ops start and end on 128-B lines of the 16-byte form)
      if (packed && ops_b > ops_a)
        CK(cudaMemcpyAsync((uint32_t*)d_pk + 2 * ops_a, (const uint32_t*)(const void*)in->ops + 2 * ops_a,
                           sizeof(uint32_t) * 2 * (size_t)(ops_b - ops_a), cudaMemcpyHostToDevice,
                           h->s_copy));
      Rng rng[] = {{packed ? nullptr : in->ops, d_ops, ops_a, ops_b, in->n_ops, 4},
                   {in->var_flags, d_vf, vf_a, vf_b, in->n_vars, 1},
                   {in->stmt_span, d_span, sp_a, sp_b, in->n_stmts, 2},
                   {in->sites, d_sites, si_a, si_b, in->n_sites, 1},
                   {in->arms, d_arms, ar_a, ar_b, in->n_arms, 2}};
      for (auto& g : rng) {
        if (!g.src) continue;
        int64_t e = g.b + 32 / g.unit;
        if (e > g.n) e = g.n;
        if (e > g.a)
          CK(cudaMemcpyAsync((int32_t*)g.dst + g.a * g.unit, g.src + g.a * g.unit,
                             sizeof(int32_t) * g.unit * (size_t)(e - g.a), cudaMemcpyHostToDevice,
                             h->s_copy));
      }
    }
    CK(cudaEventRecord(h->pev[1 + k], h->s_copy));
    if (h->trace) CK(cudaEventRecord(h->tev[3 * k], h->s_copy));
    cudaStream_t s_reg = s_regs[k & 1];
    CK(cudaStreamWaitEvent(s_reg, h->pev[1 + k], 0));
    if (packed && f0 < f1) {
      const int64_t ops_a = K == 1 ? 0 : lo(f0, &dfx_fn_desc::op_off);
      const int64_t ops_b = K == 1 || f1 == nf ? in->n_ops : lo(f1, &dfx_fn_desc::op_off);
      int rcu = dfx::unpack_ops_launch((const uint32_t*)d_pk, (int32_t*)d_ops, ops_a, ops_b, s_reg);
      if (rcu != DFX_OK) return fail(rcu, "unpack_ops launch failed");
    }
    int rc = dfx::region_launch(r, f0, f1, s_reg);
    if (rc != DFX_OK) return fail(rc, "region_kernel launch failed");
    CK(cudaMemcpyAsync(g_ready + k, h->pin_one + k, sizeof(int), cudaMemcpyHostToDevice, s_reg));
    if (h->trace) CK(cudaEventRecord(h->tev[3 * k + 1], s_reg));
  }
  CK(cudaEventRecord(h->ev0, st));
  {
    const int rc = dfx::replay_launch(r, st, &gate);
    if (rc != DFX_OK) {
      for (cudaStream_t sr : s_regs) cudaStreamSynchronize(sr);   // the ranges open; the kernel drains
      cudaStreamSynchronize(st);
      return fail(rc, "replay launch failed: %s", cudaGetErrorString(cudaGetLastError()));
    }
  }
  // once the last range is open, its region stream backfills the slots the
  // gated launch left to the region kernels (same item queue)
  cudaEvent_t ev_bf = nullptr;
  if (K > 1 && !getenv("DFX_NO_BACKFILL")) {
    cudaStream_t s_last = s_regs[(K - 1) & 1];
    if (dfx::replay_launch_backfill(r, s_last, &gate) == DFX_OK &&
        cudaEventCreateWithFlags(&ev_bf, cudaEventDisableTiming) == cudaSuccess) {
      CK(cudaEventRecord(ev_bf, s_last));
      CK(cudaStreamWaitEvent(st, ev_bf, 0));
    }
  }
  CK(cudaEventRecord(h->ev1, st));
  if (ev_bf) cudaEventDestroy(ev_bf);   // released once recorded and waited on
  // a range's region kernel never got an SM slot beside the gated launch
  // (e.g. another process holds the GPU), so its items gave up waiting:
  // replay the batch again, ungated, through the device-resident path
  //
  auto ungated = [&]() -> int {
    if (h->trace) fprintf(stderr, "dfx_replay_batch: gate timed out; replaying ungated\n");
    for (cudaStream_t sr : s_regs) cudaStreamSynchronize(sr);
    cudaStreamSynchronize(h->s_copy);
    cudaStreamSynchronize(st);
    dfx_replay* rp = nullptr;
    dfx_replay_in in16 = *in;
    std::vector<int32_t> ops16;
    if (packed) {      // the device-resident path takes the 16-byte form
      ops16.resize(4 * (size_t)in->n_ops);
      dfx::unpack_ops_host((const uint32_t*)(const void*)in->ops, ops16.data(), in->n_ops);
      in16.ops = ops16.data();
    }
    int rc = dfx_replay_create(h, &in16, out->event_cap > 0 ? out->event_cap : 1, &rp);
    if (rc) return rc;
    int64_t n_ev = 0;
    float kms = 0.f;
    rc = dfx_replay_run(h, rp, &n_ev, &kms);
    if (rc == DFX_OK || rc == DFX_E_NOSPC) {
      const int rc2 = dfx_replay_fetch(h, rp, out);
      if (rc == DFX_OK) rc = rc2;
      out->kernel_ms = kms;
    }
    dfx_replay_destroy(h, rp);
    return rc;
  };
  auto gate_timed_out = [&]() -> bool {
    int t = 0;
    return cudaMemcpy(&t, g_timeout, sizeof t, cudaMemcpyDeviceToHost) == cudaSuccess && t != 0;
  };
  // range k's events go home as soon as its last item is done
  const auto t_call = std::chrono::steady_clock::now();
  std::vector<double> t_done(K, 0.0);
  unsigned long long count = 0, done = 0;
  std::vector<int> redo;
  for (int k = 0; k < K; k++) {
    volatile unsigned long long* hd = h->host_done + k;
    if (range_items[k] > 0) {
      while (*hd == 0ull) {
        if (cudaEventQuery(h->ev1) != cudaErrorNotReady) break;   // finished (or failed)
        std::this_thread::yield();
      }
      if (*hd == 0ull) {
        CK(cudaEventSynchronize(h->ev1));
        if (*hd == 0ull) {
          if (gate_timed_out()) return ungated();
          return fail(DFX_E_CUDA, "dfx_replay_batch: range %d did not complete", k);
        }
      }
    }
    t_done[k] = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_call).count();
    const unsigned long long c = range_items[k] > 0 ? *hd - 1ull : 0ull;
    count += c;
    if ((long long)c > ev_cap[k]) { redo.push_back(k); continue; }
    unsigned long long n = c;
    if (cap <= (int64_t)done) n = 0;
    else if ((int64_t)(done + n) > cap) n = (unsigned long long)cap - done;
    if (n)
      CK(cudaMemcpyAsync(out->events + done, d_ev + ev_off[k], sizeof(dfx_event) * (size_t)n,
                         cudaMemcpyDeviceToHost, h->s_d2h));
    done += n;
  }
  CK(cudaStreamSynchronize(st));
  {
    int timed_out = 0;
    CK(cudaMemcpy(&timed_out, g_timeout, sizeof timed_out, cudaMemcpyDeviceToHost));
    if (timed_out) return ungated();
  }
  if (!redo.empty() && (int64_t)count <= cap) {
    for (int k : redo) {
      const int64_t need = (int64_t)(h->host_done[k] - 1ull);
      if (h->trace)
        fprintf(stderr, "dfx_replay_batch range %d: %lld events overflow its region of %lld; "
                "replayed into an exact-size one\n", k, (long long)need, (long long)ev_cap[k]);
      auto* d_re = (dfx_event*)dbuf(h, "events_redo", sizeof(dfx_event) * (size_t)need);
      if (!d_re) return fail(DFX_E_CUDA, "dfx_replay_batch: device allocation failed");
      CK(cudaStreamSynchronize(h->s_d2h));   // the previous redo's events are home
      dfx::ReplayDev rk = r;
      rk.item_fn = (const int32_t*)d_ifn + range_item0[k];
      rk.item_chunk = (const int32_t*)d_ich + range_item0[k];
      rk.n_items = range_items[k];
      rk.fn_lo = cut[k];
      rk.fn_hi = cut[k + 1];
      rk.events = d_re;
      rk.event_cap = need;
      rk.event_count = d_cnt + K;
      rk.next = reinterpret_cast<unsigned*>(g_next + 1);
      CK(cudaMemsetAsync(d_cnt + K, 0, sizeof(unsigned long long), st));
      const int rc = dfx::replay_launch(rk, st);   // tables rebuilt identically
      if (rc != DFX_OK) return fail(rc, "replay launch failed: %s", cudaGetErrorString(cudaGetLastError()));
      CK(cudaStreamSynchronize(st));
      CK(cudaMemcpyAsync(out->events + done, d_re, sizeof(dfx_event) * (size_t)need,
                         cudaMemcpyDeviceToHost, h->s_d2h));
      done += (unsigned long long)need;
    }
  }
  // the wide functions (rare): one ungated launch, all ranges have landed;
  // their events go into their own region (regrown once if it overflows)
  if (n_wide) {
    int64_t ops_w = 0;
    for (size_t i = 0; i < n_wide; i++)
      if (i == 0 || wide_fn[i] != wide_fn[i - 1]) ops_w += in->fns[wide_fn[i]].n_ops;
    int64_t cap_w = (int64_t)(1.25 * (double)(cap > 0 ? cap : 0) *
                              ((double)ops_w / (double)(in->n_ops > 0 ? in->n_ops : 1))) + 4096;
    for (int attempt = 0; attempt < 2; attempt++) {
      auto* d_ew = (dfx_event*)dbuf(h, "events_wide", sizeof(dfx_event) * (size_t)cap_w);
      if (!d_ew) return fail(DFX_E_CUDA, "dfx_replay_batch: device allocation failed");
      CK(cudaStreamSynchronize(h->s_d2h));
      dfx::ReplayDev rw = r;
      rw.events = d_ew;
      rw.event_cap = cap_w;
      rw.event_count = d_cnt + K + 1;
      CK(cudaMemsetAsync(d_cnt + K + 1, 0, sizeof(unsigned long long), st));
      const int rc = dfx::replay_launch_wide(rw, st);
      if (rc != DFX_OK) return fail(rc, "wide replay launch failed: %s", cudaGetErrorString(cudaGetLastError()));
      CK(cudaEventRecord(h->ev1, st));
      unsigned long long cw = 0;
      CK(cudaMemcpyAsync(&cw, d_cnt + K + 1, sizeof cw, cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      if ((int64_t)cw > cap_w && attempt == 0) { cap_w = (int64_t)cw; continue; }
      count += cw;
      unsigned long long n = cw;
      if (cap <= (int64_t)done) n = 0;
      else if ((int64_t)(done + n) > cap) n = (unsigned long long)cap - done;
      if (n)
        CK(cudaMemcpyAsync(out->events + done, d_ew, sizeof(dfx_event) * (size_t)n,
                           cudaMemcpyDeviceToHost, h->s_d2h));
      done += n;
      break;
    }
  }
  if (in->n_vars)
    CK(cudaMemcpyAsync(out->var_out, d_vout, (size_t)in->n_vars, cudaMemcpyDeviceToHost, h->s_d2h));
  CK(cudaStreamSynchronize(h->s_d2h));
  for (const dfx_event& e : host_events) {     // functions beyond the wide limits
    if ((int64_t)done < cap) out->events[done++] = e;
    count++;
  }
  float ms = 0.f;
  CK(cudaEventElapsedTime(&ms, h->ev0, h->ev1));
  if (h->trace) {
    const cudaEvent_t t0 = h->tev[3 * dfx_handle::kPipeMax];
    float k0 = 0.f;
    cudaEventElapsedTime(&k0, t0, h->ev0);
    fprintf(stderr, "dfx_replay_batch: K=%d, replay launch at %.2f ms\n", K, k0);
    for (int k = 0; k < K; k++) {
      float a = 0.f, b = 0.f;
      cudaEventElapsedTime(&a, t0, h->tev[3 * k]);
      cudaEventElapsedTime(&b, t0, h->tev[3 * k + 1]);
      fprintf(stderr, "dfx_replay_batch range %2d: functions [%d, %d) h2d done %8.2f ms, open "
              "%8.2f ms, complete %8.2f ms (host clock from launch)\n", k, cut[k], cut[k + 1],
              a, b, t_done[k]);
    }
  }
  out->kernel_ms = ms;
  out->n_events = (int64_t)count;
  if ((int64_t)count > cap) return fail(DFX_E_NOSPC, "event capacity %lld < %llu",
                                        (long long)cap, count);
  return DFX_OK;
}

// ---------------------------------------------------------------------------
// kernels (a) + (b): CSR fixpoint and transfer requirements
// ---------------------------------------------------------------------------
}  // extern "C"

struct dfx_csr {
  dfx::CsrDev p{};
  std::vector<void*> allocs;
  void* scratch = nullptr;
  size_t scratch_bytes = 0;
  int32_t* counts = nullptr;
  int64_t* offsets = nullptr;
  uint32_t* d_masks = nullptr;
  int64_t masks_cap = 0;
  uint32_t* d_occ = nullptr;
  uint16_t* d_vars = nullptr;     // requirement lists (grow-only)
  int64_t vars_cap = 0;
  uint8_t* d_b8 = nullptr;        // byte-coded requirement lists (grow-only)
  int64_t b8_cap = 0;
  int* d_bad = nullptr;           // access-list validation flag
  void* d_cnt = nullptr;
  uint8_t* flags = nullptr;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
};

namespace {

template <class T>
T* csr_alloc(dfx_csr* c, size_t n) {
  void* p = nullptr;
  if (cudaMalloc(&p, n * sizeof(T) + 16) != cudaSuccess) return nullptr;
  c->allocs.push_back(p);
  return (T*)p;
}

int csr_destroy_impl(dfx_csr* c) {
  if (!c) return DFX_OK;
  for (void* p : c->allocs) cudaFree(p);
  if (c->d_masks) cudaFree(c->d_masks);
  if (c->d_occ) cudaFree(c->d_occ);
  if (c->d_vars) cudaFree(c->d_vars);
  if (c->d_b8) cudaFree(c->d_b8);
  if (c->e0) cudaEventDestroy(c->e0);
  if (c->e1) cudaEventDestroy(c->e1);
  delete c;
  return DFX_OK;
}

// allocate every device array of a problem with n nodes, `words` words
int csr_alloc_all(dfx_csr* c, int64_t n, int words, int64_t nnz, const uint32_t* S_host) {
  dfx::CsrDev& p = c->p;
  p.n_nodes = n;
  p.words = words;
  p.nnz = nnz;
  const size_t plane = (size_t)n * words;
  p.row_ptr = csr_alloc<int32_t>(c, n + 1);
  p.col = csr_alloc<int32_t>(c, nnz > 0 ? nnz : 1);
  p.kind = csr_alloc<uint8_t>(c, n);
  p.A = csr_alloc<uint32_t>(c, plane);
  p.B = csr_alloc<uint32_t>(c, plane);
  p.USE = csr_alloc<uint32_t>(c, plane);
  p.OH = csr_alloc<uint32_t>(c, plane);
  p.OD = csr_alloc<uint32_t>(c, plane);
  p.REQ = csr_alloc<uint32_t>(c, plane);
  p.S = csr_alloc<uint32_t>(c, words);
  p.stamp = csr_alloc<int32_t>(c, n);
  p.popc = csr_alloc<int32_t>(c, n);
  p.desc = csr_alloc<int32_t>(c, (size_t)n * 8);
  p.fp_slot = csr_alloc<int32_t>(c, words / 4);
  c->counts = csr_alloc<int32_t>(c, n);
  c->offsets = csr_alloc<int64_t>(c, n + 1);
  c->scratch_bytes = dfx::scan_scratch_bytes(n);
  c->scratch = csr_alloc<uint8_t>(c, c->scratch_bytes);
  c->d_cnt = csr_alloc<uint8_t>(c, dfx::round_ctl_bytes());
  c->d_bad = csr_alloc<int>(c, 1);
  p.seen = csr_alloc<int32_t>(c, nnz > 0 ? nnz : 1);
  p.chunk_done = csr_alloc<int32_t>(c, n);
  p.seen4 = csr_alloc<int32_t>(c, 4 * (size_t)n);
  p.succ_ptr = csr_alloc<int32_t>(c, n + 1);
  p.succ = csr_alloc<int32_t>(c, nnz > 0 ? nnz : 1);
  c->flags = csr_alloc<uint8_t>(c, 2 * (size_t)n);   // >= 2 * n_chunks for chunk_nodes >= 1
  // scalar quads -> FP slots
  std::vector<int32_t> slot(words / 4, -1);
  int ns = 0;
  for (int q = 0; q < words / 4; q++) {
    const uint32_t* s = S_host + 4 * q;
    if (s[0] | s[1] | s[2] | s[3]) slot[q] = ns++;
  }
  p.n_fp_slots = ns;
  p.s_quads_low = 1;
  for (int q = 8; q < words / 4; q++)
    if (slot[q] >= 0) p.s_quads_low = 0;
  p.FPQ = csr_alloc<uint32_t>(c, (size_t)n * 4 * (ns > 0 ? ns : 1));
  for (void* a : c->allocs)
    if (!a) return fail(DFX_E_CUDA, "cudaMalloc failed for a %lld-node x %d-word problem",
                        (long long)n, words);
  if (c->allocs.size() != 26) return fail(DFX_E_CUDA, "cudaMalloc failed (%lld nodes)", (long long)n);
  CK(cudaMemcpy(p.S, S_host, sizeof(uint32_t) * words, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(p.fp_slot, slot.data(), sizeof(int32_t) * slot.size(), cudaMemcpyHostToDevice));
  CK(cudaEventCreate(&c->e0));
  CK(cudaEventCreate(&c->e1));
  return DFX_OK;
}

int check_words(int64_t n, int words) {
  if (n <= 0 || n > 0x7FFFFFFF) return fail(DFX_E_ARG, "n_nodes %lld out of range", (long long)n);
  if (words <= 0) return fail(DFX_E_ARG, "words=%d out of range", words);
  if (dfx::vpl_for(words) < 0)
    return fail(DFX_E_LIMIT, "words=%d: need a multiple of 4 and at most 512", words);
  return DFX_OK;
}

}  // namespace

extern "C" {

}  // extern "C"

namespace {
int check_nnz(int64_t nnz) {
  if (nnz < 0 || nnz > 0x7FFFFFFF) return fail(DFX_E_ARG, "nnz %lld out of range (int32 row_ptr)", (long long)nnz);
  return DFX_OK;
}

// the uploaded CSR is well formed (device check, one round trip) before any
// kernel gathers through it; a bad graph is an argument error, not a fault
int validate_csr(dfx_csr* c, cudaStream_t st) {
  CK(cudaMemsetAsync(c->d_bad, 0, sizeof(int), st));
  if (dfx::check_csr(c->p, c->d_bad, st)) return fail(DFX_E_CUDA, "check_csr launch failed");
  int bad = 0;
  CK(cudaMemcpyAsync(&bad, c->d_bad, sizeof(int), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (bad) return fail(DFX_E_ARG, "CSR: row_ptr must run from 0 to nnz without decreasing and "
                                  "every predecessor id must lie in [0, n_nodes)");
  return DFX_OK;
}

// H2D of one problem's inputs into already-allocated buffers (+ A = R|W)
int csr_upload(dfx_csr* c, const dfx_csr_in* in, cudaStream_t st) {
  dfx::CsrDev& p = c->p;
  const size_t plane = sizeof(uint32_t) * (size_t)in->n_nodes * in->words;
  CK(cudaMemcpyAsync(p.row_ptr, in->row_ptr, sizeof(int32_t) * (in->n_nodes + 1), cudaMemcpyHostToDevice, st));
  if (in->nnz) CK(cudaMemcpyAsync(p.col, in->col, sizeof(int32_t) * in->nnz, cudaMemcpyHostToDevice, st));
  int vrc = validate_csr(c, st);
  if (vrc) return vrc;
  CK(cudaMemcpyAsync(p.kind, in->node_kind, in->n_nodes, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(p.USE, in->R, plane, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(p.B, in->W, plane, cudaMemcpyHostToDevice, st));
  int rc = dfx::or_planes(p, st);
  if (!rc) rc = dfx::build_desc(p, st);
  if (!rc) rc = dfx::build_succ(p, c->scratch, c->scratch_bytes, c->counts, st);
  if (rc) return fail(rc, "or_planes/build_desc launch failed");
  return DFX_OK;
}

bool same_scalars(const dfx_csr* c, const uint32_t* S, int words) {
  std::vector<uint32_t> cur(words);
  if (cudaMemcpy(cur.data(), c->p.S, sizeof(uint32_t) * words, cudaMemcpyDeviceToHost) != cudaSuccess)
    return false;
  return std::memcmp(cur.data(), S, sizeof(uint32_t) * words) == 0;
}
}  // namespace

extern "C" {

int dfx_csr_create(dfx_handle* h, const dfx_csr_in* in, dfx_csr** out) {
  if (!h || !in || !out) return fail(DFX_E_ARG, "dfx_csr_create: null argument");
  CK(cudaSetDevice(h->device));
  int rc = check_words(in->n_nodes, in->words);
  if (!rc) rc = check_nnz(in->nnz);
  if (rc) return rc;
  if (!in->row_ptr || !in->node_kind || !in->R || !in->W || !in->S || (in->nnz && !in->col))
    return fail(DFX_E_ARG, "dfx_csr_in: null array");
  auto* c = new dfx_csr();
  rc = csr_alloc_all(c, in->n_nodes, in->words, in->nnz, in->S);
  if (!rc) rc = csr_upload(c, in, h->st());
  if (rc) { csr_destroy_impl(c); return rc; }
  *out = c;
  return DFX_OK;
}

int dfx_csr_generate_c3(dfx_handle* h, const dfx_c3_spec* spec, dfx_csr** out) {
  if (!h || !spec || !out) return fail(DFX_E_ARG, "dfx_csr_generate_c3: null argument");
  CK(cudaSetDevice(h->device));
  int rc = check_words(spec->n_nodes, spec->words);
  if (rc) return rc;
  int64_t nnz = 0;
  {  // exact edge count (host, cheap: one hash per node)
    for (int64_t n = 1; n < spec->n_nodes; n++) nnz += 1 + dfx::c3_n_extra(spec->seed, n);
  }
  std::vector<uint32_t> S(spec->words);
  for (int w = 0; w < spec->words; w++) S[w] = dfx::c3_scalar_word(spec->w0 + w, spec->n_scalar);
  auto* c = new dfx_csr();
  rc = csr_alloc_all(c, spec->n_nodes, spec->words, nnz, S.data());
  if (rc) { csr_destroy_impl(c); return rc; }
  rc = dfx::c3_generate(c->p, spec->seed, spec->w0, h->st(), c->scratch, c->scratch_bytes);
  if (!rc) rc = dfx::build_desc(c->p, h->st());
  if (!rc) rc = dfx::build_succ(c->p, c->scratch, c->scratch_bytes, c->counts, h->st());
  if (rc) { csr_destroy_impl(c); return fail(rc, "c3 generation failed"); }
  CK(cudaStreamSynchronize(h->st()));
  *out = c;
  return DFX_OK;
}

// Nodes per warp task of kernel (a): 56 (C3 sweep 32..512, scripts/tune_c3.py).
// Real programs' CFGs (cfgprog.py, scripts/diag_cfg_solve.py) measured too:
// 56 is best there as well (2.9 ms vs 3.0 at 128, 4.5 at 8 on 40 C4 units).
static int default_chunk(dfx_handle*, int64_t) { return 56; }

int dfx_csr_destroy(dfx_handle* h, dfx_csr* p) {
  if (h) cudaSetDevice(h->device);
  return csr_destroy_impl(p);
}

int dfx_csr_solve(dfx_handle* h, dfx_csr* c, int32_t chunk_nodes, dfx_csr_stats* stats) {
  if (!h || !c) return fail(DFX_E_ARG, "dfx_csr_solve: null argument");
  CK(cudaSetDevice(h->device));
  if (chunk_nodes <= 0) chunk_nodes = default_chunk(h, c->p.n_nodes);
  cudaStream_t st = h->st();
  dfx::SolveStats s{};
  CK(cudaEventRecord(c->e0, st));
  int rc = dfx::mfp_solve(c->p, c->d_cnt, c->flags, st, chunk_nodes, &s);
  if (rc) return fail(rc, "mfp_solve failed: %s", cudaGetErrorString(cudaGetLastError()));
  CK(cudaEventRecord(c->e1, st));
  CK(cudaEventSynchronize(c->e1));
  if (stats) {
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, c->e0, c->e1));
    stats->rounds_h = s.rounds[0];
    stats->rounds_d = s.rounds[1];
    stats->evaluated = s.evaluated;
    stats->rows_read = s.rows_read;
    stats->rows_written = s.rows_written;
    stats->solve_ms = ms;
    stats->kernel_ms = s.kernel_ms;
  }
  return DFX_OK;
}

int dfx_csr_solve_async(dfx_handle* h, dfx_csr* c, int32_t chunk_nodes) {
  if (!h || !c) return fail(DFX_E_ARG, "dfx_csr_solve_async: null argument");
  CK(cudaSetDevice(h->device));
  if (chunk_nodes <= 0) chunk_nodes = default_chunk(h, c->p.n_nodes);
  dfx::SolveStats s{};
  int rc = dfx::mfp_solve(c->p, c->d_cnt, c->flags, h->st(), chunk_nodes, &s, false);
  if (rc) return fail(rc, "mfp_solve failed: %s", cudaGetErrorString(cudaGetLastError()));
  return DFX_OK;
}

int dfx_csr_requirements(dfx_handle* h, dfx_csr* c, dfx_req_out* out, dfx_csr_stats* stats) {
  if (!h || !c) return fail(DFX_E_ARG, "dfx_csr_requirements: null argument");
  CK(cudaSetDevice(h->device));
  cudaStream_t st = h->st();
  const dfx::CsrDev& p = c->p;
  const int ow = 2 * ((p.words + 31) / 32);
  if (!c->d_occ) {
    CK(cudaMalloc(&c->d_occ, sizeof(uint32_t) * (size_t)p.n_nodes * ow));
  }
  int64_t want = (out && out->masks) ? out->cap : 0;
  if (want > c->masks_cap) {
    if (c->d_masks) cudaFree(c->d_masks);
    c->d_masks = nullptr;
    CK(cudaMalloc(&c->d_masks, sizeof(uint32_t) * (size_t)want));
    c->masks_cap = want;
  }
  int64_t n_out = 0;
  CK(cudaEventRecord(c->e0, st));
  int rc = dfx::requirements(p, c->counts, c->offsets, c->scratch, c->scratch_bytes, c->d_occ,
                             want ? c->d_masks : nullptr, want, &n_out, st);
  if (rc) return fail(rc, "requirements failed: %s", cudaGetErrorString(cudaGetLastError()));
  CK(cudaEventRecord(c->e1, st));
  CK(cudaStreamSynchronize(st));   // n_out is on the host now
  if (out) {
    out->n_masks = n_out;
    out->occ_words = ow;
    if (want && n_out) {
      size_t ncopy = (size_t)(n_out < want ? n_out : want);
      CK(cudaMemcpyAsync(out->masks, c->d_masks, sizeof(uint32_t) * ncopy, cudaMemcpyDeviceToHost, st));
    }
    if (want && out->occ)
      CK(cudaMemcpyAsync(out->occ, c->d_occ, sizeof(uint32_t) * (size_t)p.n_nodes * ow, cudaMemcpyDeviceToHost, st));
    if (want && out->row_off)
      CK(cudaMemcpyAsync(out->row_off, c->offsets, sizeof(int64_t) * (size_t)(p.n_nodes + 1), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
  }
  if (stats) {
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, c->e0, c->e1));
    stats->req_ms = ms;
    stats->n_masks = n_out;
  }
  if (want && n_out > want) return fail(DFX_E_NOSPC, "mask capacity %lld < %lld", (long long)want, (long long)n_out);
  return DFX_OK;
}

int dfx_csr_download(dfx_handle* h, dfx_csr* c, uint32_t* out_h, uint32_t* out_d, uint32_t* req) {
  if (!h || !c) return fail(DFX_E_ARG, "dfx_csr_download: null argument");
  CK(cudaSetDevice(h->device));
  const size_t plane = sizeof(uint32_t) * (size_t)c->p.n_nodes * c->p.words;
  cudaStream_t st = h->st();
  if (out_h) CK(cudaMemcpyAsync(out_h, c->p.OH, plane, cudaMemcpyDeviceToHost, st));
  if (out_d) CK(cudaMemcpyAsync(out_d, c->p.OD, plane, cudaMemcpyDeviceToHost, st));
  if (req) CK(cudaMemcpyAsync(req, c->p.REQ, plane, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  return DFX_OK;
}

int dfx_csr_export(dfx_handle* h, dfx_csr* c, int32_t* row_ptr, int32_t* col, uint8_t* kind,
                   uint32_t* R, uint32_t* W) {
  if (!h || !c) return fail(DFX_E_ARG, "dfx_csr_export: null argument");
  CK(cudaSetDevice(h->device));
  const dfx::CsrDev& p = c->p;
  const size_t plane = sizeof(uint32_t) * (size_t)p.n_nodes * p.words;
  cudaStream_t st = h->st();
  if (row_ptr) CK(cudaMemcpyAsync(row_ptr, p.row_ptr, sizeof(int32_t) * (p.n_nodes + 1), cudaMemcpyDeviceToHost, st));
  if (col && p.nnz) CK(cudaMemcpyAsync(col, p.col, sizeof(int32_t) * p.nnz, cudaMemcpyDeviceToHost, st));
  if (kind) CK(cudaMemcpyAsync(kind, p.kind, p.n_nodes, cudaMemcpyDeviceToHost, st));
  if (R) CK(cudaMemcpyAsync(R, p.USE, plane, cudaMemcpyDeviceToHost, st));
  if (W) CK(cudaMemcpyAsync(W, p.B, plane, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  return DFX_OK;
}

int64_t dfx_csr_nnz(dfx_csr* c) { return c ? c->p.nnz : -1; }

int dfx_mfp_csr(dfx_handle* h, const dfx_csr_in* in, dfx_req_out* out, dfx_csr_stats* stats) {
  if (!h || !in) return fail(DFX_E_ARG, "dfx_mfp_csr: null argument");
  CK(cudaSetDevice(h->device));
  {
    int vr = check_words(in->n_nodes, in->words);
    if (!vr) vr = check_nnz(in->nnz);
    if (vr) return vr;
  }
  // device buffers persist in the handle across calls of the same shape
  dfx_csr* c = h->csr_cache;
  if (c && (c->p.n_nodes != in->n_nodes || c->p.words != in->words || c->p.nnz != in->nnz ||
            !same_scalars(c, in->S, in->words))) {
    csr_destroy_impl(c);
    c = h->csr_cache = nullptr;
  }
  int rc;
  if (!c) {
    rc = dfx_csr_create(h, in, &c);
    if (rc) return rc;
    h->csr_cache = c;
  } else {
    rc = csr_upload(c, in, h->st());
    if (rc) return rc;
  }
  rc = dfx_csr_solve(h, c, 0, stats);
  if (!rc) rc = dfx_csr_requirements(h, c, out, stats);
  return rc;
}

// ---------------------------------------------------------------------------
// list forms (csrc/acc.cu): access lists in, requirement lists out
// ---------------------------------------------------------------------------
}  // extern "C"

namespace {
int check_acc_in(const dfx_acc_in* in) {
  if (!in->row_ptr || !in->node_kind || !in->acc_off || !in->S || (in->nnz && !in->col) ||
      (in->n_acc && !in->acc))
    return fail(DFX_E_ARG, "dfx_acc_in: null array");
  int rc = check_nnz(in->nnz);
  if (rc) return rc;
  if (in->n_acc < 0 || in->acc_off[0] != 0 || in->acc_off[in->n_nodes] != in->n_acc)
    return fail(DFX_E_ARG, "dfx_acc_in: acc_off must run from 0 to n_acc");
  return check_words(in->n_nodes, in->words);
}

// H2D of CSR + access lists into already-allocated buffers, then expand the
// lists into the A/B/USE planes and build the node descriptors.  The access
// lists go up in node ranges on the copy stream, each range expanded on the
// compute stream as soon as it lands; descriptors and the successor CSR are
// built meanwhile.  The validation flag is read back by check_bad().
int csr_upload_acc(dfx_handle* h, dfx_csr* c, const dfx_acc_in* in, cudaStream_t st) {
  dfx::CsrDev& p = c->p;
  int rc0;
  auto* d_off = (int64_t*)dbuf(h, "acc_off", sizeof(int64_t) * (size_t)(in->n_nodes + 1));
  auto* d_acc = (uint16_t*)dbuf(h, "acc", sizeof(uint16_t) * (size_t)(in->n_acc > 0 ? in->n_acc : 1));
  if (!d_off || !d_acc) return fail(DFX_E_CUDA, "access-list buffers: allocation failed");
  CK(h->pipeline_init());
  CK(cudaMemcpyAsync(p.row_ptr, in->row_ptr, sizeof(int32_t) * (in->n_nodes + 1), cudaMemcpyHostToDevice, st));
  if (in->nnz) CK(cudaMemcpyAsync(p.col, in->col, sizeof(int32_t) * in->nnz, cudaMemcpyHostToDevice, st));
  rc0 = validate_csr(c, st);
  if (rc0) return rc0;
  CK(cudaMemcpyAsync(p.kind, in->node_kind, in->n_nodes, cudaMemcpyHostToDevice, st));
  CK(cudaMemsetAsync(c->d_bad, 0, sizeof(int), st));
  CK(cudaEventRecord(h->pev[0], st));
  int rc = dfx::build_desc(p, st);
  if (!rc) rc = dfx::build_succ(p, c->scratch, c->scratch_bytes, c->counts, st);
  if (rc) return fail(rc, "build_desc/build_succ launch failed");
  CK(cudaStreamWaitEvent(h->s_copy, h->pev[0], 0));   // buffers free of the previous call
  const int K = in->n_nodes >= 4096 ? dfx_handle::kPipe : 1;
  for (int k = 0; k < K; k++) {
    const int64_t lo = in->n_nodes * k / K, hi = in->n_nodes * (k + 1) / K;
    const int64_t a = in->acc_off[lo], b = in->acc_off[hi];
    CK(cudaMemcpyAsync(d_off + lo, in->acc_off + lo, sizeof(int64_t) * (size_t)(hi - lo + 1),
                       cudaMemcpyHostToDevice, h->s_copy));
    if (b > a) CK(cudaMemcpyAsync(d_acc + a, in->acc + a, sizeof(uint16_t) * (size_t)(b - a),
                                  cudaMemcpyHostToDevice, h->s_copy));
    CK(cudaEventRecord(h->pev[1 + k], h->s_copy));
    CK(cudaStreamWaitEvent(st, h->pev[1 + k], 0));
    rc = dfx::expand_acc(p, d_off, d_acc, c->d_bad, lo, hi, st);
    if (rc) return fail(rc, "expand_acc launch failed");
  }
  return DFX_OK;
}

int check_acc8_in(const dfx_acc8_in* in) {
  if (!in->row_ptr || !in->node_kind || !in->byte_off || !in->S || (in->nnz && !in->col) ||
      (in->n_bytes && !in->bytes))
    return fail(DFX_E_ARG, "dfx_acc8_in: null array");
  int rc = check_nnz(in->nnz);
  if (rc) return rc;
  if (in->n_bytes < 0 || in->n_bytes > 0x7FFFFFFF || in->byte_off[0] != 0 ||
      in->byte_off[in->n_nodes] != in->n_bytes)
    return fail(DFX_E_ARG, "dfx_acc8_in: byte_off must run from 0 to n_bytes (< 2^31)");
  return check_words(in->n_nodes, in->words);
}

// csr_upload_acc for byte-coded lists: CSR first (validated), then the lists
// in node ranges on the copy stream, each range decoded into the planes on
// the compute stream as it lands.
int csr_upload_acc8(dfx_handle* h, dfx_csr* c, const dfx_acc8_in* in, cudaStream_t st) {
  dfx::CsrDev& p = c->p;
  auto* d_off = (int32_t*)dbuf(h, "b8_off", sizeof(int32_t) * (size_t)(in->n_nodes + 1));
  auto* d_bytes = (uint8_t*)dbuf(h, "b8_in", (size_t)(in->n_bytes > 0 ? in->n_bytes : 1));
  if (!d_off || !d_bytes) return fail(DFX_E_CUDA, "byte-list buffers: allocation failed");
  CK(h->pipeline_init());
  CK(cudaMemcpyAsync(p.row_ptr, in->row_ptr, sizeof(int32_t) * (in->n_nodes + 1), cudaMemcpyHostToDevice, st));
  if (in->nnz) CK(cudaMemcpyAsync(p.col, in->col, sizeof(int32_t) * in->nnz, cudaMemcpyHostToDevice, st));
  int rc = validate_csr(c, st);
  if (rc) return rc;
  CK(cudaMemcpyAsync(p.kind, in->node_kind, in->n_nodes, cudaMemcpyHostToDevice, st));
  CK(cudaMemsetAsync(c->d_bad, 0, sizeof(int), st));
  CK(cudaEventRecord(h->pev[0], st));
  rc = dfx::build_desc(p, st);
  if (!rc) rc = dfx::build_succ(p, c->scratch, c->scratch_bytes, c->counts, st);
  if (rc) return fail(rc, "build_desc/build_succ launch failed");
  CK(cudaStreamWaitEvent(h->s_copy, h->pev[0], 0));   // buffers free of the previous call
  const int K = in->n_nodes >= 4096 ? dfx_handle::kPipe : 1;
  for (int k = 0; k < K; k++) {
    const int64_t lo = in->n_nodes * k / K, hi = in->n_nodes * (k + 1) / K;
    const int64_t a = in->byte_off[lo], b = in->byte_off[hi];
    CK(cudaMemcpyAsync(d_off + lo, in->byte_off + lo, sizeof(int32_t) * (size_t)(hi - lo + 1),
                       cudaMemcpyHostToDevice, h->s_copy));
    if (b > a) CK(cudaMemcpyAsync(d_bytes + a, in->bytes + a, (size_t)(b - a), cudaMemcpyHostToDevice,
                                  h->s_copy));
    CK(cudaEventRecord(h->pev[1 + k], h->s_copy));
    CK(cudaStreamWaitEvent(st, h->pev[1 + k], 0));
    rc = dfx::expand_b8(p, d_off, d_bytes, c->d_bad, lo, hi, st);
    if (rc) return fail(rc, "expand_b8 launch failed");
  }
  return DFX_OK;
}

__global__ void offsets_i32_kernel(const int64_t* in, int32_t* out, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (int32_t)in[i];
}

// dfx_csr_requirements_list for byte-coded lists: kernel (b), byte counts,
// scan and encoding per node range, each range's bytes going home on the D2H
// stream while the next range is computed.
int requirements_b8(dfx_handle* h, dfx_csr* c, dfx_req8_list* out, dfx_csr_stats* stats) {
  CK(h->pipeline_init());
  cudaStream_t st = h->st();
  const dfx::CsrDev& p = c->p;
  const int64_t want = out->bytes ? out->cap : 0;
  if (want > c->b8_cap) {
    if (c->d_b8) cudaFree(c->d_b8);
    c->d_b8 = nullptr;
    c->b8_cap = 0;
    CK(cudaMalloc(&c->d_b8, (size_t)want));
    c->b8_cap = want;
  }
  auto* d_off32 = (int32_t*)dbuf(h, "b8_out_off", sizeof(int32_t) * (size_t)(p.n_nodes + 1));
  if (!d_off32) return fail(DFX_E_CUDA, "byte-list offsets: allocation failed");
  const int K = p.n_nodes >= 4096 && want ? dfx_handle::kPipe : 1;
  CK(cudaMemsetAsync(c->offsets, 0, sizeof(int64_t), st));
  CK(cudaEventRecord(c->e0, st));
  for (int k = 0; k < K; k++) {
    const int lo = (int)(p.n_nodes * k / K), hi = (int)(p.n_nodes * (k + 1) / K);
    int rc = dfx::requirements_range(p, c->counts, c->offsets, c->scratch, c->scratch_bytes, lo, hi,
                                     st, true);
    if (!rc && want) rc = dfx::compact_b8(p, c->offsets, c->d_b8, want, lo, hi, st);
    if (rc) return fail(rc, "requirements failed: %s", cudaGetErrorString(cudaGetLastError()));
    CK(cudaMemcpyAsync(h->pin_cnt + k, c->offsets + hi, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    CK(cudaEventRecord(h->pev[1 + dfx_handle::kPipeMax + k], st));
  }
  offsets_i32_kernel<<<148 * 4, 256, 0, st>>>(c->offsets, d_off32, p.n_nodes + 1);
  CK(cudaGetLastError());
  CK(cudaEventRecord(c->e1, st));
  int64_t done = 0;
  for (int k = 0; k < K; k++) {
    CK(cudaEventSynchronize(h->pev[1 + dfx_handle::kPipeMax + k]));
    int64_t end = (int64_t)h->pin_cnt[k];
    if (end > want) end = want;
    if (want && end > done)
      CK(cudaMemcpyAsync(out->bytes + done, c->d_b8 + done, (size_t)(end - done),
                         cudaMemcpyDeviceToHost, h->s_d2h));
    if (end > done) done = end;
  }
  const int64_t n_out = (int64_t)h->pin_cnt[K - 1];
  if (n_out > 0x7FFFFFFF) return fail(DFX_E_LIMIT, "byte-coded requirement lists exceed 2^31 bytes");
  if (out->row_off) {
    CK(cudaEventSynchronize(c->e1));
    CK(cudaMemcpyAsync(out->row_off, d_off32, sizeof(int32_t) * (size_t)(p.n_nodes + 1),
                       cudaMemcpyDeviceToHost, h->s_d2h));
  }
  CK(cudaStreamSynchronize(h->s_d2h));
  out->n_out = n_out;
  if (stats) {
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, c->e0, c->e1));
    stats->req_ms = ms;
    stats->n_masks = n_out;
  }
  if (want && n_out > want)
    return fail(DFX_E_NOSPC, "byte-list capacity %lld < %lld", (long long)want, (long long)n_out);
  return DFX_OK;
}

int check_bad(dfx_csr* c, const dfx_acc_in* in, cudaStream_t st) {
  int bad = 0;
  CK(cudaMemcpyAsync(&bad, c->d_bad, sizeof(int), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (bad) return fail(DFX_E_ARG, "access list: variable >= %d or kind 0", 32 * in->words);
  return DFX_OK;
}
}  // namespace

extern "C" {

int dfx_csr_create_acc(dfx_handle* h, const dfx_acc_in* in, dfx_csr** out) {
  if (!h || !in || !out) return fail(DFX_E_ARG, "dfx_csr_create_acc: null argument");
  CK(cudaSetDevice(h->device));
  int rc = check_acc_in(in);
  if (rc) return rc;
  auto* c = new dfx_csr();
  rc = csr_alloc_all(c, in->n_nodes, in->words, in->nnz, in->S);
  if (!rc) rc = csr_upload_acc(h, c, in, h->st());
  if (!rc) rc = check_bad(c, in, h->st());
  if (rc) { csr_destroy_impl(c); return rc; }
  *out = c;
  return DFX_OK;
}

int dfx_csr_requirements_list(dfx_handle* h, dfx_csr* c, dfx_req_list* out, dfx_csr_stats* stats) {
  if (!h || !c) return fail(DFX_E_ARG, "dfx_csr_requirements_list: null argument");
  CK(cudaSetDevice(h->device));
  CK(h->pipeline_init());
  cudaStream_t st = h->st();
  const dfx::CsrDev& p = c->p;
  const int64_t want = (out && out->vars) ? out->cap : 0;
  if (want > c->vars_cap) {
    if (c->d_vars) cudaFree(c->d_vars);
    c->d_vars = nullptr;
    c->vars_cap = 0;
    CK(cudaMalloc(&c->d_vars, sizeof(uint16_t) * (size_t)want));
    c->vars_cap = want;
  }
  // Pipeline over node ranges: kernel (b), the scan and the list compaction
  // of range k+1 run while range k's lists go back on the D2H stream.
  const int K = p.n_nodes >= 4096 && want ? dfx_handle::kPipe : 1;
  CK(cudaMemsetAsync(c->offsets, 0, sizeof(int64_t), st));
  CK(cudaEventRecord(c->e0, st));
  for (int k = 0; k < K; k++) {
    const int lo = (int)(p.n_nodes * k / K), hi = (int)(p.n_nodes * (k + 1) / K);
    int rc = dfx::requirements_range(p, c->counts, c->offsets, c->scratch, c->scratch_bytes, lo, hi, st);
    if (!rc && want) rc = dfx::compact_list(p, c->offsets, c->d_vars, want, lo, hi, st);
    if (rc) return fail(rc, "requirements failed: %s", cudaGetErrorString(cudaGetLastError()));
    CK(cudaMemcpyAsync(h->pin_cnt + k, c->offsets + hi, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    CK(cudaEventRecord(h->pev[1 + dfx_handle::kPipeMax + k], st));
  }
  CK(cudaEventRecord(c->e1, st));
  int64_t done = 0;
  for (int k = 0; k < K; k++) {
    CK(cudaEventSynchronize(h->pev[1 + dfx_handle::kPipeMax + k]));
    int64_t end = (int64_t)h->pin_cnt[k];
    if (end > want) end = want;
    if (want && end > done)
      CK(cudaMemcpyAsync(out->vars + done, c->d_vars + done, sizeof(uint16_t) * (size_t)(end - done),
                         cudaMemcpyDeviceToHost, h->s_d2h));
    if (end > done) done = end;
  }
  const int64_t n_out = (int64_t)h->pin_cnt[K - 1];
  if (out && out->row_off)
    CK(cudaMemcpyAsync(out->row_off, c->offsets, sizeof(int64_t) * (size_t)(p.n_nodes + 1),
                       cudaMemcpyDeviceToHost, h->s_d2h));
  CK(cudaStreamSynchronize(h->s_d2h));
  if (out) out->n_out = n_out;
  if (stats) {
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, c->e0, c->e1));
    stats->req_ms = ms;
    stats->n_masks = n_out;
  }
  if (want && n_out > want)
    return fail(DFX_E_NOSPC, "requirement-list capacity %lld < %lld", (long long)want, (long long)n_out);
  return DFX_OK;
}

int dfx_csr_export_acc(dfx_handle* h, dfx_csr* c, int64_t* acc_off, uint16_t* acc, int64_t cap,
                       int64_t* n_acc) {
  if (!h || !c || !n_acc) return fail(DFX_E_ARG, "dfx_csr_export_acc: null argument");
  CK(cudaSetDevice(h->device));
  cudaStream_t st = h->st();
  const dfx::CsrDev& p = c->p;
  int rc = dfx::count_acc(p, c->counts, st);
  int64_t n = 0;
  if (!rc) rc = dfx::scan_counts(p.n_nodes, c->counts, c->offsets, c->scratch, c->scratch_bytes, &n, st);
  if (rc) return fail(rc, "export_acc: count/scan failed");
  CK(cudaStreamSynchronize(st));
  *n_acc = n;
  if (acc_off)
    CK(cudaMemcpyAsync(acc_off, c->offsets, sizeof(int64_t) * (size_t)(p.n_nodes + 1),
                       cudaMemcpyDeviceToHost, st));
  if (acc) {
    if (cap < n) return fail(DFX_E_NOSPC, "access-list capacity %lld < %lld", (long long)cap, (long long)n);
    auto* d_acc = (uint16_t*)dbuf(h, "acc_export", sizeof(uint16_t) * (size_t)(n > 0 ? n : 1));
    if (!d_acc) return fail(DFX_E_CUDA, "export_acc: allocation failed");
    rc = dfx::export_acc(p, c->offsets, d_acc, st);
    if (rc) return fail(rc, "export_acc launch failed");
    if (n) CK(cudaMemcpyAsync(acc, d_acc, sizeof(uint16_t) * (size_t)n, cudaMemcpyDeviceToHost, st));
  }
  CK(cudaStreamSynchronize(st));
  return DFX_OK;
}

int dfx_mfp_acc(dfx_handle* h, const dfx_acc_in* in, dfx_req_list* out, dfx_csr_stats* stats) {
  if (!h || !in) return fail(DFX_E_ARG, "dfx_mfp_acc: null argument");
  CK(cudaSetDevice(h->device));
  int rc = check_acc_in(in);
  if (rc) return rc;
  // device buffers persist in the handle across calls of the same shape
  dfx_csr* c = h->csr_cache;
  if (c && (c->p.n_nodes != in->n_nodes || c->p.words != in->words || c->p.nnz != in->nnz ||
            !same_scalars(c, in->S, in->words))) {
    csr_destroy_impl(c);
    c = h->csr_cache = nullptr;
  }
  if (!c) {
    c = new dfx_csr();
    rc = csr_alloc_all(c, in->n_nodes, in->words, in->nnz, in->S);
    if (rc) { csr_destroy_impl(c); return rc; }
    h->csr_cache = c;
  }
  rc = csr_upload_acc(h, c, in, h->st());
  if (!rc) rc = dfx_csr_solve(h, c, 0, stats);    // synchronises: the flag is final
  if (!rc) rc = check_bad(c, in, h->st());
  if (!rc) rc = dfx_csr_requirements_list(h, c, out, stats);
  return rc;
}

int dfx_mfp_acc8(dfx_handle* h, const dfx_acc8_in* in, dfx_req8_list* out, dfx_csr_stats* stats) {
  if (!h || !in || !out) return fail(DFX_E_ARG, "dfx_mfp_acc8: null argument");
  CK(cudaSetDevice(h->device));
  int rc = check_acc8_in(in);
  if (rc) return rc;
  dfx_csr* c = h->csr_cache;
  if (c && (c->p.n_nodes != in->n_nodes || c->p.words != in->words || c->p.nnz != in->nnz ||
            !same_scalars(c, in->S, in->words))) {
    csr_destroy_impl(c);
    c = h->csr_cache = nullptr;
  }
  if (!c) {
    c = new dfx_csr();
    rc = csr_alloc_all(c, in->n_nodes, in->words, in->nnz, in->S);
    if (rc) { csr_destroy_impl(c); return rc; }
    h->csr_cache = c;
  }
  auto now = [] { return std::chrono::steady_clock::now(); };
  const auto t0 = now();
  rc = csr_upload_acc8(h, c, in, h->st());
  if (h->trace) CK(cudaStreamSynchronize(h->st()));
  const auto t1 = now();
  if (!rc) rc = dfx_csr_solve(h, c, 0, stats);    // synchronises: the flag is final
  const auto t2 = now();
  if (!rc) {
    int bad = 0;
    CK(cudaMemcpy(&bad, c->d_bad, sizeof(int), cudaMemcpyDeviceToHost));
    if (bad) rc = fail(DFX_E_ARG, "byte-coded access list: variable >= %d, kind 0 or an "
                                  "unterminated entry", 32 * in->words);
  }
  if (!rc) rc = requirements_b8(h, c, out, stats);
  if (h->trace) {
    const auto t3 = now();
    auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
    fprintf(stderr, "[dfx_mfp_acc8] upload+expand %.3f ms, solve %.3f ms, requirements+D2H %.3f ms\n",
            ms(t0, t1), ms(t1, t2), ms(t2, t3));
  }
  return rc;
}

// ---------------------------------------------------------------------------
// kernel (c): interprocedural summaries
// ---------------------------------------------------------------------------
}  // extern "C"

struct dfx_cg {
  dfx::CgDev g{};
  std::vector<int32_t> wave_off;
  std::vector<void*> allocs;
  int* d_changed = nullptr;
};

namespace {
int cg_destroy_impl(dfx_cg* c) {
  if (!c) return DFX_OK;
  for (void* p : c->allocs) cudaFree(p);
  delete c;
  return DFX_OK;
}
void* cg_alloc(dfx_cg* c, size_t bytes) {
  void* p = nullptr;
  if (cudaMalloc(&p, bytes + 16) != cudaSuccess) return nullptr;
  c->allocs.push_back(p);
  return p;
}
// pad [rows][ns] (elem bytes each) to [rows][nsp]
template <class T>
std::vector<T> pad_rows(const T* src, int rows, int ns, int nsp) {
  std::vector<T> out((size_t)rows * nsp, T(0));
  for (int r = 0; r < rows; r++) std::memcpy(&out[(size_t)r * nsp], src + (size_t)r * ns, sizeof(T) * ns);
  return out;
}
}  // namespace

extern "C" {

int dfx_cg_create(dfx_handle* h, const dfx_cg_in* in, dfx_cg** out) {
  if (!h || !in || !out) return fail(DFX_E_ARG, "dfx_cg_create: null argument");
  CK(cudaSetDevice(h->device));
  cudaStream_t st = h->st();
  const int nf = in->n_funcs, ns = in->n_slots;
  const int nsp = ((ns + 31) / 32) * 32;
  auto* c = new dfx_cg();
  dfx::CgDev& g = c->g;
  g.n_funcs = nf; g.n_slots = ns; g.nsp = nsp; g.n_params = in->n_params; g.n_waves = in->n_waves;
  g.many = in->src_off && dfx::cg_many_sources(in->src_off, nf);
  auto up = [&](const void* src, size_t bytes) -> void* {
    void* p = cg_alloc(c, bytes);
    if (p && bytes && src) cudaMemcpyAsync(p, src, bytes, cudaMemcpyHostToDevice, st);
    return p;
  };
  auto direct = pad_rows(in->direct, nf, ns, nsp);
  g.direct = (const uint8_t*)up(direct.data(), direct.size());
  g.src_off = (const int32_t*)up(in->src_off, sizeof(int32_t) * (nf + 1));
  g.src = (const int32_t*)up(in->src, sizeof(int32_t) * 4 * in->n_src);
  g.slist = (const int16_t*)up(in->slist, sizeof(int16_t) * in->n_slist);
  g.bind = (const int32_t*)up(in->bind, sizeof(int32_t) * 2 * in->n_bind);
  g.wave_fns = (const int32_t*)up(in->wave_fns, sizeof(int32_t) * nf);
  c->wave_off.assign(in->wave_off, in->wave_off + in->n_waves + 1);
  g.h_wave_off = c->wave_off.data();
  c->d_changed = (int*)cg_alloc(c, sizeof(int));
  for (void* p : c->allocs)
    if (!p) { cg_destroy_impl(c); return fail(DFX_E_CUDA, "dfx_cg_create: allocation failed"); }
  if (c->allocs.size() != 7) { cg_destroy_impl(c); return fail(DFX_E_CUDA, "dfx_cg_create: allocation failed"); }
  CK(cudaStreamSynchronize(st));
  *out = c;
  return DFX_OK;
}

int dfx_cg_destroy(dfx_handle* h, dfx_cg* c) {
  if (h) cudaSetDevice(h->device);
  return cg_destroy_impl(c);
}

int32_t dfx_cg_nsp(dfx_cg* c) { return c ? c->g.nsp : -1; }

int dfx_cg_wave(dfx_handle* h, dfx_cg* c, const dfx_cg_tables* prev, dfx_cg_tables* cur,
                int32_t wave, int32_t shard, int32_t nshards, int32_t* changed) {
  if (!h || !c || !prev || !cur) return fail(DFX_E_ARG, "dfx_cg_wave: null argument");
  if (wave < 0 || wave >= c->g.n_waves || nshards < 1 || shard < 0 || shard >= nshards)
    return fail(DFX_E_ARG, "dfx_cg_wave: bad wave/shard");
  CK(cudaSetDevice(h->device));
  cudaStream_t st = h->st();
  CK(cudaMemsetAsync(c->d_changed, 0, sizeof(int), st));
  int rc = dfx::cg_wave(c->g, prev->bits, prev->list, prev->len, cur->bits, cur->list, cur->len,
                        wave, shard, nshards, c->d_changed, st);
  if (rc) return fail(rc, "cg_wave failed: %s", cudaGetErrorString(cudaGetLastError()));
  if (changed) {
    CK(cudaMemcpyAsync(changed, c->d_changed, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
  }
  return DFX_OK;
}

// ---------------------------------------------------------------------------
// fused multi-GPU kernel (c) over peer memory (dfx_cgp_*)
// ---------------------------------------------------------------------------
}  // extern "C"

struct dfx_cgp {
  dfx_cg* cg = nullptr;                 // static arrays (direct, sources, bindings, waves)
  std::vector<int32_t> wave_off;
  int nranks = 1, rank = 0, maxp = 1, nf = 0, ns = 0, nsp = 32;
  void* block = nullptr;                // this rank's exchange block
  size_t off_bits[2], off_list[2], off_len[2], off_arrive = 0, off_changed = 0, bytes = 0;
  void* base[dfx::kMaxPeers] = {};      // every rank's block (peers opened by IPC)
  bool opened[dfx::kMaxPeers] = {};
  dfx::PeerTables tab{};
  unsigned int* blocks_done = nullptr;
  int* err = nullptr;
  unsigned long long steps = 0;         // waves completed over all solves
  int gen = 0;                          // solves started
  const dfx_cg_in* in = nullptr;        // host inputs (init tables), kept by the caller
};

namespace {
int cgp_destroy_impl(dfx_cgp* p) {
  if (!p) return DFX_OK;
  for (int r = 0; r < p->nranks && r < dfx::kMaxPeers; r++)
    if (p->opened[r]) cudaIpcCloseMemHandle(p->base[r]);
  if (p->block) cudaFree(p->block);
  if (p->blocks_done) cudaFree(p->blocks_done);
  if (p->err) cudaFree(p->err);
  if (p->cg) cg_destroy_impl(p->cg);
  delete p;
  return DFX_OK;
}
size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }
}  // namespace

extern "C" {

int dfx_cgp_create(dfx_handle* h, const dfx_cg_in* in, int32_t nranks, int32_t rank, dfx_cgp** out) {
  if (!h || !in || !out) return fail(DFX_E_ARG, "dfx_cgp_create: null argument");
  if (nranks < 1 || nranks > dfx::kMaxPeers || rank < 0 || rank >= nranks)
    return fail(DFX_E_ARG, "dfx_cgp_create: rank %d of %d (at most %d ranks)", rank, nranks, dfx::kMaxPeers);
  CK(cudaSetDevice(h->device));
  auto* p = new dfx_cgp();
  int rc = dfx_cg_create(h, in, &p->cg);
  if (rc) { delete p; return rc; }
  p->nranks = nranks; p->rank = rank; p->in = in;
  p->nf = in->n_funcs; p->ns = in->n_slots; p->nsp = p->cg->g.nsp;
  p->maxp = in->max_passes > 0 ? in->max_passes : 1;
  p->wave_off.assign(in->wave_off, in->wave_off + in->n_waves + 1);
  p->cg->g.h_wave_off = p->wave_off.data();
  const size_t rows = (size_t)(p->nf > 0 ? p->nf : 1);
  size_t o = 0;
  for (int k = 0; k < 2; k++) {
    p->off_bits[k] = o; o = align256(o + rows * p->nsp);
    p->off_list[k] = o; o = align256(o + 2 * rows * p->nsp);
    p->off_len[k] = o; o = align256(o + 4 * rows);
  }
  p->off_arrive = o; o = align256(o + sizeof(unsigned long long));
  p->off_changed = o; o = align256(o + sizeof(int) * (size_t)(p->maxp + 2));
  p->bytes = o;
  if (cudaMalloc(&p->block, p->bytes) != cudaSuccess || cudaMalloc(&p->blocks_done, 64) != cudaSuccess ||
      cudaMalloc(&p->err, 64) != cudaSuccess) {
    cgp_destroy_impl(p);
    return fail(DFX_E_CUDA, "dfx_cgp_create: allocation failed");
  }
  // counters and flags start at zero and are never cleared afterwards
  CK(cudaMemset(p->block, 0, p->bytes));
  CK(cudaMemset(p->err, 0, 64));
  CK(cudaDeviceSynchronize());
  *out = p;
  return DFX_OK;
}

int dfx_cgp_handle(dfx_cgp* p, void* ipc_handle) {
  if (!p || !ipc_handle) return fail(DFX_E_ARG, "dfx_cgp_handle: null argument");
  cudaIpcMemHandle_t hd;
  CK(cudaIpcGetMemHandle(&hd, p->block));
  static_assert(sizeof(hd) == DFX_IPC_HANDLE_BYTES, "IPC handle size");
  std::memcpy(ipc_handle, &hd, sizeof hd);
  return DFX_OK;
}

int dfx_cgp_connect(dfx_handle* h, dfx_cgp* p, const void* ipc_handles) {
  if (!h || !p || !ipc_handles) return fail(DFX_E_ARG, "dfx_cgp_connect: null argument");
  CK(cudaSetDevice(h->device));
  for (int r = 0; r < p->nranks; r++) {
    if (r == p->rank) { p->base[r] = p->block; continue; }
    cudaIpcMemHandle_t hd;
    std::memcpy(&hd, (const char*)ipc_handles + (size_t)r * DFX_IPC_HANDLE_BYTES, sizeof hd);
    CK(cudaIpcOpenMemHandle(&p->base[r], hd, cudaIpcMemLazyEnablePeerAccess));
    p->opened[r] = true;
  }
  for (int r = 0; r < p->nranks; r++) {
    char* b = (char*)p->base[r];
    for (int k = 0; k < 2; k++) {
      p->tab.bits[r][k] = (uint8_t*)(b + p->off_bits[k]);
      p->tab.list[r][k] = (int16_t*)(b + p->off_list[k]);
      p->tab.len[r][k] = (int32_t*)(b + p->off_len[k]);
    }
    p->tab.arrive[r] = (unsigned long long*)(b + p->off_arrive);
    p->tab.changed[r] = (int*)(b + p->off_changed);
  }
  return DFX_OK;
}

int dfx_cgp_solve(dfx_handle* h, dfx_cgp* p, dfx_cg_out* out) {
  if (!h || !p || !out) return fail(DFX_E_ARG, "dfx_cgp_solve: null argument");
  if (!p->base[p->rank]) return fail(DFX_E_ARG, "dfx_cgp_solve: not connected");
  CK(cudaSetDevice(h->device));
  cudaStream_t st = h->st();
  const dfx_cg_in* in = p->in;
  const int nf = p->nf, ns = p->ns, nsp = p->nsp;
  const int gen = ++p->gen;
  // pass-0 tables into t0 (local; peers only write t1 during pass 1)
  auto* d_stage = (uint8_t*)dbuf(h, "cgp_stage", 2 * (size_t)(nf > 0 ? nf : 1) * nsp + 16);
  if (!d_stage) return fail(DFX_E_CUDA, "dfx_cgp_solve: allocation failed");
  if (nf && ns) {
    const size_t nb = (size_t)nf * ns;
    int rc0 = 0;
    CK(cudaMemcpyAsync(d_stage, in->init_bits, nb, cudaMemcpyHostToDevice, st));
    rc0 |= dfx::repitch(d_stage, ns, p->tab.bits[p->rank][0], nsp, ns, nf, st);
    CK(cudaMemcpyAsync(d_stage, in->init_list, 2 * nb, cudaMemcpyHostToDevice, st));
    rc0 |= dfx::repitch(d_stage, 2 * (size_t)ns, p->tab.list[p->rank][0], 2 * (size_t)nsp, 2 * (size_t)ns, nf, st);
    if (rc0) return fail(DFX_E_CUDA, "dfx_cgp_solve: repitch failed");
  }
  if (nf) CK(cudaMemcpyAsync(p->tab.len[p->rank][0], in->init_len, sizeof(int32_t) * nf, cudaMemcpyHostToDevice, st));
  const int n_waves = (int)p->wave_off.size() - 1;
  const long long spins = 20000000;       // ~4 s of polling before a peer is declared lost
  int passes = 0, launches = 0;
  CK(cudaEventRecord(h->ev0, st));
  for (int pass = 1; pass <= p->maxp; pass++) {
    passes = pass;
    const int cur = pass & 1;              // pass 1 reads t0, writes t1
    for (int w = 0; w < n_waves; w++) {
      int rc = dfx::cg_peer_wave(p->cg->g, p->tab, cur, w, p->rank, p->nranks, pass, gen,
                                 p->blocks_done, st);
      p->steps++;
      if (!rc) rc = dfx::cg_peer_wait(p->tab.arrive[p->rank], p->steps * (unsigned long long)p->nranks,
                                      spins, p->err, st);
      if (rc) return fail(rc, "cg_peer_wave failed: %s", cudaGetErrorString(cudaGetLastError()));
      launches += 2;
    }
    int flag = 0, err = 0;
    CK(cudaMemcpyAsync(&flag, p->tab.changed[p->rank] + pass, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(&err, p->err, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (err) return fail(DFX_E_CUDA, "dfx_cgp_solve: a peer did not arrive (pass %d)", pass);
    if (flag != gen) break;                // no rank changed a set in this pass
  }
  CK(cudaEventRecord(h->ev1, st));
  const int last = passes & 1;
  if (nf && ns) {
    const size_t nb = (size_t)nf * ns;
    int rc0 = dfx::repitch(p->tab.bits[p->rank][last], nsp, d_stage, ns, ns, nf, st);
    if (rc0) return fail(rc0, "dfx_cgp_solve: repitch failed");
    CK(cudaMemcpyAsync(out->bits, d_stage, nb, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    rc0 = dfx::repitch(p->tab.list[p->rank][last], 2 * (size_t)nsp, d_stage, 2 * (size_t)ns, 2 * (size_t)ns, nf, st);
    if (rc0) return fail(rc0, "dfx_cgp_solve: repitch failed");
    CK(cudaMemcpyAsync(out->list, d_stage, 2 * nb, cudaMemcpyDeviceToHost, st));
  }
  if (nf) CK(cudaMemcpyAsync(out->len, p->tab.len[p->rank][last], sizeof(int32_t) * nf, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  float ms = 0.f;
  CK(cudaEventElapsedTime(&ms, h->ev0, h->ev1));
  out->kernel_ms = ms;
  out->passes = passes;
  out->launches = launches;
  return DFX_OK;
}

int dfx_cgp_destroy(dfx_handle* h, dfx_cgp* p) {
  if (h) cudaSetDevice(h->device);
  return cgp_destroy_impl(p);
}

// replaces dartomp.interproc.summarize_all (pkg/src/dartomp/interproc.py:90-144)
}  // extern "C"

namespace {
// NCCL, loaded at run time: the process's libnccl.so.2 (torch's, when torch
// has loaded one) or the system's; no link-time dependency of libdfx.so
struct Nccl {
  bool ok = false;
  std::string why;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

const Nccl& nccl() {
  static Nccl n = [] {
    Nccl x;
    void* lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!lib) lib = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!lib) { x.why = dlerror() ? dlerror() : "libnccl.so.2 not found"; return x; }
    auto sym = [&](const char* name) { return dlsym(lib, name); };
    x.GetUniqueId = (decltype(x.GetUniqueId))sym("ncclGetUniqueId");
    x.CommInitRank = (decltype(x.CommInitRank))sym("ncclCommInitRank");
    x.CommDestroy = (decltype(x.CommDestroy))sym("ncclCommDestroy");
    x.AllReduce = (decltype(x.AllReduce))sym("ncclAllReduce");
    x.AllGather = (decltype(x.AllGather))sym("ncclAllGather");
    x.GetErrorString = (decltype(x.GetErrorString))sym("ncclGetErrorString");
    x.ok = x.GetUniqueId && x.CommInitRank && x.CommDestroy && x.AllReduce && x.AllGather &&
           x.GetErrorString;
    if (!x.ok) x.why = "libnccl.so.2 lacks a required symbol";
    return x;
  }();
  return n;
}

#define NK(expr)                                                                          \
  do {                                                                                    \
    ncclResult_t r_ = (expr);                                                             \
    if (r_ != ncclSuccess)                                                                \
      return fail(DFX_E_CUDA, "%s: %s (%s:%d)", #expr, nccl().GetErrorString(r_), __FILE__, \
                  __LINE__);                                                              \
  } while (0)

// Device state of one summaries solve (grow-only handle buffers).
struct CgRun {
  dfx::CgDev g{};
  int nf = 0, ns = 0, nsp = 0, maxp = 1;
  int32_t* d_woff = nullptr;
  int* d_flags = nullptr;
  uint8_t* tb[2] = {};
  int16_t* tl[2] = {};
  int32_t* tn[2] = {};
  uint8_t* d_stage = nullptr;
};

// Upload the graph and pass-0 tables; `wave_off`/`wave_fns` (host) are the
// schedule this rank runs (the whole graph's, or its owned functions').
int cg_setup(dfx_handle* h, const dfx_cg_in* in, const int32_t* wave_off, const int32_t* wave_fns,
             int n_waves, int n_wave_fns, CgRun& R) {
  cudaStream_t st = h->st();
  const int nf = in->n_funcs, ns = in->n_slots;
  R.nf = nf; R.ns = ns;
  R.nsp = ((ns + 31) / 32) * 32;                  // padded row (16-B quads, 32-bit seen words)
  const int nsp = R.nsp;
  R.maxp = in->max_passes > 0 ? in->max_passes : 1;
  const int maxp = R.maxp;
  const size_t rows = (size_t)(nf > 0 ? nf : 1);
  auto* d_direct = (uint8_t*)dbuf(h, "cg_direct", rows * nsp + 16);
  auto* d_srcoff = (int32_t*)dbuf(h, "cg_srcoff", sizeof(int32_t) * (rows + 1));
  auto* d_src = (int32_t*)dbuf(h, "cg_src", sizeof(int32_t) * 4 * (size_t)(in->n_src + 1));
  auto* d_slist = (int16_t*)dbuf(h, "cg_slist", sizeof(int16_t) * (size_t)(in->n_slist + 1));
  auto* d_bind = (int32_t*)dbuf(h, "cg_bind", sizeof(int32_t) * 2 * (size_t)(in->n_bind + 1));
  auto* d_wfns = (int32_t*)dbuf(h, "cg_wfns", sizeof(int32_t) * (size_t)(n_wave_fns + 1));
  R.d_woff = (int32_t*)dbuf(h, "cg_woff", sizeof(int32_t) * (size_t)(n_waves + 1));
  R.d_flags = (int*)dbuf(h, "cg_flags", sizeof(int) * (size_t)(maxp + 2));
  R.tb[0] = (uint8_t*)dbuf(h, "cg_b0", rows * nsp + 16);
  R.tb[1] = (uint8_t*)dbuf(h, "cg_b1", rows * nsp + 16);
  R.tl[0] = (int16_t*)dbuf(h, "cg_l0", sizeof(int16_t) * rows * nsp + 16);
  R.tl[1] = (int16_t*)dbuf(h, "cg_l1", sizeof(int16_t) * rows * nsp + 16);
  R.tn[0] = (int32_t*)dbuf(h, "cg_n0", sizeof(int32_t) * rows);
  R.tn[1] = (int32_t*)dbuf(h, "cg_n1", sizeof(int32_t) * rows);
  // dense rows go up contiguously into a staging buffer and are re-pitched
  // to the padded layout on the device (one DMA per array)
  R.d_stage = (uint8_t*)dbuf(h, "cg_stage", sizeof(int16_t) * rows * nsp + 16);
  if (!d_direct || !d_srcoff || !d_src || !d_slist || !d_bind || !d_wfns || !R.d_woff ||
      !R.d_flags || !R.tb[0] || !R.tb[1] || !R.tl[0] || !R.tl[1] || !R.tn[0] || !R.tn[1] ||
      !R.d_stage)
    return fail(DFX_E_CUDA, "dfx_summaries: device allocation failed");
  if (nf && ns) {
    const size_t nb = (size_t)nf * ns;
    int rc0 = 0;
    CK(cudaMemcpyAsync(R.d_stage, in->direct, nb, cudaMemcpyHostToDevice, st));
    rc0 |= dfx::repitch(R.d_stage, ns, d_direct, nsp, ns, nf, st);
    CK(cudaMemcpyAsync(R.d_stage, in->init_bits, nb, cudaMemcpyHostToDevice, st));
    rc0 |= dfx::repitch(R.d_stage, ns, R.tb[0], nsp, ns, nf, st);
    CK(cudaMemcpyAsync(R.d_stage, in->init_list, 2 * nb, cudaMemcpyHostToDevice, st));
    rc0 |= dfx::repitch(R.d_stage, 2 * (size_t)ns, R.tl[0], 2 * (size_t)nsp, 2 * (size_t)ns, nf, st);
    if (rc0) return fail(DFX_E_CUDA, "dfx_summaries: repitch failed");
  }
  if (nf) CK(cudaMemcpyAsync(R.tn[0], in->init_len, sizeof(int32_t) * nf, cudaMemcpyHostToDevice, st));
  // the solve writes a row's list only up to its length; the download reads
  // whole rows (the host keeps the first len entries), so the second table
  // starts defined (a few MB; compute-sanitizer initcheck)
  CK(cudaMemsetAsync(R.tb[1], 0, rows * nsp, st));
  CK(cudaMemsetAsync(R.tl[1], 0, sizeof(int16_t) * rows * nsp, st));
  CK(cudaMemcpyAsync(d_srcoff, in->src_off, sizeof(int32_t) * (size_t)(nf + 1), cudaMemcpyHostToDevice, st));
  if (in->n_src) CK(cudaMemcpyAsync(d_src, in->src, sizeof(int32_t) * 4 * (size_t)in->n_src, cudaMemcpyHostToDevice, st));
  if (in->n_slist) CK(cudaMemcpyAsync(d_slist, in->slist, sizeof(int16_t) * (size_t)in->n_slist, cudaMemcpyHostToDevice, st));
  if (in->n_bind) CK(cudaMemcpyAsync(d_bind, in->bind, sizeof(int32_t) * 2 * (size_t)in->n_bind, cudaMemcpyHostToDevice, st));
  if (n_wave_fns) CK(cudaMemcpyAsync(d_wfns, wave_fns, sizeof(int32_t) * n_wave_fns, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(R.d_woff, wave_off, sizeof(int32_t) * (size_t)(n_waves + 1), cudaMemcpyHostToDevice, st));
  CK(cudaMemsetAsync(R.d_flags, 0, sizeof(int) * (size_t)(maxp + 2), st));
  dfx::CgDev& g = R.g;
  g.n_funcs = nf; g.n_slots = ns; g.nsp = nsp; g.n_params = in->n_params; g.n_waves = n_waves;
  g.many = in->src_off && dfx::cg_many_sources(in->src_off, nf);
  g.direct = d_direct; g.src_off = d_srcoff; g.src = d_src; g.slist = d_slist; g.bind = d_bind;
  g.wave_fns = d_wfns;
  g.h_wave_off = wave_off;
  return DFX_OK;
}

// D2H of table `last` as dense rows (re-pitched on the device)
int cg_download(dfx_handle* h, CgRun& R, int last, dfx_cg_out* out) {
  cudaStream_t st = h->st();
  const int nf = R.nf, ns = R.ns, nsp = R.nsp;
  const size_t rows = (size_t)(nf > 0 ? nf : 1);
  if (nf && ns) {
    const size_t nb = (size_t)nf * ns;
    int rc0 = dfx::repitch(R.tb[last], nsp, R.d_stage, ns, ns, nf, st);
    if (rc0) return fail(rc0, "dfx_summaries: repitch failed");
    CK(cudaMemcpyAsync(out->bits, R.d_stage, nb, cudaMemcpyDeviceToHost, st));
    auto* d_stage2 = (uint8_t*)dbuf(h, "cg_stage2", sizeof(int16_t) * rows * nsp + 16);
    if (!d_stage2) return fail(DFX_E_CUDA, "dfx_summaries: device allocation failed");
    rc0 = dfx::repitch(R.tl[last], 2 * (size_t)nsp, d_stage2, 2 * (size_t)ns, 2 * (size_t)ns, nf, st);
    if (rc0) return fail(rc0, "dfx_summaries: repitch failed");
    CK(cudaMemcpyAsync(out->list, d_stage2, 2 * nb, cudaMemcpyDeviceToHost, st));
  }
  if (nf) CK(cudaMemcpyAsync(out->len, R.tn[last], sizeof(int32_t) * nf, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  return DFX_OK;
}
}  // namespace

extern "C" {

int dfx_summaries(dfx_handle* h, const dfx_cg_in* in, dfx_cg_out* out) {
  if (!h || !in || !out) return fail(DFX_E_ARG, "dfx_summaries: null argument");
  if (in->n_funcs < 0 || in->n_slots < 0 || in->n_waves < 0)
    return fail(DFX_E_ARG, "dfx_summaries: negative size");
  CK(cudaSetDevice(h->device));
  cudaStream_t st = h->st();
  CgRun R;
  int rc = cg_setup(h, in, in->wave_off, in->wave_fns, in->n_waves, in->n_funcs, R);
  if (rc) return rc;
  // all passes in one persistent cooperative launch (waves separated by grid
  // barriers); passes alternate tables t0 -> t1 -> t0 ...
  CK(cudaEventRecord(h->ev0, st));
  rc = dfx::cg_solve(R.g, R.tb[0], R.tl[0], R.tn[0], R.tb[1], R.tl[1], R.tn[1], R.d_woff, R.maxp,
                     R.d_flags, R.d_flags + R.maxp + 1, st);
  CK(cudaEventRecord(h->ev1, st));
  if (rc) return fail(rc, "cg_solve failed: %s", cudaGetErrorString(cudaGetLastError()));
  int passes = 0;
  CK(cudaMemcpyAsync(&passes, R.d_flags + R.maxp + 1, sizeof(int), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  rc = cg_download(h, R, passes & 1, out);       // the table the last pass wrote
  if (rc) return rc;
  float ms = 0.f;
  CK(cudaEventElapsedTime(&ms, h->ev0, h->ev1));
  out->kernel_ms = ms;
  out->passes = passes;
  out->launches = 1;
  return DFX_OK;
}

// ---------------------------------------------------------------------------
// NCCL on the handle, and kernel (c) sharded by call-graph components
// ---------------------------------------------------------------------------
int dfx_comm_unique_id(void* id_out) {
  if (!id_out) return fail(DFX_E_ARG, "dfx_comm_unique_id: null argument");
  const Nccl& n = nccl();
  if (!n.ok) return fail(DFX_E_CUDA, "NCCL unavailable: %s", n.why.c_str());
  ncclUniqueId id;
  NK(n.GetUniqueId(&id));
  std::memcpy(id_out, &id, sizeof id);
  return DFX_OK;
}

int dfx_comm_init(dfx_handle* h, const void* unique_id, int32_t nranks, int32_t rank) {
  if (!h || !unique_id) return fail(DFX_E_ARG, "dfx_comm_init: null argument");
  if (nranks < 1 || rank < 0 || rank >= nranks)
    return fail(DFX_E_ARG, "dfx_comm_init: rank %d of %d", rank, nranks);
  const Nccl& n = nccl();
  if (!n.ok) return fail(DFX_E_CUDA, "NCCL unavailable: %s", n.why.c_str());
  CK(cudaSetDevice(h->device));
  dfx_comm_destroy(h);
  ncclUniqueId id;
  std::memcpy(&id, unique_id, sizeof id);
  NK(n.CommInitRank(&h->comm, nranks, id, rank));
  h->comm_rank = rank;
  h->comm_size = nranks;
  return DFX_OK;
}

int dfx_comm_destroy(dfx_handle* h) {
  if (!h || !h->comm) return DFX_OK;
  nccl().CommDestroy(h->comm);
  h->comm = nullptr;
  h->comm_rank = 0;
  h->comm_size = 1;
  return DFX_OK;
}

// Kernel (c) across the ranks of the handle's communicator, sharded by
// call-graph component: owner[f] is the rank that rebuilds f.  The caller
// guarantees that a function and every function it calls share an owner (a
// union of connected components of the call graph), so no rank ever reads a
// row another rank produces while the passes run.  Per pass each rank runs
// its own functions' waves (the reference's order, interproc.py:105-143,
// restricted to them) in one cooperative launch, then ONE ncclAllReduce(MAX)
// of the pass's changed flag decides, on every rank alike, whether another
// pass follows -- the reference's global termination test, so every
// component runs exactly the reference's number of passes (insertion orders
// may still evolve after a component's sets settle).  After the last pass
// ONE ncclAllGather of the owned rows gives every rank every summary.
int dfx_summaries_sharded(dfx_handle* h, const dfx_cg_in* in, const int32_t* owner,
                          dfx_cg_out* out, int32_t* n_collectives) {
  if (!h || !in || !out || !owner) return fail(DFX_E_ARG, "dfx_summaries_sharded: null argument");
  if (!h->comm) return fail(DFX_E_ARG, "dfx_summaries_sharded: no communicator (dfx_comm_init)");
  if (in->n_funcs < 0 || in->n_slots < 0 || in->n_waves < 0)
    return fail(DFX_E_ARG, "dfx_summaries_sharded: negative size");
  CK(cudaSetDevice(h->device));
  cudaStream_t st = h->st();
  const Nccl& nc = nccl();
  const int nf = in->n_funcs, me = h->comm_rank, world = h->comm_size;
  for (int f = 0; f < nf; f++)
    if (owner[f] < 0 || owner[f] >= world)
      return fail(DFX_E_ARG, "dfx_summaries_sharded: owner[%d] = %d of %d ranks", f, owner[f], world);
  // this rank's schedule: its functions, wave by wave in the reference order
  std::vector<int32_t> woff(1, 0), wfns;
  for (int w = 0; w < in->n_waves; w++) {
    for (int i = in->wave_off[w]; i < in->wave_off[w + 1]; i++)
      if (owner[in->wave_fns[i]] == me) wfns.push_back(in->wave_fns[i]);
    if ((int)wfns.size() > woff.back()) woff.push_back((int32_t)wfns.size());
  }
  const int n_waves = (int)woff.size() - 1;
  CgRun R;
  int rc = cg_setup(h, in, woff.data(), wfns.data(), n_waves, (int)wfns.size(), R);
  if (rc) return rc;
  int collectives = 0;
  CK(cudaEventRecord(h->ev0, st));
  int passes = 0;
  int* d_pass = R.d_flags + R.maxp + 1;
  for (int p = 1; p <= R.maxp; p++) {
    if (n_waves > 0) {
      rc = dfx::cg_solve(R.g, R.tb[0], R.tl[0], R.tn[0], R.tb[1], R.tl[1], R.tn[1], R.d_woff, p,
                         R.d_flags, d_pass, st, p);
      if (rc) return fail(rc, "cg_solve failed: %s", cudaGetErrorString(cudaGetLastError()));
    }
    NK(nc.AllReduce(R.d_flags + p, R.d_flags + p, 1, ncclInt32, ncclMax, h->comm, st));
    collectives++;
    int changed = 0;
    CK(cudaMemcpyAsync(&changed, R.d_flags + p, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    passes = p;
    if (!changed) break;
  }
  const int last = passes & 1;
  // final exchange: every rank's owned rows to every rank
  std::vector<int32_t> cnt(world, 0);
  for (int f = 0; f < nf; f++) cnt[owner[f]]++;
  const int per = *std::max_element(cnt.begin(), cnt.end());
  if (world > 1 && per > 0) {
    const int rowb = 3 * R.nsp + 4;
    std::vector<int32_t> lists;      // rank r's functions at [r * per, r * per + cnt[r])
    lists.assign((size_t)world * per, 0);
    std::vector<int> fill(world, 0);
    for (int f = 0; f < nf; f++) lists[(size_t)owner[f] * per + fill[owner[f]]++] = f;
    auto* d_lists = (int32_t*)dbuf(h, "cg_xlists", sizeof(int32_t) * lists.size() + 16);
    auto* d_send = (uint8_t*)dbuf(h, "cg_xsend", (size_t)per * rowb + 16);
    auto* d_recv = (uint8_t*)dbuf(h, "cg_xrecv", (size_t)world * per * rowb + 16);
    if (!d_lists || !d_send || !d_recv) return fail(DFX_E_CUDA, "dfx_summaries_sharded: allocation failed");
    CK(cudaMemcpyAsync(d_lists, lists.data(), sizeof(int32_t) * lists.size(), cudaMemcpyHostToDevice, st));
    rc = dfx::cg_pack(R.tb[last], R.tl[last], R.tn[last], R.nsp, d_lists + (size_t)me * per, cnt[me],
                      d_send, rowb, false, st);
    if (rc) return fail(rc, "cg_pack failed");
    NK(nc.AllGather(d_send, d_recv, (size_t)per * rowb, ncclUint8, h->comm, st));
    collectives++;
    for (int r = 0; r < world; r++) {
      if (r == me) continue;
      rc = dfx::cg_pack(R.tb[last], R.tl[last], R.tn[last], R.nsp, d_lists + (size_t)r * per, cnt[r],
                        d_recv + (size_t)r * per * rowb, rowb, true, st);
      if (rc) return fail(rc, "cg_unpack failed");
    }
  }
  CK(cudaEventRecord(h->ev1, st));
  rc = cg_download(h, R, last, out);
  if (rc) return rc;
  float ms = 0.f;
  CK(cudaEventElapsedTime(&ms, h->ev0, h->ev1));
  out->kernel_ms = ms;
  out->passes = passes;
  out->launches = n_waves > 0 ? passes : 0;
  if (n_collectives) *n_collectives = collectives;
  return DFX_OK;
}

// ---------------------------------------------------------------------------
// transfer simulator (sim.cu): replaces dartomp.simulator.simulate
// (simulator.py:180-708) for a batch of lowered programs
// ---------------------------------------------------------------------------
int dfx_sim_batch(dfx_handle* h, const dfx_sim_in* in, dfx_sim_out* out) {
  if (!h || !in || !out) return fail(DFX_E_ARG, "dfx_sim_batch: null argument");
  if (in->n_progs < 0 || in->n_ops < 0 || in->n_vars < 0 || in->n_ops > INT32_MAX ||
      in->n_vars > INT32_MAX)
    return fail(DFX_E_ARG, "dfx_sim_batch: bad sizes");
  if (in->n_progs && (!in->progs || !in->ops || !in->arg64))
    return fail(DFX_E_ARG, "dfx_sim_batch: null input array");
  if (in->n_vars && !out->vars) return fail(DFX_E_ARG, "dfx_sim_batch: null vars output");
  std::vector<int32_t> item_prog, item_chunk;
  for (int i = 0; i < in->n_progs; i++) {
    const dfx_sim_prog& p = in->progs[i];
    if (p.op_off < 0 || p.n_ops < 1 || (int64_t)p.op_off + p.n_ops > in->n_ops || p.var_off < 0 ||
        p.n_vars < 0 || (int64_t)p.var_off + p.n_vars > in->n_vars)
      return fail(DFX_E_ARG, "dfx_sim_batch: program %d out of range", i);
    for (int c = 0; c < (p.n_vars + 31) / 32; c++) {
      item_prog.push_back(i);
      item_chunk.push_back(c);
    }
  }
  CK(cudaSetDevice(h->device));
  cudaStream_t st = h->st();
  const int n_items = (int)item_prog.size();
  const int64_t cap = out->rec_cap > 0 ? out->rec_cap : 0;
  auto* d_progs = (dfx_sim_prog*)dbuf(h, "sim_progs", sizeof(dfx_sim_prog) * in->n_progs + 16);
  auto* d_ops = (int32_t*)dbuf(h, "sim_ops", sizeof(int32_t) * 4 * in->n_ops + 16);
  auto* d_arg = (int64_t*)dbuf(h, "sim_arg", sizeof(int64_t) * in->n_ops + 16);
  auto* d_items = (int32_t*)dbuf(h, "sim_items", sizeof(int32_t) * 2 * (size_t)n_items + 16);
  auto* d_vars = (dfx_sim_var*)dbuf(h, "sim_vars", sizeof(dfx_sim_var) * in->n_vars + 16);
  auto* d_recs = (dfx_sim_rec*)dbuf(h, "sim_recs", sizeof(dfx_sim_rec) * cap + 16);
  auto* d_ctr = (unsigned long long*)dbuf(h, "sim_ctr", 64);
  if (!d_progs || !d_ops || !d_arg || !d_items || !d_vars || !d_recs || !d_ctr)
    return fail(DFX_E_CUDA, "dfx_sim_batch: allocation failed");
  if (in->n_progs) {
    CK(cudaMemcpyAsync(d_progs, in->progs, sizeof(dfx_sim_prog) * in->n_progs, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(d_ops, in->ops, sizeof(int32_t) * 4 * in->n_ops, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(d_arg, in->arg64, sizeof(int64_t) * in->n_ops, cudaMemcpyHostToDevice, st));
  }
  if (n_items) {
    CK(cudaMemcpyAsync(d_items, item_prog.data(), sizeof(int32_t) * n_items, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(d_items + n_items, item_chunk.data(), sizeof(int32_t) * n_items,
                       cudaMemcpyHostToDevice, st));
  }
  CK(cudaMemsetAsync(d_ctr, 0, 64, st));
  dfx::SimDev s;
  s.progs = d_progs; s.ops = d_ops; s.arg64 = d_arg;
  s.item_prog = d_items; s.item_chunk = d_items + n_items; s.n_items = n_items;
  s.vars = d_vars; s.recs = d_recs; s.rec_cap = cap;
  s.rec_count = d_ctr; s.next = reinterpret_cast<unsigned*>(d_ctr + 1);
  CK(cudaEventRecord(h->ev0, st));
  int rc = dfx::sim_launch(s, st);
  CK(cudaEventRecord(h->ev1, st));
  if (rc) return fail(rc, "sim_launch failed: %s", cudaGetErrorString(cudaGetLastError()));
  unsigned long long nrec = 0;
  CK(cudaMemcpyAsync(&nrec, d_ctr, sizeof nrec, cudaMemcpyDeviceToHost, st));
  if (in->n_vars)
    CK(cudaMemcpyAsync(out->vars, d_vars, sizeof(dfx_sim_var) * in->n_vars, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  out->n_recs = (int64_t)nrec;
  float ms = 0.f;
  CK(cudaEventElapsedTime(&ms, h->ev0, h->ev1));
  out->kernel_ms = ms;
  if ((int64_t)nrec > cap) return fail(DFX_E_NOSPC, "dfx_sim_batch: %llu records, capacity %lld", nrec, (long long)cap);
  if (nrec) CK(cudaMemcpy(out->recs, d_recs, sizeof(dfx_sim_rec) * nrec, cudaMemcpyDeviceToHost));
  return DFX_OK;
}

}  // extern "C"
