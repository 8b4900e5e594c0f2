// api.cu -- C ABI of libdfx.so (include/dfx.h): handles, buffers, entry points.
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <unordered_map>
#include <vector>

#include <cuda_runtime.h>

#include "../../include/dfx.h"
#include "dfx_internal.h"

struct dfx_handle {
  int device = 0;
  cudaStream_t stream = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
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
  if (h->stream) cudaStreamDestroy(h->stream);
  delete h;
  return DFX_OK;
}

// ---------------------------------------------------------------------------
// E1: dfx_replay_batch  (replaces dartomp.dataflow.analyze_function,
// pkg/src/dartomp/dataflow.py:737-740, batched over functions)
// ---------------------------------------------------------------------------
int dfx_replay_batch(dfx_handle* h, const dfx_replay_in* in, dfx_replay_out* out) {
  if (!h || !in || !out) return fail(DFX_E_ARG, "dfx_replay_batch: null argument");
  CK(cudaSetDevice(h->device));
  const int nf = in->n_funcs;
  // work items: one warp per (function, 32-variable chunk); at least one per
  // function so statically known errors surface even without variables
  std::vector<int32_t> item_fn, item_chunk;
  int max_slots = 2;
  for (int f = 0; f < nf; f++) {
    const dfx_fn_desc& d = in->fns[f];
    if (d.n_slots > 64 || d.max_loop_depth > 24 || d.max_br_depth > 48 || d.max_arms > 192)
      return fail(DFX_E_LIMIT, "function %d exceeds replay limits (slots %d, loops %d, "
                  "branches %d, arms %d)", f, d.n_slots, d.max_loop_depth, d.max_br_depth,
                  d.max_arms);
    if (d.n_slots > max_slots) max_slots = d.n_slots;
    int chunks = (d.n_vars + 31) / 32;
    if (chunks == 0) chunks = 1;
    for (int c = 0; c < chunks; c++) {
      item_fn.push_back(f);
      item_chunk.push_back(c);
    }
  }
  const size_t n_items = item_fn.size();
  struct Part { const char* name; const void* src; size_t bytes; void** dst; };
  void *d_fns, *d_ops, *d_vf, *d_span, *d_sites, *d_arms, *d_ifn, *d_ich;
  Part parts[] = {
      {"fns", in->fns, sizeof(dfx_fn_desc) * (size_t)nf, &d_fns},
      {"ops", in->ops, sizeof(int32_t) * 4 * (size_t)in->n_ops, &d_ops},
      {"vf", in->var_flags, sizeof(int32_t) * (size_t)in->n_vars, &d_vf},
      {"span", in->stmt_span, sizeof(int32_t) * 2 * (size_t)in->n_stmts, &d_span},
      {"sites", in->sites, sizeof(int32_t) * (size_t)in->n_sites, &d_sites},
      {"arms", in->arms, sizeof(int32_t) * 2 * (size_t)in->n_arms, &d_arms},
      {"ifn", item_fn.data(), sizeof(int32_t) * n_items, &d_ifn},
      {"ich", item_chunk.data(), sizeof(int32_t) * n_items, &d_ich},
  };
  for (auto& p : parts) {
    *p.dst = dbuf(h, p.name, p.bytes + 16);
    if (!*p.dst) return fail(DFX_E_CUDA, "cudaMalloc %s (%zu B) failed", p.name, p.bytes);
    if (p.bytes) CK(cudaMemcpyAsync(*p.dst, p.src, p.bytes, cudaMemcpyHostToDevice, h->stream));
  }
  const int64_t cap = out->event_cap;
  auto* d_ev = (dfx_event*)dbuf(h, "events", sizeof(dfx_event) * (size_t)(cap > 0 ? cap : 1));
  auto* d_cnt = (unsigned long long*)dbuf(h, "evcount", sizeof(unsigned long long));
  auto* d_vout = (uint8_t*)dbuf(h, "vout", (size_t)in->n_vars + 1);
  if (!d_ev || !d_cnt || !d_vout) return fail(DFX_E_CUDA, "cudaMalloc outputs failed");
  CK(cudaMemsetAsync(d_cnt, 0, sizeof(unsigned long long), h->stream));
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
  r.max_slots = max_slots;
  r.events = d_ev;
  r.event_cap = cap;
  r.event_count = d_cnt;
  r.var_out = d_vout;
  CK(cudaEventRecord(h->ev0, h->stream));
  int rc = dfx::replay_launch(r, h->stream);
  if (rc != DFX_OK) return fail(rc, "replay launch failed: %s", cudaGetErrorString(cudaGetLastError()));
  CK(cudaEventRecord(h->ev1, h->stream));
  unsigned long long count = 0;
  CK(cudaMemcpyAsync(&count, d_cnt, sizeof count, cudaMemcpyDeviceToHost, h->stream));
  CK(cudaStreamSynchronize(h->stream));
  size_t ncopy = count < (unsigned long long)cap ? (size_t)count : (size_t)cap;
  if (ncopy)
    CK(cudaMemcpyAsync(out->events, d_ev, sizeof(dfx_event) * ncopy, cudaMemcpyDeviceToHost,
                       h->stream));
  if (in->n_vars)
    CK(cudaMemcpyAsync(out->var_out, d_vout, (size_t)in->n_vars, cudaMemcpyDeviceToHost,
                       h->stream));
  CK(cudaStreamSynchronize(h->stream));
  float ms = 0.f;
  CK(cudaEventElapsedTime(&ms, h->ev0, h->ev1));
  out->kernel_ms = ms;
  out->n_events = (int64_t)count;
  if ((int64_t)count > cap) return fail(DFX_E_NOSPC, "event capacity %lld < %llu",
                                        (long long)cap, count);
  return DFX_OK;
}

}  // extern "C"
