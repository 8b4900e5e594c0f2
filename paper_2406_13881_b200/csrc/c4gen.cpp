// c4gen.cpp -- configuration C4 generator: batches of synthetic structured
// functions emitted directly as E1 replay programs (the format lower.py
// produces), so 100k functions need no C front end.  Each function is a
// random structured body -- statements with host or device accesses,
// if/else, switch, for/while/do loops nested up to 3 deep, kernels with
// firstprivate-eligible scalars, Algorithm-1 hoist tables for every read --
// with N_f ~ U[n_min, n_max] statement nodes and V_f drawn from a list of
// variable counts.  Counter-based hashing: function f of seed s is the same
// on every host and in every shard.
#include <cstdint>
#include <cstring>
#include <thread>
#include <vector>

#include "../../include/dfx.h"

namespace {

struct Rng {
  uint64_t s;
  explicit Rng(uint64_t seed) : s(seed) {}
  uint64_t next() {
    uint64_t x = (s += 0x9E3779B97F4A7C15ull);
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
  }
  int below(int n) { return n <= 1 ? 0 : (int)(next() % (uint64_t)n); }
  bool chance(double p) { return (next() >> 11) * (1.0 / 9007199254740992.0) < p; }
};

struct FnGen {
  Rng r;
  int V;
  int target;
  int stmts = 0;
  int pos = 0;
  std::vector<int32_t> ops, span, sites, arms;
  std::vector<int> loop_ids;      // enclosing for-loops (stmt ids)
  int loop_depth = 0, max_loop = 0, br_depth = 0, max_br = 0, max_arms = 0;
  int live = 1, max_live = 1;
  int region_start = -1;
  std::vector<uint8_t> scalar;

  FnGen(uint64_t seed, int v, int n) : r(seed), V(v), target(n), scalar(v) {
    for (int i = 0; i < V; i++) scalar[i] = r.chance(0.2);
  }
  int new_stmt(int len) {
    int id = (int)span.size() / 2;
    span.push_back(pos);
    span.push_back(pos + len);
    pos += len + 1;
    stmts++;
    return id;
  }
  void close_stmt(int id) { span[2 * id + 1] = pos; pos++; }
  void emit(int op, int a = 0, int b = 0, int c = 0) {
    ops.push_back(op); ops.push_back(a); ops.push_back(b); ops.push_back(c);
  }
  int var() { return r.below(V); }
  // hoist table for a read at stmt s (bounds.py:134-193 inputs)
  int site(int s) {
    int off = (int)sites.size();
    bool sub = r.chance(0.8);
    int n = sub ? (int)loop_ids.size() : 0;
    sites.push_back(n);
    sites.push_back(s);
    for (int i = 0; i < n; i++) {
      int lid = loop_ids[i];
      int code = lid;
      if (r.chance(0.7)) code |= DFX_AC_QUAL;
      if (r.chance(0.8)) code |= DFX_AC_CLEAN;
      sites.push_back(span[2 * lid]);
      sites.push_back(code);
    }
    return off;
  }
  void hold(int n) { live += n; if (live + 1 > max_live) max_live = live + 1; }

  void host_stmt() {
    int s = new_stmt(12 + r.below(30));
    int k = 1 + r.below(3);
    for (int i = 0; i < k; i++) {
      int v = var();
      int c = r.below(10);
      if (c < 5) emit(DFX_OP_HR, v, s, site(s));
      else if (c < 8) emit(DFX_OP_HW, v, s, 0);
      else { emit(DFX_OP_HR, v, s, site(s)); emit(DFX_OP_HW, v, s, 0); }
    }
  }
  void kernel_stmt() {
    int s = new_stmt(60 + r.below(60));
    if (region_start < 0) region_start = span[2 * s];
    int nr = 1 + r.below(4), nw = 1 + r.below(3);
    std::vector<int> rd, wr;
    for (int i = 0; i < nw; i++) wr.push_back(var());
    for (int i = 0; i < nr; i++) rd.push_back(var());
    for (int v : rd) {
      bool written = false;
      for (int w : wr) written |= w == v;
      int fl = DFX_OP_DR | ((scalar[v] && !written) ? DFX_F_FP : 0);
      emit(fl, v, s, site(s));
    }
    for (int v : wr) emit(DFX_OP_DW, v, s, 0);
  }
  int anchor_kind() { return r.chance(0.5) ? DFX_ARM_BEFORE : DFX_ARM_AFTER; }
  void block(int n, int depth) {
    for (int i = 0; i < n && stmts < target; i++) stmt(depth);
  }
  void stmt(int depth) {
    double x = (r.next() >> 11) * (1.0 / 9007199254740992.0);
    if (depth < 4 && x < 0.10) {                       // if / else
      int s = new_stmt(8);
      emit(DFX_OP_HR, var(), s, site(s));
      emit(DFX_OP_BR_BEGIN);
      br_depth++; if (br_depth > max_br) max_br = br_depth;
      live++;
      emit(DFX_OP_ARM_FORK | DFX_F_CAPTURE); hold(2);
      block(1 + r.below(3), depth + 1);
      int a0 = (int)span.size() / 2 - 1;
      bool has_else = r.chance(0.5);
      int a1 = s;
      if (has_else) {
        emit(DFX_OP_ARM_FORK | DFX_F_CAPTURE); hold(2);
        block(1 + r.below(2), depth + 1);
        a1 = (int)span.size() / 2 - 1;
        live--;
      } else {
        emit(DFX_OP_ARM_PASSIVE); hold(1);
      }
      live--;
      close_stmt(s);
      int off = (int)arms.size() / 2;
      arms.push_back(anchor_kind()); arms.push_back(a0);
      arms.push_back(has_else ? anchor_kind() : DFX_ARM_BEFORE); arms.push_back(a1);
      emit(DFX_OP_BR_END, off, 2, 0);
      br_depth--;
      if (2 > max_arms) max_arms = 2;
      live -= 3;
      return;
    }
    if (depth < 4 && x < 0.13) {                       // switch
      int s = new_stmt(8);
      emit(DFX_OP_HR, var(), s, site(s));
      emit(DFX_OP_BR_BEGIN);
      br_depth++; if (br_depth > max_br) max_br = br_depth;
      live++;
      int k = 1 + r.below(3);
      std::vector<int> anchors;
      for (int g = 0; g < k; g++) {
        emit(DFX_OP_ARM_FORK); hold(1);
        block(r.below(3), depth + 1);
        emit(DFX_OP_ARM_CLOSE); hold(1); live--;
        anchors.push_back((int)span.size() / 2 - 1);
      }
      bool dflt = r.chance(0.5);
      if (!dflt) { emit(DFX_OP_ARM_PASSIVE); hold(1); anchors.push_back(s); }
      close_stmt(s);
      int off = (int)arms.size() / 2;
      for (int a : anchors) { arms.push_back(anchor_kind()); arms.push_back(a); }
      emit(DFX_OP_BR_END, off, (int)anchors.size(), 0);
      br_depth--;
      if ((int)anchors.size() > max_arms) max_arms = (int)anchors.size();
      live -= 1 + (int)anchors.size();
      return;
    }
    if (loop_depth < 3 && x < 0.25) {                  // for / while / do
      int kind = r.below(10);
      int s = new_stmt(16);
      int iv = var();
      bool is_for = kind < 7;
      if (is_for) {
        emit(DFX_OP_HW, iv, s, 0);                     // init
        emit(DFX_OP_HR, iv, s, site(s));               // cond (entry edge)
        loop_ids.push_back(s);
      } else if (kind < 9) {
        emit(DFX_OP_HR, iv, s, site(s));
      }
      int begin = (int)ops.size() / 4;
      emit(DFX_OP_LOOP_BEGIN | (kind < 9 ? DFX_F_MAY_SKIP : 0), s, 0, 0);
      loop_depth++; if (loop_depth > max_loop) max_loop = loop_depth;
      hold(2);
      block(1 + r.below(4), depth + 1);
      if (is_for) emit(DFX_OP_HW, iv, s, 0);           // increment
      emit(DFX_OP_HR | DFX_F_OVR, iv, s, s);           // cond (back edge, BODY_END)
      emit(DFX_OP_LOOP_END, begin + 1, 0, 0);
      live -= 2;
      loop_depth--;
      if (is_for) loop_ids.pop_back();
      close_stmt(s);
      return;
    }
    if (x < 0.45) kernel_stmt();
    else host_stmt();
  }
};

}  // namespace

extern "C" {

static void c4_shape(uint64_t seed, int32_t f, int32_t n_min, int32_t n_max,
                     const int32_t* var_choices, int32_t n_choices, uint64_t* fseed, int* N, int* V) {
  *fseed = seed * 0x100000001B3ull + (uint64_t)f * 0x9E3779B97F4A7C15ull + 1;
  Rng pick(*fseed ^ 0xC4C4C4C4ull);
  *N = n_min + pick.below(n_max - n_min + 1);
  *V = var_choices[pick.below(n_choices)];
}

// Shapes (statement nodes N_f, variables V_f) of functions [0, n): cheap,
// for cost-based sharding before generation.
int dfx_gen_c4_shapes(uint64_t seed, int32_t n, int32_t n_min, int32_t n_max,
                      const int32_t* var_choices, int32_t n_choices, int32_t* N, int32_t* V) {
  for (int32_t f = 0; f < n; f++) {
    uint64_t fs;
    c4_shape(seed, f, n_min, n_max, var_choices, n_choices, &fs, N + f, V + f);
  }
  return DFX_OK;
}

// Generate the functions listed in fids[0..n) of a C4 batch.  Two-pass
// protocol: call with NULL arrays to get the sizes (returned in *sizes: ops,
// vars, stmts, sites, arms), then with arrays of at least those sizes.
// facts_out gets sum(N_f * V_f).
int dfx_gen_c4(uint64_t seed, const int32_t* fids, int32_t n, int32_t n_min, int32_t n_max,
               const int32_t* var_choices, int32_t n_choices, dfx_fn_desc* fns, int32_t* ops,
               int32_t* var_flags, int32_t* stmt_span, int32_t* sites, int32_t* arms,
               int64_t* sizes, int64_t* facts_out) {
  // per-function sizes (pass 1) or placement (pass 2); functions are
  // generated in parallel across host threads, each independently seeded
  struct Sz { int64_t ops, vars, stmts, sites, arms, facts; };
  std::vector<Sz> sz((size_t)n);
  const bool place = fns != nullptr;
  std::vector<int64_t> off_o, off_v, off_st, off_si, off_ar;
  if (place) {   // offsets need the sizes: regenerate sizes cheaply first
    int64_t o = 0, v = 0, st = 0, si = 0, ar = 0;
    off_o.resize(n); off_v.resize(n); off_st.resize(n); off_si.resize(n); off_ar.resize(n);
    (void)o; (void)v; (void)st; (void)si; (void)ar;
  }
  auto gen_one = [&](int32_t i, bool write) {
    uint64_t fseed;
    int N, V;
    c4_shape(seed, fids[i], n_min, n_max, var_choices, n_choices, &fseed, &N, &V);
    FnGen g(fseed, V, N);
    while (g.stmts < N) g.stmt(0);
    g.emit(DFX_OP_END);
    const int nst = (int)g.span.size() / 2;
    sz[i] = Sz{(int64_t)g.ops.size() / 4, V, nst, (int64_t)g.sites.size(),
               (int64_t)g.arms.size() / 2, (int64_t)N * V};
    if (!write) return;
    dfx_fn_desc& d = fns[i];
    std::memset(&d, 0, sizeof d);
    d.op_off = (int32_t)off_o[i];
    d.n_ops = (int32_t)(g.ops.size() / 4);
    d.var_off = (int32_t)off_v[i];
    d.n_vars = V;
    d.stmt_off = (int32_t)off_st[i];
    d.n_stmts = nst;
    d.site_off = (int32_t)off_si[i];
    d.arm_off = (int32_t)off_ar[i];
    d.region_begin_start = g.region_start;
    d.n_slots = g.max_live + 2 * g.max_loop + 2;
    d.max_loop_depth = g.max_loop;
    d.max_br_depth = g.max_br;
    d.max_arms = g.max_arms;
    d.flags = DFX_FN_NO_ERR_SITES;   // no hoist code or arm carries a braces error
    std::memcpy(ops + 4 * off_o[i], g.ops.data(), g.ops.size() * sizeof(int32_t));
    for (int k = 0; k < V; k++) {
      int fl = g.scalar[k] ? DFX_V_SCALAR : 0;
      if (k % 2) fl |= DFX_V_NONLOCAL;
      var_flags[off_v[i] + k] = fl | (((k * 7919) % V) << 16);   // distinct name ranks
    }
    std::memcpy(stmt_span + 2 * off_st[i], g.span.data(), g.span.size() * sizeof(int32_t));
    std::memcpy(sites + off_si[i], g.sites.data(), g.sites.size() * sizeof(int32_t));
    std::memcpy(arms + 2 * off_ar[i], g.arms.data(), g.arms.size() * sizeof(int32_t));
  };
  unsigned nt = std::thread::hardware_concurrency();
  if (nt < 1) nt = 1;
  if (nt > 64) nt = 64;
  auto parallel = [&](bool write) {
    std::vector<std::thread> th;
    for (unsigned t = 0; t < nt; t++)
      th.emplace_back([&, t] {
        for (int32_t i = (int32_t)t; i < n; i += (int32_t)nt) gen_one(i, write);
      });
    for (auto& x : th) x.join();
  };
  parallel(false);
  int64_t o = 0, v = 0, st = 0, si = 0, ar = 0, facts = 0;
  if (place) {
    for (int32_t i = 0; i < n; i++) {
      off_o[i] = o; off_v[i] = v; off_st[i] = st; off_si[i] = si; off_ar[i] = ar;
      o += sz[i].ops; v += sz[i].vars; st += sz[i].stmts; si += sz[i].sites; ar += sz[i].arms;
    }
    parallel(true);
  }
  o = v = st = si = ar = 0;
  for (int32_t i = 0; i < n; i++) {
    o += sz[i].ops; v += sz[i].vars; st += sz[i].stmts; si += sz[i].sites; ar += sz[i].arms;
    facts += sz[i].facts;
  }
  if (sizes) {
    sizes[0] = o; sizes[1] = v; sizes[2] = st; sizes[3] = si; sizes[4] = ar;
  }
  if (facts_out) *facts_out = facts;
  return DFX_OK;
}

}  // extern "C"

// Dynamic op visits of each function's replay program: the number of ops the
// reference schedule executes (`_Analyzer` visit order), i.e. the final value
// of E1's visit counter -- loops run their body twice (dry round + planning
// round, dataflow.py:566-590: 3 + 2 x content), branches once (2 + content).
// Host-side accounting for the C4 roofline (algorithmic bytes per fact-visit).
extern "C" int dfx_program_visits(const dfx_fn_desc* fns, int32_t n, const int32_t* ops,
                                  int64_t* visits) {
  if (!fns || !ops || !visits || n < 0) return DFX_E_ARG;
  unsigned nt = std::thread::hardware_concurrency();
  if (nt == 0) nt = 1;
  if (nt > 32) nt = 32;
  std::vector<std::thread> th;
  for (unsigned t = 0; t < nt; t++)
    th.emplace_back([&, t] {
      std::vector<int64_t> stk;
      std::vector<char> is_loop;
      for (int32_t f = (int32_t)t; f < n; f += (int32_t)nt) {
        const int32_t* o = ops + 4 * fns[f].op_off;
        int64_t cur = 0;
        stk.clear(); is_loop.clear();
        for (int32_t pc = 0; pc < fns[f].n_ops; pc++) {
          const int code = o[4 * pc] & 0xFF;
          if (code == DFX_OP_END) break;
          if (code == DFX_OP_BR_BEGIN || code == DFX_OP_LOOP_BEGIN) {
            stk.push_back(cur); is_loop.push_back(code == DFX_OP_LOOP_BEGIN);
            cur = 0;
          } else if ((code == DFX_OP_BR_END || code == DFX_OP_LOOP_END) && !stk.empty()) {
            const int64_t dyn = is_loop.back() ? 3 + 2 * cur : 2 + cur;
            cur = stk.back() + dyn;
            stk.pop_back(); is_loop.pop_back();
          } else {
            cur++;
          }
        }
        visits[f] = cur;
      }
    });
  for (auto& x : th) x.join();
  return DFX_OK;
}
