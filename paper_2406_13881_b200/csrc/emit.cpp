// emit.cpp -- batched directive emission: the reference's
// rewriter (`rewriter.apply_plans`, dartomp/rewriter.py:255-274, with
// `_FunctionRewriter` :118-252 and `detect_indent_unit` :55-74) and report
// (`report.plan_lines`, dartomp/report.py:13-39) as native host code over
// flattened plans, for many translation units in one call.
//
// Text is UTF-32 (one code point per element), so every offset is the
// reference's Python string index.  Output is byte-identical to the
// reference: the same insertions, ordered by (offset, priority, per-function
// sequence, emission order) exactly like the reference's stable sort.
// Errors come back per unit as the reference would raise them:
//   1 PreconditionError at a loop without a braced body (rewriter.py:102-110)
//   2 InternalError "conflicting update directions ..." (rewriter.py:204-208)
//   3 InternalError on a plan position the rewriter does not place
// and, in the report, an AFTER update (report.py:35 has no key for it: the
// reference raises KeyError) unless DFX_EMIT_AFTER_LINES asks for an
// "after line N" line instead.
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <map>
#include <set>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/dfx.h"

namespace {

using U32 = std::u32string;

// Python str.isspace() for the code points str.strip() removes
bool py_space(uint32_t c) {
  return (c >= 9 && c <= 13) || (c >= 28 && c <= 32) || c == 133 || c == 160 || c == 5760 ||
         (c >= 8192 && c <= 8202) || c == 8232 || c == 8233 || c == 8239 || c == 8287 || c == 12288;
}

struct Src {
  const uint32_t* t;
  int64_t n;
  std::vector<int64_t> starts;   // SourceFile.line_starts
  Src(const uint32_t* text, int64_t len) : t(text), n(len) {
    starts.push_back(0);
    for (int64_t i = 0; i < n; i++)
      if (t[i] == '\n') starts.push_back(i + 1);
  }
  int64_t line_idx(int64_t off) const {   // bisect_right(starts, off) - 1
    return (int64_t)(std::upper_bound(starts.begin(), starts.end(), off) - starts.begin()) - 1;
  }
  int64_t line_of(int64_t off) const { return line_idx(off) + 1; }
  int64_t line_start(int64_t off) const { return starts[line_idx(off)]; }
  int64_t line_end(int64_t off) const {
    const int64_t l = line_idx(off);
    return l + 1 < (int64_t)starts.size() ? starts[l + 1] : n;
  }
  U32 indent_at(int64_t off) const {
    const int64_t s = line_start(off);
    int64_t i = s;
    while (i < n && (t[i] == ' ' || t[i] == '\t')) i++;
    return U32(t + s, t + i);
  }
  bool blank(int64_t a, int64_t b) const {   // not text[a:b].strip()
    for (int64_t i = a; i < b; i++)
      if (!py_space(t[i])) return false;
    return true;
  }
  int64_t find_nl(int64_t from) const {
    for (int64_t i = from < 0 ? 0 : from; i < n; i++)
      if (t[i] == '\n') return i;
    return -1;
  }
};

U32 ascii(const char* s) { return U32(s, s + std::strlen(s)); }
U32 dec(int64_t v) { return ascii(std::to_string(v).c_str()); }

// detect_indent_unit (rewriter.py:55-74)
U32 detect_unit(const Src& s) {
  std::vector<std::pair<int64_t, int64_t>> deltas;   // (delta, count), insertion order
  int64_t prev = 0;
  for (int64_t st : s.starts) {
    const int64_t end = s.line_end(st);
    if (s.blank(st, end)) continue;
    if (st < s.n && s.t[st] == '\t') return ascii("\t");
    int64_t w = 0;
    while (st + w < end && s.t[st + w] == ' ') w++;
    if (w > prev) {
      const int64_t d = w - prev;
      bool found = false;
      for (auto& kv : deltas)
        if (kv.first == d) { kv.second++; found = true; break; }
      if (!found) deltas.push_back({d, 1});
    }
    prev = w;
  }
  if (deltas.empty()) return ascii("    ");
  // Counter.most_common(1): the largest count, first inserted on ties
  auto best = deltas[0];
  for (auto& kv : deltas)
    if (kv.second > best.second) best = kv;
  return U32((size_t)best.first, U' ');
}

struct Ins {            // an insertion; its text is arena[a, a + len)
  int64_t offset;
  int prio;
  int64_t seq;
  int64_t order;
  int64_t a, len;
};
enum { kOpen = 0, kUpdate = 1, kClause = 2, kReindent = 3, kClose = 4 };

struct Ctx {
  const dfx_emit_in* in;
  U32 str(int32_t id) const {
    return U32(in->strpool + in->str_off[id], in->strpool + in->str_off[id + 1]);
  }
};

U32 join_names(const std::vector<U32>& v) {
  U32 out;
  for (size_t i = 0; i < v.size(); i++) {
    if (i) out += U", ";
    out += v[i];
  }
  return out;
}

}  // namespace

extern "C" int dfx_emit_batch(const dfx_emit_in* in, dfx_emit_out* out) {
  if (!in || !out || in->n_units < 0 || in->n_fns < 0 || in->n_plans < 0) return DFX_E_ARG;
  Ctx cx{in};
  const bool after_lines = (in->flags & DFX_EMIT_AFTER_LINES) != 0;
  // functions and plans of each unit (functions in order, plans in order)
  std::vector<std::vector<int32_t>> unit_fns(in->n_units);
  for (int32_t f = 0; f < in->n_fns; f++) {
    const int32_t u = in->fn_unit[f];
    if (u < 0 || u >= in->n_units) return DFX_E_ARG;
    unit_fns[u].push_back(f);
  }
  std::vector<std::vector<int32_t>> fn_plans(in->n_fns);
  for (int32_t p = 0; p < in->n_plans; p++) {
    const int32_t f = in->plan[6 * p];
    if (f < 0 || f >= in->n_fns) return DFX_E_ARG;
    fn_plans[f].push_back(p);
  }
  int64_t text_need = 0, ins_need = 0, rep_need = 0;
  std::vector<U32> texts(in->n_units), reports(in->n_units);
  std::vector<std::vector<std::pair<int64_t, int64_t>>> placed(in->n_units);
  for (int32_t u = 0; u < in->n_units; u++) {
    out->err_kind[u] = 0;
    out->err_offset[u] = -1;
    const Src s(in->text + in->text_off[u], in->text_off[u + 1] - in->text_off[u]);
    U32 unit = in->unit_len[u] >= 0
                   ? U32(in->unit_text + in->unit_off[u], in->unit_text + in->unit_off[u] + in->unit_len[u])
                   : detect_unit(s);
    std::vector<Ins> ins;
    U32 arena;
    arena.reserve(1 << 12);
    const int64_t unit_a = 0, unit_n = (int64_t)unit.size();
    arena += unit;                 // the reindent pad, shared by every covered line
    int64_t order = 0;
    U32 err_msg;
    for (int32_t f : unit_fns[u]) {
      if (out->err_kind[u]) break;
      int64_t seq = 0;
      auto add = [&](int64_t off, int prio, const U32& text) {
        ins.push_back(Ins{off, prio, seq++, order++, (int64_t)arena.size(), (int64_t)text.size()});
        arena += text;
      };
      auto add_unit = [&](int64_t off, int prio) {
        ins.push_back(Ins{off, prio, seq++, order++, unit_a, unit_n});
      };
      const int64_t rb = in->fn_region[2 * f], re = in->fn_region[2 * f + 1];
      int64_t first_line = -1, last_line = -1;
      if (rb >= 0) {
        first_line = s.line_start(rb);
        last_line = s.line_start(re - 1);
      }
      auto in_region_lines = [&](int64_t ls) { return first_line <= ls && ls <= last_line; };
      // emit_region (rewriter.py:141-159)
      if (rb >= 0) {
        const int64_t begin_off = s.line_start(rb);
        const U32 indent = s.indent_at(rb);
        const U32 clauses = cx.str(in->fn_clause[f]);
        add(begin_off, kOpen, indent + U"#pragma omp target data " + clauses + U"\n" + indent + U"{\n");
        const int64_t close_off = s.line_end(re - 1);
        U32 closer = indent + U"}\n";
        if (close_off == s.n && !(s.n > 0 && s.t[s.n - 1] == '\n')) closer = U"\n" + closer;
        add(close_off, kClose, closer);
        int64_t off = begin_off;
        while (off <= last_line) {
          const int64_t end = s.line_end(off);
          if (!s.blank(off, end)) add_unit(off, kReindent);
          if (end <= off) break;
          off = end;
        }
      }
      // emit_updates (rewriter.py:167-224): one directive per (point,
      // position, direction), names merged
      struct Key { int64_t off; int pos, kind; };
      std::vector<Key> keys;
      std::vector<std::set<U32>> groups;
      std::map<int64_t, std::pair<U32, U32>> after_ctx;
      std::map<std::tuple<int64_t, int, int>, int> key_idx;
      auto find_key = [&](int64_t off, int pos, int kind) -> int {
        auto it = key_idx.find(std::make_tuple(off, pos, kind));
        return it == key_idx.end() ? -1 : it->second;
      };
      std::vector<int32_t> kplans;
      for (int32_t p : fn_plans[f]) {
        const int32_t* pp = in->plan + 6 * p;
        const int64_t* pos64 = in->plan_pos + 3 * p;
        if (pp[1] == 1) { kplans.push_back(p); continue; }   // kernel clause
        const int kind = pp[2], position = pp[3];
        int64_t off;
        if (position == DFX_POS_BODY_END) {
          if (pos64[2] < 0) {                 // _body_brace_offset: braces required
            out->err_kind[u] = DFX_EMIT_ERR_BRACES;
            out->err_offset[u] = pos64[0];
            break;
          }
          off = s.line_start(pos64[2]);
        } else if (position == DFX_POS_BEFORE) {
          off = s.line_start(pos64[0]);
        } else if (position == DFX_POS_AFTER) {
          const int64_t nl = s.find_nl(pos64[1]);
          U32 prefix;
          if (nl < 0) { off = s.n; prefix = U"\n"; }
          else off = nl + 1;
          const int64_t line = s.line_start(pos64[1]);
          const U32 pad = in_region_lines(line) ? unit : U32();
          after_ctx[off] = {prefix, pad + s.indent_at(line)};
        } else {
          out->err_kind[u] = DFX_EMIT_ERR_POSITION;   // err_offset: the plan
          out->err_offset[u] = p;
          break;
        }
        int k = find_key(off, position, kind);
        if (k < 0) {
          keys.push_back(Key{off, position, kind});
          groups.emplace_back();
          k = (int)keys.size() - 1;
          key_idx[std::make_tuple(off, position, kind)] = k;
        }
        for (int64_t i = in->plan_names_off[p]; i < in->plan_names_off[p + 1]; i++)
          groups[k].insert(cx.str(in->name_idx[i]));
      }
      if (out->err_kind[u]) break;
      for (size_t k = 0; k < keys.size() && !out->err_kind[u]; k++) {
        const Key& K = keys[k];
        std::vector<U32> names(groups[k].begin(), groups[k].end());   // sorted
        const int tw = find_key(K.off, K.pos, K.kind == DFX_EMIT_TO ? DFX_EMIT_FROM : DFX_EMIT_TO);
        if (tw >= 0) {
          std::vector<U32> clash;
          for (const U32& nme : names)
            if (groups[tw].count(nme)) clash.push_back(nme);
          if (!clash.empty()) {
            out->err_kind[u] = DFX_EMIT_ERR_CLASH;
            err_msg = join_names(clash);
            break;
          }
        }
        const U32 body = U32(K.kind == DFX_EMIT_TO ? U"to(" : U"from(") + join_names(names) + U")";
        if (K.pos == DFX_POS_BODY_END) {
          const U32 extra = in_region_lines(K.off) ? unit : U32();
          add(K.off, kUpdate, extra + s.indent_at(K.off) + unit + U"#pragma omp target update " + body + U"\n");
        } else if (K.pos == DFX_POS_AFTER) {
          const auto& ctx = after_ctx[K.off];
          add(K.off, kUpdate, ctx.first + ctx.second + U"#pragma omp target update " + body + U"\n");
        } else {
          U32 indent = s.indent_at(K.off);
          if (in_region_lines(K.off)) indent = unit + indent;
          add(K.off, kUpdate, indent + U"#pragma omp target update " + body + U"\n");
        }
      }
      if (out->err_kind[u]) break;
      // emit_kernel_clauses (rewriter.py:226-244): per kernel (first-seen
      // order), kinds in clause order, names merged and sorted
      std::vector<int32_t> kgroup;
      std::map<int32_t, int> group_idx;
      std::vector<int64_t> kstart;
      std::vector<std::map<int, std::set<U32>>> kkinds;
      for (int32_t p : kplans) {
        const int32_t* pp = in->plan + 6 * p;
        if (pp[3] != DFX_POS_KERNEL) {
          out->err_kind[u] = DFX_EMIT_ERR_POSITION;
          out->err_offset[u] = p;
          break;
        }
        auto gi = group_idx.find(pp[4]);
        size_t g = gi == group_idx.end() ? kgroup.size() : (size_t)gi->second;
        if (g == kgroup.size()) {
          group_idx[pp[4]] = (int)g;
          kgroup.push_back(pp[4]);
          kstart.push_back(in->plan_pos[3 * p]);
          kkinds.emplace_back();
        }
        auto& st = kkinds[g][pp[2]];
        for (int64_t i = in->plan_names_off[p]; i < in->plan_names_off[p + 1]; i++)
          st.insert(cx.str(in->name_idx[i]));
      }
      if (out->err_kind[u]) break;
      static const char32_t* fmt[5] = {U"map(to: ", U"map(tofrom: ", U"map(from: ", U"map(alloc: ",
                                       U"firstprivate("};
      for (size_t g = 0; g < kgroup.size(); g++) {
        U32 parts;
        for (int kind = 0; kind < 5; kind++) {
          auto it = kkinds[g].find(kind);
          if (it == kkinds[g].end()) continue;
          std::vector<U32> names(it->second.begin(), it->second.end());
          if (!parts.empty()) parts += U" ";
          parts += U32(fmt[kind]) + join_names(names) + U")";
        }
        // _pragma_end: the newline ending a (possibly continued) pragma
        int64_t i = kstart[g], off;
        for (;;) {
          const int64_t j = s.find_nl(i);
          if (j < 0) { off = s.n; break; }
          if (j > 0 && s.t[j - 1] == '\\') { i = j + 1; continue; }
          off = j;
          break;
        }
        add(off, kClause, U" " + parts);
      }
    }
    // report lines (report.py:13-39)
    U32 rep;
    bool after_err = false;
    if (in->flags & DFX_EMIT_REPORT) {
      bool any = false;
      auto line = [&](const U32& l) { rep += l; rep += U"\n"; any = true; };
      for (int32_t f : unit_fns[u]) {
        line(U"function\t" + cx.str(in->fn_name[f]));
        const int64_t rb = in->fn_region[2 * f], re = in->fn_region[2 * f + 1];
        if (rb >= 0)
          line(U"region\t" + dec(s.line_of(rb)) + U".." + dec(s.line_of(re - 1)) + U"\t" +
               cx.str(in->fn_clause[f]));
        static const char32_t* kfmt[5] = {U"map(to: ", U"map(tofrom: ", U"map(from: ", U"map(alloc: ",
                                          U"firstprivate("};
        for (int32_t p : fn_plans[f]) {
          const int32_t* pp = in->plan + 6 * p;
          if (pp[1] != 1) continue;
          std::vector<U32> names;
          for (int64_t i = in->plan_names_off[p]; i < in->plan_names_off[p + 1]; i++)
            names.push_back(cx.str(in->name_idx[i]));
          line(U"kernel-clause\t" + dec(s.line_of(in->plan_pos[3 * p])) + U"\t" + U32(kfmt[pp[2]]) +
               join_names(names) + U")");
        }
        for (int32_t p : fn_plans[f]) {
          const int32_t* pp = in->plan + 6 * p;
          if (pp[1] != 0) continue;
          std::vector<U32> names;
          for (int64_t i = in->plan_names_off[p]; i < in->plan_names_off[p + 1]; i++)
            names.push_back(cx.str(in->name_idx[i]));
          U32 where;
          if (pp[3] == DFX_POS_BEFORE) where = U"before";
          else if (pp[3] == DFX_POS_BODY_END) where = U"end-of-body";
          else if (pp[3] == DFX_POS_AFTER && after_lines) where = U"after";
          else { after_err = true; break; }
          line(U"update\t" + U32(pp[2] == DFX_EMIT_TO ? U"to(" : U"from(") + join_names(names) + U")\t" +
               where + U" line " + dec(s.line_of(in->plan_pos[3 * p])));
        }
        if (after_err) break;
        for (int64_t i = in->fn_supp_off[f]; i < in->fn_supp_off[f + 1]; i++)
          line(U"suppressed\t" + cx.str(in->supp_idx[i]));
      }
      if (!any && !after_err) line(U"no kernels; nothing to map");
    }
    out->report_err[u] = after_err ? 1 : 0;
    if (after_err) rep.clear();
    if (out->err_kind[u]) {
      texts[u] = err_msg;           // the clash names (InternalError message)
    } else {
      std::stable_sort(ins.begin(), ins.end(), [](const Ins& a, const Ins& b) {
        return std::tie(a.offset, a.prio, a.seq, a.order) < std::tie(b.offset, b.prio, b.seq, b.order);
      });
      U32 o;
      int64_t extra = 0;
      for (const Ins& x : ins) extra += x.len;
      o.resize((size_t)(s.n + extra));
      char32_t* w = &o[0];
      int64_t pos = 0;
      placed[u].reserve(ins.size());
      for (const Ins& x : ins) {
        std::memcpy(w, s.t + pos, sizeof(char32_t) * (size_t)(x.offset - pos));
        w += x.offset - pos;
        placed[u].push_back({(int64_t)(w - &o[0]), x.len});
        std::memcpy(w, arena.data() + x.a, sizeof(char32_t) * (size_t)x.len);
        w += x.len;
        pos = x.offset;
      }
      std::memcpy(w, s.t + pos, sizeof(char32_t) * (size_t)(s.n - pos));
      texts[u] = std::move(o);
    }
    reports[u] = std::move(rep);
    text_need += (int64_t)texts[u].size();
    ins_need += (int64_t)placed[u].size();
    rep_need += (int64_t)reports[u].size();
  }
  out->text_need = text_need;
  out->ins_need = ins_need;
  out->report_need = rep_need;
  if (text_need > out->text_cap || ins_need > out->ins_cap || rep_need > out->report_cap)
    return DFX_E_NOSPC;
  int64_t a = 0, b = 0, c = 0;
  for (int32_t u = 0; u < in->n_units; u++) {
    out->text_off[u] = a;
    std::copy(texts[u].begin(), texts[u].end(), out->text + a);
    a += (int64_t)texts[u].size();
    out->ins_off[u] = b;
    for (auto& pr : placed[u]) { out->ins[2 * b] = pr.first; out->ins[2 * b + 1] = pr.second; b++; }
    out->report_off[u] = c;
    std::copy(reports[u].begin(), reports[u].end(), out->report + c);
    c += (int64_t)reports[u].size();
  }
  out->text_off[in->n_units] = a;
  out->ins_off[in->n_units] = b;
  out->report_off[in->n_units] = c;
  return DFX_OK;
}
