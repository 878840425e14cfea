// Host planner: Alg. 1 Parts 1-2 of PackInfer (arXiv 2602.06072) and the
// packed execution domain ("union of valid query-key regions").
//
// Part 1 and Part 2 follow the same readings as the oracle (R1-R9) and must
// agree with it BIT-EXACTLY (tests/test_plan_parity.py); the work/row/span tables are
// implementation-side and are checked by the coverage invariant instead.
//
// Pure integer host code: no device work, no allocation visible to the caller (scratch lives
// in std::vector; the result goes into the caller's host arena).

#ifndef PI_LPT_BUCKET_SHIFT
#define PI_LPT_BUCKET_SHIFT 5
#endif
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "packinfer.h"
#include "common.h"

namespace pi {

namespace {

struct Piece {
  int32_t request, piece, kv_begin, kv_len, prefix, group;
};

struct Group {
  int64_t load = 0;
  std::vector<int32_t> members;  // piece indices, assignment order
  std::vector<int32_t> held;     // prefix ids held (small, linear scan)
  int64_t base = 0;
  int64_t cap = 0;
  bool holds(int32_t p) const {
    for (int32_t x : held)
      if (x == p) return true;
    return false;
  }
};

struct Entry {       // one member of a group buffer, in entry order
  int32_t piece;     // piece index
  int32_t ctx;       // shared prefix id (prefix entry member) or -1 (singleton entry)
  bool first_of_ctx; // first member of its prefix entry
};

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

}  // namespace

pi_status plan_impl(int32_t n, const int32_t* kv_len, const int32_t* q_len,
                    const int32_t* prefix_id, int32_t n_prefix, const int32_t* prefix_len,
                    const int32_t* appended, const pi_config* cfg, void* arena, size_t arena_bytes,
                    pi_plan* out) {
  if (!cfg || !out) return fail(PI_EINVAL, "cfg and out must be non-NULL");
  if (n < 0 || n_prefix < 0) return fail(PI_EINVAL, "negative n / n_prefix");
  if (n > 0 && (!kv_len || !q_len)) return fail(PI_EINVAL, "kv_len/q_len NULL with n > 0");
  if (n_prefix > 0 && !prefix_len) return fail(PI_EINVAL, "prefix_len NULL with n_prefix > 0");
  const int64_t C = cfg->capacity;
  const int64_t delta = cfg->headroom;
  const int32_t r = cfg->gqa_ratio;
  const int32_t TQ = cfg->tile_q, TK = cfg->tile_k;
  const int64_t chunk = cfg->decode_chunk;
  const bool no_qpack = (cfg->flags & PI_PLAN_NO_QPACK) != 0;
  if (C < 1) return fail(PI_EINVAL, "capacity must be >= 1");
  if (delta < 0 || cfg->num_groups < 0 || cfg->mem_cap < 0)
    return fail(PI_EINVAL, "negative headroom / num_groups / mem_cap");
  if (cfg->mem_cap > 0 && cfg->mem_cap < C + delta)
    return fail(PI_EINVAL, "mem_cap must be 0 or >= capacity + headroom");
  if (TQ != 128 || TK != 128) return fail(PI_EINVAL, "tile_q and tile_k must be 128");
  if (chunk < TK || chunk % TK) return fail(PI_EINVAL, "decode_chunk must be a positive multiple of tile_k");
  if (r < 1 || r > 16) return fail(PI_EINVAL, "gqa_ratio must be in [1, 16]");
  if (cfg->flags & ~PI_PLAN_NO_QPACK) return fail(PI_EINVAL, "unknown pi_config.flags bits");
  int64_t total_q = 0;
  for (int32_t i = 0; i < n; ++i) {
    const int32_t L = kv_len[i], q = q_len[i];
    const int32_t p = prefix_id ? prefix_id[i] : -1;
    if (L < 1) return fail(PI_EINVAL, "kv_len[" + std::to_string(i) + "] < 1");
    if (q < 1 || q > L) return fail(PI_EINVAL, "q_len[" + std::to_string(i) + "] not in [1, kv_len]");
    if (p < -1 || p >= n_prefix) return fail(PI_EINVAL, "prefix_id[" + std::to_string(i) + "] out of range");
    if (p >= 0 && (prefix_len[p] < 1 || prefix_len[p] > L - q))
      return fail(PI_EINVAL, "prefix_len[" + std::to_string(p) + "] must be in [1, kv_len - q_len] of request " +
                                 std::to_string(i));
    total_q += q;
  }
  if (total_q > INT32_MAX) return fail(PI_EINVAL, "total_q exceeds int32");
  // Decode-loop steps since the last consolidation: appended[i] new tokens of decode
  // request i sit in its suffix headroom; the layout (Parts 1-2) is planned from kv_len, the
  // execution domain from kv_len + appended.
  int64_t total_appended = 0;
  for (int32_t i = 0; appended && i < n; ++i) {
    if (appended[i] < 0) return fail(PI_EINVAL, "appended[" + std::to_string(i) + "] < 0");
    if (appended[i] > 0 && q_len[i] != 1)
      return fail(PI_EINVAL, "appended tokens are only defined for decode requests (q_len == 1)");
    if (appended[i] > delta)
      return fail(PI_EREGROUP, "appended[" + std::to_string(i) + "] exceeds the headroom: re-plan (regroup)");
    total_appended += appended[i];
  }
  auto app = [&](int32_t i) -> int64_t { return appended ? appended[i] : 0; };

  // ---------------- pieces (reading R5: split into C-token pieces, prefix dropped) ---------
  std::vector<Piece> pieces;
  std::vector<int32_t> first_piece(n + 1, 0);
  for (int32_t i = 0; i < n; ++i) {
    first_piece[i] = (int32_t)pieces.size();
    const int64_t L = kv_len[i];
    const int32_t p = prefix_id ? prefix_id[i] : -1;
    if (L <= C) {
      pieces.push_back({i, 0, 0, (int32_t)L, p, -1});
    } else {
      int32_t a = 0;
      for (int64_t b = 0; b < L; b += C, ++a)
        pieces.push_back({i, a, (int32_t)b, (int32_t)std::min<int64_t>(C, L - b), -1, -1});
    }
  }
  first_piece[n] = (int32_t)pieces.size();
  const int32_t NP = (int32_t)pieces.size();

  std::vector<Group> groups;
  int32_t G0 = 0;
  std::vector<int32_t> order(NP);
  if (n > 0) {
    // ---------------- Alg. 1 line 1 (reading R2: prefix-deduplicated L_total) -------------
    int64_t L_total = 0;
    std::vector<int64_t> n_p(n_prefix, 0);
    for (const Piece& pc : pieces) {
      L_total += pc.kv_len;
      if (pc.prefix >= 0) n_p[pc.prefix] += 1;
    }
    for (int32_t p = 0; p < n_prefix; ++p)
      if (n_p[p] > 0) L_total -= (n_p[p] - 1) * (int64_t)prefix_len[p];
    G0 = cfg->num_groups > 0 ? cfg->num_groups : (int32_t)std::max<int64_t>(1, ceil_div(L_total, C));
    groups.resize(G0);
    // ---------------- Alg. 1 line 3 (reading R3: -len, request, piece) ----------------------
    for (int32_t k = 0; k < NP; ++k) order[k] = k;
    std::sort(order.begin(), order.end(), [&](int32_t a, int32_t b) {
      const Piece &x = pieces[a], &y = pieces[b];
      if (x.kv_len != y.kv_len) return x.kv_len > y.kv_len;
      if (x.request != y.request) return x.request < y.request;
      return x.piece < y.piece;
    });
    // ---------------- Alg. 1 lines 4-9 (readings R1, R4, R6) ------------------------------
    for (int32_t k : order) {
      Piece& pc = pieces[k];
      int32_t best_g = -1;
      int64_t best_load = 0, best_c = 0;
      for (int32_t g = 0; g < (int32_t)groups.size(); ++g) {
        const Group& grp = groups[g];
        const int64_t shared = (pc.prefix >= 0 && grp.holds(pc.prefix)) ? prefix_len[pc.prefix] : 0;
        const int64_t c = pc.kv_len - shared;
        if (grp.load + c > C) continue;
        if (cfg->mem_cap > 0 && grp.load + c + delta * ((int64_t)grp.members.size() + 1) > cfg->mem_cap) continue;
        if (best_g < 0 || grp.load + c < best_load) {  // strict: lowest g wins ties
          best_g = g;
          best_load = grp.load + c;
          best_c = c;
        }
      }
      if (best_g < 0) {
        groups.emplace_back();
        best_g = (int32_t)groups.size() - 1;
        best_c = pc.kv_len;
      }
      Group& grp = groups[best_g];
      grp.load += best_c;
      grp.members.push_back(k);
      if (pc.prefix >= 0 && !grp.holds(pc.prefix)) grp.held.push_back(pc.prefix);
      pc.group = best_g;
    }
  }
  const int32_t G = (int32_t)groups.size();

  // ---------------- Alg. 1 Part 2 (readings R7, R8, R9) -------------------------------------
  std::vector<pi_offset> offsets(NP);
  std::vector<pi_copy> copies;
  std::vector<std::vector<Entry>> entries(G);
  int64_t base = 0;
  std::vector<int32_t> cnt(n_prefix, 0), emitted(n_prefix, 0);
  for (int32_t g = 0; g < G; ++g) {
    Group& grp = groups[g];
    grp.base = base;
    for (int32_t k : grp.members)
      if (pieces[k].prefix >= 0) cnt[pieces[k].prefix] += 1;
    int64_t d = 0;
    for (int32_t k : grp.members) {
      const Piece& pc = pieces[k];
      const int32_t p = pc.prefix;
      if (p >= 0 && cnt[p] >= 2) {
        if (emitted[p]) continue;
        emitted[p] = 1;
        const int64_t LP = prefix_len[p];
        copies.push_back({1, p, 0, (int32_t)LP, base + d});
        const int64_t dp = d;
        d += LP;
        bool first = true;
        for (int32_t k2 : grp.members) {
          const Piece& pc2 = pieces[k2];
          if (pc2.prefix != p) continue;
          const int64_t LQ = pc2.kv_len - LP;
          copies.push_back({0, pc2.request, (int32_t)(pc2.kv_begin + LP), (int32_t)LQ, base + d});
          offsets[k2] = {(int32_t)dp, (int32_t)LP, (int32_t)d, (int32_t)LQ};
          entries[g].push_back({k2, p, first});
          first = false;
          d += LQ + delta;
        }
      } else {
        copies.push_back({0, pc.request, pc.kv_begin, pc.kv_len, base + d});
        offsets[k] = {(int32_t)d, 0, (int32_t)d, pc.kv_len};
        entries[g].push_back({k, -1, true});
        d += pc.kv_len + delta;
      }
    }
    for (int32_t k : grp.members)
      if (pieces[k].prefix >= 0) { cnt[pieces[k].prefix] = 0; emitted[pieces[k].prefix] = 0; }
    grp.cap = d;
    base += d;
  }
  const int64_t buffer_tokens = base;
  if (buffer_tokens > INT32_MAX - 4 * (int64_t)TK)
    return fail(PI_EINVAL, "buffer_tokens exceeds int32 range");

  // ---------------- packed execution domain: prefill work (rows = tokens) ------------------
  std::vector<int64_t> q_off(n + 1, 0);
  for (int32_t i = 0; i < n; ++i) q_off[i + 1] = q_off[i] + q_len[i];
  std::vector<pi_work> pwork, dwork;
  std::vector<pi_row> rows;
  std::vector<pi_span> spans;
  auto piece_buf = [&](int32_t k) -> int64_t {  // global buffer start of a piece's suffix
    return groups[pieces[k].group].base + offsets[k].d_suffix;
  };
  auto add_span = [&](int64_t b, int64_t len) { spans.push_back({(int32_t)b, (int32_t)len}); };
  int64_t valid_cells = 0, tile_cells = 0;

  struct OpenTile {
    bool open = false;
    int32_t g = -1, ctx = -1, nrows = 0;
    std::vector<std::pair<int32_t, std::pair<int32_t, int32_t>>> members;  // piece, [a0, a1)
  } ot;

  auto emit_tile = [&](int32_t g, int32_t ctx,
                       const std::vector<std::pair<int32_t, std::pair<int32_t, int32_t>>>& mem) {
    pi_work w{};
    w.kind = 0;
    w.group = g;
    w.row_begin = (int32_t)rows.size();
    w.span_begin = (int32_t)spans.size();
    const int32_t k0 = mem.front().first;
    const int32_t i0 = pieces[k0].request;
    const bool split = first_piece[i0 + 1] - first_piece[i0] > 1;
    int64_t full_keys = 0;
    if (split) {  // earlier pieces of a split request: fully visible spans
      for (int32_t k = first_piece[i0]; k < k0; ++k) {
        add_span(piece_buf(k), pieces[k].kv_len);
        full_keys += pieces[k].kv_len;
      }
    }
    if (ctx >= 0) {  // shared prefix entry: the prefix span is visible to every row
      const int64_t pb = groups[g].base + offsets[k0].d_prefix;
      add_span(pb, offsets[k0].l_prefix);
      full_keys += offsets[k0].l_prefix;
    }
    int64_t hull_lo = INT64_MAX, hull_hi = INT64_MIN;
    for (const auto& m : mem) {
      const int32_t k = m.first;
      const Piece& pc = pieces[k];
      const int32_t i = pc.request;
      const int64_t lo = piece_buf(k);
      const int64_t first_pos = (int64_t)kv_len[i] - q_len[i];
      for (int32_t pos = m.second.first; pos < m.second.second; ++pos) {
        const int64_t hi = lo + (pos - pc.kv_begin - offsets[k].l_prefix) + 1;
        rows.push_back({(int32_t)(q_off[i] + (pos - first_pos)), (int32_t)lo, (int32_t)hi, 0});
        hull_lo = std::min(hull_lo, lo);
        hull_hi = std::max(hull_hi, hi);
        valid_cells += full_keys + (hi - lo);
      }
    }
    add_span(hull_lo, hull_hi - hull_lo);
    w.row_count = (int32_t)rows.size() - w.row_begin;
    w.span_count = (int32_t)spans.size() - w.span_begin;
    int64_t nk = 0;
    for (int32_t s = w.span_begin; s < (int32_t)spans.size(); ++s) nk += ceil_div(spans[s].len, TK);
    w.n_ktiles = (int32_t)nk;
    tile_cells += nk * TQ * TK;
    pwork.push_back(w);
  };
  auto close_tile = [&]() {
    if (ot.open && !ot.members.empty()) emit_tile(ot.g, ot.ctx, ot.members);
    ot.open = false;
    ot.members.clear();
    ot.nrows = 0;
  };

  for (int32_t g = 0; g < G; ++g) {
    for (const Entry& e : entries[g]) {
      const Piece& pc = pieces[e.piece];
      const int32_t i = pc.request;
      if (q_len[i] == 1) { close_tile(); continue; }  // decode member
      const int32_t a0 = std::max<int32_t>(pc.kv_begin, kv_len[i] - q_len[i]);
      const int32_t a1 = pc.kv_begin + pc.kv_len;
      if (a0 >= a1) { close_tile(); continue; }       // piece holds no query rows
      const int32_t nrows = a1 - a0;
      const bool split = first_piece[i + 1] - first_piece[i] > 1;
      if (split || nrows >= TQ || no_qpack) {
        close_tile();
        for (int32_t c = a0; c < a1; c += TQ)
          emit_tile(g, e.ctx, {{e.piece, {c, std::min(a1, c + TQ)}}});
        continue;
      }
      if (!(ot.open && ot.g == g && ot.ctx == e.ctx && ot.nrows + nrows <= TQ)) {
        close_tile();
        ot.open = true;
        ot.g = g;
        ot.ctx = e.ctx;
      }
      ot.members.push_back({e.piece, {a0, a1}});
      ot.nrows += nrows;
    }
    close_tile();
  }

  // ---------------- decode work (rows = (request, GQA head); q_len == 1) -------------------
  std::vector<int32_t> dcount(n, 0);
  std::vector<std::vector<int32_t>> item_members;  // decode requests of each decode item
  auto emit_decode = [&](int32_t g, const std::vector<int32_t>& reqs, int64_t b, int64_t len) {
    for (int64_t c0 = 0; c0 < len; c0 += chunk) {
      const int64_t cl = std::min<int64_t>(chunk, len - c0);
      pi_work w{};
      w.kind = 1;
      w.group = g;
      w.row_begin = (int32_t)rows.size();
      w.span_begin = (int32_t)spans.size();
      add_span(b + c0, cl);
      for (int32_t i : reqs) {
        for (int32_t h = 0; h < r; ++h)
          rows.push_back({(int32_t)q_off[i], (int32_t)(b + c0), (int32_t)(b + c0 + cl), h});
        dcount[i] += 1;
      }
      w.row_count = (int32_t)rows.size() - w.row_begin;
      w.span_count = 1;
      w.n_ktiles = (int32_t)ceil_div(cl, TK);
      dwork.push_back(w);
      item_members.push_back(reqs);
    }
  };
  const int32_t per_block = std::max(1, TQ / r);
  for (int32_t g = 0; g < G; ++g) {
    const auto& ent = entries[g];
    for (size_t a = 0; a < ent.size(); ++a) {
      const Entry& e = ent[a];
      if (e.ctx >= 0 && e.first_of_ctx) {  // shared prefix: read once for all decode members
        std::vector<int32_t> dm;
        for (size_t b = a; b < ent.size() && ent[b].ctx == e.ctx; ++b)
          if (q_len[pieces[ent[b].piece].request] == 1) dm.push_back(pieces[ent[b].piece].request);
        const int64_t pb = groups[g].base + offsets[e.piece].d_prefix;
        for (size_t s = 0; s < dm.size(); s += per_block) {
          std::vector<int32_t> blk(dm.begin() + s, dm.begin() + std::min(dm.size(), s + per_block));
          emit_decode(g, blk, pb, offsets[e.piece].l_prefix);
        }
      }
      const Piece& pc = pieces[e.piece];
      if (q_len[pc.request] != 1) continue;
      const bool last_piece = e.piece == first_piece[pc.request + 1] - 1;
      emit_decode(g, {pc.request}, piece_buf(e.piece), offsets[e.piece].l_suffix + (last_piece ? app(pc.request) : 0));
    }
  }
  // partial slots for rows with more than one decode item (reading R10 / Q19)
  std::vector<int32_t> slot_base(n, -1), occ(n, 0);
  std::vector<pi_merge> merges;
  int32_t n_slots = 0;
  for (int32_t i = 0; i < n; ++i) {
    if (dcount[i] > 1) {
      slot_base[i] = n_slots;
      merges.push_back({(int32_t)q_off[i], n_slots, dcount[i], 0});
      n_slots += dcount[i];
    }
  }
  for (size_t w = 0; w < dwork.size(); ++w) {
    int32_t row = dwork[w].row_begin;
    for (int32_t i : item_members[w]) {
      const int32_t slot = slot_base[i] >= 0 ? slot_base[i] + occ[i]++ : -1;
      for (int32_t h = 0; h < r; ++h, ++row) rows[row].out = ((slot + 1) << 4) | h;
    }
  }
  // LPT order (cost descending, stable).  Prefill items are sorted by cost bucket (32 key tiles
  // wide) and keep emission order (group, request, Q tile) inside a bucket: the ~150 units in
  // flight then cover few requests, so their K/V spans stay in L2, while the per-CTA totals of
  // the snake schedule stay balanced (units within a bucket differ by < 32 key tiles).  cfg2:
  // prefill DRAM reads 1.64 GB -> 0.84 GB per launch (Q 0.45 + K/V 0.22 GB algorithmic), same
  // kernel time (scripts/ab_lpt.sh).
  auto lpt = [](std::vector<pi_work>& v, int shift) {
    std::stable_sort(v.begin(), v.end(), [shift](const pi_work& a, const pi_work& b) {
      return (a.n_ktiles >> shift) > (b.n_ktiles >> shift);
    });
  };
  lpt(pwork, PI_LPT_BUCKET_SHIFT);
  lpt(dwork, 0);

  // ---------------- decode loop: next append slot per request, group drift (Eq. 4) ----------
  std::vector<int32_t> append_pos(std::max(n, 1), -1);
  std::vector<int64_t> gload(G, 0);
  for (int32_t g = 0; g < G; ++g) gload[g] = groups[g].load;
  for (int32_t i = 0; i < n; ++i) {
    const int32_t k = first_piece[i + 1] - 1;  // last piece holds the growing suffix
    const Piece& pc = pieces[k];
    if (q_len[i] == 1) {
      gload[pc.group] += app(i);
      if (app(i) < delta)
        append_pos[i] = (int32_t)(groups[pc.group].base + offsets[k].d_suffix + offsets[k].l_suffix + app(i));
    }
  }
  int64_t drift = 0;
  if (G > 0) {
    int64_t mx = gload[0], mn = gload[0];
    for (int64_t x : gload) { mx = std::max(mx, x); mn = std::min(mn, x); }
    drift = mx - mn;
  }

  // ---------------- reported quantities ------------------------------------------------------
  int64_t sumL2 = 0;
  for (int32_t i = 0; i < n; ++i) sumL2 += (int64_t)kv_len[i] * kv_len[i];
  int64_t disc = 0;
  if (G > 0) {
    int64_t mx = groups[0].load, mn = groups[0].load;
    for (const Group& g : groups) { mx = std::max(mx, g.load); mn = std::min(mn, g.load); }
    disc = mx - mn;
  }
  // copy_prefix: cumsum of the buffer cells each copy covers (its tokens, plus the headroom after
  // a suffix) -> the copies tile [0, buffer_tokens) exactly; copy_tokens is Eq. 5's volume.
  int64_t copy_tokens = 0;
  std::vector<int64_t> copy_prefix(copies.size() + 1, 0);
  for (size_t c = 0; c < copies.size(); ++c) {
    copy_prefix[c + 1] = copy_prefix[c] + copies[c].len + (copies[c].src_kind == 0 ? delta : 0);
    copy_tokens += copies[c].len;
  }

  // ---------------- arena layout (every table 256-byte aligned) ---------------------------
  size_t off = 0;
  auto reserve = [&](size_t bytes) { size_t o = off; off = align_up(off + bytes, 256); return o; };
  const size_t o_pieces = reserve(sizeof(pi_piece) * NP);
  const size_t o_offsets = reserve(sizeof(pi_offset) * NP);
  const size_t o_groups = reserve(sizeof(pi_group) * G);
  const size_t o_copies = reserve(sizeof(pi_copy) * copies.size());
  const size_t o_cprefix = reserve(sizeof(int64_t) * copy_prefix.size());
  const size_t o_pwork = reserve(sizeof(pi_work) * pwork.size());
  const size_t o_dwork = reserve(sizeof(pi_work) * dwork.size());
  const size_t o_rows = reserve(sizeof(pi_row) * rows.size());
  const size_t o_spans = reserve(sizeof(pi_span) * spans.size());
  const size_t o_merges = reserve(sizeof(pi_merge) * merges.size());
  const size_t o_append = reserve(sizeof(int32_t) * std::max(n, 1));
  const size_t need = std::max<size_t>(off, 256);

  std::memset(out, 0, sizeof(*out));
  out->n_pieces = NP;
  out->n_groups = G;
  out->g0 = G0;
  out->n_copies = (int32_t)copies.size();
  out->n_prefill_work = (int32_t)pwork.size();
  out->n_decode_work = (int32_t)dwork.size();
  out->n_rows = (int32_t)rows.size();
  out->n_spans = (int32_t)spans.size();
  out->n_merges = (int32_t)merges.size();
  out->n_partial_slots = n_slots;
  out->buffer_tokens = buffer_tokens;
  out->copy_tokens = copy_tokens;
  out->n_requests = n;
  out->n_prefix = n_prefix;
  out->total_q = (int32_t)total_q;
  out->gqa_ratio = r;
  out->eta_num = sumL2;
  out->eta_den = (int64_t)std::max(G, 1) * TK * TK;
  out->valid_cells = valid_cells;
  out->tile_cells = tile_cells;
  out->discrepancy = (int32_t)disc;
  out->drift = drift;
  out->appended_total = total_appended;
  out->arena_bytes = need;
  if (!arena || arena_bytes < need) {
    out->arena = nullptr;
    return fail(PI_ENOSPC, "host arena too small: need " + std::to_string(need) + " bytes");
  }
  char* A = static_cast<char*>(arena);
  std::memset(A, 0, need);
  out->arena = arena;
  out->pieces = reinterpret_cast<pi_piece*>(A + o_pieces);
  out->offsets = reinterpret_cast<pi_offset*>(A + o_offsets);
  out->groups = reinterpret_cast<pi_group*>(A + o_groups);
  out->copies = reinterpret_cast<pi_copy*>(A + o_copies);
  out->copy_prefix = reinterpret_cast<int64_t*>(A + o_cprefix);
  out->prefill_work = reinterpret_cast<pi_work*>(A + o_pwork);
  out->decode_work = reinterpret_cast<pi_work*>(A + o_dwork);
  out->rows = reinterpret_cast<pi_row*>(A + o_rows);
  out->spans = reinterpret_cast<pi_span*>(A + o_spans);
  out->merges = reinterpret_cast<pi_merge*>(A + o_merges);
  out->append_pos = reinterpret_cast<int32_t*>(A + o_append);
  for (int32_t k = 0; k < NP; ++k) {
    const Piece& pc = pieces[k];
    out->pieces[k] = {pc.request, pc.piece, pc.kv_begin, pc.kv_len, pc.group};
    out->offsets[k] = offsets[k];
  }
  for (int32_t g = 0; g < G; ++g)
    out->groups[g] = {groups[g].base, (int32_t)groups[g].load, (int32_t)groups[g].members.size(),
                      (int32_t)groups[g].cap, 0};
  if (!copies.empty()) std::memcpy(out->copies, copies.data(), sizeof(pi_copy) * copies.size());
  std::memcpy(out->copy_prefix, copy_prefix.data(), sizeof(int64_t) * copy_prefix.size());
  if (!pwork.empty()) std::memcpy(out->prefill_work, pwork.data(), sizeof(pi_work) * pwork.size());
  if (!dwork.empty()) std::memcpy(out->decode_work, dwork.data(), sizeof(pi_work) * dwork.size());
  if (!rows.empty()) std::memcpy(out->rows, rows.data(), sizeof(pi_row) * rows.size());
  if (!spans.empty()) std::memcpy(out->spans, spans.data(), sizeof(pi_span) * spans.size());
  if (!merges.empty()) std::memcpy(out->merges, merges.data(), sizeof(pi_merge) * merges.size());
  std::memcpy(out->append_pos, append_pos.data(), sizeof(int32_t) * std::max(n, 1));
  return PI_OK;
}

}  // namespace pi
