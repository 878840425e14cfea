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
  const bool dpack = (cfg->flags & PI_PLAN_DPACK) != 0;
  const bool paged = (cfg->flags & PI_PLAN_PAGED) != 0;
  if (C < 1) return fail(PI_EINVAL, "capacity must be >= 1");
  if (delta < 0 || cfg->num_groups < 0 || cfg->mem_cap < 0)
    return fail(PI_EINVAL, "negative headroom / num_groups / mem_cap");
  if (cfg->mem_cap > 0 && cfg->mem_cap < C + delta)
    return fail(PI_EINVAL, "mem_cap must be 0 or >= capacity + headroom");
  if (TQ != 128 || TK != 128) return fail(PI_EINVAL, "tile_q and tile_k must be 128");
  if (chunk < TK || chunk % TK) return fail(PI_EINVAL, "decode_chunk must be a positive multiple of tile_k");
  if (r < 1 || r > 16) return fail(PI_EINVAL, "gqa_ratio must be in [1, 16]");
  if (cfg->flags & ~(PI_PLAN_NO_QPACK | PI_PLAN_DPACK | PI_PLAN_PAGED | PI_PLAN_LPT_EXACT))
    return fail(PI_EINVAL, "unknown pi_config.flags bits");
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
    if ((cfg->flags & PI_PLAN_PAGED) && q != 1)
      return fail(PI_EINVAL, "PI_PLAN_PAGED plans decode batches only (q_len == 1)");
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
    // Without M_max the argmin (resulting load, g) over feasible groups needs no scan: every
    // non-holder of the piece's prefix gets load_g + len, every holder load_g + len - L_P < that,
    // and feasibility (resulting load <= C) is monotone in the resulting load, so the answer is the
    // best of (a) the holders (a short list per prefix) and (b) the least-loaded group overall
    // (lowest g on ties) when it is not a holder; if that best is infeasible, none is.  A
    // tournament tree over (load_g, g) gives (b) in O(1) and updates in O(log G): O(N log G)
    // instead of O(N G) (cfg3: 338 pieces x 143 groups).  With M_max > 0 feasibility also depends
    // on member counts, so the plain scan below is used.  Both are the same argmin (R1).
    const bool fast = cfg->mem_cap == 0;
    int32_t TS = 1;
    while (TS < G0 + NP) TS <<= 1;
    std::vector<int32_t> tree(fast ? 2 * TS : 0, -1);   // leaf g at TS + g; -1 = no group
    std::vector<int64_t> tload(fast ? TS : 0, 0);
    auto better = [&](int32_t a, int32_t b) -> int32_t {   // (load, g) lexicographic min
      if (a < 0) return b;
      if (b < 0) return a;
      return (tload[b] < tload[a] || (tload[b] == tload[a] && b < a)) ? b : a;
    };
    auto tree_set = [&](int32_t g, int64_t load) {
      tload[g] = load;
      int32_t x = TS + g;
      tree[x] = g;
      for (x >>= 1; x >= 1; x >>= 1) tree[x] = better(tree[2 * x], tree[2 * x + 1]);
    };
    std::vector<std::vector<int32_t>> holders(fast ? n_prefix : 0);   // groups holding prefix p
    if (fast) {
      for (int32_t g = 0; g < G0; ++g) tree[TS + g] = g;
      for (int32_t x = TS - 1; x >= 1; --x) tree[x] = better(tree[2 * x], tree[2 * x + 1]);
    }
    for (int32_t k : order) {
      Piece& pc = pieces[k];
      int32_t best_g = -1;
      int64_t best_load = 0, best_c = 0;
      if (fast) {
        const int32_t m = tree[1];
        if (m >= 0 && !(pc.prefix >= 0 && groups[m].holds(pc.prefix))) {
          best_g = m;
          best_load = tload[m] + pc.kv_len;
          best_c = pc.kv_len;
        }
        if (pc.prefix >= 0) {
          const int64_t c = pc.kv_len - prefix_len[pc.prefix];
          for (int32_t g : holders[pc.prefix]) {
            const int64_t v = tload[g] + c;
            if (best_g < 0 || v < best_load || (v == best_load && g < best_g)) {
              best_g = g;
              best_load = v;
              best_c = c;
            }
          }
        }
        if (best_g >= 0 && best_load > C) best_g = -1;
      }
      for (int32_t g = 0; !fast && g < (int32_t)groups.size(); ++g) {
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
      if (pc.prefix >= 0 && !grp.holds(pc.prefix)) {
        grp.held.push_back(pc.prefix);
        if (fast) holders[pc.prefix].push_back(best_g);
      }
      if (fast) tree_set(best_g, grp.load);
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
  std::vector<pi_rowseg> segs;   // row segments (the per-row table is expanded on the device)
  int32_t n_rows = 0;
  std::vector<pi_span> spans;
  auto piece_buf = [&](int32_t k) -> int64_t {  // global buffer start of a piece's suffix
    return groups[pieces[k].group].base + offsets[k].d_suffix;
  };
  auto add_span = [&](int64_t b, int64_t len) { spans.push_back({(int32_t)b, (int32_t)len}); };
  int64_t valid_cells = 0, tile_cells = 0;

  using Member = std::pair<int32_t, std::pair<int32_t, int32_t>>;   // piece, [a0, a1)
  struct OpenTile {
    bool open = false;
    int32_t g = -1, ctx = -1, nrows = 0;
    std::vector<Member> members;
  } ot;
  ot.members.reserve(TQ);
  segs.reserve(2 * (size_t)NP + (size_t)total_q / TQ + 16);

  auto emit_tile = [&](int32_t g, int32_t ctx, const Member* mem, int32_t n_mem) {
    pi_work w{};
    w.kind = 0;
    w.group = g;
    w.row_begin = n_rows;
    w.span_begin = (int32_t)spans.size();
    const int32_t k0 = mem[0].first;
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
    // one row segment per member: rows pos = a0 .. a1-1 are (q_token0 + j, lo, hi0 + j) (the
    // causal own-suffix grows by one key per row); the device expands them (packinfer_plan_upload)
    int64_t hull_lo = INT64_MAX, hull_hi = INT64_MIN;
    for (int32_t mi = 0; mi < n_mem; ++mi) {
      const Member& m = mem[mi];
      const int32_t k = m.first;
      const Piece& pc = pieces[k];
      const int32_t i = pc.request;
      const int64_t lo = piece_buf(k);
      const int64_t first_pos = (int64_t)kv_len[i] - q_len[i];
      const int64_t cnt = m.second.second - m.second.first;
      if (cnt <= 0) continue;
      const int64_t hi0 = lo + (m.second.first - pc.kv_begin - offsets[k].l_prefix) + 1;
      segs.push_back({n_rows, (int32_t)cnt, (int32_t)(q_off[i] + (m.second.first - first_pos)), (int32_t)lo,
                      (int32_t)hi0, 0, PI_SEG_PREFILL, 0});
      n_rows += (int32_t)cnt;
      hull_lo = std::min(hull_lo, lo);
      hull_hi = std::max(hull_hi, hi0 + cnt - 1);
      valid_cells += cnt * (full_keys + hi0 - lo) + cnt * (cnt - 1) / 2;
    }
    add_span(hull_lo, hull_hi - hull_lo);
    w.row_count = n_rows - w.row_begin;
    w.span_count = (int32_t)spans.size() - w.span_begin;
    int64_t nk = 0;
    for (int32_t s = w.span_begin; s < (int32_t)spans.size(); ++s) nk += ceil_div(spans[s].len, TK);
    w.n_ktiles = (int32_t)nk;
    tile_cells += nk * TQ * TK;
    pwork.push_back(w);
  };
  auto close_tile = [&]() {
    if (ot.open && !ot.members.empty()) emit_tile(ot.g, ot.ctx, ot.members.data(), (int32_t)ot.members.size());
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
        for (int32_t c = a0; c < a1; c += TQ) {
          const Member one{e.piece, {c, std::min(a1, c + TQ)}};
          emit_tile(g, e.ctx, &one, 1);
        }
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
  std::vector<int32_t> item_seg;   // first row segment of each decode item: one segment per member
  std::vector<int32_t> dm;         // scratch: decode members of a prefix entry
  auto emit_decode = [&](int32_t g, const int32_t* reqs, int32_t n_reqs, int64_t b, int64_t len) {
    // ceil(len / chunk) chunks of near-equal tile counts (not full chunks + a short remainder):
    // the chunks of one span then sit next to each other in the LPT order, so a split row's last
    // partial lands with the others instead of in the launch's tail
    const int64_t n_tiles = ceil_div(len, TK), n_chunks = std::max<int64_t>(1, ceil_div(len, chunk));
    for (int64_t q = 0, c0 = 0; q < n_chunks && c0 < len; ++q) {
      const int64_t tiles_q = n_tiles / n_chunks + (q < n_tiles % n_chunks ? 1 : 0);
      const int64_t cl = std::min<int64_t>(tiles_q * TK, len - c0);
      pi_work w{};
      w.kind = 1;
      w.group = g;
      w.row_begin = n_rows;
      w.span_begin = (int32_t)spans.size();
      add_span(b + c0, cl);
      item_seg.push_back((int32_t)segs.size());
      for (int32_t mi = 0; mi < n_reqs; ++mi) {   // r rows (request i, GQA sub-head h = 0..r-1); out set below
        const int32_t i = reqs[mi];
        // reserved holds the request until the slot pass below (then 0)
        segs.push_back({n_rows, r, (int32_t)q_off[i], (int32_t)(b + c0), (int32_t)(b + c0 + cl), 0, PI_SEG_DECODE, i});
        n_rows += r;
        dcount[i] += 1;
      }
      w.row_count = n_rows - w.row_begin;
      w.span_count = 1;
      w.n_ktiles = (int32_t)ceil_div(cl, TK);
      dwork.push_back(w);
      c0 += cl;
    }
  };
  const int32_t per_block = std::max(1, TQ / r);
  {  // upper bound of the decode items: every entry's span (plus appended keys) in chunks
    size_t est = 0;
    for (int32_t g = 0; g < G; ++g) est += (size_t)(groups[g].cap / chunk) + 2 * entries[g].size();
    dwork.reserve(est);
    item_seg.reserve(est);
    spans.reserve(spans.size() + est);
    segs.reserve(segs.size() + est + (size_t)n);
  }
  // PI_PLAN_DPACK (default): packed decode items (the decode analogue of packed prefill tiles,
  // P:150): consecutive decode suffixes of one group - adjacent in B_g up to the headroom between
  // them - share ONE item whose key span is their hull (<= decode_chunk keys, <= kDpackRows rows);
  // each row sees only its own suffix [lo, hi).  Every key is still read once, and one unit
  // epilogue serves several requests (configs[3] decode kernel -7 %, profiles/r03b).
  constexpr int64_t kDpackRows = 32;
  struct PackMember { int32_t req; int64_t b, len; };
  std::vector<PackMember> pack;
  auto flush_pack = [&](int32_t g) {
    if (pack.empty()) return;
    if (pack.size() == 1) {
      emit_decode(g, &pack[0].req, 1, pack[0].b, pack[0].len);
    } else {
      const int64_t hb = pack.front().b, he = pack.back().b + pack.back().len;
      pi_work w{};
      w.kind = 1;
      w.group = g;
      w.row_begin = n_rows;
      w.span_begin = (int32_t)spans.size();
      add_span(hb, he - hb);
      item_seg.push_back((int32_t)segs.size());
      for (const PackMember& m : pack) {
        segs.push_back({n_rows, r, (int32_t)q_off[m.req], (int32_t)m.b, (int32_t)(m.b + m.len), 0, PI_SEG_DECODE, m.req});
        n_rows += r;
        dcount[m.req] += 1;
      }
      w.row_count = n_rows - w.row_begin;
      w.span_count = 1;
      w.n_ktiles = (int32_t)ceil_div(he - hb, TK);
      dwork.push_back(w);
    }
    pack.clear();
  };
  // PI_PLAN_PAGED (NEXT-4 "no packed I/O" baseline, Fig. breakdown): decode items over
  // each request's LOGICAL tokens [0, kv_len + appended) read straight from the paged cache
  // (packinfer_attention_decode_paged): no consolidation, no prefix co-location; the block-table
  // row rides in pi_work.reserved.  Chunk boundaries are multiples of tile_k, so with page_size
  // a multiple of 128 a 128-key tile never crosses a page.
  for (int32_t i = 0; paged && i < n; ++i) {
    const int64_t b0 = (int64_t)dwork.size();
    emit_decode(-1, &i, 1, 0, (int64_t)kv_len[i] + app(i));
    for (int64_t w = b0; w < (int64_t)dwork.size(); ++w) dwork[w].reserved = i;
  }
  for (int32_t g = 0; !paged && g < G; ++g) {
    const auto& ent = entries[g];
    for (size_t a = 0; a < ent.size(); ++a) {
      const Entry& e = ent[a];
      if (e.ctx >= 0 && e.first_of_ctx) {  // shared prefix: read once for all decode members
        flush_pack(g);
        dm.clear();
        for (size_t b = a; b < ent.size() && ent[b].ctx == e.ctx; ++b)
          if (q_len[pieces[ent[b].piece].request] == 1) dm.push_back(pieces[ent[b].piece].request);
        const int64_t pb = groups[g].base + offsets[e.piece].d_prefix;
        for (size_t s = 0; s < dm.size(); s += per_block)
          emit_decode(g, dm.data() + s, (int32_t)(std::min(dm.size(), s + per_block) - s), pb,
                      offsets[e.piece].l_prefix);
      }
      const Piece& pc = pieces[e.piece];
      if (q_len[pc.request] != 1) {   // a prefill suffix sits between: not adjacent any more
        flush_pack(g);
        continue;
      }
      const bool last_piece = e.piece == first_piece[pc.request + 1] - 1;
      const int64_t b = piece_buf(e.piece), len = offsets[e.piece].l_suffix + (last_piece ? app(pc.request) : 0);
      if (!dpack || len >= chunk) {   // one item per suffix (default), or a long suffix chunked on its own
        flush_pack(g);
        emit_decode(g, &pc.request, 1, b, len);
        continue;
      }
      // <= kDpackRows rows: the kernel lane-slices decode units of <= 32 rows (every softmax warp
      // takes 16 keys of each tile); larger units run with only their rows' lane quarters busy
      if (!pack.empty() && (b + len - pack.front().b > chunk || (int64_t)(pack.size() + 1) * r > kDpackRows))
        flush_pack(g);
      pack.push_back({pc.request, b, len});
    }
    flush_pack(g);
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
    const int32_t s_end = w + 1 < dwork.size() ? item_seg[w + 1] : (int32_t)segs.size();
    for (int32_t sg = item_seg[w]; sg < s_end; ++sg) {
      const int32_t i = segs[sg].reserved;
      segs[sg].reserved = 0;
      const int32_t slot = slot_base[i] >= 0 ? slot_base[i] + occ[i]++ : -1;
      segs[sg].out = (slot + 1) << 4;   // row h of the segment: out | h
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
  lpt(pwork, (cfg->flags & PI_PLAN_LPT_EXACT) ? 0 : PI_LPT_BUCKET_SHIFT);
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
  const size_t o_segs = reserve(sizeof(pi_rowseg) * segs.size());
  const size_t o_spans = reserve(sizeof(pi_span) * spans.size());
  const size_t o_merges = reserve(sizeof(pi_merge) * merges.size());
  const size_t o_slot_merge = reserve(sizeof(int32_t) * (size_t)n_slots);
  const size_t o_append = reserve(sizeof(int32_t) * std::max(n, 1));
  const size_t need = std::max<size_t>(off, 256);
  // device arena = the host arena's tables + the expanded row table behind them
  const size_t o_rows = need;
  const size_t o_sched = align_up(o_rows + sizeof(pi_row) * (size_t)n_rows, 256);
  const size_t dev_need = o_sched + 256;

  std::memset(out, 0, sizeof(*out));
  out->n_pieces = NP;
  out->n_groups = G;
  out->g0 = G0;
  out->n_copies = (int32_t)copies.size();
  out->n_prefill_work = (int32_t)pwork.size();
  out->n_decode_work = (int32_t)dwork.size();
  out->n_rows = n_rows;
  out->n_segs = (int32_t)segs.size();
  out->rows_offset = o_rows;
  out->sched_offset = o_sched;
  out->device_arena_bytes = dev_need;
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
  out->segs = reinterpret_cast<pi_rowseg*>(A + o_segs);
  out->spans = reinterpret_cast<pi_span*>(A + o_spans);
  out->merges = reinterpret_cast<pi_merge*>(A + o_merges);
  out->slot_merge = reinterpret_cast<int32_t*>(A + o_slot_merge);
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
  if (!segs.empty()) std::memcpy(out->segs, segs.data(), sizeof(pi_rowseg) * segs.size());
  if (!spans.empty()) std::memcpy(out->spans, spans.data(), sizeof(pi_span) * spans.size());
  if (!merges.empty()) std::memcpy(out->merges, merges.data(), sizeof(pi_merge) * merges.size());
  for (int32_t m = 0; m < (int32_t)merges.size(); ++m)   // slot -> its merge entry (in-kernel merge)
    for (int32_t b = 0; b < merges[m].slot_count; ++b) out->slot_merge[merges[m].slot_begin + b] = m;
  std::memcpy(out->append_pos, append_pos.data(), sizeof(int32_t) * std::max(n, 1));
  return PI_OK;
}

}  // namespace pi

extern "C" pi_status packinfer_plan_rows(const pi_plan* plan, pi_row* rows, int32_t cap) {
  if (!plan) return pi::fail(PI_EINVAL, "plan is NULL");
  if (plan->n_rows > 0 && (!plan->segs || !rows)) return pi::fail(PI_EINVAL, "plan has no segments / rows is NULL");
  if (cap < plan->n_rows) return pi::fail(PI_ENOSPC, "rows capacity < n_rows = " + std::to_string(plan->n_rows));
  for (int32_t s = 0; s < plan->n_segs; ++s) {
    const pi_rowseg& g = plan->segs[s];
    for (int32_t j = 0; j < g.count; ++j)
      rows[g.row_begin + j] = g.kind == PI_SEG_PREFILL ? pi_row{g.q_token + j, g.lo, g.hi + j, g.out}
                                                       : pi_row{g.q_token, g.lo, g.hi, g.out | j};
  }
  return pi::ok();
}
