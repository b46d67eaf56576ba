// Propagation-blocking layout of one part's PageRank rows (config C3; the
// binned step in csrc/k_graph.cu). Built once per graph and part on the host.
//
// The pull CSR (rows = destinations) of the part's rows [lo, hi) is turned
// into two streams that the two phases of a step read sequentially:
//   * push order: the part's edges sorted by source. Consecutive sources are
//     cut into CHUNKS of <= chunk_edges edges spanning <= span_max source ids
//     (a source with more edges is split into single-source pieces). Inside a
//     chunk the edges are regrouped by destination BIN (bin_rows consecutive
//     destination rows); src_local[] holds, in that order, each edge's source
//     as an offset from the chunk's first source.
//   * bin-major order: bin j's entries are the segments (chunk 0, j),
//     (chunk 1, j), ... back to back, each segment sorted by destination (so
//     a hub row's entries form runs the gather adds up before its atomics);
//     gtab[s][j] is where segment (s, j)
//     starts, gtab[S][j] where bin j's entries end. dst16[] holds each entry's
//     destination as an offset inside its bin, bank-folded (o ^ ((o >> 5) & 31) ^
//     ((o >> 10) & 31): the gather's accumulator word, an involution). Bins start at multiples of 8
//     entries (padding entries: destination 0, value 0, which adds nothing).
//   * per chunk, a descriptor for the scatter: for every 32-entry window of
//     the chunk's bin-grouped entries {bitmap of the entries that start a
//     non-empty segment, segments started before the window}, then per
//     non-empty segment delta = (bin-major start) - (chunk-local start), so
//     entry f goes to vals[delta[k] + f] without any search on the device.
// Phase 1 (scatter) turns chunk s's gather inputs c[u0 .. u0+span) into the
// values of its segments; phase 2 (gather) streams a bin's values and dst16
// into a shared-memory accumulator of the bin's rows. The gather UNITS split
// heavy bins (R-MAT hubs) into several units of <= unit_edges entries that
// combine through a global accumulator slot.
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <numeric>
#include <thread>
#include <vector>

#include "hcl_datagen.h"

namespace {

struct Bins {
  hcl_pr_bins_info info{};
  std::vector<int32_t> chunks;     // 8 per chunk: u0, span, src_off, n_edges, desc_off, n_seg, 0, 0
  std::vector<uint32_t> cdesc;     // per chunk: 2 per window {bitmap, k_base}, then n_seg deltas (each part 16-byte aligned)
  std::vector<uint16_t> src_local; // per chunk, padded to multiples of 8 entries
  std::vector<uint32_t> gtab;      // (n_chunks + 1) x gstride
  std::vector<uint16_t> dst16;     // n_entries
  std::vector<int32_t> units;      // 4 per unit: bin, e0, e1, slot (-1: the unit is the whole bin)
  std::vector<int32_t> slot_units; // units per accumulator slot
};

inline int64_t align8(int64_t x) { return (x + 7) & ~int64_t(7); }

// f(first, last) over [0, n) split across the host's cores
template <typename F>
void parallel_chunks(int64_t n, F&& f) {
  const int64_t t = std::max<int64_t>(1, std::min<int64_t>(std::thread::hardware_concurrency(), (n + 63) / 64));
  if (t == 1) {
    f(0, n);
    return;
  }
  std::vector<std::thread> ts;
  for (int64_t i = 0; i < t; ++i) ts.emplace_back([&, i] { f(n * i / t, n * (i + 1) / t); });
  for (auto& th : ts) th.join();
}

}  // namespace

extern "C" {

void* hcl_pagerank_bins_build(const int32_t* row_ptr, const int32_t* col_idx, int64_t v, int64_t lo, int64_t hi,
                              int64_t bin_rows, int64_t chunk_edges, int64_t span_max, int64_t unit_edges,
                              hcl_pr_bins_info* info) {
  if (!row_ptr || !col_idx || v < 1 || lo < 0 || hi < lo || hi > v || bin_rows < 8 || bin_rows > 65536 ||
      chunk_edges < 8 || chunk_edges > 65536 || span_max < 1 || span_max > 65536 || unit_edges < 8)
    return nullptr;
  auto* b = new Bins();
  hcl_pr_bins_info& I = b->info;
  I.lo = lo;
  I.hi = hi;
  I.bin_rows = bin_rows;
  I.chunk_edges = chunk_edges;
  I.span_max = span_max;
  I.unit_edges = unit_edges;
  const int64_t p_lo = row_ptr[lo], p_hi = row_ptr[hi];
  const int64_t E = p_hi - p_lo;
  I.n_edges = E;
  const int64_t B = (hi - lo + bin_rows - 1) / bin_rows;
  I.n_bins = B;
  const int64_t gs = (B + 4) & ~int64_t(3);  // gtab row stride: >= B+1 entries, 16-byte aligned rows
  I.gstride = gs;

  // 1. push order (sources ascending; per source, destinations ascending)
  std::vector<int64_t> off(static_cast<size_t>(v) + 1, 0);
  for (int64_t p = p_lo; p < p_hi; ++p) ++off[static_cast<size_t>(col_idx[p]) + 1];
  for (int64_t u = 0; u < v; ++u) off[u + 1] += off[u];
  std::vector<int32_t> push_dst(static_cast<size_t>(E));
  {
    std::vector<int64_t> cur(off.begin(), off.end() - 1);
    for (int64_t r = lo; r < hi; ++r)
      for (int32_t p = row_ptr[r]; p < row_ptr[r + 1]; ++p) push_dst[cur[col_idx[p]]++] = static_cast<int32_t>(r);
  }

  // 2. chunks: {u0, span, push-order first edge, edges}
  struct Chunk {
    int64_t u0, span, e0, n;
  };
  std::vector<Chunk> ch;
  {
    int64_t u = 0;
    while (u < v) {
      const int64_t d = off[u + 1] - off[u];
      if (d == 0) {
        ++u;
        continue;
      }
      if (d > chunk_edges) {  // a hub: single-source pieces of (nearly) equal size
        const int64_t k = (d + chunk_edges - 1) / chunk_edges;
        for (int64_t i = 0; i < k; ++i) {
          const int64_t a = off[u] + d * i / k, e = off[u] + d * (i + 1) / k;
          ch.push_back({u, 1, a, e - a});
        }
        ++u;
        continue;
      }
      const int64_t u0 = u, e0 = off[u];
      int64_t last = u;
      ++u;
      while (u < v && u - u0 < span_max) {
        const int64_t du = off[u + 1] - off[u];
        if (du > chunk_edges || off[u + 1] - e0 > chunk_edges) break;
        if (du) last = u;
        ++u;
      }
      ch.push_back({u0, last - u0 + 1, e0, off[last + 1] - e0});
      u = last + 1;
    }
  }
  const int64_t S = static_cast<int64_t>(ch.size());
  I.n_chunks = S;

  // 3. segment lengths -> bin-major positions (column scan over the chunks)
  b->gtab.assign(static_cast<size_t>((S + 1) * gs), 0);
  uint32_t* G = b->gtab.data();
  parallel_chunks(S, [&](int64_t s0, int64_t s1) {
    for (int64_t s = s0; s < s1; ++s)
      for (int64_t e = ch[s].e0; e < ch[s].e0 + ch[s].n; ++e) ++G[s * gs + (push_dst[e] - lo) / bin_rows];
  });
  int64_t pos = 0;
  std::vector<int64_t> bin_start(static_cast<size_t>(B) + 1);
  for (int64_t j = 0; j < B; ++j) {
    bin_start[j] = pos;
    for (int64_t s = 0; s < S; ++s) {
      const uint32_t n = G[s * gs + j];
      G[s * gs + j] = static_cast<uint32_t>(pos);
      pos += n;
    }
    G[S * gs + j] = static_cast<uint32_t>(pos);
    pos = align8(pos);
  }
  for (int64_t j = B; j < gs; ++j)  // unused row tail: empty segments
    for (int64_t s = 0; s <= S; ++s) G[s * gs + j] = static_cast<uint32_t>(pos);
  bin_start[B] = pos;
  I.n_entries = pos;

  // 4. per chunk: src_local (chunk-local, bin-grouped) and dst16 (bin-major),
  //    each segment sorted by (destination, source); the scatter descriptor
  b->chunks.assign(static_cast<size_t>(8 * S), 0);
  std::vector<int64_t> src_off(static_cast<size_t>(S) + 1, 0), desc_off(static_cast<size_t>(S) + 1, 0);
  for (int64_t s = 0; s < S; ++s) {
    src_off[s + 1] = src_off[s] + align8(ch[s].n);
    int64_t nseg = 0;
    for (int64_t j = 0; j < B; ++j) nseg += G[(s + 1) * gs + j] > G[s * gs + j];
    // windows, then deltas, each part a multiple of 4 words (16-byte bulk copies)
    const int64_t words = ((2 * ((ch[s].n + 31) / 32) + 3) & ~int64_t(3)) + ((nseg + 3) & ~int64_t(3));
    desc_off[s + 1] = desc_off[s] + words;
  }
  b->src_local.assign(static_cast<size_t>(src_off[S]), 0);
  b->dst16.assign(static_cast<size_t>(pos), 0);
  b->cdesc.assign(static_cast<size_t>(desc_off[S]), 0);
  I.n_src = src_off[S];
  I.n_desc = desc_off[S];
  parallel_chunks(S, [&](int64_t s0, int64_t s1) {
    std::vector<int64_t> loc(static_cast<size_t>(B) + 1), fill(static_cast<size_t>(B));
    std::vector<uint32_t> key;
    for (int64_t s = s0; s < s1; ++s) {
      const Chunk& c = ch[s];
      loc[0] = 0;
      for (int64_t j = 0; j < B; ++j) loc[j + 1] = loc[j] + (G[(s + 1) * gs + j] - G[s * gs + j]);
      std::fill(fill.begin(), fill.end(), 0);
      key.assign(static_cast<size_t>(c.n), 0);
      // sources of the chunk in push order: walk u from u0 over [e0, e0+n)
      int64_t u = c.u0;
      for (int64_t e = c.e0; e < c.e0 + c.n; ++e) {
        while (off[u + 1] <= e) ++u;
        const int64_t r = push_dst[e] - lo, j = r / bin_rows;
        key[loc[j] + fill[j]++] = static_cast<uint32_t>((r - j * bin_rows) << 16 | (u - c.u0));
      }
      const int64_t nwin = (c.n + 31) / 32;
      uint32_t* win = &b->cdesc[desc_off[s]];
      int32_t* dl = reinterpret_cast<int32_t*>(win + ((2 * nwin + 3) & ~int64_t(3)));
      int64_t k = 0;
      for (int64_t j = 0; j < B; ++j) {
        if (loc[j + 1] == loc[j]) continue;
        if (loc[j + 1] - loc[j] > 1) std::sort(key.begin() + loc[j], key.begin() + loc[j + 1]);
        for (int64_t q = loc[j]; q < loc[j + 1]; ++q) {
          b->src_local[src_off[s] + q] = static_cast<uint16_t>(key[q] & 0xffffu);
          // stored bank-folded (pb_swz in csrc/k_graph.cu, an involution inside each
          // 32-row block): the gather indexes its accumulator with it directly
          const uint32_t d = key[q] >> 16;
          b->dst16[G[s * gs + j] + (q - loc[j])] = static_cast<uint16_t>(d ^ ((d >> 5) & 31u) ^ ((d >> 10) & 31u));
        }
        win[2 * (loc[j] / 32)] |= 1u << (loc[j] % 32);
        dl[k++] = static_cast<int32_t>(static_cast<int64_t>(G[s * gs + j]) - loc[j]);
      }
      uint32_t before = 0;
      for (int64_t w = 0; w < nwin; ++w) {
        win[2 * w + 1] = before;
        before += static_cast<uint32_t>(__builtin_popcount(win[2 * w]));
      }
      int32_t* o = &b->chunks[8 * s];
      o[0] = static_cast<int32_t>(c.u0);
      o[1] = static_cast<int32_t>(c.span);
      o[2] = static_cast<int32_t>(src_off[s]);
      o[3] = static_cast<int32_t>(c.n);
      o[4] = static_cast<int32_t>(desc_off[s]);
      o[5] = static_cast<int32_t>(k);
    }
  });

  // 5. gather units, largest first (heavy bins split; they combine in a slot)
  struct Unit {
    int32_t bin, e0, e1, slot;
  };
  std::vector<Unit> us;
  int32_t slots = 0;
  for (int64_t j = 0; j < B; ++j) {
    const int64_t a = bin_start[j], e = align8(G[S * gs + j]), n = e - a;
    if (n <= unit_edges) {
      us.push_back({static_cast<int32_t>(j), static_cast<int32_t>(a), static_cast<int32_t>(e), -1});
      continue;
    }
    const int64_t k = (n + unit_edges - 1) / unit_edges;
    int64_t prev = a;
    for (int64_t i = 1; i <= k; ++i) {
      const int64_t nx = i == k ? e : a + align8(n * i / k);
      us.push_back({static_cast<int32_t>(j), static_cast<int32_t>(prev), static_cast<int32_t>(nx), slots});
      prev = nx;
    }
    b->slot_units.push_back(static_cast<int32_t>(k));
    ++slots;
  }
  std::stable_sort(us.begin(), us.end(), [](const Unit& x, const Unit& y) { return x.e1 - x.e0 > y.e1 - y.e0; });
  b->units.resize(4 * us.size());
  for (size_t i = 0; i < us.size(); ++i) std::memcpy(&b->units[4 * i], &us[i], 16);
  I.n_units = static_cast<int64_t>(us.size());
  I.n_slots = slots;
  *info = I;
  return b;
}

int hcl_pagerank_bins_export(void* h, int32_t* chunks, uint16_t* src_local, uint32_t* gtab, uint16_t* dst16,
                             int32_t* units, int32_t* slot_units, uint32_t* cdesc) {
  if (!h) return 1000 + 9;
  const Bins* b = static_cast<const Bins*>(h);
  auto put = [](auto* dst, const auto& v) {
    if (dst && !v.empty()) std::memcpy(dst, v.data(), v.size() * sizeof(v[0]));
  };
  put(chunks, b->chunks);
  put(src_local, b->src_local);
  put(gtab, b->gtab);
  put(dst16, b->dst16);
  put(units, b->units);
  put(slot_units, b->slot_units);
  put(cdesc, b->cdesc);
  return 0;
}

void hcl_pagerank_bins_free(void* h) { delete static_cast<Bins*>(h); }

}  // extern "C"
