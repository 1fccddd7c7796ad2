// Host planning: actor layout -> chunked bucket image, and the work-descriptor tables the kernels
// consume (pack units, chain-hop tiles, pull copy tiles).  Written for the library; the oracle's
// definitions live elsewhere and share nothing with this file.
//
// Image format ("chunks them", L1467 "divided into k smaller
// chunks"): rank regions in rank order, each holding the rank's FSDP segments in tensor order at
// 256-B aligned offsets, region length rounded to 256 B, cut into chunks of C bytes (last short),
// regions placed chunk-aligned.
#include <algorithm>
#include <map>

#include "lam_internal.h"

namespace lam {

uint64_t ImagePlan::chunk_len(uint64_t g) const {
  uint32_t r = chunk_rank[g];
  uint64_t j = g - chunk_base[r];
  uint64_t rem = region_len[r] - j * C;
  return rem < C ? rem : C;
}

bool build_image_plan(const std::vector<Tensor>& ts, int N, int layout, uint64_t C, ImagePlan* out) {
  if (N < 1 || N > LAM_MAX_RANKS || C == 0 || C % kChunkAlign) return false;
  ImagePlan p;
  p.C = C;
  p.N = N;
  p.by_tensor.assign(ts.size(), {});
  // per rank: (tensor, elem0, count)
  std::vector<std::vector<Segment>> per(N);
  if (layout == LAM_FSDP2_DIM0) {
    for (uint32_t t = 0; t < ts.size(); ++t) {
      uint64_t d0 = ts[t].d0, row = ts[t].d1, rows = cdiv(d0, N);
      for (int r = 0; r < N; ++r) {
        uint64_t a = (uint64_t)r * rows, b = std::min<uint64_t>(d0, (uint64_t)(r + 1) * rows);
        if (b > a) per[r].push_back({t, (uint32_t)r, a * row, (b - a) * row, 0});
      }
    }
  } else if (layout == LAM_FSDP1_FLAT) {
    uint64_t P = 0;
    std::vector<uint64_t> start(ts.size() + 1, 0);
    for (size_t t = 0; t < ts.size(); ++t) start[t + 1] = start[t] + ts[t].numel();
    P = start.back();
    uint64_t each = cdiv(P, N);
    for (int r = 0; r < N; ++r) {
      uint64_t a = (uint64_t)r * each, b = std::min<uint64_t>(P, (uint64_t)(r + 1) * each);
      for (uint32_t t = 0; t < ts.size(); ++t) {
        uint64_t lo = std::max(a, start[t]), hi = std::min(b, start[t + 1]);
        if (hi > lo) per[r].push_back({t, (uint32_t)r, lo - start[t], hi - lo, 0});
      }
    }
  } else {
    return false;
  }
  uint64_t base = 0;
  for (int r = 0; r < N; ++r) {
    uint64_t off = 0;
    for (auto s : per[r]) {
      off = align_up(off, kSegAlign);
      s.off = off;
      off += 2 * s.count;
      p.by_tensor[s.tensor].push_back((uint32_t)p.segs.size());
      p.segs.push_back(s);
    }
    uint64_t L = align_up(off, kSegAlign);
    p.region_len.push_back(L);
    p.n_chunks.push_back(cdiv(L, C));
    p.chunk_base.push_back(base);
    base += p.n_chunks.back();
    for (uint64_t j = 0; j < p.n_chunks.back(); ++j) p.chunk_rank.push_back((uint32_t)r);
  }
  p.total_chunks = base;
  if (p.total_chunks >= (1ull << 32)) return false;
  *out = std::move(p);
  return true;
}

bool build_pack_units(const ImagePlan& p, const std::vector<Tensor>& ts, int rank,
                      const std::vector<lam_shard>& shards, uint64_t region_base_in_part,
                      std::vector<PackUnit>* units, std::vector<uint32_t>* units_per_chunk,
                      std::string* err) {
  (void)ts;
  units->clear();
  units_per_chunk->assign(p.total_chunks, 0);
  std::map<uint32_t, std::vector<uint32_t>> by_t;
  for (uint32_t i = 0; i < shards.size(); ++i) by_t[shards[i].tensor_id].push_back(i);
  for (const Segment& s : p.segs) {
    if ((int)s.rank != rank) continue;
    // find the shard covering [elem0, elem0+count)
    int found = -1;
    for (uint32_t i : by_t[s.tensor]) {
      const lam_shard& sh = shards[i];
      if (sh.elem_offset <= s.elem0 && s.elem0 + s.count <= sh.elem_offset + sh.elem_count) {
        found = (int)i;
        break;
      }
    }
    if (found < 0) {
      *err = "no shard covers tensor " + std::to_string(s.tensor) + " elements [" +
             std::to_string(s.elem0) + ", " + std::to_string(s.elem0 + s.count) + ") of rank " +
             std::to_string(rank);
      return false;
    }
    uint64_t src0 = s.elem0 - shards[found].elem_offset;
    uint64_t e = 0;
    while (e < s.count) {
      uint64_t byte = s.off + 2 * e;                 // region offset of this unit's first output byte
      uint64_t g = p.chunk_base[rank] + byte / p.C;
      uint64_t chunk_end = (byte / p.C + 1) * p.C;   // region offset where the chunk ends
      uint64_t n = std::min<uint64_t>(kPackUnitElems, s.count - e);
      n = std::min<uint64_t>(n, (chunk_end - byte) / 2);
      PackUnit u;
      u.src_elem = src0 + e;
      u.dst_off = region_base_in_part + byte;
      u.shard = (uint32_t)found;
      u.n = (uint32_t)n;
      u.chunk = (uint32_t)g;
      u.word0 = (uint32_t)((byte % p.C) / 4);
      units->push_back(u);
      (*units_per_chunk)[g]++;
      e += n;
    }
  }
  return true;
}

void build_hop_tiles(const ImagePlan& p, const std::vector<int>& ranks, std::vector<HopTile>* tiles,
                     std::vector<uint32_t>* tiles_per_chunk) {
  tiles->clear();
  tiles_per_chunk->assign(p.total_chunks, 0);
  for (int r : ranks) {
    for (uint64_t j = 0; j < p.n_chunks[r]; ++j) {
      uint64_t g = p.chunk_base[r] + j;
      uint64_t len = p.chunk_len(g);
      for (uint64_t o = 0; o < len; o += kHopTileBytes) {
        HopTile t;
        t.region_off = j * p.C + o;
        t.chunk = (uint32_t)g;
        t.rank = (uint32_t)r;
        t.bytes = (uint32_t)std::min<uint64_t>(kHopTileBytes, len - o);
        t.word0 = (uint32_t)(o / 4);
        tiles->push_back(t);
        (*tiles_per_chunk)[g]++;
      }
    }
  }
  // order tiles so the pipeline advances chunk by chunk across all ranks of the part: chunk j of
  // every rank region before chunk j + 1 of any (the regions are produced side by side)
  std::stable_sort(tiles->begin(), tiles->end(), [&](const HopTile& a, const HopTile& b) {
    return chunk_order(p, a.chunk, 0) < chunk_order(p, b.chunk, 0);
  });
  for (size_t i = 0; i < tiles->size(); ++i) (*tiles)[i].tile = (uint32_t)i;
}

std::vector<HopTile> tree_hop_tiles(const std::vector<HopTile>& tiles, int R, int node, uint64_t peer_mask, int N) {
  std::vector<std::pair<uint32_t, uint32_t>> runs;   // chunk runs [begin, end) of the tile list
  for (uint32_t i = 0; i < tiles.size(); ++i)
    if (runs.empty() || tiles[runs.back().first].chunk != tiles[i].chunk) runs.push_back({i, i + 1});
    else runs.back().second = i + 1;
  std::vector<HopTile> out;
  out.reserve(tiles.size());
  for (size_t g0 = 0; g0 < runs.size(); g0 += (size_t)R) {
    const size_t gn = std::min<size_t>((size_t)R, runs.size() - g0);
    for (size_t k = 0; k < gn; ++k) {
      const size_t j = (k + (size_t)(node - 1)) % gn;   // owner of the group's j-th chunk run: relay j + 1
      const auto& run = runs[g0 + j];
      const int owner = (int)j + 1;
      for (uint32_t i = run.first; i < run.second; ++i) {
        HopTile t = tiles[i];
        const int src = owner != node && (peer_mask >> owner & 1ull) ? owner : 0;
        t.rank += (uint32_t)(src * N);
        out.push_back(t);
      }
    }
  }
  return out;
}

static uint32_t widest_align(uint64_t a, uint64_t b, uint64_t c, uint64_t d, uint64_t e) {
  uint64_t x = a | b | c | d | e;
  if (x % 16 == 0) return 16;
  if (x % 4 == 0) return 4;
  return 2;
}

// Emit the 2-D block {rows x row_bytes} in tiles of <= kPullTileBytes.
static void emit_block(std::vector<CopyTile>* out, uint32_t rank, uint64_t src_off, uint64_t dst,
                       uint64_t src_pitch, uint64_t dst_pitch, uint64_t rows, uint64_t row_bytes) {
  if (rows == 0 || row_bytes == 0) return;
  if (row_bytes >= kPullTileBytes || rows == 1) {
    for (uint64_t r = 0; r < rows; ++r)
      for (uint64_t o = 0; o < row_bytes; o += kPullTileBytes) {
        uint64_t n = std::min<uint64_t>(kPullTileBytes, row_bytes - o);
        CopyTile t{src_off + r * src_pitch + o, dst + r * dst_pitch + o, 0, 0, 1, (uint32_t)n, rank, 0};
        t.align = widest_align(t.src_off, t.dst, n, 0, 0);
        out->push_back(t);
      }
    return;
  }
  uint64_t per = std::max<uint64_t>(1, kPullTileBytes / row_bytes);
  for (uint64_t r = 0; r < rows; r += per) {
    uint64_t n = std::min<uint64_t>(per, rows - r);
    CopyTile t{src_off + r * src_pitch, dst + r * dst_pitch, (uint32_t)src_pitch, (uint32_t)dst_pitch,
               (uint32_t)n, (uint32_t)row_bytes, rank, 0};
    t.align = widest_align(t.src_off, t.dst, row_bytes, src_pitch, dst_pitch);
    out->push_back(t);
  }
}

// Transposed (K-major) part: source rows [r0, r1) x cols [c0, c1) of tensor t, element (i, c) to
// dbase + (c - c0) * tpitch + (row0 + i - r0) * 2.  Whole rows inside a segment become tiles of
// <= kPullTRows rows x kPullTCols columns (the kernel moves them as 8x8 register transposes); rows
// cut by a segment boundary (FSDP1 flat cuts) become single-row tiles.
static void emit_transposed_part(std::vector<CopyTile>* out, const ImagePlan& p, const Tensor& t, uint32_t tid,
                                 int64_t r0, int64_t r1, int64_t c0, int64_t c1, uint64_t dbase, uint64_t row0,
                                 uint64_t tpitch, uint64_t* bytes) {
  const uint64_t d1 = (uint64_t)t.d1, w = (uint64_t)(c1 - c0);
  auto tile = [&](uint32_t rank, uint64_t src_off, uint64_t i, uint64_t col, uint64_t rows, uint64_t cols) {
    // rows [i, i + rows) (source row numbers), columns [col, col + cols) relative to c0
    CopyTile x{src_off, dbase + col * tpitch + (row0 + i - (uint64_t)r0) * 2, (uint32_t)(d1 * 2), (uint32_t)tpitch,
               (uint32_t)rows, (uint32_t)(cols * 2), rank, 0};
    if (rows == 1) x.src_pitch = 0;
    x.align = widest_align(x.src_off, x.dst, x.src_pitch, x.dst_pitch, 0) | LAM_TILE_TRANSPOSE;
    out->push_back(x);
    *bytes += rows * cols * 2;
  };
  for (uint32_t si : p.by_tensor[tid]) {
    const Segment& s = p.segs[si];
    const uint64_t e0 = s.elem0, e1 = s.elem0 + s.count;
    // source rows of the slice that intersect [e0, e1)
    const uint64_t ia = std::max<uint64_t>((uint64_t)r0, e0 / d1), ib = std::min<uint64_t>((uint64_t)r1, cdiv(e1, d1));
    uint64_t i = ia;
    while (i < ib) {
      const uint64_t a = i * d1 + (uint64_t)c0, b = i * d1 + (uint64_t)c1;
      const uint64_t lo = std::max(a, e0), hi = std::min(b, e1);
      if (lo >= hi) { ++i; continue; }
      if (lo != a || hi != b) {   // row cut by the segment: one row, columns [lo - a, hi - a)
        tile(s.rank, s.off + (lo - e0) * 2, i, lo - a, 1, hi - lo);
        ++i;
        continue;
      }
      uint64_t j = i;   // maximal run of whole rows inside the segment
      while (j < ib && j * d1 + (uint64_t)c0 >= e0 && j * d1 + (uint64_t)c1 <= e1) ++j;
      for (uint64_t col = 0; col < w; col += kPullTCols)
        for (uint64_t r = i; r < j; r += kPullTRows)
          tile(s.rank, s.off + (r * d1 + (uint64_t)c0 + col - e0) * 2, r, col, std::min<uint64_t>(kPullTRows, j - r),
               std::min<uint64_t>(kPullTCols, w - col));
      i = j;
    }
  }
}

bool build_copy_tiles(const ImagePlan& p, const std::vector<Tensor>& ts, const lam_tp_layout& L,
                      std::vector<CopyTile>* tiles, uint64_t* bytes, std::string* err) {
  tiles->clear();
  *bytes = 0;
  if (L.tp_size < 1 || L.tp_rank < 0 || L.tp_rank >= L.tp_size || L.n_dsts < 0 || (L.n_dsts && !L.dsts)) {
    *err = "bad tp layout";
    return false;
  }
  for (int k = 0; k < L.n_dsts; ++k) {
    const lam_dst& d = L.dsts[k];
    if (!d.dst || d.n_parts < 1 || !d.parts) { *err = "dst " + std::to_string(k) + ": empty"; return false; }
    // total destination rows (needed by the K-major pitch) and a check of every part
    int64_t width = -1;
    uint64_t total_rows = 0;
    bool two_d = false;
    for (int q = 0; q < d.n_parts; ++q) {
      if (d.parts[q].tensor_id >= ts.size()) { *err = "bad tensor id"; return false; }
      const Tensor& t = ts[d.parts[q].tensor_id];
      int64_t r0, r1, c0, c1, pad;
      if (!part_slice(t, d.parts[q].rule, L.tp_size, L.tp_rank, &r0, &r1, &c0, &c1, &pad)) {
        *err = "rule not applicable to " + t.name;
        return false;
      }
      if (width >= 0 && c1 - c0 != width) { *err = "parts of different widths in one dst"; return false; }
      width = c1 - c0;
      two_d = two_d || t.ndim == 2;
      total_rows += (uint64_t)(r1 - r0 + pad);
    }
    const bool transpose = d.transpose && two_d;
    const uint64_t w = (uint64_t)width;
    uint64_t dpitch;
    if (transpose) {
      dpitch = d.dst_row_pitch_bytes ? (uint64_t)d.dst_row_pitch_bytes : total_rows * 2;
      if (dpitch < total_rows * 2) { *err = "K-major row pitch smaller than the rows"; return false; }
    } else {
      dpitch = d.dst_row_pitch_bytes ? (uint64_t)d.dst_row_pitch_bytes : w * 2;
      if (dpitch < w * 2) { *err = "row pitch smaller than the row"; return false; }
    }
    if (dpitch >= (1ull << 32)) { *err = "row pitch too large"; return false; }
    const uint64_t dbase = (uint64_t)(uintptr_t)d.dst;
    uint64_t row0 = 0;   // destination row where the current part starts
    for (int q = 0; q < d.n_parts; ++q) {
      const Tensor& t = ts[d.parts[q].tensor_id];
      int64_t r0, r1, c0, c1, pad;
      part_slice(t, d.parts[q].rule, L.tp_size, L.tp_rank, &r0, &r1, &c0, &c1, &pad);
      const uint64_t real = (uint64_t)(r1 - r0);
      if (pad) {   // vocabulary padding rows: zero-filled by the pull (R15)
        const size_t first = tiles->size();
        if (transpose)  // K-major: in every destination row c, the run of pad entries after the real rows
          emit_block(tiles, LAM_TILE_ZERO, 0, dbase + (row0 + real) * 2, 0, dpitch, w, (uint64_t)pad * 2);
        else
          emit_block(tiles, LAM_TILE_ZERO, 0, dbase + (row0 + real) * dpitch, 0, dpitch, (uint64_t)pad, w * 2);
        for (size_t i = first; i < tiles->size(); ++i) (*tiles)[i].src_pitch = 0;
        *bytes += (uint64_t)pad * w * 2;
      }
      if (transpose) {
        emit_transposed_part(tiles, p, t, d.parts[q].tensor_id, r0, r1, c0, c1, dbase, row0, dpitch, bytes);
        row0 += real + (uint64_t)pad;
        continue;
      }
      // The slice as runs in the flattened source tensor: run k = [start_k, start_k + run) with
      // start_k = (r0 + k) * d1 + c0; a full-row slice is one contiguous run.
      bool full = (c0 == 0 && c1 == t.d1);
      uint64_t run = full ? real * t.d1 : w;
      uint64_t nrun = full ? 1 : real;
      uint64_t first = (uint64_t)r0 * t.d1 + c0, stride = (uint64_t)t.d1;
      for (uint32_t si : p.by_tensor[d.parts[q].tensor_id]) {
        if (real == 0) break;
        const Segment& s = p.segs[si];
        uint64_t e0 = s.elem0, e1 = s.elem0 + s.count;
        // runs overlapping [e0, e1): start_k + run > e0 and start_k < e1
        uint64_t klo = 0, khi = nrun;  // [klo, khi)
        if (nrun > 1) {
          klo = (e0 + 1 > first + run) ? (e0 + 1 - run - first + stride - 1) / stride : 0;
          khi = (e1 > first) ? std::min<uint64_t>(nrun, (e1 - first + stride - 1) / stride) : 0;
        } else if (!(first + run > e0 && first < e1)) {
          continue;
        }
        auto dst_of = [&](uint64_t k, uint64_t col) {   // dst address of run k, element col
          return full ? dbase + (row0 * w + col) * 2  // contiguous: col indexes the run
                      : dbase + (row0 + k) * dpitch + col * 2;
        };
        auto src_of = [&](uint64_t el) { return s.off + (el - e0) * 2; };
        uint64_t k = klo;
        while (k < khi) {
          uint64_t a = first + k * stride, b = a + run;  // run k's elements
          uint64_t lo = std::max(a, e0), hi = std::min(b, e1);
          if (lo >= hi) { ++k; continue; }
          if (lo == a && hi == b && !full) {
            // maximal stretch of whole runs inside the segment
            uint64_t k2 = k;
            while (k2 < khi && first + k2 * stride >= e0 && first + k2 * stride + run <= e1) ++k2;
            emit_block(tiles, s.rank, src_of(a), dst_of(k, 0), stride * 2, dpitch, k2 - k, run * 2);
            *bytes += (k2 - k) * run * 2;
            k = k2;
            continue;
          }
          if (full && dpitch != w * 2) {
            // pitched destination with full-row source: emit row by row pieces
            for (uint64_t el = lo; el < hi;) {
              uint64_t row = el / t.d1, col = el % t.d1;
              uint64_t n = std::min<uint64_t>(hi - el, t.d1 - col);
              emit_block(tiles, s.rank, src_of(el), dbase + (row0 + row - r0) * dpitch + col * 2, 0, 0, 1, n * 2);
              el += n;
            }
          } else {
            emit_block(tiles, s.rank, src_of(lo), dst_of(k, lo - a), 0, 0, 1, (hi - lo) * 2);
          }
          *bytes += (hi - lo) * 2;
          ++k;
        }
      }
      row0 += real + (uint64_t)pad;
    }
  }
  return true;
}

// Source chunk of a copy tile (tiles never straddle chunks after split_by_chunk).  Zero tiles
// read nothing; split_by_chunk parks the chunk they are launched with in src_off.
uint32_t chunk_of(const ImagePlan& p, const CopyTile& t) {
  if (t.zero()) return (uint32_t)t.src_off;
  return (uint32_t)(p.chunk_base[t.src_rank] + t.src_off / p.C);
}

// Launch order of source chunks for a pull: chunk j of every rank region before chunk j + 1 of any
// (FSDP ranks pack, and relays receive, their regions side by side, so the j-th chunks become
// available together), ranks rotated by `rot` so that concurrent pullers read from different GPUs
// (sorting rank-major made every TP rank read the same peer at once: 4 x slower NVLink gathers).
uint64_t chunk_order(const ImagePlan& p, uint32_t g, int rot) {
  const uint32_t r = p.chunk_rank[g];
  const uint64_t j = g - p.chunk_base[r];
  return j * (uint64_t)p.N + (uint64_t)((r + p.N - (uint32_t)(rot % p.N)) % p.N);
}

// Cut copy tiles at source-chunk boundaries (whole rows where possible, a row crossing a boundary
// is split in two) and order them by chunk_order, so a pull can be launched chunk by chunk.  K-major
// tiles are cut at 8-row groups so every piece keeps the 16-B destination alignment of the 8x8
// transposes; a group holding a boundary is cut into single rows.  Zero tiles go first.
std::vector<CopyTile> split_by_chunk(const ImagePlan& p, const std::vector<CopyTile>& in, int rot) {
  const uint64_t C = p.C;
  std::vector<CopyTile> out, zeros;
  out.reserve(in.size());
  auto widest = [](uint64_t x) -> uint32_t { return x % 16 == 0 ? 16 : (x % 4 == 0 ? 4 : 2); };
  // destination step of one source row / one byte of a row
  auto row_step = [](const CopyTile& t) -> uint64_t { return t.transposed() ? 2 : t.dst_pitch; };
  auto piece = [&](const CopyTile& t, uint64_t r0, uint64_t nrows) {
    CopyTile u = t;
    u.src_off = t.src_off + r0 * t.src_pitch;
    u.dst = t.dst + r0 * row_step(t);
    u.rows = (uint32_t)nrows;
    if (nrows == 1) {
      u.src_pitch = 0;
      if (!t.transposed()) u.dst_pitch = 0;
    }
    out.push_back(u);
  };
  auto cut_row = [&](const CopyTile& t, uint64_t r) {   // one row, cut at every chunk boundary
    uint64_t a = t.src_off + r * t.src_pitch, dst = t.dst + r * row_step(t), left = t.row_bytes;
    while (left > 0) {
      const uint64_t n = std::min<uint64_t>(left, (a / C + 1) * C - a);
      CopyTile u = t;
      u.src_off = a;
      u.dst = dst;
      u.rows = 1;
      u.row_bytes = (uint32_t)n;
      u.src_pitch = 0;
      if (t.transposed()) {
        u.align = std::min<uint32_t>(t.align & 0xFF, widest(a | dst)) | LAM_TILE_TRANSPOSE;
        dst += n / 2 * t.dst_pitch;
      } else {
        u.dst_pitch = 0;
        u.align = n == t.row_bytes && t.rows == 1 ? t.align : std::min(t.align, widest(a | dst | n));
        dst += n;
      }
      out.push_back(u);
      a += n;
      left -= n;
    }
  };
  for (const CopyTile& t : in) {
    if (t.zero()) { zeros.push_back(t); continue; }
    if (t.rows == 1) { cut_row(t, 0); continue; }
    const uint64_t grp = t.transposed() ? 8 : 1;   // rows cut only at multiples of grp
    uint64_t r0 = 0;
    for (uint64_t g = 0; g < t.rows; g += grp) {
      const uint64_t ge = std::min<uint64_t>(t.rows, g + grp);
      const uint64_t a = t.src_off + g * t.src_pitch, b = t.src_off + (ge - 1) * t.src_pitch + t.row_bytes;
      const bool crosses = a / C != (b - 1) / C;
      const bool new_chunk = g > r0 && a / C != (t.src_off + r0 * t.src_pitch) / C;
      if (new_chunk || crosses) {
        if (g > r0) piece(t, r0, g - r0);
        r0 = g;
      }
      if (crosses) {
        for (uint64_t r = g; r < ge; ++r) cut_row(t, r);
        r0 = ge;
      }
    }
    if (t.rows > r0) piece(t, r0, t.rows - r0);
  }
  std::stable_sort(out.begin(), out.end(), [&](const CopyTile& x, const CopyTile& y) {
    return chunk_order(p, chunk_of(p, x), rot) < chunk_order(p, chunk_of(p, y), rot);
  });
  const uint64_t first = out.empty() ? 0 : chunk_of(p, out.front());
  for (CopyTile& z : zeros) z.src_off = first;
  out.insert(out.begin(), zeros.begin(), zeros.end());
  return out;
}

}  // namespace lam

using namespace lam;

extern "C" int64_t lam_plan_segments(const lam_model_dims* d, int32_t layout, int32_t N, uint64_t C,
                                     lam_segment_info* out, int64_t cap) {
  if (!d || !model_valid(*d)) return LAM_EINVAL;
  ImagePlan p;
  if (!build_image_plan(model_tensors(*d), N, layout, C, &p)) return LAM_EINVAL;
  if (out) {
    for (size_t i = 0; i < p.segs.size() && (int64_t)i < cap; ++i) {
      const Segment& s = p.segs[i];
      out[i] = lam_segment_info{s.tensor, s.rank, s.elem0, s.count, p.chunk_base[s.rank] * p.C + s.off};
    }
  }
  return (int64_t)p.segs.size();
}

extern "C" int64_t lam_plan_tree_tiles(const lam_model_dims* d, int32_t layout, int32_t N, uint64_t C,
                                       int32_t n_relays, int32_t node, uint64_t peer_mask, lam_hop_tile_info* out,
                                       int64_t cap) {
  if (!d || !model_valid(*d) || n_relays < 1 || node < 1 || node > n_relays) return LAM_EINVAL;
  std::vector<Tensor> ts = model_tensors(*d);
  ImagePlan p;
  if (!build_image_plan(ts, N, layout, C, &p)) return LAM_EINVAL;
  std::vector<int> all(N);
  for (int r = 0; r < N; ++r) all[r] = r;
  std::vector<HopTile> tiles;
  std::vector<uint32_t> tpc;
  build_hop_tiles(p, all, &tiles, &tpc);
  tiles = tree_hop_tiles(tiles, n_relays, node, peer_mask, N);
  if (out)
    for (size_t i = 0; i < tiles.size() && (int64_t)i < cap; ++i)
      out[i] = lam_hop_tile_info{tiles[i].region_off, tiles[i].chunk, tiles[i].rank % (uint32_t)N, tiles[i].bytes,
                                 tiles[i].rank / (uint32_t)N};
  return (int64_t)tiles.size();
}

extern "C" int64_t lam_plan_copy_tiles(const lam_model_dims* d, int32_t layout, int32_t N, uint64_t C,
                                       const lam_tp_layout* L, lam_copy_tile_info* out, int64_t cap) {
  if (!d || !L || !model_valid(*d)) return LAM_EINVAL;
  std::vector<Tensor> ts = model_tensors(*d);
  ImagePlan p;
  if (!build_image_plan(ts, N, layout, C, &p)) return LAM_EINVAL;
  std::vector<CopyTile> tiles;
  uint64_t bytes = 0;
  std::string err;
  if (!build_copy_tiles(p, ts, *L, &tiles, &bytes, &err)) return LAM_EINVAL;
  tiles = split_by_chunk(p, tiles, pull_rotation(p, *L));
  if (out) {
    for (size_t i = 0; i < tiles.size() && (int64_t)i < cap; ++i) {
      const CopyTile& t = tiles[i];
      out[i] = lam_copy_tile_info{t.src_off, t.dst, t.src_pitch, t.dst_pitch, t.rows, t.row_bytes, t.src_rank, t.align};
    }
  }
  return (int64_t)tiles.size();
}
