// mapio.cu -- map / scene input and activity export on the device
// (reference mapio.hpp:19-38; SPEC.md mapio module, lines 323-390).
//
// Parsing.  The whole text goes up once (the bytes a caller would otherwise
// turn into an occupancy array on the host) and the device does the rest:
//   1. k_newlines<false>: per 8 KB chunk, count '\n' (4 bytes per compare with
//      __vcmpeq4); k_scan: chunk offsets; k_newlines<true>: every newline's
//      byte offset, in file order (block-level exclusive scan).
//   2. k_line_scan: one thread per line -> the last non-empty line, the first
//      non-empty line past the header's height and the first line's length.
//   3. k_rows<FMT>: one warp per row: length check, character classes ->
//      occupancy bytes, first error (line, column) by a 64-bit atomicMin on
//      a file-order key, per-row 'S' / 'T' counts (ASCII scenes).
//   4. ASCII scenes: k_scan over the row counts, then k_scene_coords writes the
//      source / target coordinates in row-major order (ballot ranks).
// The Moving AI header (4 short lines) is parsed on the host before the body
// goes up: it fixes the body's offset and the expected dimensions.
//
// Pins (P11-P13; the reference headers leave these open):
//   P11 line ends: '\n' or "\r\n"; the final newline is optional and trailing
//       empty lines are ignored.  A '\r' anywhere else is an unknown byte.
//   P12 header: exactly `type octile`, `height H`, `width W`, `map`, in this
//       order, tokens separated by spaces or tabs, H and W decimal in 1..65535.
//   P13 PGM samples: round-half-up of v * maxval / max (integer arithmetic),
//       header "P5\n<W> <H>\n<maxval>\n", 16-bit samples big-endian.
#include <algorithm>
#include <cstring>
#include <new>
#include <string>

#include "am_host.hpp"

struct am_scene {
  uint32_t W = 0, H = 0, format = 0;
  uint8_t* d_occ = nullptr;  // dense H x W, nonzero = obstacle
  uint32_t* d_src = nullptr;  // (row, col) pairs, row-major order
  uint32_t* d_tgt = nullptr;
  uint64_t n_src = 0, n_tgt = 0, obstacles = 0;
};

namespace am {

constexpr int kTextChunk = 8192;  // bytes per CTA of the newline scan (256 threads x 32 B)
constexpr int kTextPad = 64;      // zero bytes after the text (unguarded word loads)

// error kinds of the row kernel (packed into the low byte of the key's kind field)
enum : uint32_t { kErrChar = 1, kErrLong = 2, kErrShort = 3 };

__device__ __forceinline__ uint64_t err_key(uint32_t line, uint32_t col, uint32_t kind, uint32_t ch) {
  return ((uint64_t)line << 40) | ((uint64_t)col << 16) | (kind << 8) | ch;
}

// inclusive warp scan
__device__ __forceinline__ uint32_t warp_incl(uint32_t v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t o = __shfl_up_sync(0xffffffffu, v, d);
    if (lane >= d) v += o;
  }
  return v;
}

// Newline count (WRITE = false) or newline offsets (WRITE = true) of one
// 8 KB chunk per CTA; thread t owns bytes [32 t, 32 t + 32) of the chunk.
template <bool WRITE>
__global__ void __launch_bounds__(256) k_newlines(const uint8_t* __restrict__ text, uint64_t n,
                                                  uint64_t* __restrict__ counts, const uint64_t* __restrict__ offs,
                                                  uint64_t* __restrict__ nl) {
  __shared__ uint32_t wsum[8];
  const uint64_t base = (uint64_t)blockIdx.x * kTextChunk + threadIdx.x * 32;
  uint32_t m[8];
  uint32_t cnt = 0;
  if (base < n) {
    const uint4* p = reinterpret_cast<const uint4*>(text + base);  // 32-byte aligned (pool allocation + padding)
    const uint4 a = p[0], b = p[1];
    const uint32_t w[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      m[i] = __vcmpeq4(w[i], 0x0A0A0A0Au);
      if (base + 4 * i + 4 > n) {  // bytes past the text (the zero padding) are not newlines anyway
        const uint64_t left = n > base + 4 * i ? n - base - 4 * i : 0;
        m[i] &= left >= 4 ? 0xffffffffu : ((1u << (8 * left)) - 1u);
      }
      cnt += __popc(m[i]) >> 3;
    }
  } else {
#pragma unroll
    for (int i = 0; i < 8; ++i) m[i] = 0;
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const uint32_t incl = warp_incl(cnt);
  if (lane == 31) wsum[wid] = incl;
  __syncthreads();
  if (!WRITE) {
    if (threadIdx.x == 0) {
      uint32_t t = 0;
      for (int i = 0; i < 8; ++i) t += wsum[i];
      counts[blockIdx.x] = t;
    }
    return;
  }
  if (!cnt) return;
  uint32_t before = 0;
  for (int i = 0; i < wid; ++i) before += wsum[i];
  uint64_t pos = offs[blockIdx.x] + before + incl - cnt;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    uint32_t x = m[i];
    while (x) {
      const int k = (__ffs(x) - 1) >> 3;
      nl[pos++] = base + 4 * i + k;
      x &= ~(0xffu << (8 * k));
    }
  }
}

struct Line {
  uint64_t start;
  uint32_t len;  // without the terminator and a trailing '\r' (clamped to 2^32-1)
};

__device__ __forceinline__ Line line_at(const uint8_t* text, uint64_t n, const uint64_t* nl, uint64_t n_nl,
                                        uint64_t i) {
  const uint64_t s = i ? nl[i - 1] + 1 : 0;
  const uint64_t e = i < n_nl ? nl[i] : n;
  uint64_t len = e - s;
  if (len && text[e - 1] == '\r') --len;
  return Line{s, (uint32_t)std::min<uint64_t>(len, 0xffffffffull)};
}

// out[0] = 1 + index of the last non-empty line (atomicMax), out[1] = first
// non-empty line index >= h_expect (atomicMin; h_expect = 0: unused),
// out[2] = length of line 0
__global__ void k_line_scan(const uint8_t* __restrict__ text, uint64_t n, const uint64_t* __restrict__ nl,
                            uint64_t n_nl, uint64_t n_lines, uint64_t h_expect, unsigned long long* out) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_lines) return;
  const Line l = line_at(text, n, nl, n_nl, i);
  if (i == 0) out[2] = l.len;
  if (!l.len) return;
  atomicMax(&out[0], (unsigned long long)(i + 1));
  if (h_expect && i >= h_expect) atomicMin(&out[1], (unsigned long long)i);
}

// character class: 0 free, 1 obstacle, 2 source (free), 3 target (free), 4 unknown
template <int FMT>
__device__ __forceinline__ uint32_t char_class(uint32_t ch) {
  if (FMT == AM_FORMAT_MOVINGAI) {  // mapio.hpp:19-21
    if (ch == '.' || ch == 'G') return 0;
    if (ch == '@' || ch == 'O' || ch == 'T' || ch == 'S' || ch == 'W') return 1;
    return 4;
  } else {  // mapio.hpp:28-29
    if (ch == '.') return 0;
    if (ch == '#') return 1;
    if (ch == 'S') return 2;
    if (ch == 'T') return 3;
    return 4;
  }
}

// one warp per row: occupancy bytes, first error, 'S' / 'T' counts
template <int FMT>
__global__ void __launch_bounds__(256) k_rows(const uint8_t* __restrict__ text, uint64_t n,
                                              const uint64_t* __restrict__ nl, uint64_t n_nl, uint32_t H,
                                              uint32_t W, uint32_t line_base, uint8_t* __restrict__ occ,
                                              uint64_t* __restrict__ row_s, uint64_t* __restrict__ row_t,
                                              unsigned long long* __restrict__ err,
                                              unsigned long long* __restrict__ obstacles) {
  const uint32_t r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (r >= H) return;
  const Line l = line_at(text, n, nl, n_nl, r);
  const uint32_t use = std::min(l.len, W);
  uint32_t bad = 0xffffffffu, bad_ch = 0, ns = 0, nt = 0, nobs = 0;
  uint8_t* orow = occ + (size_t)r * W;
  const uint32_t* t32 = reinterpret_cast<const uint32_t*>(text);
  for (uint32_t c0 = 0; c0 < use; c0 += 128) {
    const uint32_t c = c0 + 4 * lane;
    if (c < use) {
      const uint64_t at = l.start + c;
      const uint32_t w0 = t32[at >> 2], w1 = t32[(at >> 2) + 1];  // padded text: in bounds
      const uint32_t w = __funnelshift_r(w0, w1, 8 * (uint32_t)(at & 3));
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        if (c + k < use) {
          const uint32_t ch = (w >> (8 * k)) & 0xffu;
          const uint32_t cls = char_class<FMT>(ch);
          if (cls == 4 && bad == 0xffffffffu) {
            bad = c + k;
            bad_ch = ch;
          }
          orow[c + k] = cls == 1;
          nobs += cls == 1;
          ns += cls == 2;
          nt += cls == 3;
        }
      }
    }
  }
  // first bad column of the warp (lanes scan disjoint columns; take the smallest)
  uint32_t best = bad;
#pragma unroll
  for (int d = 16; d; d >>= 1) best = min(best, __shfl_xor_sync(0xffffffffu, best, d));
  const uint32_t best_ch = __shfl_sync(0xffffffffu, bad_ch, __ffs(__ballot_sync(0xffffffffu, bad == best)) - 1);
#pragma unroll
  for (int d = 16; d; d >>= 1) {
    ns += __shfl_xor_sync(0xffffffffu, ns, d);
    nt += __shfl_xor_sync(0xffffffffu, nt, d);
    nobs += __shfl_xor_sync(0xffffffffu, nobs, d);
  }
  if (lane) return;
  if (row_s) row_s[r] = ns;
  if (row_t) row_t[r] = nt;
  atomicAdd(obstacles, (unsigned long long)nobs);
  const uint32_t line = line_base + r;
  if (best != 0xffffffffu) {
    atomicMin(err, err_key(line, best + 1, kErrChar, best_ch));
  } else if (l.len > W) {
    atomicMin(err, err_key(line, W + 1, kErrLong, 0));
  } else if (l.len < W) {
    atomicMin(err, err_key(line, l.len + 1, kErrShort, 0));
  }
}

// ASCII scenes: (row, col) of every 'S' and 'T' in row-major order
__global__ void __launch_bounds__(256) k_scene_coords(const uint8_t* __restrict__ text, uint64_t n,
                                                      const uint64_t* __restrict__ nl, uint64_t n_nl, uint32_t H,
                                                      uint32_t W, const uint64_t* __restrict__ s_off,
                                                      const uint64_t* __restrict__ t_off, uint32_t* __restrict__ src,
                                                      uint32_t* __restrict__ tgt) {
  const uint32_t r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (r >= H) return;
  uint64_t sp = s_off[r], tp = t_off[r];
  if (sp == s_off[r + 1] && tp == t_off[r + 1]) return;
  const Line l = line_at(text, n, nl, n_nl, r);
  const uint32_t lt = (1u << lane) - 1u;
  for (uint32_t c0 = 0; c0 < W; c0 += 32) {
    const uint32_t c = c0 + lane;
    const uint32_t ch = c < W ? text[l.start + c] : 0u;
    const uint32_t bs = __ballot_sync(0xffffffffu, ch == 'S'), bt = __ballot_sync(0xffffffffu, ch == 'T');
    if (ch == 'S') {
      const uint64_t k = sp + __popc(bs & lt);
      src[2 * k] = r;
      src[2 * k + 1] = c;
    }
    if (ch == 'T') {
      const uint64_t k = tp + __popc(bt & lt);
      tgt[2 * k] = r;
      tgt[2 * k + 1] = c;
    }
    sp += __popc(bs);
    tp += __popc(bt);
  }
}

// ---- emission (mapio.hpp:24-27, 32-33) ----
// one thread per 4 cells of a row; row r's text starts at r * (W + 1)
__global__ void k_emit_rows(const uint8_t* __restrict__ occ, uint32_t W, uint32_t H, uint8_t free_ch,
                            uint8_t obst_ch, uint8_t* __restrict__ out) {
  const uint32_t r = blockIdx.y;
  const uint32_t c = (blockIdx.x * blockDim.x + threadIdx.x) * 4;
  if (c > W) return;
  uint8_t* o = out + (size_t)r * (W + 1);
  const uint8_t* in = occ + (size_t)r * W;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    if (c + k < W) o[c + k] = in[c + k] ? obst_ch : free_ch;
    if (c + k == W) o[W] = '\n';
  }
}

__global__ void k_emit_marks(const uint32_t* __restrict__ rc, uint64_t n, uint32_t W, uint8_t ch,
                             uint8_t* __restrict__ out) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  out[(size_t)rc[2 * i] * (W + 1) + rc[2 * i + 1]] = ch;
}

// ---- PGM export (mapio.hpp:35-38) ----
template <int CB>
__device__ __forceinline__ uint32_t decode_cell(uint32_t v, uint32_t rollback) {
  const uint32_t flagbit = CB == 16 ? kFlag16 : kFlag32;
  const uint32_t low = CB == 16 ? 0x7FFFu : kLow32;
  const uint32_t a = v & low;
  return ((v & flagbit) && a) ? a - rollback : 0u;
}

// CB = 0: plain dense uint32 map (caller-uploaded); 16 / 32: the encoded field
template <int CB>
__device__ __forceinline__ uint32_t map_value(const void* val, const Geo& g, uint32_t r, uint32_t c,
                                              uint32_t rollback) {
  if (CB == 0) return static_cast<const uint32_t*>(val)[(size_t)r * g.W + c];
  if (CB == 16) return decode_cell<16>(static_cast<const uint16_t*>(val)[g.idx(r, c)], rollback);
  return decode_cell<32>(static_cast<const uint32_t*>(val)[g.idx(r, c)], rollback);
}

template <int CB>
__global__ void __launch_bounds__(256) k_map_max(Geo g, const void* __restrict__ val, uint32_t rollback,
                                                 uint32_t* __restrict__ mx) {
  uint32_t m = 0;
  const uint32_t r = blockIdx.y;
  for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < g.W; c += gridDim.x * blockDim.x)
    m = max(m, map_value<CB>(val, g, r, c, rollback));
#pragma unroll
  for (int d = 16; d; d >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, d));
  if ((threadIdx.x & 31) == 0 && m) atomicMax(mx, m);
}

// sample = round-half-up(v * maxval / max) (pin P13): float estimate, exact integer correction
template <int CB>
__global__ void __launch_bounds__(256) k_pgm(Geo g, const void* __restrict__ val, uint32_t rollback, uint32_t mx,
                                             uint32_t maxval, uint8_t* __restrict__ out) {
  const uint32_t r = blockIdx.y;
  const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= g.W) return;
  const uint32_t v = map_value<CB>(val, g, r, c, rollback);
  uint32_t q = 0;
  if (mx) {
    const uint64_t num = 2ull * v * maxval + mx, den = 2ull * mx;  // q = floor(num / den)
    q = (uint32_t)__float2uint_rn((float)v * ((float)maxval / (float)mx));
    if ((uint64_t)q * den > num) --q;
    else if ((uint64_t)(q + 1) * den <= num) ++q;
  }
  const size_t i = (size_t)r * g.W + c;
  if (maxval == 255) {
    out[i] = (uint8_t)q;
  } else {
    out[2 * i] = (uint8_t)(q >> 8);
    out[2 * i + 1] = (uint8_t)q;
  }
}

static dim3 rows_grid(uint32_t W, uint32_t H, int bx) { return dim3((W + bx - 1) / bx, H); }

}  // namespace am

using am::fail;

// ------------------------------------------------------------- host side
namespace {

void set_err(am_parse_info* info, uint64_t line, uint64_t col, const char* fmt, ...) {
  if (!info) return;
  info->error_line = line;
  info->error_column = col;
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(info->error, sizeof info->error, fmt, ap);
  va_end(ap);
}

// one header line of the Moving AI format: [pos, end of line) with '\r' stripped
struct HLine {
  const char* p;
  size_t len;
};

bool next_line(const char* text, uint64_t len, uint64_t* pos, HLine* out) {
  if (*pos >= len) return false;
  const char* s = text + *pos;
  const void* nlp = memchr(s, '\n', len - *pos);
  const size_t l = nlp ? (size_t)((const char*)nlp - s) : (size_t)(len - *pos);
  *pos += l + (nlp ? 1 : 0);
  out->p = s;
  out->len = (l && s[l - 1] == '\r') ? l - 1 : l;
  return true;
}

// tokens separated by spaces / tabs; returns count (<= 3) and their 1-based columns
int tokens(const HLine& l, std::string tok[3], size_t col[3]) {
  int k = 0;
  size_t i = 0;
  while (i < l.len) {
    while (i < l.len && (l.p[i] == ' ' || l.p[i] == '\t')) ++i;
    if (i >= l.len) break;
    const size_t b = i;
    while (i < l.len && l.p[i] != ' ' && l.p[i] != '\t') ++i;
    if (k < 3) {
      tok[k] = std::string(l.p + b, i - b);
      col[k] = b + 1;
    }
    ++k;
  }
  return k;
}

}  // namespace

extern "C" {

am_status am_movingai_header(const char* text, uint64_t len, am_parse_info* info, uint64_t* body_offset) {
  if (!text && len) return AM_EINVAL;
  am_parse_info local{};
  if (!info) info = &local;
  *info = am_parse_info{};
  uint64_t pos = 0;
  static const char* const kKey[4] = {"type", "height", "width", "map"};
  uint32_t dims[2] = {0, 0};
  for (int ln = 0; ln < 4; ++ln) {
    HLine l{};
    if (!next_line(text, len, &pos, &l)) {
      set_err(info, ln + 1, 1, "Moving AI header: missing `%s` line", kKey[ln]);
      return AM_EINVAL;
    }
    std::string tok[3];
    size_t col[3] = {1, 1, 1};
    const int k = tokens(l, tok, col);
    const int want = ln == 3 ? 1 : 2;
    if (k == 0 || tok[0] != kKey[ln]) {
      set_err(info, ln + 1, k ? col[0] : 1, "Moving AI header: expected `%s`", kKey[ln]);
      return AM_EINVAL;
    }
    if (k != want) {
      set_err(info, ln + 1, k > want ? col[want] : l.len + 1, "Moving AI header: `%s` takes %d value(s)", kKey[ln],
              want - 1);
      return AM_EINVAL;
    }
    if (ln == 0 && tok[1] != "octile") {
      set_err(info, 1, col[1], "Moving AI header: map type must be `octile`");
      return AM_EINVAL;
    }
    if (ln == 1 || ln == 2) {
      const std::string& t = tok[1];
      uint64_t v = 0;
      for (size_t i = 0; i < t.size(); ++i) {
        if (t[i] < '0' || t[i] > '9') {
          set_err(info, ln + 1, col[1] + i, "Moving AI header: %s is not a decimal number", kKey[ln]);
          return AM_EINVAL;
        }
        v = std::min<uint64_t>(v * 10 + (uint64_t)(t[i] - '0'), 65536);  // saturate: only the range matters
      }
      if (v < 1 || v > 65535) {
        set_err(info, ln + 1, col[1], "Moving AI header: %s outside 1..65535", kKey[ln]);
        return AM_EINVAL;
      }
      dims[ln - 1] = (uint32_t)v;
    }
  }
  info->height = dims[0];
  info->width = dims[1];
  if (body_offset) *body_offset = pos;
  return AM_OK;
}

}  // extern "C"

namespace {

// text bytes -> device copy (zero-padded), newline offsets, line count
struct TextDev {
  uint8_t* text = nullptr;
  uint64_t n = 0;
  uint64_t* counts = nullptr;  // per chunk, then exclusive offsets (nchunks + 1)
  uint64_t* offs = nullptr;
  uint64_t* nl = nullptr;
  uint64_t n_nl = 0, n_lines = 0;
  unsigned long long* scal = nullptr;  // [0..2] k_line_scan, [3] error key, [4] obstacles
  void release(am_ctx* ctx) {
    am::dfree(ctx, text);
    am::dfree(ctx, counts);
    am::dfree(ctx, offs);
    am::dfree(ctx, nl);
    am::dfree(ctx, scal);
    *this = TextDev{};
  }
};

#define CKT(call)                                                                                   \
  do {                                                                                              \
    cudaError_t e_ = (call);                                                                        \
    if (e_ != cudaSuccess) {                                                                        \
      (void)cudaGetLastError();                                                                     \
      td.release(ctx);                                                                              \
      return am::fail(ctx, e_ == cudaErrorMemoryAllocation ? AM_EOOM : AM_ECUDA, "%s: %s", #call,   \
                      cudaGetErrorString(e_));                                                      \
    }                                                                                               \
  } while (0)

am_status upload_lines(am_ctx* ctx, const char* body, uint64_t n, uint64_t h_expect, TextDev& td,
                       unsigned long long scal_h[3]) {
  cudaStream_t s = ctx->stream;
  td.n = n;
  const uint64_t nchunks = std::max<uint64_t>(1, (n + am::kTextChunk - 1) / am::kTextChunk);
  CKT(am::dmalloc(ctx, &td.text, n + am::kTextPad));
  CKT(am::dmalloc(ctx, &td.counts, nchunks * 8));
  CKT(am::dmalloc(ctx, &td.offs, (nchunks + 1) * 8));
  CKT(am::dmalloc(ctx, &td.scal, 8 * 8));
  CKT(cudaMemsetAsync(td.text + n, 0, am::kTextPad, s));
  if (n) CKT(cudaMemcpyAsync(td.text, body, n, cudaMemcpyHostToDevice, s));
  am::k_newlines<false><<<(unsigned)nchunks, 256, 0, s>>>(td.text, n, td.counts, nullptr, nullptr);
  ++ctx->launches;
  am::launch_scan(td.counts, nchunks, td.offs, s);
  ++ctx->launches;
  CKT(cudaPeekAtLastError());
  CKT(cudaMemcpyAsync(&td.n_nl, td.offs + nchunks, 8, cudaMemcpyDeviceToHost, s));
  CKT(cudaStreamSynchronize(s));
  CKT(am::dmalloc(ctx, &td.nl, std::max<uint64_t>(1, td.n_nl) * 8));
  if (td.n_nl) {
    am::k_newlines<true><<<(unsigned)nchunks, 256, 0, s>>>(td.text, n, nullptr, td.offs, td.nl);
    ++ctx->launches;
  }
  // a final line without terminator counts; an empty tail after the last '\n' does not
  uint64_t last_nl = 0;
  if (td.n_nl) CKT(cudaMemcpyAsync(&last_nl, td.nl + td.n_nl - 1, 8, cudaMemcpyDeviceToHost, s));
  CKT(cudaStreamSynchronize(s));
  td.n_lines = td.n_nl + ((td.n_nl ? last_nl + 1 : 0) < n ? 1 : 0);
  const unsigned long long init[3] = {0ull, ~0ull, 0ull};
  CKT(cudaMemcpyAsync(td.scal, init, sizeof init, cudaMemcpyHostToDevice, s));
  CKT(cudaMemsetAsync(td.scal + 3, 0xFF, 8, s));
  CKT(cudaMemsetAsync(td.scal + 4, 0, 8, s));
  if (td.n_lines) {
    am::k_line_scan<<<(unsigned)((td.n_lines + 255) / 256), 256, 0, s>>>(td.text, n, td.nl, td.n_nl, td.n_lines,
                                                                          h_expect, td.scal);
    ++ctx->launches;
  }
  CKT(cudaPeekAtLastError());
  CKT(cudaMemcpyAsync(scal_h, td.scal, 3 * 8, cudaMemcpyDeviceToHost, s));
  CKT(cudaStreamSynchronize(s));
  return AM_OK;
}

void scene_free(am_ctx* ctx, am_scene* sc) {
  if (!sc) return;
  am::dfree(ctx, sc->d_occ);
  am::dfree(ctx, sc->d_src);
  am::dfree(ctx, sc->d_tgt);
  delete sc;
}

// row-kernel error key -> message
am_status row_error(am_ctx* ctx, am_parse_info* info, unsigned long long key, uint32_t W, const char* what) {
  const uint32_t line = (uint32_t)(key >> 40), col = (uint32_t)((key >> 16) & 0xffffffu);
  const uint32_t kind = (uint32_t)((key >> 8) & 0xffu), ch = (uint32_t)(key & 0xffu);
  if (kind == am::kErrChar)
    set_err(info, line, col, "%s: unexpected byte 0x%02x", what, ch);
  else if (kind == am::kErrLong)
    set_err(info, line, col, "%s: row longer than %u cells", what, W);
  else
    set_err(info, line, col, "%s: row shorter than %u cells", what, W);
  return fail(ctx, AM_EINVAL, "%s (line %u, column %u)", info->error, line, col);
}

}  // namespace

extern "C" {

am_status am_scene_parse(am_ctx* ctx, const char* text, uint64_t len, uint32_t format, am_scene** out,
                         am_parse_info* info) {
  if (!ctx || !out || (!text && len)) return AM_EINVAL;
  *out = nullptr;
  am_parse_info local{};
  if (!info) info = &local;
  *info = am_parse_info{};
  if (format != AM_FORMAT_MOVINGAI && format != AM_FORMAT_ASCII_SCENE)
    return fail(ctx, AM_EINVAL, "unknown text format %u", format);
  CK(cudaSetDevice(ctx->device));
  cudaStream_t s = ctx->stream;
  const bool mai = format == AM_FORMAT_MOVINGAI;
  uint64_t body = 0;
  uint32_t W = 0, H = 0, line_base = 1;
  if (mai) {
    const am_status st = am_movingai_header(text, len, info, &body);
    if (st) return fail(ctx, st, "%s (line %llu, column %llu)", info->error, (unsigned long long)info->error_line,
                        (unsigned long long)info->error_column);
    W = info->width;
    H = info->height;
    line_base = 5;
  }
  TextDev td;
  unsigned long long scal[3];
  if (am_status st = upload_lines(ctx, text + body, len - body, mai ? H : 0, td, scal)) return st;
  const char* what = mai ? "Moving AI map" : "ASCII scene";
  auto reject = [&](uint64_t line, uint64_t col, const char* msg) {
    set_err(info, line, col, "%s: %s", what, msg);
    td.release(ctx);
    return fail(ctx, AM_EINVAL, "%s (line %llu, column %llu)", info->error, (unsigned long long)line,
                (unsigned long long)col);
  };
  uint32_t rows_present = 0;  // rows the body holds (Moving AI: missing rows are reported after row errors)
  if (mai) {
    rows_present = (uint32_t)std::min<uint64_t>(td.n_lines, H);
  } else {
    if (scal[0] == 0) return reject(1, 1, "no rows");
    if (scal[2] == 0) return reject(1, 1, "empty first row");
    if (scal[2] > 65535) return reject(1, 65536, "row longer than 65535 cells");
    if (scal[0] > 65535) return reject(65536, 1, "more than 65535 rows");
    H = (uint32_t)scal[0];
    W = (uint32_t)scal[2];
    rows_present = H;
  }
  am_scene* sc = new (std::nothrow) am_scene();
  if (!sc) {
    td.release(ctx);
    return AM_EOOM;
  }
  sc->W = W;
  sc->H = H;
  sc->format = format;
  uint64_t* row_cnt = nullptr;  // [2][H + 1] counts, then [2][H + 1] offsets
  auto fail_sc = [&](cudaError_t e) {
    (void)cudaGetLastError();
    am::dfree(ctx, row_cnt);
    td.release(ctx);
    scene_free(ctx, sc);
    return fail(ctx, e == cudaErrorMemoryAllocation ? AM_EOOM : AM_ECUDA, "scene parse: %s", cudaGetErrorString(e));
  };
  cudaError_t e = am::dmalloc(ctx, &sc->d_occ, (size_t)W * H);
  if (!e && !mai) e = am::dmalloc(ctx, &row_cnt, (size_t)4 * (H + 1) * 8);
  if (!e && mai && rows_present < H) e = cudaMemsetAsync(sc->d_occ, 0, (size_t)W * H, s);
  if (e) return fail_sc(e);
  if (rows_present) {
    const uint64_t threads = (uint64_t)rows_present * 32;
    const unsigned blocks = (unsigned)((threads + 255) / 256);
    if (mai)
      am::k_rows<AM_FORMAT_MOVINGAI><<<blocks, 256, 0, s>>>(td.text, td.n, td.nl, td.n_nl, rows_present, W, line_base,
                                                            sc->d_occ, nullptr, nullptr, td.scal + 3, td.scal + 4);
    else
      am::k_rows<AM_FORMAT_ASCII_SCENE><<<blocks, 256, 0, s>>>(td.text, td.n, td.nl, td.n_nl, rows_present, W,
                                                               line_base, sc->d_occ, row_cnt, row_cnt + (H + 1),
                                                               td.scal + 3, td.scal + 4);
    ++ctx->launches;
  }
  unsigned long long tail[2] = {~0ull, 0};
  e = cudaPeekAtLastError();
  if (!e) e = cudaMemcpyAsync(tail, td.scal + 3, 16, cudaMemcpyDeviceToHost, s);
  if (!e) e = cudaStreamSynchronize(s);
  if (e) return fail_sc(e);
  sc->obstacles = tail[1];
  if (tail[0] != ~0ull) {
    am::dfree(ctx, row_cnt);
    scene_free(ctx, sc);
    td.release(ctx);
    return row_error(ctx, info, tail[0], W, what);
  }
  if (mai && td.n_lines < H) {
    am::dfree(ctx, row_cnt);
    scene_free(ctx, sc);
    char msg[96];
    snprintf(msg, sizeof msg, "body has %llu rows, the header says %u", (unsigned long long)td.n_lines, H);
    return reject(line_base + td.n_lines, 1, msg);
  }
  if (mai && scal[1] != ~0ull) {
    am::dfree(ctx, row_cnt);
    scene_free(ctx, sc);
    char msg[96];
    snprintf(msg, sizeof msg, "more rows than the header's height %u", H);
    return reject(line_base + scal[1], 1, msg);
  }
  if (!mai) {
    uint64_t* s_off = row_cnt + 2 * (H + 1);
    uint64_t* t_off = row_cnt + 3 * (H + 1);
    am::launch_scan(row_cnt, H, s_off, s);
    am::launch_scan(row_cnt + (H + 1), H, t_off, s);
    ctx->launches += 2;
    uint64_t tot[2] = {0, 0};
    e = cudaPeekAtLastError();
    if (!e) e = cudaMemcpyAsync(&tot[0], s_off + H, 8, cudaMemcpyDeviceToHost, s);
    if (!e) e = cudaMemcpyAsync(&tot[1], t_off + H, 8, cudaMemcpyDeviceToHost, s);
    if (!e) e = cudaStreamSynchronize(s);
    if (e) return fail_sc(e);
    sc->n_src = tot[0];
    sc->n_tgt = tot[1];
    if (!sc->n_src) {
      am::dfree(ctx, row_cnt);
      scene_free(ctx, sc);
      td.release(ctx);
      set_err(info, 0, 0, "ASCII scene: no source ('S') cell");
      return fail(ctx, AM_EINVAL, "%s", info->error);
    }
    e = am::dmalloc(ctx, &sc->d_src, sc->n_src * 8);
    if (!e && sc->n_tgt) e = am::dmalloc(ctx, &sc->d_tgt, sc->n_tgt * 8);
    if (e) return fail_sc(e);
    am::k_scene_coords<<<(unsigned)(((uint64_t)H * 32 + 255) / 256), 256, 0, s>>>(
        td.text, td.n, td.nl, td.n_nl, H, W, s_off, t_off, sc->d_src, sc->d_tgt);
    ++ctx->launches;
    e = cudaPeekAtLastError();
    if (e) return fail_sc(e);
  }
  am::dfree(ctx, row_cnt);
  td.release(ctx);
  info->width = W;
  info->height = H;
  info->n_sources = sc->n_src;
  info->n_targets = sc->n_tgt;
  info->obstacles = sc->obstacles;
  *out = sc;
  return AM_OK;
}

am_status am_scene_destroy(am_ctx* ctx, am_scene* sc) {
  if (!ctx) return AM_EINVAL;
  if (!sc) return AM_OK;
  CK(cudaSetDevice(ctx->device));
  scene_free(ctx, sc);
  return AM_OK;
}

am_status am_scene_download(am_ctx* ctx, const am_scene* sc, uint8_t* occupancy, uint32_t* src_rc, uint32_t* tgt_rc) {
  if (!ctx || !sc) return AM_EINVAL;
  CK(cudaSetDevice(ctx->device));
  cudaStream_t s = ctx->stream;
  if (occupancy) CK(cudaMemcpyAsync(occupancy, sc->d_occ, (size_t)sc->W * sc->H, cudaMemcpyDeviceToHost, s));
  if (src_rc && sc->n_src) CK(cudaMemcpyAsync(src_rc, sc->d_src, sc->n_src * 8, cudaMemcpyDeviceToHost, s));
  if (tgt_rc && sc->n_tgt) CK(cudaMemcpyAsync(tgt_rc, sc->d_tgt, sc->n_tgt * 8, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  return AM_OK;
}

am_status am_grid_create_scene(am_ctx* ctx, const am_scene* sc, const uint32_t* src_rc, uint64_t n_src,
                               am_grid** out) {
  if (!ctx || !sc || !out) return AM_EINVAL;
  if (!src_rc) {
    if (!sc->n_src) return fail(ctx, AM_EINVAL, "SourceSet must be nonempty (the map carries no sources)");
    return am_grid_create_device(ctx, sc->W, sc->H, sc->d_occ, sc->d_src, sc->n_src, out);
  }
  if (!n_src) return fail(ctx, AM_EINVAL, "SourceSet must be nonempty");
  CK(cudaSetDevice(ctx->device));
  uint32_t* d = nullptr;
  CK(am::dmalloc(ctx, &d, n_src * 8));
  cudaError_t e = cudaMemcpyAsync(d, src_rc, n_src * 8, cudaMemcpyHostToDevice, ctx->stream);
  const am_status st = e ? fail(ctx, AM_ECUDA, "source upload: %s", cudaGetErrorString(e))
                         : am_grid_create_device(ctx, sc->W, sc->H, sc->d_occ, d, n_src, out);
  am::dfree(ctx, d);
  return st;
}

// ---------------------------------------------------------------- emitters
am_status am_emit_text(am_ctx* ctx, uint32_t format, uint32_t W, uint32_t H, const uint8_t* occupancy,
                       const uint32_t* src_rc, uint64_t n_src, const uint32_t* tgt_rc, uint64_t n_tgt, char* out,
                       uint64_t capacity, uint64_t* length) {
  if (!ctx || !length || !am::dims_ok(W, H) || (!occupancy && W)) return AM_EINVAL;
  if (format != AM_FORMAT_MOVINGAI && format != AM_FORMAT_ASCII_SCENE)
    return fail(ctx, AM_EINVAL, "unknown text format %u", format);
  const bool mai = format == AM_FORMAT_MOVINGAI;
  char head[96] = "";
  if (mai) snprintf(head, sizeof head, "type octile\nheight %u\nwidth %u\nmap\n", H, W);
  const size_t hl = strlen(head);
  const uint64_t body = (uint64_t)H * (W + 1);
  *length = hl + body;
  if (!out) return AM_OK;
  if (capacity < *length) return fail(ctx, AM_EINVAL, "output buffer of %llu bytes < %llu",
                                      (unsigned long long)capacity, (unsigned long long)*length);
  // the coordinate lists must name in-bounds cells (Scene invariant)
  auto inb = [&](const uint32_t* rc, uint64_t n) {
    for (uint64_t i = 0; i < n; ++i)
      if (rc[2 * i] >= H || rc[2 * i + 1] >= W) return false;
    return true;
  };
  if (!mai && ((n_src && (!src_rc || !inb(src_rc, n_src))) || (n_tgt && (!tgt_rc || !inb(tgt_rc, n_tgt)))))
    return fail(ctx, AM_EINVAL, "scene point out of bounds");
  CK(cudaSetDevice(ctx->device));
  cudaStream_t s = ctx->stream;
  uint8_t *d_occ = nullptr, *d_txt = nullptr;
  uint32_t* d_rc = nullptr;
  const uint64_t npts = mai ? 0 : n_src + n_tgt;
  cudaError_t e = am::dmalloc(ctx, &d_occ, (size_t)W * H);
  if (!e) e = am::dmalloc(ctx, &d_txt, body);
  if (!e && npts) e = am::dmalloc(ctx, &d_rc, npts * 8);
  if (!e) e = cudaMemcpyAsync(d_occ, occupancy, (size_t)W * H, cudaMemcpyHostToDevice, s);
  if (!e && n_src && !mai) e = cudaMemcpyAsync(d_rc, src_rc, n_src * 8, cudaMemcpyHostToDevice, s);
  if (!e && n_tgt && !mai) e = cudaMemcpyAsync(d_rc + 2 * n_src, tgt_rc, n_tgt * 8, cudaMemcpyHostToDevice, s);
  if (!e) {
    am::k_emit_rows<<<am::rows_grid(W / 4 + 1, H, 128), 128, 0, s>>>(d_occ, W, H, '.', mai ? '@' : '#', d_txt);
    ++ctx->launches;
    // targets first, then sources: a cell listed as both is written 'S'
    if (!mai && n_tgt) {
      am::k_emit_marks<<<(unsigned)((n_tgt + 255) / 256), 256, 0, s>>>(d_rc + 2 * n_src, n_tgt, W, 'T', d_txt);
      ++ctx->launches;
    }
    if (!mai && n_src) {
      am::k_emit_marks<<<(unsigned)((n_src + 255) / 256), 256, 0, s>>>(d_rc, n_src, W, 'S', d_txt);
      ++ctx->launches;
    }
    e = cudaPeekAtLastError();
  }
  memcpy(out, head, hl);
  if (!e) e = cudaMemcpyAsync(out + hl, d_txt, body, cudaMemcpyDeviceToHost, s);
  if (!e) e = cudaStreamSynchronize(s);
  am::dfree(ctx, d_occ);
  am::dfree(ctx, d_txt);
  am::dfree(ctx, d_rc);
  if (e) {
    (void)cudaGetLastError();
    return fail(ctx, AM_ECUDA, "emit: %s", cudaGetErrorString(e));
  }
  return AM_OK;
}

}  // extern "C"

// ---------------------------------------------------------------- PGM export
namespace {

am_status pgm_impl(am_ctx* ctx, const am::Geo& geo, int cb, const void* val, uint32_t rollback, uint8_t* out,
                   uint64_t capacity, uint64_t* length) {
  cudaStream_t s = ctx->stream;
  uint32_t* d_max = nullptr;
  CK(am::dmalloc(ctx, &d_max, 4));
  uint32_t mx = 0;
  cudaError_t e = cudaMemsetAsync(d_max, 0, 4, s);
  if (!e) {
    const dim3 grid((geo.W + 1023) / 1024, geo.H);
    if (cb == 0) am::k_map_max<0><<<grid, 256, 0, s>>>(geo, val, rollback, d_max);
    else if (cb == 16) am::k_map_max<16><<<grid, 256, 0, s>>>(geo, val, rollback, d_max);
    else am::k_map_max<32><<<grid, 256, 0, s>>>(geo, val, rollback, d_max);
    ++ctx->launches;
    e = cudaPeekAtLastError();
  }
  if (!e) e = cudaMemcpyAsync(&mx, d_max, 4, cudaMemcpyDeviceToHost, s);
  if (!e) e = cudaStreamSynchronize(s);
  am::dfree(ctx, d_max);
  if (e) {
    (void)cudaGetLastError();
    return fail(ctx, AM_ECUDA, "pgm max: %s", cudaGetErrorString(e));
  }
  const uint32_t maxval = mx > 255 ? 65535u : 255u;  // mapio.hpp:35-36
  char head[64];
  snprintf(head, sizeof head, "P5\n%u %u\n%u\n", geo.W, geo.H, maxval);
  const size_t hl = strlen(head);
  const uint64_t body = (uint64_t)geo.W * geo.H * (maxval == 255 ? 1 : 2);
  *length = hl + body;
  if (!out) return AM_OK;
  if (capacity < *length)
    return fail(ctx, AM_EINVAL, "output buffer of %llu bytes < %llu", (unsigned long long)capacity,
                (unsigned long long)*length);
  uint8_t* d_out = nullptr;
  CK(am::dmalloc(ctx, &d_out, body));
  const dim3 grid = am::rows_grid(geo.W, geo.H, 256);
  if (cb == 0) am::k_pgm<0><<<grid, 256, 0, s>>>(geo, val, rollback, mx, maxval, d_out);
  else if (cb == 16) am::k_pgm<16><<<grid, 256, 0, s>>>(geo, val, rollback, mx, maxval, d_out);
  else am::k_pgm<32><<<grid, 256, 0, s>>>(geo, val, rollback, mx, maxval, d_out);
  ++ctx->launches;
  e = cudaPeekAtLastError();
  memcpy(out, head, hl);
  if (!e) e = cudaMemcpyAsync(out + hl, d_out, body, cudaMemcpyDeviceToHost, s);
  if (!e) e = cudaStreamSynchronize(s);
  am::dfree(ctx, d_out);
  if (e) {
    (void)cudaGetLastError();
    return fail(ctx, AM_ECUDA, "pgm: %s", cudaGetErrorString(e));
  }
  return AM_OK;
}

}  // namespace

extern "C" {

am_status am_activity_export_pgm(am_ctx* ctx, am_grid* g, uint8_t* out, uint64_t capacity, uint64_t* length) {
  if (!ctx || !g || !length) return AM_EINVAL;
  if (!g->have_map) return fail(ctx, AM_EINVAL, "no activity map: call am_propagate first");
  if (g->slab) return fail(ctx, AM_EINVAL, "PGM export of a slab grid: gather it first");
  CK(cudaSetDevice(ctx->device));
  if (am_status jst = am::join_map(ctx, g)) return jst;
  if (g->plain_active) return pgm_impl(ctx, g->g, 0, g->plain, 0, out, capacity, length);
  return pgm_impl(ctx, g->g, g->cell_bits, g->val[g->cur], g->computed - g->layers_used, out, capacity, length);
}

am_status am_export_pgm(am_ctx* ctx, uint32_t W, uint32_t H, const uint32_t* values, uint8_t* out,
                        uint64_t capacity, uint64_t* length) {
  if (!ctx || !length || !values || !am::dims_ok(W, H)) return AM_EINVAL;
  CK(cudaSetDevice(ctx->device));
  am::Geo geo{};
  geo.W = W;
  geo.H = H;
  uint32_t* d = nullptr;
  CK(am::dmalloc(ctx, &d, (size_t)W * H * 4));
  cudaError_t e = cudaMemcpyAsync(d, values, (size_t)W * H * 4, cudaMemcpyHostToDevice, ctx->stream);
  const am_status st = e ? fail(ctx, AM_ECUDA, "pgm upload: %s", cudaGetErrorString(e))
                         : pgm_impl(ctx, geo, 0, d, 0, out, capacity, length);
  am::dfree(ctx, d);
  return st;
}

}  // extern "C"
