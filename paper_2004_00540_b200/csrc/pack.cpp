// pack.cpp -- host side of the packed occupancy upload (upload.cu): one byte per cell
// (grid.hpp:56, nonzero = obstacle, grid.hpp:20) to one bit per cell, 32 cells per word.  The widest
// vector compare the host CPU has is picked at run time (AVX-512BW: one test-mask per 64 bytes; AVX2: a
// compare + movemask per 32; SSE2 otherwise); AM_PACK_ISA=sse2|avx2|avx512 forces one.
#include <immintrin.h>

#include <cstdint>
#include <cstdlib>
#include <cstring>

namespace am {

namespace {

inline uint32_t tail_word(const uint8_t* row, uint32_t c0, uint32_t W) {
  uint32_t v = 0;
  for (uint32_t c = c0; c < W; ++c) v |= (row[c] != 0 ? 1u : 0u) << (c & 31);
  return v;
}

void pack_sse2(const uint8_t* occ, uint32_t W, uint32_t r0, uint32_t r1, uint32_t pw, uint32_t* out) {
  const __m128i z = _mm_setzero_si128();
  const uint32_t full = W / 32;
  for (uint32_t r = r0; r < r1; ++r) {
    const uint8_t* row = occ + (size_t)r * W;
    uint32_t* o = out + (size_t)(r - r0) * pw;
    for (uint32_t w = 0; w < full; ++w) {
      const __m128i a = _mm_loadu_si128(reinterpret_cast<const __m128i*>(row + 32 * w));
      const __m128i b = _mm_loadu_si128(reinterpret_cast<const __m128i*>(row + 32 * w + 16));
      const uint32_t fa = (uint32_t)_mm_movemask_epi8(_mm_cmpeq_epi8(a, z));  // 1: free
      const uint32_t fb = (uint32_t)_mm_movemask_epi8(_mm_cmpeq_epi8(b, z));
      o[w] = ~(fa | fb << 16);
    }
    if (full < pw) o[full] = tail_word(row, 32 * full, W);
  }
}

__attribute__((target("avx2"))) void pack_avx2(const uint8_t* occ, uint32_t W, uint32_t r0, uint32_t r1,
                                                uint32_t pw, uint32_t* out) {
  const __m256i z = _mm256_setzero_si256();
  const uint32_t full = W / 32;
  for (uint32_t r = r0; r < r1; ++r) {
    const uint8_t* row = occ + (size_t)r * W;
    uint32_t* o = out + (size_t)(r - r0) * pw;
    for (uint32_t w = 0; w < full; ++w) {
      const __m256i a = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(row + 32 * w));
      o[w] = ~(uint32_t)_mm256_movemask_epi8(_mm256_cmpeq_epi8(a, z));
    }
    if (full < pw) o[full] = tail_word(row, 32 * full, W);
  }
}

__attribute__((target("avx2,avx512f,avx512bw"))) void pack_avx512(const uint8_t* occ, uint32_t W, uint32_t r0,
                                                              uint32_t r1, uint32_t pw, uint32_t* out) {
  const uint32_t full = W / 32, pairs = full / 2;
  for (uint32_t r = r0; r < r1; ++r) {
    const uint8_t* row = occ + (size_t)r * W;
    uint32_t* o = out + (size_t)(r - r0) * pw;
    for (uint32_t p = 0; p < pairs; ++p) {
      const __m512i a = _mm512_loadu_si512(row + 64 * p);
      const uint64_t m = _mm512_test_epi8_mask(a, a);  // 1: nonzero byte = obstacle
      std::memcpy(o + 2 * p, &m, 8);
    }
    if (2 * pairs < full) {
      const __m256i a = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(row + 64 * pairs));
      o[2 * pairs] = ~(uint32_t)_mm256_movemask_epi8(_mm256_cmpeq_epi8(a, _mm256_setzero_si256()));
    }
    if (full < pw) o[full] = tail_word(row, 32 * full, W);
  }
}

using PackFn = void (*)(const uint8_t*, uint32_t, uint32_t, uint32_t, uint32_t, uint32_t*);

int pick_isa() {  // 0 sse2, 1 avx2, 2 avx512
  const char* e = getenv("AM_PACK_ISA");
  __builtin_cpu_init();
  const bool has512 = __builtin_cpu_supports("avx512bw") && __builtin_cpu_supports("avx512f");
  const bool has2 = __builtin_cpu_supports("avx2");
  if (e && !strcmp(e, "sse2")) return 0;
  if (e && !strcmp(e, "avx2") && has2) return 1;
  if (e && !strcmp(e, "avx512") && has512) return 2;
  return has512 ? 2 : has2 ? 1 : 0;
}

}  // namespace

int pack_isa() {
  static const int isa = pick_isa();
  return isa;
}

// Packs rows [r0, r1) of a W-wide byte grid: bit c of word w of a row is 1 if cell 32w + c is an obstacle
// (nonzero byte); bits past W are 0.  pw words per packed row.
void pack_rows(const uint8_t* occ, uint32_t W, uint32_t r0, uint32_t r1, uint32_t pw, uint32_t* out) {
  static const PackFn fn = pack_isa() == 2 ? pack_avx512 : pack_isa() == 1 ? pack_avx2 : pack_sse2;
  fn(occ, W, r0, r1, pw, out);
}

}  // namespace am
