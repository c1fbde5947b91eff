// Host-side narrowing of int32 count rows into the narrowest wire storage
// (GNB_X_U4 nibbles / GNB_X_U8 / GNB_X_U16) for the host pipeline
// (predict_host_impl in api.cu).  The e2e path on int32 host buffers is bound
// by how fast host threads can read the int32 rows, so the row loop is
// explicit AVX2 (runtime-dispatched) with a scalar fallback; both write the
// same bytes.  Returns whether every count of rows [r0, r1) fits BITS bits
// (negative counts never fit).  Pitch padding of each output row is zeroed.
#include <cstdint>
#include <cstdlib>
#include <cstring>

#if defined(__x86_64__)
#include <immintrin.h>
#endif

namespace gnb {

namespace {

template <int BITS>
bool narrow_scalar(const int32_t* s, int32_t F, int64_t ldx, uint8_t* d, int64_t dpitch,
                   int64_t r0, int64_t r1, int32_t j0) {
  uint32_t acc = 0;
  for (int64_t r = r0; r < r1; ++r) {
    const int32_t* a = s + r * ldx;
    uint8_t* o = d + r * dpitch;
    if constexpr (BITS == 4) {
      int32_t j = j0;
      for (; j + 1 < F; j += 2) {
        const uint32_t lo = static_cast<uint32_t>(a[j]), hi = static_cast<uint32_t>(a[j + 1]);
        acc |= lo | hi;
        o[j / 2] = static_cast<uint8_t>(lo | (hi << 4));
      }
      if (j < F) {
        const uint32_t lo = static_cast<uint32_t>(a[j]);
        acc |= lo;
        o[j / 2] = static_cast<uint8_t>(lo);
      }
      const int64_t used = (F + 1) / 2;
      if (dpitch > used) std::memset(o + used, 0, static_cast<size_t>(dpitch - used));
    } else if constexpr (BITS == 8) {
      for (int32_t j = j0; j < F; ++j) {
        const uint32_t v = static_cast<uint32_t>(a[j]);
        acc |= v;
        o[j] = static_cast<uint8_t>(v);
      }
      if (dpitch > F) std::memset(o + F, 0, static_cast<size_t>(dpitch - F));
    } else {
      uint16_t* o16 = reinterpret_cast<uint16_t*>(o);
      for (int32_t j = j0; j < F; ++j) {
        const uint32_t v = static_cast<uint32_t>(a[j]);
        acc |= v;
        o16[j] = static_cast<uint16_t>(v);
      }
      if (dpitch > 2 * int64_t(F)) std::memset(o + 2 * int64_t(F), 0, static_cast<size_t>(dpitch - 2 * int64_t(F)));
    }
  }
  return (acc >> BITS) == 0;
}

#if defined(__x86_64__)
// 16 counts per step: OR-accumulate (for the fit check), pack with unsigned
// saturation (exact for counts that fit; anything else fails the check).
template <int BITS>
__attribute__((target("avx2"))) bool narrow_avx2(const int32_t* s, int32_t F, int64_t ldx,
                                                 uint8_t* d, int64_t dpitch, int64_t r0,
                                                 int64_t r1) {
  const int32_t F16 = F / 16 * 16;
  __m256i acc = _mm256_setzero_si256();
  const __m128i nib = _mm_set1_epi16(0x1001);  // maddubs weights (1, 16) per byte pair
  for (int64_t r = r0; r < r1; ++r) {
    const int32_t* a = s + r * ldx;
    uint8_t* o = d + r * dpitch;
    for (int32_t j = 0; j < F16; j += 16) {
      const __m256i x0 = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(a + j));
      const __m256i x1 = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(a + j + 8));
      acc = _mm256_or_si256(acc, _mm256_or_si256(x0, x1));
      // [x0 0-3, x1 0-3, x0 4-7, x1 4-7] as u16 -> in order
      const __m256i w = _mm256_permute4x64_epi64(_mm256_packus_epi32(x0, x1), 0xD8);
      if constexpr (BITS == 16) {
        _mm256_storeu_si256(reinterpret_cast<__m256i*>(o + 2 * j), w);
      } else {
        const __m128i b = _mm_packus_epi16(_mm256_castsi256_si128(w),
                                           _mm256_extracti128_si256(w, 1));
        if constexpr (BITS == 8) {
          _mm_storeu_si128(reinterpret_cast<__m128i*>(o + j), b);
        } else {
          const __m128i p = _mm_maddubs_epi16(b, nib);  // e0 + 16 e1 per pair (< 256)
          _mm_storel_epi64(reinterpret_cast<__m128i*>(o + j / 2), _mm_packus_epi16(p, p));
        }
      }
    }
    if (F16 < F && !narrow_scalar<BITS>(s, F, ldx, d, dpitch, r, r + 1, F16)) return false;
    if (F16 == F) {  // pitch padding (the scalar tail zeroes it otherwise)
      const int64_t used = BITS == 4 ? (F + 1) / 2 : BITS == 8 ? F : 2 * int64_t(F);
      if (dpitch > used) std::memset(o + used, 0, static_cast<size_t>(dpitch - used));
    }
  }
  alignas(32) uint32_t lanes[8];
  _mm256_store_si256(reinterpret_cast<__m256i*>(lanes), acc);
  uint32_t all = 0;
  for (uint32_t v : lanes) all |= v;
  return (all >> BITS) == 0;
}

// 16 counts per step with AVX-512: saturating down-conversion (vpmovusdb /
// vpmovusdw) straight from the 512-bit load.
template <int BITS>
__attribute__((target("avx512f,avx512bw"))) bool narrow_avx512(const int32_t* s, int32_t F,
                                                               int64_t ldx, uint8_t* d,
                                                               int64_t dpitch, int64_t r0,
                                                               int64_t r1) {
  const int32_t F16 = F / 16 * 16;
  __m512i acc = _mm512_setzero_si512();
  const __m128i nib = _mm_set1_epi16(0x1001);
  for (int64_t r = r0; r < r1; ++r) {
    const int32_t* a = s + r * ldx;
    uint8_t* o = d + r * dpitch;
    for (int32_t j = 0; j < F16; j += 16) {
      const __m512i x = _mm512_loadu_si512(a + j);
      acc = _mm512_or_si512(acc, x);
      if constexpr (BITS == 16) {
        _mm256_storeu_si256(reinterpret_cast<__m256i*>(o + 2 * j), _mm512_cvtusepi32_epi16(x));
      } else {
        const __m128i b = _mm512_cvtusepi32_epi8(x);
        if constexpr (BITS == 8) {
          _mm_storeu_si128(reinterpret_cast<__m128i*>(o + j), b);
        } else {
          const __m128i p = _mm_maddubs_epi16(b, nib);
          _mm_storel_epi64(reinterpret_cast<__m128i*>(o + j / 2), _mm_packus_epi16(p, p));
        }
      }
    }
    if (F16 < F && !narrow_scalar<BITS>(s, F, ldx, d, dpitch, r, r + 1, F16)) return false;
    if (F16 == F) {
      const int64_t used = BITS == 4 ? (F + 1) / 2 : BITS == 8 ? F : 2 * int64_t(F);
      if (dpitch > used) std::memset(o + used, 0, static_cast<size_t>(dpitch - used));
    }
  }
  return (static_cast<uint32_t>(_mm512_reduce_or_epi32(acc)) >> BITS) == 0;
}

bool have_avx2() {
  static const bool v = __builtin_cpu_supports("avx2");
  return v;
}

// GNB_NARROW_ISA=avx2 / scalar: force a narrower instruction set (A/B)
int isa() {
  static const int v = [] {
    const char* e = getenv("GNB_NARROW_ISA");
    if (e && !strcmp(e, "scalar")) return 0;
    if (__builtin_cpu_supports("avx512bw") && !(e && !strcmp(e, "avx2"))) return 2;
    return have_avx2() ? 1 : 0;
  }();
  return v;
}
#endif

}  // namespace

bool narrow_rows_block(int bits, const int32_t* s, int32_t F, int64_t ldx, uint8_t* d,
                       int64_t dpitch, int64_t r0, int64_t r1) {
#if defined(__x86_64__)
  const int level = isa();
  if (level == 2) {
    switch (bits) {
      case 4: return narrow_avx512<4>(s, F, ldx, d, dpitch, r0, r1);
      case 8: return narrow_avx512<8>(s, F, ldx, d, dpitch, r0, r1);
      default: return narrow_avx512<16>(s, F, ldx, d, dpitch, r0, r1);
    }
  }
  if (level == 1) {
    switch (bits) {
      case 4: return narrow_avx2<4>(s, F, ldx, d, dpitch, r0, r1);
      case 8: return narrow_avx2<8>(s, F, ldx, d, dpitch, r0, r1);
      default: return narrow_avx2<16>(s, F, ldx, d, dpitch, r0, r1);
    }
  }
#endif
  switch (bits) {
    case 4: return narrow_scalar<4>(s, F, ldx, d, dpitch, r0, r1, 0);
    case 8: return narrow_scalar<8>(s, F, ldx, d, dpitch, r0, r1, 0);
    default: return narrow_scalar<16>(s, F, ldx, d, dpitch, r0, r1, 0);
  }
}

}  // namespace gnb
