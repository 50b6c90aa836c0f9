// Host-side u64 -> int32 narrowing for pinned uploads (runtime.cu ring_upload).
// The link, not the GPU, bounds a host-buffer solve (DESIGN.md §3 e2e): host
// threads narrow part of in_src to 4 B per edge while the DMA engine moves the
// rest raw.  AVX-512 VPMOVQD + unsigned compare + non-temporal stores: the
// pinned staging buffer is written without being read first (no RFO), which
// leaves host DRAM bandwidth to the concurrent DMA.
#include <immintrin.h>
#include <omp.h>

#include <cstdint>

namespace {

__attribute__((target("avx512f"))) int narrow_avx512(const uint64_t* in, int32_t* out, int64_t begin,
                                                     int64_t end, uint64_t bound) {
  const __m512i vb = _mm512_set1_epi64((long long)bound);
  __mmask8 bad = 0;
  int64_t i = begin;
  for (; i < end && ((uintptr_t)(out + i) & 31); ++i) bad |= in[i] >= bound, out[i] = (int32_t)in[i];
  for (; i + 16 <= end; i += 16) {
    const __m512i a = _mm512_loadu_si512(in + i);
    const __m512i b = _mm512_loadu_si512(in + i + 8);
    bad |= _mm512_cmpge_epu64_mask(a, vb) | _mm512_cmpge_epu64_mask(b, vb);
    _mm256_stream_si256(reinterpret_cast<__m256i*>(out + i), _mm512_cvtepi64_epi32(a));
    _mm256_stream_si256(reinterpret_cast<__m256i*>(out + i + 8), _mm512_cvtepi64_epi32(b));
  }
  for (; i < end; ++i) bad |= in[i] >= bound, out[i] = (int32_t)in[i];
  _mm_sfence();  // streaming stores visible before the DMA reads the buffer
  return bad != 0;
}

int narrow_scalar(const uint64_t* in, int32_t* out, int64_t begin, int64_t end, uint64_t bound) {
  int bad = 0;
  for (int64_t i = begin; i < end; ++i) {
    bad |= in[i] >= bound ? 1 : 0;
    out[i] = (int32_t)in[i];
  }
  return bad;
}

}  // namespace

namespace fprb {

// out[i] = (int32)in[i] for i < count; returns true if any in[i] >= bound.
bool host_narrow_ids(const uint64_t* in, int32_t* out, int64_t count, uint64_t bound) {
  static const bool avx512 = __builtin_cpu_supports("avx512f");
  int bad = 0;
#pragma omp parallel reduction(| : bad)
  {
    const int nt = omp_get_num_threads(), t = omp_get_thread_num();
    // 64-element aligned slices so every thread's stores start 32-B aligned
    const int64_t blocks = (count + 63) / 64;
    const int64_t b0 = blocks * t / nt, b1 = blocks * (t + 1) / nt;
    const int64_t lo = b0 * 64, hi = b1 * 64 < count ? b1 * 64 : count;
    if (lo < hi) bad |= avx512 ? narrow_avx512(in, out, lo, hi, bound) : narrow_scalar(in, out, lo, hi, bound);
  }
  return bad != 0;
}

}  // namespace fprb
