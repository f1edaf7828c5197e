// fvb_hostcopy.cpp -- see fvb_hostcopy.h.  Host code only (g++).
#include "fvb_hostcopy.h"

#include <immintrin.h>

#include <cstring>

namespace fvb {
namespace {

constexpr size_t kStreamMin = 64 * 1024;  // below this, plain stores (cache-resident)

bool has_avx2() {
    static const bool v = __builtin_cpu_supports("avx2");
    return v;
}

__attribute__((target("avx2"))) void stream_copy(char* d, const char* s, size_t n) {
    size_t head = (32 - (reinterpret_cast<uintptr_t>(d) & 31)) & 31;
    if (head > n) head = n;
    std::memcpy(d, s, head);
    d += head;
    s += head;
    n -= head;
    size_t i = 0;
    for (; i + 128 <= n; i += 128) {
        const __m256i a = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(s + i));
        const __m256i b = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(s + i + 32));
        const __m256i c = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(s + i + 64));
        const __m256i e = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(s + i + 96));
        _mm256_stream_si256(reinterpret_cast<__m256i*>(d + i), a);
        _mm256_stream_si256(reinterpret_cast<__m256i*>(d + i + 32), b);
        _mm256_stream_si256(reinterpret_cast<__m256i*>(d + i + 64), c);
        _mm256_stream_si256(reinterpret_cast<__m256i*>(d + i + 96), e);
    }
    std::memcpy(d + i, s + i, n - i);
    _mm_sfence();  // streaming stores are weakly ordered: drain before returning
}

void plain_fill(char* d, uint64_t bits, size_t width, size_t n) {
    if (bits == 0) {
        std::memset(d, 0, n);
        return;
    }
    for (size_t i = 0; i + width <= n; i += width) std::memcpy(d + i, &bits, width);
}

__attribute__((target("avx2"))) void stream_fill(char* d, uint64_t bits, size_t width, size_t n) {
    if (reinterpret_cast<uintptr_t>(d) % width) {  // the vector pattern needs element alignment
        plain_fill(d, bits, width, n);
        return;
    }
    size_t head = (32 - (reinterpret_cast<uintptr_t>(d) & 31)) & 31;  // a multiple of width
    if (head > n) head = n;
    plain_fill(d, bits, width, head);
    d += head;
    n -= head;
    const __m256i v = width == 8 ? _mm256_set1_epi64x(static_cast<long long>(bits))
                                 : _mm256_set1_epi32(static_cast<int>(static_cast<uint32_t>(bits)));
    size_t i = 0;
    for (; i + 128 <= n; i += 128) {
        _mm256_stream_si256(reinterpret_cast<__m256i*>(d + i), v);
        _mm256_stream_si256(reinterpret_cast<__m256i*>(d + i + 32), v);
        _mm256_stream_si256(reinterpret_cast<__m256i*>(d + i + 64), v);
        _mm256_stream_si256(reinterpret_cast<__m256i*>(d + i + 96), v);
    }
    plain_fill(d + i, bits, width, n - i);
    _mm_sfence();
}

}  // namespace

void host_copy(char* dst, const char* src, size_t n) {
    if (n >= kStreamMin && has_avx2())
        stream_copy(dst, src, n);
    else
        std::memcpy(dst, src, n);
}

void host_fill(char* dst, uint64_t bits, size_t width, size_t n) {
    if (n >= kStreamMin && has_avx2())
        stream_fill(dst, bits, width, n);
    else
        plain_fill(dst, bits, width, n);
}

}  // namespace fvb
