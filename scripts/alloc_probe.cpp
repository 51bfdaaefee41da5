// Host allocation cost of a 10M-element std::vector<std::complex<double>>
// result (160 MB): fresh mmap (default), heap-recycled (M_MMAP_THRESHOLD),
// and transparent huge pages (madvise before first touch).
#include <malloc.h>
#include <sys/mman.h>
#include <chrono>
#include <complex>
#include <cstdio>
#include <cstring>
#include <vector>
using cplx = std::complex<double>;
static double ms(std::chrono::steady_clock::time_point a) {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - a).count();
}
int main() {
  const size_t n = 10000000;
  for (int r = 0; r < 3; ++r) {
    auto t = std::chrono::steady_clock::now();
    std::vector<cplx> v(n);
    printf("default  rep %d: %.1f ms\n", r, ms(t));
  }
  for (int r = 0; r < 3; ++r) {
    auto t = std::chrono::steady_clock::now();
    std::vector<cplx> v;
    v.reserve(n);
    char* b = reinterpret_cast<char*>(v.data());
    char* a0 = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(b) + (2u << 20) - 1) & ~uintptr_t((2u << 20) - 1));
    madvise(a0, (n * 16 - (a0 - b)) & ~size_t((2u << 20) - 1), MADV_HUGEPAGE);
    v.resize(n);
    printf("thp      rep %d: %.1f ms\n", r, ms(t));
  }
  mallopt(M_MMAP_THRESHOLD, 1 << 30);
  mallopt(M_TRIM_THRESHOLD, 1 << 30);
  for (int r = 0; r < 3; ++r) {
    auto t = std::chrono::steady_clock::now();
    std::vector<cplx> v(n);
    printf("heap     rep %d: %.1f ms\n", r, ms(t));
  }
  return 0;
}
