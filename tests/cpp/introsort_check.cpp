// Host check: sg::isort::sort reproduces libstdc++ std::sort with a
// key-only comparator (the scipy csr_sort_indices order), including the
// heap-sort fallback.
#include "../../paper_2604_26441_b200/csrc/sg_introsort.cuh"
#include <algorithm>
#include <cstdio>
#include <random>
#include <vector>

int main() {
  std::mt19937 rng(12345);
  long bad = 0, total = 0;
  auto cmp = [](uint16_t x, uint16_t y) { return (x >> 8) < (y >> 8); };
  for (int trial = 0; trial < 100000; ++trial) {
    int n = rng() % 260;
    int nk = 1 + rng() % 90;
    std::vector<uint16_t> a(n);
    for (int i = 0; i < n; ++i) a[i] = uint16_t(((rng() % nk) << 8) | (i & 255));
    if (trial % 5 == 1) std::sort(a.begin(), a.end());
    if (trial % 5 == 2) std::reverse(a.begin(), a.end());
    std::vector<uint16_t> b = a;
    std::sort(a.begin(), a.end(), cmp);
    sg::isort::sort(b.data(), n);
    ++total;
    bad += (a != b);
  }
  for (int trial = 0; trial < 20000; ++trial) {  // heap fallback in isolation
    int n = 1 + rng() % 200;
    std::vector<uint16_t> a(n);
    for (int i = 0; i < n; ++i) a[i] = uint16_t(((rng() % 20) << 8) | (i & 255));
    std::vector<uint16_t> b = a;
    std::make_heap(a.begin(), a.end(), cmp);
    std::sort_heap(a.begin(), a.end(), cmp);
    sg::isort::heap_sort(b.data(), n);
    ++total;
    bad += (a != b);
  }
  printf("introsort mismatches %ld / %ld\n", bad, total);
  return bad != 0;
}
