// Exact emulation of libstdc++'s std::sort (introsort, median-of-3 pivot,
// threshold 16, heap-sort fallback, final insertion sort) on an array of
// uint16 items compared by their high byte only.
//
// scipy's csr_sort_indices sorts (column, value) pairs with std::sort and a
// key-only comparator (kv_pair_less); the order in which equal-column
// duplicates end up -- and therefore the summation order of
// csr_sum_duplicates -- is a deterministic function of the key sequence.
// Reproducing it is what makes the level-1 Galerkin operator bit-identical
// to the reference's canonical_csr(coo) (transfer.py:33-39, :166-174).
// Mirrors bits/stl_algo.h and bits/stl_heap.h (GCC 13).
#pragma once
#include <cstdint>

#ifndef __CUDACC__
#ifndef __host__
#define __host__
#endif
#ifndef __device__
#define __device__
#endif
#ifndef __forceinline__
#define __forceinline__ inline
#endif
#endif

namespace sg {
namespace isort {

using Item = uint16_t;

__host__ __device__ __forceinline__ bool lt(Item a, Item b) { return (a >> 8) < (b >> 8); }
__host__ __device__ __forceinline__ void swp(Item* v, int a, int b) {
  Item t = v[a];
  v[a] = v[b];
  v[b] = t;
}

__host__ __device__ inline void push_heap(Item* f, int hole, int top, Item value) {
  int parent = (hole - 1) / 2;
  while (hole > top && lt(f[parent], value)) {
    f[hole] = f[parent];
    hole = parent;
    parent = (hole - 1) / 2;
  }
  f[hole] = value;
}

__host__ __device__ inline void adjust_heap(Item* f, int hole, int len, Item value) {
  const int top = hole;
  int second = hole;
  while (second < (len - 1) / 2) {
    second = 2 * (second + 1);
    if (lt(f[second], f[second - 1])) second--;
    f[hole] = f[second];
    hole = second;
  }
  if ((len & 1) == 0 && second == (len - 2) / 2) {
    second = 2 * (second + 1);
    f[hole] = f[second - 1];
    hole = second - 1;
  }
  push_heap(f, hole, top, value);
}

__host__ __device__ inline void heap_sort(Item* f, int n) {
  if (n >= 2) {  // make_heap
    int parent = (n - 2) / 2;
    while (true) {
      adjust_heap(f, parent, n, f[parent]);
      if (parent == 0) break;
      parent--;
    }
  }
  int last = n;
  while (last > 1) {  // sort_heap
    --last;
    Item value = f[last];
    f[last] = f[0];
    adjust_heap(f, 0, last, value);
  }
}

__host__ __device__ inline void move_median_to_first(Item* v, int r, int a, int b, int c) {
  if (lt(v[a], v[b])) {
    if (lt(v[b], v[c])) swp(v, r, b);
    else if (lt(v[a], v[c])) swp(v, r, c);
    else swp(v, r, a);
  } else if (lt(v[a], v[c])) {
    swp(v, r, a);
  } else if (lt(v[b], v[c])) {
    swp(v, r, c);
  } else {
    swp(v, r, b);
  }
}

__host__ __device__ inline int unguarded_partition(Item* v, int first, int last, int pivot) {
  while (true) {
    while (lt(v[first], v[pivot])) ++first;
    --last;
    while (lt(v[pivot], v[last])) --last;
    if (!(first < last)) return first;
    swp(v, first, last);
    ++first;
  }
}

__host__ __device__ inline void unguarded_linear_insert(Item* v, int last) {
  Item val = v[last];
  int next = last - 1;
  while (lt(val, v[next])) {
    v[last] = v[next];
    last = next;
    --next;
  }
  v[last] = val;
}

__host__ __device__ inline void insertion_sort(Item* v, int first, int last) {
  if (first == last) return;
  for (int i = first + 1; i != last; ++i) {
    if (lt(v[i], v[first])) {
      Item val = v[i];
      for (int q = i; q > first; --q) v[q] = v[q - 1];
      v[first] = val;
    } else {
      unguarded_linear_insert(v, i);
    }
  }
}

__host__ __device__ inline int lg(int n) {
  int r = 0;
  while (n > 1) {
    n >>= 1;
    ++r;
  }
  return r;
}

// std::sort(v, v + n, key-only comparator).  Sub-ranges produced by a
// partition are disjoint, so processing them from an explicit stack yields
// exactly the recursive __introsort_loop result.
__host__ __device__ inline void sort(Item* v, int n) {
  if (n <= 0) return;
  int st_first[64], st_last[64], st_depth[64];
  int sp = 0;
  st_first[0] = 0;
  st_last[0] = n;
  st_depth[0] = lg(n) * 2;
  sp = 1;
  while (sp > 0) {
    --sp;
    const int first = st_first[sp];
    int last = st_last[sp];
    int depth = st_depth[sp];
    while (last - first > 16) {
      if (depth == 0) {
        heap_sort(v + first, last - first);
        break;
      }
      --depth;
      const int mid = first + (last - first) / 2;
      move_median_to_first(v, first, first + 1, mid, last - 1);
      const int cut = unguarded_partition(v, first + 1, last, first);
      st_first[sp] = cut;
      st_last[sp] = last;
      st_depth[sp] = depth;
      ++sp;
      last = cut;
    }
  }
  if (n > 16) {  // __final_insertion_sort
    insertion_sort(v, 0, 16);
    for (int i = 16; i != n; ++i) unguarded_linear_insert(v, i);
  } else {
    insertion_sort(v, 0, n);
  }
}

}  // namespace isort
}  // namespace sg
