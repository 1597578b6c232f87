// gapkit_b200: a fresh std::vector<T>(n) whose pages are faulted in by
// several threads before the (serial) value-initialisation.
//
// The reference's surface returns results by value as std::vector
// (ParentArray, types.hpp:20), so every call builds an n-entry vector.  On
// the GPU box's host, value-initialising 0.5 GB (kron27's ParentArray)
// through one thread's page faults costs ~184 ms; touching one byte per page
// from 16 threads first and then resizing costs ~57 ms
// (tools/bench_mem/hostcopy.cu).  The result is an ordinary
// std::vector<T>(n) of value-initialised elements.  Used by both
// gapkit::Bfs (bfs.hpp) and gapkit::b200::Bfs (ref_binding.hpp), so it
// depends on nothing but the standard library.
#ifndef GAPKIT_B200_FRESH_VECTOR_HPP_
#define GAPKIT_B200_FRESH_VECTOR_HPP_

#include <algorithm>
#include <cstddef>
#include <thread>
#include <type_traits>
#include <vector>

namespace gk_host {

template <class T>
std::vector<T> FreshVector(size_t n) {
  static_assert(std::is_trivial_v<T>, "pages are touched before the elements exist");
  std::vector<T> v;
  const size_t bytes = n * sizeof(T);
  if (bytes < (size_t(64) << 20)) {  // small arrays: faults are cheap, threads are not
    v.resize(n);
    return v;
  }
  v.reserve(n);
  const unsigned hw = std::thread::hardware_concurrency();
  const unsigned nt = std::max(1u, std::min(16u, hw ? hw : 1u));
  // Write one byte per 4 KiB page of the reserved (not yet constructed)
  // storage; the first write is what maps the page.  T is trivial, and the
  // resize below value-initialises every element afterwards.
  volatile char* base = reinterpret_cast<volatile char*>(v.data());
  std::vector<std::thread> pool;
  for (unsigned t = 0; t < nt; t++)
    pool.emplace_back([=] {
      const size_t lo = (bytes * t / nt) & ~size_t(4095), hi = bytes * (t + 1) / nt;
      for (size_t o = lo; o < hi; o += 4096) base[o] = 0;
    });
  for (auto& th : pool) th.join();
  v.resize(n);
  return v;
}

}  // namespace gk_host

#endif  // GAPKIT_B200_FRESH_VECTOR_HPP_
