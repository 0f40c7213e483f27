// Device workspace heap (see common.cuh: dev_malloc / dev_free).
//
// The solver objects of a refresh (Ozaki GEMM batches, root-inverse batches, the low-rank path) are
// built per refresh with sizes that drift with the step count.  cudaMalloc/cudaFree in that path
// measured 25-1500 ms per call on a busy device (and cudaFree synchronises the device), so the
// workspaces come from a few large slabs carved by a best-fit heap with coalescing: after the first
// refreshes no CUDA allocation call happens any more.  Slabs are kept until process exit.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <iterator>
#include <map>
#include <mutex>
#include <unordered_map>
#include <vector>

#include "common.cuh"

namespace shampoo {

namespace {
constexpr size_t kSlab = size_t(4) << 30;  // minimum slab size
constexpr size_t kAlign = 256;

struct Heap {
  std::mutex mu;
  std::vector<std::pair<char*, size_t>> slabs;      // base, size
  std::map<char*, size_t> free_by_addr;             // free segments
  std::multimap<size_t, char*> free_by_size;
  std::unordered_map<void*, size_t> live;           // allocated segments
  bool log = false;

  Heap() {
    const char* e = std::getenv("SHAMPOO_DEVMEM_LOG");  // debug: every slab allocation
    log = e && std::atoi(e) != 0;
  }
  int slab_of(char* p) const {
    for (size_t i = 0; i < slabs.size(); ++i)
      if (p >= slabs[i].first && p < slabs[i].first + slabs[i].second) return (int)i;
    return -1;
  }
  void add_free(char* p, size_t sz) {
    free_by_addr.emplace(p, sz);
    free_by_size.emplace(sz, p);
  }
  void remove_free(std::map<char*, size_t>::iterator it) {
    auto range = free_by_size.equal_range(it->second);
    for (auto s = range.first; s != range.second; ++s)
      if (s->second == it->first) {
        free_by_size.erase(s);
        break;
      }
    free_by_addr.erase(it);
  }
};

Heap& heap() {
  static Heap* h = new Heap();  // never destroyed: device memory outlives static destructors
  return *h;
}
}  // namespace

cudaError_t dev_malloc_bytes(void** p, size_t bytes) {
  Heap& H = heap();
  const size_t want = ((bytes ? bytes : 1) + kAlign - 1) & ~(kAlign - 1);
  std::lock_guard<std::mutex> lk(H.mu);
  auto it = H.free_by_size.lower_bound(want);
  if (it == H.free_by_size.end()) {
    const size_t sz = std::max(kSlab, want);
    char* base = nullptr;
    const auto t0 = std::chrono::steady_clock::now();
    cudaError_t e = cudaMalloc(&base, sz);
    if (e != cudaSuccess) {  // give back the slabs that are entirely idle, then retry once
      cudaGetLastError();
      for (size_t i = 0; i < H.slabs.size();) {
        auto it2 = H.free_by_addr.find(H.slabs[i].first);
        if (it2 != H.free_by_addr.end() && it2->second == H.slabs[i].second) {
          H.remove_free(it2);
          cudaFree(H.slabs[i].first);
          H.slabs.erase(H.slabs.begin() + i);
        } else {
          ++i;
        }
      }
      e = cudaMalloc(&base, sz);
      if (e != cudaSuccess) return e;
    }
    if (H.log)
      std::fprintf(stderr, "[devmem] slab %zu: %.2f GB in %.1f ms\n", H.slabs.size(), sz / 1e9,
                   std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
    H.slabs.push_back({base, sz});
    H.add_free(base, sz);
    it = H.free_by_size.lower_bound(want);
  }
  char* seg = it->second;
  const size_t sz = it->first;
  H.remove_free(H.free_by_addr.find(seg));
  if (sz > want) H.add_free(seg + want, sz - want);
  H.live[seg] = want;
  *p = seg;
  return cudaSuccess;
}

void dev_free(void* ptr) {
  if (!ptr) return;
  Heap& H = heap();
  std::lock_guard<std::mutex> lk(H.mu);
  auto lv = H.live.find(ptr);
  if (lv == H.live.end()) {  // not from the heap
    cudaFree(ptr);
    return;
  }
  char* p = static_cast<char*>(ptr);
  size_t sz = lv->second;
  H.live.erase(lv);
  const int slab = H.slab_of(p);
  // coalesce with the following and the preceding free segments of the same slab
  auto nx = H.free_by_addr.find(p + sz);
  if (nx != H.free_by_addr.end() && H.slab_of(nx->first) == slab) {
    sz += nx->second;
    H.remove_free(nx);
  }
  auto pv = H.free_by_addr.lower_bound(p);
  if (pv != H.free_by_addr.begin()) {
    pv = std::prev(pv);
    if (pv->first + pv->second == p && H.slab_of(pv->first) == slab) {
      p = pv->first;
      sz += pv->second;
      H.remove_free(pv);
    }
  }
  H.add_free(p, sz);
}

}  // namespace shampoo
