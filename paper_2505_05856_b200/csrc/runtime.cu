// Runtime side of the C-ABI: error state, device init, the swap engine's
// pinned-host transfers and the co-located / peer boundary copies.
//
// Swap (memopt `swap` actions, memopt.py:208,282): D2H on the stage's copy
// stream after the producer's forward, H2D prefetch on the same stream before
// the first backward reader; ordering is carried by CUDA events recorded on the
// compute stream and waited on the copy stream (and vice versa).
#include "common.cuh"
#include "../../include/dawnpiper.h"

#include <algorithm>
#include <map>
#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>

namespace dpn {
namespace {
thread_local std::string g_err;
}
void set_error(const std::string& msg) { g_err = msg; }
const char* last_error() { return g_err.c_str(); }
}  // namespace dpn

using namespace dpn;

extern "C" const char* dpn_last_error(void) { return dpn::last_error(); }

extern "C" int dpn_version(void) { return DPN_ABI_VERSION; }

extern "C" int dpn_init(int device) {
  DPN_CHECK_CUDA(cudaSetDevice(device));
  cudaDeviceProp prop;
  DPN_CHECK_CUDA(cudaGetDeviceProperties(&prop, device));
  DPN_REQUIRE(prop.major == 10 && prop.minor == 0,
              std::string("sm_100a kernels need a B200-class device, got ") + prop.name +
                  " (sm_" + std::to_string(prop.major) + std::to_string(prop.minor) + ")");
  DPN_CHECK_CUDA(cudaFree(nullptr));
  return 0;
}

extern "C" int dpn_host_alloc(int64_t bytes, void** out) {
  DPN_REQUIRE(out != nullptr, "null out");
  DPN_CHECK_CUDA(cudaHostAlloc(out, (size_t)bytes, cudaHostAllocPortable));
  return 0;
}

extern "C" int dpn_host_free(void* p) {
  DPN_CHECK_CUDA(cudaFreeHost(p));
  return 0;
}

extern "C" int dpn_swap_out(void* host_dst, const void* dev_src, int64_t bytes, void* copy_stream,
                            void* ready_event, void* done_event) {
  cudaStream_t s = (cudaStream_t)copy_stream;
  if (ready_event) DPN_CHECK_CUDA(cudaStreamWaitEvent(s, (cudaEvent_t)ready_event, 0));
  DPN_CHECK_CUDA(cudaMemcpyAsync(host_dst, dev_src, (size_t)bytes, cudaMemcpyDeviceToHost, s));
  if (done_event) DPN_CHECK_CUDA(cudaEventRecord((cudaEvent_t)done_event, s));
  return 0;
}

extern "C" int dpn_swap_in(void* dev_dst, const void* host_src, int64_t bytes, void* copy_stream,
                           void* ready_event, void* done_event) {
  cudaStream_t s = (cudaStream_t)copy_stream;
  if (ready_event) DPN_CHECK_CUDA(cudaStreamWaitEvent(s, (cudaEvent_t)ready_event, 0));
  DPN_CHECK_CUDA(cudaMemcpyAsync(dev_dst, host_src, (size_t)bytes, cudaMemcpyHostToDevice, s));
  if (done_event) DPN_CHECK_CUDA(cudaEventRecord((cudaEvent_t)done_event, s));
  return 0;
}

extern "C" int dpn_p2p_copy(void* dst, int dst_dev, const void* src, int src_dev, int64_t bytes,
                            void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (dst_dev == src_dev) {
    DPN_CHECK_CUDA(cudaMemcpyAsync(dst, src, (size_t)bytes, cudaMemcpyDeviceToDevice, s));
  } else {
    DPN_CHECK_CUDA(cudaMemcpyPeerAsync(dst, dst_dev, src, src_dev, (size_t)bytes, s));
  }
  return 0;
}

extern "C" int dpn_enable_peer(int dev, int peer) {
  int can = 0;
  DPN_CHECK_CUDA(cudaDeviceCanAccessPeer(&can, dev, peer));
  DPN_REQUIRE(can, "peer access not supported between devices");
  int cur = 0;
  DPN_CHECK_CUDA(cudaGetDevice(&cur));
  DPN_CHECK_CUDA(cudaSetDevice(dev));
  cudaError_t e = cudaDeviceEnablePeerAccess(peer, 0);
  if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
  else DPN_CHECK_CUDA(e);
  DPN_CHECK_CUDA(cudaSetDevice(cur));
  return 0;
}

extern "C" int dpn_memset_async(void* dst, int value, int64_t bytes, void* stream) {
  DPN_CHECK_CUDA(cudaMemsetAsync(dst, value, (size_t)bytes, (cudaStream_t)stream));
  return 0;
}

// ---------------------------------------------------------------------------
// Per-stage device arenas: one cudaMalloc of `cap` bytes per arena, carved by
// a first-fit free list with coalescing.  torch's caching allocator sits on
// top through a MemPool whose pluggable allocator is dpn_arena_malloc /
// dpn_arena_free (runtime/arena.py): the stage's caching-allocator segments
// come out of its arena, so the arena IS the stage's device-memory cap (an
// allocation past it fails like a real OOM on a GPU of that size) and its
// high-water mark is the stage's measured peak.  The arena serving a
// malloc is the calling thread's current one (dpn_arena_select).
namespace {
constexpr size_t kArenaAlign = 512;
struct Arena {
  int dev = 0;
  char* base = nullptr;
  size_t cap = 0, used = 0, peak = 0;
  std::map<size_t, size_t> free_;          // offset -> size
  std::unordered_map<char*, size_t> live;  // pointer -> size
};
std::mutex g_arena_mu;
std::vector<Arena*> g_arenas;
thread_local int g_current_arena = -1;

Arena* arena_at(int h) {
  return (h >= 0 && h < (int)g_arenas.size()) ? g_arenas[h] : nullptr;
}
}  // namespace

extern "C" int dpn_arena_create(int device, int64_t cap_bytes, int* handle) {
  DPN_REQUIRE(handle != nullptr && cap_bytes > 0, "dpn_arena_create: bad arguments");
  int cur = 0;
  DPN_CHECK_CUDA(cudaGetDevice(&cur));
  DPN_CHECK_CUDA(cudaSetDevice(device));
  void* base = nullptr;
  const size_t cap = ((size_t)cap_bytes + kArenaAlign - 1) / kArenaAlign * kArenaAlign;
  cudaError_t e = cudaMalloc(&base, cap);
  cudaSetDevice(cur);
  DPN_CHECK_CUDA(e);
  Arena* a = new Arena();
  a->dev = device;
  a->base = static_cast<char*>(base);
  a->cap = cap;
  a->free_[0] = cap;
  std::lock_guard<std::mutex> lk(g_arena_mu);
  g_arenas.push_back(a);
  *handle = (int)g_arenas.size() - 1;
  return 0;
}

extern "C" int dpn_arena_destroy(int handle) {
  std::lock_guard<std::mutex> lk(g_arena_mu);
  Arena* a = arena_at(handle);
  DPN_REQUIRE(a != nullptr, "dpn_arena_destroy: unknown arena");
  DPN_REQUIRE(a->live.empty(), "dpn_arena_destroy: arena still has live allocations");
  int cur = 0;
  cudaGetDevice(&cur);
  cudaSetDevice(a->dev);
  cudaFree(a->base);
  cudaSetDevice(cur);
  delete a;
  g_arenas[handle] = nullptr;
  return 0;
}

extern "C" int dpn_arena_select(int handle) {
  DPN_REQUIRE(handle == -1 || arena_at(handle) != nullptr, "dpn_arena_select: unknown arena");
  g_current_arena = handle;
  return 0;
}

extern "C" int dpn_arena_stats(int handle, int64_t* in_use, int64_t* peak, int64_t* cap) {
  std::lock_guard<std::mutex> lk(g_arena_mu);
  Arena* a = arena_at(handle);
  DPN_REQUIRE(a != nullptr, "dpn_arena_stats: unknown arena");
  if (in_use) *in_use = (int64_t)a->used;
  if (peak) *peak = (int64_t)a->peak;
  if (cap) *cap = (int64_t)a->cap;
  return 0;
}

extern "C" int dpn_arena_reset_peak(int handle) {
  std::lock_guard<std::mutex> lk(g_arena_mu);
  Arena* a = arena_at(handle);
  DPN_REQUIRE(a != nullptr, "dpn_arena_reset_peak: unknown arena");
  a->peak = a->used;
  return 0;
}

// torch CUDAPluggableAllocator entry points (signatures fixed by torch).
extern "C" void* dpn_arena_malloc(size_t size, int device, void* /*stream*/) {
  std::lock_guard<std::mutex> lk(g_arena_mu);
  Arena* a = arena_at(g_current_arena);
  if (a == nullptr || a->dev != device) return nullptr;  // no arena selected: refuse
  const size_t need = std::max<size_t>(kArenaAlign, (size + kArenaAlign - 1) / kArenaAlign * kArenaAlign);
  for (auto it = a->free_.begin(); it != a->free_.end(); ++it) {
    if (it->second < need) continue;
    const size_t off = it->first, sz = it->second;
    a->free_.erase(it);
    if (sz > need) a->free_[off + need] = sz - need;
    char* p = a->base + off;
    a->live[p] = need;
    a->used += need;
    a->peak = std::max(a->peak, a->used);
    return p;
  }
  return nullptr;  // the stage's cap is exhausted: torch raises OutOfMemoryError
}

extern "C" void dpn_arena_free(void* ptr, size_t /*size*/, int /*device*/, void* /*stream*/) {
  std::lock_guard<std::mutex> lk(g_arena_mu);
  for (Arena* a : g_arenas) {
    if (a == nullptr) continue;
    char* p = static_cast<char*>(ptr);
    auto it = a->live.find(p);
    if (it == a->live.end()) continue;
    size_t off = (size_t)(p - a->base), sz = it->second;
    a->live.erase(it);
    a->used -= sz;
    auto nx = a->free_.lower_bound(off);
    if (nx != a->free_.end() && off + sz == nx->first) {  // merge with the next free block
      sz += nx->second;
      nx = a->free_.erase(nx);
    }
    if (nx != a->free_.begin()) {  // and with the previous one
      auto pv = std::prev(nx);
      if (pv->first + pv->second == off) {
        pv->second += sz;
        return;
      }
    }
    a->free_[off] = sz;
    return;
  }
}

// Release every arena this library created (the process' dpn state) after a
// device synchronize; allocations still live in an arena are reported.
extern "C" int dpn_destroy(void) {
  cudaDeviceSynchronize();
  std::lock_guard<std::mutex> lk(g_arena_mu);
  size_t leaked = 0;
  for (Arena*& a : g_arenas) {
    if (a == nullptr) continue;
    leaked += a->live.size();
    int cur = 0;
    cudaGetDevice(&cur);
    cudaSetDevice(a->dev);
    cudaFree(a->base);
    cudaSetDevice(cur);
    delete a;
    a = nullptr;
  }
  g_arenas.clear();
  g_current_arena = -1;
  DPN_REQUIRE(leaked == 0, "dpn_destroy: " + std::to_string(leaked) + " arena allocations were still live");
  return 0;
}
