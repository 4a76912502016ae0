// Runtime side of the C-ABI: error state, device init, the swap engine's
// pinned-host transfers and the co-located / peer boundary copies.
//
// Swap (memopt `swap` actions, memopt.py:208,282): D2H on the stage's copy
// stream after the producer's forward, H2D prefetch on the same stream before
// the first backward reader; ordering is carried by CUDA events recorded on the
// compute stream and waited on the copy stream (and vice versa).
#include "common.cuh"
#include "../../include/dawnpiper.h"

#include <string>

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
