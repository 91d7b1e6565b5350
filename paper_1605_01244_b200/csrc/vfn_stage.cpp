// Pageable host buffers at pinned speed (vfn_internal.cuh, HostStager).
// A reference user hands NufftPlan.evaluate fresh numpy arrays; a
// cudaMemcpyAsync from pageable memory is synchronous and single-threaded in
// the driver, and the first touch of a fresh output array page-faults.  Here
// the bytes move through rings of pinned pieces: host threads copy a piece
// while the DMA engine moves the previous one.
#include <algorithm>
#include <cstring>
#include <map>
#include <mutex>
#include <thread>
#include <vector>

#include "vfn_internal.cuh"

namespace vfn {

namespace {
constexpr size_t kPiece = (size_t)64 << 20;  // bytes per pinned piece
constexpr int kRing = 3;                     // pieces per direction
}  // namespace

struct HostStager {
  std::mutex mu;  // one transfer at a time (device stagers are shared by plan builds and rectilinear calls)
  char* in[kRing] = {};
  char* out[kRing] = {};
  cudaEvent_t ev_in[kRing] = {}, ev_out[kRing] = {};
  bool used_in[kRing] = {}, used_out[kRing] = {};
  bool ok = false;
  int threads = 8;
};

bool is_pageable(const void* ptr) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, ptr) != cudaSuccess) {
    cudaGetLastError();
    return true;
  }
  return a.type == cudaMemoryTypeUnregistered;
}

HostStager* stager_create() {
  HostStager* st = new HostStager();
  st->ok = true;
  for (int i = 0; i < kRing && st->ok; ++i) {
    st->ok = cudaMallocHost(&st->in[i], kPiece) == cudaSuccess && cudaMallocHost(&st->out[i], kPiece) == cudaSuccess &&
             cudaEventCreateWithFlags(&st->ev_in[i], cudaEventDisableTiming) == cudaSuccess &&
             cudaEventCreateWithFlags(&st->ev_out[i], cudaEventDisableTiming) == cudaSuccess;
  }
  if (!st->ok) cudaGetLastError();
  st->threads = (int)std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
  return st;
}

void stager_destroy(HostStager* st) {
  if (!st) return;
  for (int i = 0; i < kRing; ++i) {
    if (st->in[i]) cudaFreeHost(st->in[i]);
    if (st->out[i]) cudaFreeHost(st->out[i]);
    if (st->ev_in[i]) cudaEventDestroy(st->ev_in[i]);
    if (st->ev_out[i]) cudaEventDestroy(st->ev_out[i]);
  }
  delete st;
}

HostStager* device_stager(int device) {
  static std::mutex mu;
  static std::map<int, HostStager*> st;
  std::lock_guard<std::mutex> lock(mu);
  HostStager*& s = st[device];
  if (!s) s = stager_create();
  return s;
}

static void par_copy(char* dst, const char* src, size_t n, int threads) {
  const int nt = (int)std::min<size_t>((size_t)threads, std::max<size_t>(1, n >> 22));  // >= 4 MB per thread
  if (nt <= 1) {
    std::memcpy(dst, src, n);
    return;
  }
  std::vector<std::thread> th;
  th.reserve(nt);
  for (int k = 0; k < nt; ++k)
    th.emplace_back([=] {
      const size_t lo = n * k / nt, hi = n * (k + 1) / nt;
      std::memcpy(dst + lo, src + lo, hi - lo);
    });
  for (auto& x : th) x.join();
}

int stage_h2d(HostStager* st, void* dst_dev, const void* src_host, size_t bytes, cudaStream_t s) {
  if (!st || !st->ok) {
    VFN_CUDA(cudaMemcpyAsync(dst_dev, src_host, bytes, cudaMemcpyHostToDevice, s));
    return VFN_OK;
  }
  std::lock_guard<std::mutex> lock(st->mu);
  const char* src = static_cast<const char*>(src_host);
  char* dst = static_cast<char*>(dst_dev);
  for (size_t off = 0, k = 0; off < bytes; off += kPiece, ++k) {
    const int r = (int)(k % kRing);
    const size_t n = std::min(kPiece, bytes - off);
    if (st->used_in[r]) VFN_CUDA(cudaEventSynchronize(st->ev_in[r]));  // its previous H2D is done
    par_copy(st->in[r], src + off, n, st->threads);
    VFN_CUDA(cudaMemcpyAsync(dst + off, st->in[r], n, cudaMemcpyHostToDevice, s));
    VFN_CUDA(cudaEventRecord(st->ev_in[r], s));
    st->used_in[r] = true;
  }
  return VFN_OK;
}

int stage_d2h(HostStager* st, void* dst_host, const void* src_dev, size_t bytes, cudaStream_t s) {
  if (!st || !st->ok) {
    VFN_CUDA(cudaMemcpyAsync(dst_host, src_dev, bytes, cudaMemcpyDeviceToHost, s));
    VFN_CUDA(cudaStreamSynchronize(s));
    return VFN_OK;
  }
  std::lock_guard<std::mutex> lock(st->mu);
  const char* src = static_cast<const char*>(src_dev);
  char* dst = static_cast<char*>(dst_host);
  const size_t np = (bytes + kPiece - 1) / kPiece;
  // D2H of piece k is enqueued kRing - 1 pieces ahead of its host copy
  auto drain = [&](size_t k) -> int {
    const int r = (int)(k % kRing);
    const size_t off = k * kPiece, n = std::min(kPiece, bytes - off);
    VFN_CUDA(cudaEventSynchronize(st->ev_out[r]));
    par_copy(dst + off, st->out[r], n, st->threads);
    return VFN_OK;
  };
  for (size_t k = 0; k < np; ++k) {
    if (k >= (size_t)kRing) VFN_CHECK(drain(k - kRing));
    const int r = (int)(k % kRing);
    const size_t off = k * kPiece, n = std::min(kPiece, bytes - off);
    VFN_CUDA(cudaMemcpyAsync(st->out[r], src + off, n, cudaMemcpyDeviceToHost, s));
    VFN_CUDA(cudaEventRecord(st->ev_out[r], s));
    st->used_out[r] = true;
  }
  for (size_t k = np > (size_t)kRing ? np - kRing : 0; k < np; ++k) VFN_CHECK(drain(k));
  return VFN_OK;
}

}  // namespace vfn
