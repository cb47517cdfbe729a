// fs_pipeline.cu — native interactive-recompute loop (C++ runtime around the kernels).
//
// The service's recompute worker (fs/service.py:110-175) recomputes the working set
// frame after frame.  ShardedEnsemble.run_frames does this from Python (and carries the
// multi-GPU exchange); this is the same single-device loop without the interpreter:
// frame f+1's device work — fused recompute, Jaccard + outlier kernels, D2H of the
// partials — is queued while host worker threads run frame f's complete-linkage merge,
// with a ring of `depth` frame buffers (device outputs + pinned host slots + events).
//
// Multi-GPU: an fs_comm (an NCCL communicator, libnccl loaded at run time — the copy
// torch already mapped when there is one) attached with fs_pipeline_set_comm sums the
// row bands' int64 [bins | Gram] partials with one ncclAllReduce on the ensemble stream
// inside every frame (north_star: partial Gram matrices summed with NCCL allreduce), so
// each rank's loop runs frame after frame without returning to Python.
#include <dlfcn.h>

#include <condition_variable>
#include <cstring>
#include <deque>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include <cuda_runtime.h>

#include "../../include/floodstream.h"
#include "fs_internal.h"

// ---------------------------------------------------------------------------
// NCCL, resolved at run time (no link-time dependency; ABI of nccl.h 2.x)
// ---------------------------------------------------------------------------
namespace {

struct NcclUniqueId {
  char internal[128];
};
using ncclComm_t = void *;
constexpr int kNcclInt64 = 4, kNcclSum = 0;  // ncclInt64, ncclSum

struct NcclApi {
  int (*get_unique_id)(NcclUniqueId *) = nullptr;
  int (*comm_init_rank)(ncclComm_t *, int, NcclUniqueId, int) = nullptr;
  int (*comm_destroy)(ncclComm_t) = nullptr;
  int (*all_reduce)(const void *, void *, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  const char *(*error_string)(int) = nullptr;
  std::string error;
  bool ok = false;
};

const NcclApi &nccl() {
  static const NcclApi api = [] {
    NcclApi a;
    void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);  // torch's copy, if mapped
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_LOCAL);
    if (!h) {
      const char *e = dlerror();
      a.error = std::string("libnccl not found: ") + (e ? e : "dlopen failed");
      return a;
    }
    a.get_unique_id = reinterpret_cast<decltype(a.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
    a.comm_init_rank = reinterpret_cast<decltype(a.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
    a.comm_destroy = reinterpret_cast<decltype(a.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
    a.all_reduce = reinterpret_cast<decltype(a.all_reduce)>(dlsym(h, "ncclAllReduce"));
    a.error_string = reinterpret_cast<decltype(a.error_string)>(dlsym(h, "ncclGetErrorString"));
    a.ok = a.get_unique_id && a.comm_init_rank && a.comm_destroy && a.all_reduce;
    if (!a.ok) a.error = "libnccl lacks ncclGetUniqueId/ncclCommInitRank/ncclAllReduce";
    return a;
  }();
  return api;
}

std::string nccl_msg(const char *what, int r) {
  const NcclApi &a = nccl();
  return std::string(what) + ": " + (a.error_string ? a.error_string(r) : "nccl error") +
         " (" + std::to_string(r) + ")";
}

}  // namespace

struct fs_comm {
  ncclComm_t comm = nullptr;
  int nranks = 1, rank = 0, device = 0;
};

namespace {

struct Frame {
  void *d_counts = nullptr, *d_rgba = nullptr, *d_part = nullptr, *d_sim = nullptr,
       *d_scores = nullptr;
  void *h_part = nullptr, *h_sim = nullptr, *h_scores = nullptr;
  std::vector<int32_t> labels;
  cudaEvent_t done = nullptr;
  bool busy = false;
  int64_t seq = -1;
};

}  // namespace

struct fs_pipeline {
  fs_ensemble *ens = nullptr;
  std::vector<uint32_t> slots;
  std::vector<uint32_t> id_rank;
  uint32_t k = 0;
  int engine = 0;
  double tau = 0.8;
  uint64_t pixels = 0;
  int device = 0;
  fs_comm *comm = nullptr;  // optional: sum [bins | Gram] over the row bands every frame
  cudaStream_t side = nullptr;
  std::vector<Frame> frames;
  std::vector<std::thread> workers;
  std::mutex mu;
  std::condition_variable cv_job, cv_free;
  std::deque<int> jobs;
  bool stop = false;
  int err = FS_OK;
  std::string err_msg;
};

namespace {

void worker_loop(fs_pipeline *p) {
  for (;;) {
    int idx;
    {
      std::unique_lock<std::mutex> lk(p->mu);
      p->cv_job.wait(lk, [&] { return p->stop || !p->jobs.empty(); });
      if (p->jobs.empty()) return;  // stop requested and nothing left
      idx = p->jobs.front();
      p->jobs.pop_front();
    }
    Frame &f = p->frames[(size_t)idx];
    int rc = FS_OK;
    std::string msg;
    cudaError_t e = cudaEventSynchronize(f.done);
    if (e != cudaSuccess) {
      rc = FS_ECUDA;
      msg = std::string("frame D2H: ") + cudaGetErrorString(e);
    } else if (p->k > 0) {
      rc = fs_cluster_complete_linkage(static_cast<const double *>(f.h_sim), p->k,
                                       p->id_rank.data(), p->tau, f.labels.data());
      if (rc) msg = fs_last_error();
    }
    std::lock_guard<std::mutex> lk(p->mu);
    if (rc && p->err == FS_OK) {
      p->err = rc;
      p->err_msg = msg;
    }
    f.busy = false;
    p->cv_free.notify_all();
  }
}

int fail(int code, const std::string &m) { return fs::set_error(code, m); }

}  // namespace

extern "C" {

int fs_pipeline_create(fs_ensemble *ens, const uint32_t *slots, uint32_t k, int engine, double tau,
                       const uint32_t *id_rank, uint32_t depth, fs_pipeline **out) {
  if (!ens || !slots || !id_rank || !out || k == 0) return fail(FS_EINVAL, "bad argument");
  if (!(tau > 0.0 && tau <= 1.0)) return fail(FS_EINVAL, "tau must be in (0, 1]");
  if (depth < 2) depth = 2;
  auto p = std::make_unique<fs_pipeline>();
  p->ens = ens;
  p->slots.assign(slots, slots + k);
  p->id_rank.assign(id_rank, id_rank + k);
  p->k = k;
  p->engine = engine;
  p->tau = tau;
  uint32_t cap = 0;
  uint64_t wpm = 0;
  int rc = fs_ensemble_info(ens, &p->pixels, &cap, &wpm, &p->device);
  if (rc) return rc;
  for (uint32_t s : p->slots)
    if (s >= cap) return fail(FS_EINVAL, "slot index out of range");
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(p->device);
  auto cleanup_fail = [&](const char *what, cudaError_t e) {
    for (auto &f : p->frames) {
      cudaFree(f.d_counts);
      cudaFree(f.d_rgba);
      cudaFree(f.d_part);
      cudaFree(f.d_sim);
      cudaFree(f.d_scores);
      cudaFreeHost(f.h_part);
      cudaFreeHost(f.h_sim);
      cudaFreeHost(f.h_scores);
      if (f.done) cudaEventDestroy(f.done);
    }
    if (p->side) cudaStreamDestroy(p->side);
    cudaGetLastError();
    cudaSetDevice(prev);
    return fail(e == cudaErrorMemoryAllocation ? FS_ENOMEM : FS_ECUDA,
                std::string(what) + ": " + cudaGetErrorString(e));
  };
  cudaError_t e;
  if ((e = cudaStreamCreateWithFlags(&p->side, cudaStreamNonBlocking)) != cudaSuccess)
    return cleanup_fail("stream", e);
  const size_t P = p->pixels, nb = k + 1, part = (nb + (size_t)k * k) * 8;
  p->frames.resize(depth);
  for (auto &f : p->frames) {
    f.labels.resize(k);
    if ((e = cudaMalloc(&f.d_counts, P * 4)) != cudaSuccess ||
        (e = cudaMalloc(&f.d_rgba, P * 4)) != cudaSuccess ||
        (e = cudaMalloc(&f.d_part, part)) != cudaSuccess ||
        (e = cudaMalloc(&f.d_sim, (size_t)k * k * 8)) != cudaSuccess ||
        (e = cudaMalloc(&f.d_scores, (size_t)k * 8)) != cudaSuccess ||
        (e = cudaHostAlloc(&f.h_part, part, cudaHostAllocPortable)) != cudaSuccess ||
        (e = cudaHostAlloc(&f.h_sim, (size_t)k * k * 8, cudaHostAllocPortable)) != cudaSuccess ||
        (e = cudaHostAlloc(&f.h_scores, (size_t)k * 8, cudaHostAllocPortable)) != cudaSuccess ||
        (e = cudaEventCreateWithFlags(&f.done, cudaEventDisableTiming)) != cudaSuccess)
      return cleanup_fail("frame buffers", e);
  }
  cudaSetDevice(prev);
  fs_pipeline *raw = p.get();
  for (uint32_t i = 0; i < depth; ++i) p->workers.emplace_back(worker_loop, raw);
  *out = p.release();
  return FS_OK;
}

int fs_pipeline_run(fs_pipeline *p, uint32_t n_frames, int64_t *bins, int64_t *gram, double *sim,
                    double *scores, int32_t *labels, double *device_ms) {
  if (!p) return fail(FS_EINVAL, "null pipeline");
  if (n_frames == 0) return FS_OK;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(p->device);
  void *sk = nullptr;
  int rc = fs_ensemble_stream_handle(p->ens, &sk);
  if (rc) return rc;
  cudaEvent_t t0, t1, ready;
  cudaEventCreate(&t0);
  cudaEventCreate(&t1);
  cudaEventCreateWithFlags(&ready, cudaEventDisableTiming);
  cudaEventRecord(t0, (cudaStream_t)sk);
  const uint32_t k = p->k;
  const size_t nb = k + 1, part = (nb + (size_t)k * k) * 8;
  int last = -1;
  for (uint32_t fi = 0; fi < n_frames && rc == FS_OK; ++fi) {
    const int idx = (int)(fi % p->frames.size());
    Frame &f = p->frames[(size_t)idx];
    {
      std::unique_lock<std::mutex> lk(p->mu);
      p->cv_free.wait(lk, [&] { return !f.busy; });
      if (p->err) break;
      f.busy = true;
      f.seq = fi;
    }
    int fused = 0;
    rc = fs_ensemble_recompute(p->ens, p->slots.data(), k, p->engine,
                               static_cast<uint32_t *>(f.d_counts), static_cast<int64_t *>(f.d_part),
                               static_cast<uint8_t *>(f.d_rgba),
                               static_cast<int64_t *>(f.d_part) + nb, 1, &fused);
    if (rc) {
      std::lock_guard<std::mutex> lk(p->mu);
      f.busy = false;
      break;
    }
    if (p->comm != nullptr) {
      // the exact int64 sum of every band's [bins | Gram] (one bucket per frame)
      const int r = nccl().all_reduce(f.d_part, f.d_part, nb + (size_t)k * k, kNcclInt64, kNcclSum,
                                      p->comm->comm, (cudaStream_t)sk);
      if (r != 0) {
        rc = fail(FS_ECUDA, nccl_msg("ncclAllReduce", r));
        std::lock_guard<std::mutex> lk(p->mu);
        f.busy = false;
        break;
      }
    }
    // Jaccard + outliers and the small D2H on the side stream, behind the recompute
    cudaEventRecord(ready, (cudaStream_t)sk);
    cudaStreamWaitEvent(p->side, ready, 0);
    rc = fs_similarity_outliers_device(static_cast<const int64_t *>(f.d_part) + nb, k,
                                       static_cast<double *>(f.d_sim),
                                       k >= 2 ? static_cast<double *>(f.d_scores) : nullptr,
                                       (void *)p->side);
    if (rc) {
      std::lock_guard<std::mutex> lk(p->mu);
      f.busy = false;
      break;
    }
    cudaMemcpyAsync(f.h_part, f.d_part, part, cudaMemcpyDeviceToHost, p->side);
    cudaMemcpyAsync(f.h_sim, f.d_sim, (size_t)k * k * 8, cudaMemcpyDeviceToHost, p->side);
    if (k >= 2) cudaMemcpyAsync(f.h_scores, f.d_scores, (size_t)k * 8, cudaMemcpyDeviceToHost, p->side);
    cudaEventRecord(f.done, p->side);
    {
      std::lock_guard<std::mutex> lk(p->mu);
      p->jobs.push_back(idx);
    }
    p->cv_job.notify_one();
    last = idx;
  }
  // drain: every queued frame's linkage has finished when its slot is free again
  {
    std::unique_lock<std::mutex> lk(p->mu);
    p->cv_free.wait(lk, [&] {
      for (auto &f : p->frames)
        if (f.busy) return false;
      return true;
    });
    if (rc == FS_OK && p->err) {
      rc = fail(p->err, p->err_msg);
      p->err = FS_OK;
    }
  }
  cudaEventRecord(t1, (cudaStream_t)sk);
  cudaEventSynchronize(t1);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, t0, t1);
  if (device_ms) *device_ms = ms;
  cudaEventDestroy(t0);
  cudaEventDestroy(t1);
  cudaEventDestroy(ready);
  if (rc == FS_OK && last >= 0) {
    Frame &f = p->frames[(size_t)last];
    if (bins) std::memcpy(bins, f.h_part, nb * 8);
    if (gram) std::memcpy(gram, static_cast<int64_t *>(f.h_part) + nb, (size_t)k * k * 8);
    if (sim) std::memcpy(sim, f.h_sim, (size_t)k * k * 8);
    if (scores && k >= 2) std::memcpy(scores, f.h_scores, (size_t)k * 8);
    if (labels) std::memcpy(labels, f.labels.data(), (size_t)k * 4);
  }
  cudaSetDevice(prev);
  return rc;
}

int fs_pipeline_set_comm(fs_pipeline *p, fs_comm *c) {
  if (!p) return fail(FS_EINVAL, "null pipeline");
  if (c != nullptr && c->device != p->device)
    return fail(FS_EINVAL, "communicator and pipeline are on different devices");
  p->comm = c;
  return FS_OK;
}

int fs_comm_unique_id(uint8_t *out) {
  if (!out) return fail(FS_EINVAL, "null out");
  const NcclApi &a = nccl();
  if (!a.ok) return fail(FS_ECUDA, a.error);
  NcclUniqueId id;
  const int r = a.get_unique_id(&id);
  if (r != 0) return fail(FS_ECUDA, nccl_msg("ncclGetUniqueId", r));
  std::memcpy(out, id.internal, sizeof(id.internal));
  return FS_OK;
}

int fs_comm_create(const uint8_t *id, int nranks, int rank, fs_comm **out) {
  if (!id || !out || nranks < 1 || rank < 0 || rank >= nranks)
    return fail(FS_EINVAL, "bad communicator arguments");
  const NcclApi &a = nccl();
  if (!a.ok) return fail(FS_ECUDA, a.error);
  auto c = std::make_unique<fs_comm>();
  c->nranks = nranks;
  c->rank = rank;
  if (cudaGetDevice(&c->device) != cudaSuccess) return fail(FS_ENODEV, "no CUDA device");
  NcclUniqueId uid;
  std::memcpy(uid.internal, id, sizeof(uid.internal));
  const int r = a.comm_init_rank(&c->comm, nranks, uid, rank);
  if (r != 0) return fail(FS_ECUDA, nccl_msg("ncclCommInitRank", r));
  *out = c.release();
  return FS_OK;
}

int fs_comm_allreduce_i64(fs_comm *c, int64_t *buf, uint64_t n, void *stream) {
  if (!c || (!buf && n)) return fail(FS_EINVAL, "bad allreduce arguments");
  if (n == 0) return FS_OK;
  const int r = nccl().all_reduce(buf, buf, (size_t)n, kNcclInt64, kNcclSum, c->comm,
                                  (cudaStream_t)stream);
  return r == 0 ? FS_OK : fail(FS_ECUDA, nccl_msg("ncclAllReduce", r));
}

int fs_comm_destroy(fs_comm *c) {
  if (!c) return FS_OK;
  int r = 0;
  if (c->comm) r = nccl().comm_destroy(c->comm);
  delete c;
  return r == 0 ? FS_OK : fail(FS_ECUDA, nccl_msg("ncclCommDestroy", r));
}

int fs_pipeline_destroy(fs_pipeline *p) {
  if (!p) return FS_OK;
  {
    std::lock_guard<std::mutex> lk(p->mu);
    p->stop = true;
  }
  p->cv_job.notify_all();
  for (auto &t : p->workers) t.join();
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(p->device);
  cudaStreamSynchronize(p->side);
  for (auto &f : p->frames) {
    cudaFree(f.d_counts);
    cudaFree(f.d_rgba);
    cudaFree(f.d_part);
    cudaFree(f.d_sim);
    cudaFree(f.d_scores);
    cudaFreeHost(f.h_part);
    cudaFreeHost(f.h_sim);
    cudaFreeHost(f.h_scores);
    cudaEventDestroy(f.done);
  }
  cudaStreamDestroy(p->side);
  cudaSetDevice(prev);
  delete p;
  return FS_OK;
}

}  // extern "C"
