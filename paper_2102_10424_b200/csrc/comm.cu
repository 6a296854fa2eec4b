// comm.cu -- collectives of the GIST round (see comm.h): NCCL, or the loopback test transport.
#include "comm.h"

#include <condition_variable>
#include <cstring>
#include <mutex>

struct gist_loopback {
  int W = 0;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t gen = 0;
  std::vector<const void*> ptr;  // per rank: the buffer published for the current collective
  std::vector<int> joined;
  // comm_alltoallv: per source rank, per destination rank, its sends in order
  std::vector<std::vector<std::vector<std::pair<const void*, size_t>>>> a2a;
};

extern "C" gist_status gist_loopback_create(int32_t world_size, gist_loopback** out) {
  if (!out || world_size < 1) return GIST_E_ARG;
  gist_loopback* lb = new gist_loopback();
  lb->W = world_size;
  lb->ptr.assign(world_size, nullptr);
  lb->joined.assign(world_size, 0);
  *out = lb;
  return GIST_OK;
}

extern "C" void gist_loopback_destroy(gist_loopback* lb) { delete lb; }

namespace gist {
namespace {

// host rendezvous of the W rank threads (generation counting: reusable back to back)
void lb_barrier(gist_loopback* lb) {
  std::unique_lock<std::mutex> lk(lb->mu);
  const uint64_t g = lb->gen;
  if (++lb->arrived == lb->W) {
    lb->arrived = 0;
    ++lb->gen;
    lb->cv.notify_all();
  } else {
    lb->cv.wait(lk, [&] { return lb->gen != g; });
  }
}

void publish(gist_loopback* lb, int rank, const void* p) {
  std::lock_guard<std::mutex> lk(lb->mu);
  lb->ptr[rank] = p;
}

gist_status cuda_fail(cudaError_t e, const char* what, std::string* err) {
  if (err) *err = std::string(what) + ": " + cudaGetErrorString(e);
  return e == cudaErrorMemoryAllocation ? GIST_E_OOM : GIST_E_CUDA;
}
gist_status nccl_fail(ncclResult_t r, const char* what, std::string* err) {
  if (err) *err = std::string(what) + ": " + ncclGetErrorString(r);
  return GIST_E_NCCL;
}

#define CKC(x, what)                                  \
  do {                                                \
    cudaError_t e_ = (x);                             \
    if (e_ != cudaSuccess) return cuda_fail(e_, what, err); \
  } while (0)

}  // namespace

gist_status loopback_join(gist_loopback* lb, int rank, int world) {
  if (!lb || lb->W != world || rank < 0 || rank >= world) return GIST_E_ARG;
  std::lock_guard<std::mutex> lk(lb->mu);
  if (lb->joined[rank]) return GIST_E_ARG;  // one context per rank
  lb->joined[rank] = 1;
  return GIST_OK;
}

void loopback_leave(gist_loopback* lb, int rank) {
  if (!lb || rank < 0 || rank >= lb->W) return;
  std::lock_guard<std::mutex> lk(lb->mu);
  lb->joined[rank] = 0;
}

gist_status comm_allgather(const Comm& c, const void* send, void* recv, size_t bytes, cudaStream_t s,
                           std::string* err) {
  if (c.world == 1) {
    if (send != recv && bytes) CKC(cudaMemcpyAsync(recv, send, bytes, cudaMemcpyDeviceToDevice, s), "allgather copy");
    return GIST_OK;
  }
  if (c.nccl) {
    ncclResult_t r = ncclAllGather(send, recv, bytes, ncclChar, c.nccl, s);
    return r == ncclSuccess ? GIST_OK : nccl_fail(r, "ncclAllGather", err);
  }
  gist_loopback* lb = c.lb;
  CKC(cudaStreamSynchronize(s), "loopback allgather: sync");  // this rank's send buffer is final
  publish(lb, c.rank, send);
  lb_barrier(lb);
  for (int r = 0; r < c.world; ++r) {
    char* dst = static_cast<char*>(recv) + (size_t)r * bytes;
    if (lb->ptr[r] != dst && bytes)
      CKC(cudaMemcpyAsync(dst, lb->ptr[r], bytes, cudaMemcpyDeviceToDevice, s), "loopback allgather: copy");
  }
  CKC(cudaStreamSynchronize(s), "loopback allgather: sync");
  lb_barrier(lb);  // no rank reuses its send buffer before every peer has copied it
  return GIST_OK;
}

gist_status comm_allreduce_sum(const Comm& c, void* buf, size_t count, bool f64, cudaStream_t s, std::string* err) {
  if (c.world == 1 || count == 0) return GIST_OK;
  if (c.nccl) {
    ncclResult_t r = ncclAllReduce(buf, buf, count, f64 ? ncclDouble : ncclFloat, ncclSum, c.nccl, s);
    return r == ncclSuccess ? GIST_OK : nccl_fail(r, "ncclAllReduce", err);
  }
  gist_loopback* lb = c.lb;
  const size_t es = f64 ? 8 : 4;
  CKC(cudaStreamSynchronize(s), "loopback allreduce: sync");
  publish(lb, c.rank, buf);
  lb_barrier(lb);
  std::vector<double> acc(count, 0.0);
  std::vector<char> tmp(count * es);
  for (int r = 0; r < c.world; ++r) {  // fixed rank order
    CKC(cudaMemcpyAsync(tmp.data(), lb->ptr[r], count * es, cudaMemcpyDeviceToHost, s), "loopback allreduce: copy");
    CKC(cudaStreamSynchronize(s), "loopback allreduce: sync");
    for (size_t i = 0; i < count; ++i) {
      if (f64) {
        double v;
        std::memcpy(&v, tmp.data() + i * 8, 8);
        acc[i] += v;
      } else {
        float v;
        std::memcpy(&v, tmp.data() + i * 4, 4);
        acc[i] = (double)((float)acc[i] + v);  // fp32 accumulation, like an fp32 reduction
      }
    }
  }
  lb_barrier(lb);  // every rank has read every input before any rank overwrites its own
  for (size_t i = 0; i < count; ++i) {
    if (f64) {
      std::memcpy(tmp.data() + i * 8, &acc[i], 8);
    } else {
      const float v = (float)acc[i];
      std::memcpy(tmp.data() + i * 4, &v, 4);
    }
  }
  CKC(cudaMemcpyAsync(buf, tmp.data(), count * es, cudaMemcpyHostToDevice, s), "loopback allreduce: copy");
  CKC(cudaStreamSynchronize(s), "loopback allreduce: sync");
  return GIST_OK;
}

gist_status comm_barrier(const Comm& c, float* word_dev, cudaStream_t s, std::string* err) {
  if (c.world == 1) return GIST_OK;
  if (c.nccl) {
    ncclResult_t r = ncclAllReduce(word_dev, word_dev, 1, ncclFloat, ncclSum, c.nccl, s);
    return r == ncclSuccess ? GIST_OK : nccl_fail(r, "ncclAllReduce (barrier)", err);
  }
  CKC(cudaStreamSynchronize(s), "loopback barrier: sync");
  lb_barrier(c.lb);
  return GIST_OK;
}

gist_status comm_alltoallv(const Comm& c, const std::vector<Xfer>& sends, const std::vector<Xfer>& recvs,
                           cudaStream_t s, std::string* err) {
  if (c.nccl) {
    ncclResult_t r = ncclGroupStart();
    for (const Xfer& x : sends)
      if (r == ncclSuccess && x.bytes) r = ncclSend(x.ptr, x.bytes, ncclChar, x.peer, c.nccl, s);
    for (const Xfer& x : recvs)
      if (r == ncclSuccess && x.bytes) r = ncclRecv(x.ptr, x.bytes, ncclChar, x.peer, c.nccl, s);
    const ncclResult_t e = ncclGroupEnd();
    if (r == ncclSuccess) r = e;
    return r == ncclSuccess ? GIST_OK : nccl_fail(r, "ncclSend/ncclRecv (all-to-all)", err);
  }
  if (c.world == 1) {  // only self transfers
    size_t k = 0;
    for (const Xfer& x : recvs) {
      if (k >= sends.size() || sends[k].bytes != x.bytes) {
        if (err) *err = "alltoallv: unmatched self transfer";
        return GIST_E_ARG;
      }
      if (x.bytes && x.ptr != sends[k].ptr)
        CKC(cudaMemcpyAsync(x.ptr, sends[k].ptr, x.bytes, cudaMemcpyDeviceToDevice, s), "alltoallv self copy");
      ++k;
    }
    return GIST_OK;
  }
  gist_loopback* lb = c.lb;
  CKC(cudaStreamSynchronize(s), "loopback alltoallv: sync");  // this rank's send buffers are final
  {
    std::lock_guard<std::mutex> lk(lb->mu);
    if (lb->a2a.size() != (size_t)c.world) lb->a2a.assign(c.world, {});
    auto& mine = lb->a2a[c.rank];
    mine.assign(c.world, {});
    for (const Xfer& x : sends) mine[x.peer].push_back({x.ptr, x.bytes});
  }
  lb_barrier(lb);
  std::vector<size_t> next(c.world, 0);
  bool match = true;
  cudaError_t ce = cudaSuccess;
  for (const Xfer& x : recvs) {
    const auto& from = lb->a2a[x.peer][c.rank];
    const size_t k = next[x.peer]++;
    if (k >= from.size() || from[k].second != x.bytes) {
      match = false;
      continue;
    }
    if (x.bytes && ce == cudaSuccess) ce = cudaMemcpyAsync(x.ptr, from[k].first, x.bytes, cudaMemcpyDeviceToDevice, s);
  }
  const cudaError_t ce2 = cudaStreamSynchronize(s);
  lb_barrier(lb);  // no rank reuses its send buffers before every peer has copied them
  if (ce != cudaSuccess) return cuda_fail(ce, "loopback alltoallv: copy", err);
  if (ce2 != cudaSuccess) return cuda_fail(ce2, "loopback alltoallv: sync", err);
  if (!match) {
    if (err) *err = "alltoallv: send / recv lists do not match";
    return GIST_E_ARG;
  }
  return GIST_OK;
}

gist_status comm_exchange_ptr(const Comm& c, void* mine, std::vector<void*>& all, std::string* err) {
  all.assign(c.world, nullptr);
  if (c.world == 1) {
    all[0] = mine;
    return GIST_OK;
  }
  if (!c.lb) {
    if (err) *err = "pointer exchange needs the loopback transport (NCCL ranks exchange IPC handles)";
    return GIST_E_UNSUPPORTED;
  }
  publish(c.lb, c.rank, mine);
  lb_barrier(c.lb);
  for (int r = 0; r < c.world; ++r) all[r] = const_cast<void*>(c.lb->ptr[r]);
  lb_barrier(c.lb);
  return GIST_OK;
}

}  // namespace gist
