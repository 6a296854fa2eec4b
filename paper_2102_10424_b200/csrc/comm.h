// comm.h -- the collectives of the GIST round structure (subAgg all-gather, eval all-reduce,
// barriers of the peer-store subAgg), behind one interface with two transports:
//   NCCL      one process per GPU (the product path)
//   loopback  W contexts of ONE process on one device stand in for W ranks (tests): the host
//             rendezvouses the W calling threads and moves the bytes with device-to-device
//             copies, so the library's W > 1 code (slot ownership, packing offsets, unpack /
//             scatter, peer stores, row-split eval) runs unchanged on one GPU.  No kernel ever
//             waits on another rank: every wait is a host-side stream synchronise + barrier.
#pragma once
#include <cuda_runtime.h>
#include <nccl.h>

#include <cstddef>
#include <string>
#include <vector>

#include "../../include/gist.h"

namespace gist {

struct Comm {
  ncclComm_t nccl = nullptr;
  gist_loopback* lb = nullptr;
  int rank = 0, world = 1;
};

// recv[r * bytes .. (r+1) * bytes) = rank r's send (in place allowed: send == recv + rank * bytes)
gist_status comm_allgather(const Comm& c, const void* send, void* recv, size_t bytes, cudaStream_t s,
                           std::string* err);
// elementwise sum over ranks, in place; f64 = double elements, else float
gist_status comm_allreduce_sum(const Comm& c, void* buf, size_t count, bool f64, cudaStream_t s, std::string* err);
// every rank's stream work issued before the call has completed before any rank's work after it
// (NCCL: a one-word all-reduce on `word_dev`, which orders the streams device-side)
gist_status comm_barrier(const Comm& c, float* word_dev, cudaStream_t s, std::string* err);
// point-to-point exchange of variable-size pieces (the owner-sharded Theta's re-partition and
// subAgg): `sends` / `recvs` list (peer, device pointer, bytes); the k-th send of rank a to rank b
// is matched with the k-th recv of rank b from rank a (both sides enumerate in the same order).
// NCCL: one grouped ncclSend / ncclRecv; loopback: device-to-device copies by the receiver.
struct Xfer {
  int peer;
  void* ptr;
  size_t bytes;
};
gist_status comm_alltoallv(const Comm& c, const std::vector<Xfer>& sends, const std::vector<Xfer>& recvs,
                           cudaStream_t s, std::string* err);
// loopback only: every rank's pointer (the P2P subAgg replica regions of one process)
gist_status comm_exchange_ptr(const Comm& c, void* mine, std::vector<void*>& all, std::string* err);
// loopback: attach / validate a context's rank
gist_status loopback_join(gist_loopback* lb, int rank, int world);
void loopback_leave(gist_loopback* lb, int rank);

}  // namespace gist
