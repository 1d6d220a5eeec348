// kfvm_loopback.cuh — in-process loopback transport for the slab
// decomposition: several rank handles in ONE process (each driven by its own
// host thread, as MPI ranks would be), exchanging their halo planes,
// KXRCF edge flags, dt maxima and SSP(4,3) error planes by device-to-device
// cudaMemcpyAsync between their buffers instead of NCCL.  It runs the
// library's multi-rank code (halo(), k_halo_local, the rank-offset boundary
// and IC code, the overlapped schedule, the collectives) with nranks > 1 on a
// single GPU, with the NCCL call semantics the library relies on:
//   * send/recv inside a group are matched per (sender, receiver) pair in
//     posting order; a group's sends are all posted before any receive
//     waits, so a group never deadlocks;
//   * a send completes (on the sender's stream) only when the receiver's copy
//     has completed, so the sender may overwrite its buffer afterwards;
//   * allreduce(max, uint64) and allgather(double) are in place / ordered on
//     the caller's stream like the NCCL collectives.
// Host-side rendezvous: cross-stream ordering is by CUDA events recorded and
// waited before a peer is allowed to proceed, so nothing here is capturable
// in a CUDA graph — loopback handles always run the eager schedule.
// Included by kfvm_gpu.cu (outside namespace kfvm_b200).
#ifndef KFVM_LOOPBACK_CUH_
#define KFVM_LOOPBACK_CUH_

#include <atomic>
#include <condition_variable>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <tuple>
#include <vector>

namespace kfvm_loop {

__global__ void k_max_slots(unsigned long long* out, const unsigned long long* slots, int n) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    unsigned long long m = slots[0];
    for (int i = 1; i < n; ++i) m = slots[i] > m ? slots[i] : m;
    *out = m;
  }
}

struct Msg {
  const void* src = nullptr;
  size_t bytes = 0;
  cudaEvent_t ready = nullptr, done = nullptr;
  bool copied = false;  // the receiver has enqueued the copy and recorded `done`
};

struct Group {
  int nranks = 0, device = 0;
  std::mutex mu;
  std::condition_variable cv;
  std::map<std::tuple<int, int, long long>, std::shared_ptr<Msg>> mbox;  // (src, dst, seq)
  std::vector<long long> send_seq, recv_seq;                            // [src * n + dst]
  // collectives: per-rank op counters, the event each rank recorded after
  // writing / after reading the shared slots of its current op
  std::vector<long long> wrote, read;  // op index whose write / read is posted
  std::vector<cudaEvent_t> ev_wrote, ev_read;
  unsigned long long* slots_u64 = nullptr;
  double* slots_f64 = nullptr;
  size_t f64_count = 0;
  int users = 0;
};

struct Pending {
  bool send;
  void* ptr;
  size_t bytes;
  int peer;
  cudaStream_t st;
};

// Group ids travel in kfvm_dist.nccl_id: the magic "KFVMLOOP" and a key.
inline bool is_id(const unsigned char* id) { return std::memcmp(id, "KFVMLOOP", 8) == 0; }
inline unsigned long long id_key(const unsigned char* id) {
  unsigned long long k;
  std::memcpy(&k, id + 8, sizeof(k));
  return k;
}
inline void make_id(unsigned char* id) {
  static std::atomic<unsigned long long> next{1};
  std::memset(id, 0, 128);
  std::memcpy(id, "KFVMLOOP", 8);
  const unsigned long long k = next++;
  std::memcpy(id + 8, &k, sizeof(k));
}

inline std::mutex& registry_mu() {
  static std::mutex m;
  return m;
}
inline std::map<unsigned long long, Group*>& registry() {
  static std::map<unsigned long long, Group*> r;
  return r;
}

// join (or create) the group `key` as one of `nranks` ranks on `device`
inline Group* join(unsigned long long key, int nranks, int device) {
  std::lock_guard<std::mutex> lk(registry_mu());
  Group*& g = registry()[key];
  if (!g) {
    g = new Group();
    g->nranks = nranks;
    g->device = device;
    g->send_seq.assign((size_t)nranks * nranks, 0);
    g->recv_seq.assign((size_t)nranks * nranks, 0);
    g->wrote.assign(nranks, -1);
    g->read.assign(nranks, -1);
    g->ev_wrote.assign(nranks, nullptr);
    g->ev_read.assign(nranks, nullptr);
    for (int r = 0; r < nranks; ++r) {
      cudaEventCreateWithFlags(&g->ev_wrote[r], cudaEventDisableTiming);
      cudaEventCreateWithFlags(&g->ev_read[r], cudaEventDisableTiming);
    }
    cudaMalloc(&g->slots_u64, sizeof(unsigned long long) * nranks);
  }
  if (g->nranks != nranks || g->device != device) return nullptr;
  g->users++;
  return g;
}

inline void leave(unsigned long long key, Group* g) {
  std::lock_guard<std::mutex> lk(registry_mu());
  if (--g->users > 0) return;
  for (auto& kv : g->mbox) {
    cudaEventDestroy(kv.second->ready);
    cudaEventDestroy(kv.second->done);
  }
  for (int r = 0; r < g->nranks; ++r) {
    cudaEventDestroy(g->ev_wrote[r]);
    cudaEventDestroy(g->ev_read[r]);
  }
  cudaFree(g->slots_u64);
  cudaFree(g->slots_f64);
  registry().erase(key);
  delete g;
}

// Execute one group of point-to-point operations of `rank` (in posting order).
inline int group_end(Group* g, int rank, std::vector<Pending>& ops) {
  const int n = g->nranks;
  std::vector<std::shared_ptr<Msg>> mine;
  std::unique_lock<std::mutex> lk(g->mu);
  // 1. post every send: its data is ready when the sender's stream reaches here
  for (const Pending& o : ops) {
    if (!o.send) continue;
    auto m = std::make_shared<Msg>();
    m->src = o.ptr;
    m->bytes = o.bytes;
    if (cudaEventCreateWithFlags(&m->ready, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&m->done, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventRecord(m->ready, o.st) != cudaSuccess)
      return 1;
    const long long s = g->send_seq[(size_t)rank * n + o.peer]++;
    g->mbox[{rank, o.peer, s}] = m;
    mine.push_back(m);
  }
  g->cv.notify_all();
  // 2. receive in posting order: wait for the matching send, copy on my stream
  for (const Pending& o : ops) {
    if (o.send) continue;
    const long long s = g->recv_seq[(size_t)o.peer * n + rank]++;
    const auto key = std::make_tuple(o.peer, rank, s);
    g->cv.wait(lk, [&] { return g->mbox.count(key) != 0; });
    std::shared_ptr<Msg> m = g->mbox[key];
    if (m->bytes != o.bytes) return 2;
    if (cudaStreamWaitEvent(o.st, m->ready, 0) != cudaSuccess ||
        cudaMemcpyAsync(o.ptr, m->src, o.bytes, cudaMemcpyDeviceToDevice, o.st) != cudaSuccess ||
        cudaEventRecord(m->done, o.st) != cudaSuccess)
      return 1;
    m->copied = true;
    g->mbox.erase(key);
    g->cv.notify_all();
  }
  // 3. a send completes when its receiver's copy has (ordered on my stream)
  size_t k = 0;
  for (const Pending& o : ops) {
    if (!o.send) continue;
    std::shared_ptr<Msg> m = mine[k++];
    g->cv.wait(lk, [&] { return m->copied; });
    if (cudaStreamWaitEvent(o.st, m->done, 0) != cudaSuccess) return 1;
    cudaEventDestroy(m->ready);  // released once the pending work completes
    cudaEventDestroy(m->done);
  }
  return 0;
}

// Collective skeleton: every rank writes its contribution into the shared
// slots (after all ranks have finished reading the previous op's slots),
// waits for all contributions, then reads.  `op` is the rank's op counter.
template <typename Write, typename Read>
inline int collective(Group* g, int rank, long long& op, cudaStream_t st, Write write, Read read) {
  const int n = g->nranks;
  std::unique_lock<std::mutex> lk(g->mu);
  const long long me = ++op;
  // everyone has read op me-1 (so its slots are free on the device too)
  g->cv.wait(lk, [&] {
    for (int r = 0; r < n; ++r)
      if (g->read[r] < me - 1) return false;
    return true;
  });
  for (int r = 0; r < n; ++r)
    if (r != rank && cudaStreamWaitEvent(st, g->ev_read[r], 0) != cudaSuccess) return 1;
  if (write()) return 1;
  if (cudaEventRecord(g->ev_wrote[rank], st) != cudaSuccess) return 1;
  g->wrote[rank] = me;
  g->cv.notify_all();
  g->cv.wait(lk, [&] {
    for (int r = 0; r < n; ++r)
      if (g->wrote[r] < me) return false;
    return true;
  });
  for (int r = 0; r < n; ++r)
    if (r != rank && cudaStreamWaitEvent(st, g->ev_wrote[r], 0) != cudaSuccess) return 1;
  if (read()) return 1;
  if (cudaEventRecord(g->ev_read[rank], st) != cudaSuccess) return 1;
  g->read[rank] = me;
  g->cv.notify_all();
  return 0;
}

// in-place max over ranks of one uint64 (the dt wavespeed reduction)
inline int allreduce_max_u64(Group* g, int rank, long long& op, unsigned long long* p,
                             cudaStream_t st) {
  return collective(
      g, rank, op, st,
      [&] {
        return cudaMemcpyAsync(g->slots_u64 + rank, p, sizeof(unsigned long long),
                               cudaMemcpyDeviceToDevice, st) != cudaSuccess;
      },
      [&] {
        k_max_slots<<<1, 32, 0, st>>>(p, g->slots_u64, g->nranks);
        return cudaGetLastError() != cudaSuccess;
      });
}

// allgather of `count` doubles per rank into dst[nranks * count]
inline int allgather_f64(Group* g, int rank, long long& op, const double* src, double* dst,
                         size_t count, cudaStream_t st) {
  {
    std::lock_guard<std::mutex> lk(g->mu);
    if (!g->slots_f64) {
      if (cudaMalloc(&g->slots_f64, sizeof(double) * count * g->nranks) != cudaSuccess) return 1;
      g->f64_count = count;
    }
    if (count != g->f64_count) return 2;
  }
  return collective(
      g, rank, op, st,
      [&] {
        return cudaMemcpyAsync(g->slots_f64 + (size_t)rank * count, src, sizeof(double) * count,
                               cudaMemcpyDeviceToDevice, st) != cudaSuccess;
      },
      [&] {
        return cudaMemcpyAsync(dst, g->slots_f64, sizeof(double) * count * g->nranks,
                               cudaMemcpyDeviceToDevice, st) != cudaSuccess;
      });
}

}  // namespace kfvm_loop

#endif
