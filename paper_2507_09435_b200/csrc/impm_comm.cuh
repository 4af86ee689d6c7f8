// Collectives of the slab-decomposed Newton step.
//
// The reference is single-process (mpm_solver.hpp:56-477 owns all state);
// its DofMap numbering (grid.hpp:69-86) and ±2-node Jacobian coupling
// (jacobian.hpp:36-65) are what make an axis-0 slab decomposition exact:
// every owned row needs only owned + two ghost particle layers and a 2-plane
// vector halo. The traffic per Newton iteration is:
//   - a 2-plane halo of one node vector before each SpMV / residual / tangent;
//   - an elementwise sum of the fixed-size reduction-partial arrays that every
//     dot product already produces (the fixed-order finalize that follows is
//     then global and identical on every rank, so all ranks take the same
//     Krylov / Newton decisions without a host round trip);
//   - min / max of a few status words (DomainError ids, max particle mass).
//
// Two transports implement it:
//   NcclComm  - one process per GPU, ncclAllReduce + grouped ncclSend/ncclRecv
//               on the simulation stream (NVLink 5 / NVSwitch on a B200 node);
//   LocalComm - ranks as host threads of one process sharing one device:
//               every collective is host-ordered (stream sync + barrier +
//               device copies), no kernel ever waits on another rank. This is
//               the single-GPU test transport for the multi-rank code path.
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>

#include <condition_variable>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

namespace impm_gpu {

enum class RedOp { Sum, Max, Min };
enum class RedType { F64, I64, I32 };

struct CommError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

struct Comm {
  int rank = 0, nranks = 1;
  struct Msg {
    int peer;
    void* buf;
    size_t bytes;
  };
  virtual ~Comm() = default;
  // in-place elementwise reduction over ranks, ordered on `s`; the result is
  // bitwise identical on every rank
  virtual void allreduce(void* d, size_t n, RedType t, RedOp op, cudaStream_t s) = 0;
  // grouped point-to-point: all sends and receives of one halo / migration
  // round; byte counts must match pairwise (zero-byte messages are skipped by
  // both sides)
  virtual void exchange(const std::vector<Msg>& sends, const std::vector<Msg>& recvs, cudaStream_t s) = 0;
  virtual const char* kind() const = 0;
};

// ------------------------------------------------------------------ NCCL --
#define NCK(call)                                                                                      \
  do {                                                                                                 \
    ncclResult_t r_ = (call);                                                                          \
    if (r_ != ncclSuccess) throw CommError(std::string("NCCL error ") + ncclGetErrorString(r_) + " at " + \
                                           __FILE__ + ":" + std::to_string(__LINE__));                 \
  } while (0)

struct NcclComm final : Comm {
  ncclComm_t c = nullptr;
  NcclComm(const ncclUniqueId& id, int r, int n) {
    rank = r;
    nranks = n;
    NCK(ncclCommInitRank(&c, n, id, r));
  }
  ~NcclComm() override {
    if (c) ncclCommDestroy(c);
  }
  static ncclDataType_t dt(RedType t) {
    return t == RedType::F64 ? ncclFloat64 : (t == RedType::I64 ? ncclInt64 : ncclInt32);
  }
  static ncclRedOp_t op(RedOp o) { return o == RedOp::Sum ? ncclSum : (o == RedOp::Max ? ncclMax : ncclMin); }
  void allreduce(void* d, size_t n, RedType t, RedOp o, cudaStream_t s) override {
    if (nranks == 1 || n == 0) return;
    NCK(ncclAllReduce(d, d, n, dt(t), op(o), c, s));
  }
  void exchange(const std::vector<Msg>& sends, const std::vector<Msg>& recvs, cudaStream_t s) override {
    NCK(ncclGroupStart());
    for (const auto& m : sends)
      if (m.bytes) NCK(ncclSend(m.buf, m.bytes, ncclUint8, m.peer, c, s));
    for (const auto& m : recvs)
      if (m.bytes) NCK(ncclRecv(m.buf, m.bytes, ncclUint8, m.peer, c, s));
    NCK(ncclGroupEnd());
  }
  const char* kind() const override { return "nccl"; }
};

// ------------------------------------------------------- in-process group --
template <class T, int OP>
__global__ void k_reduce_ranks(int nr, const void* const* __restrict__ src, size_t n, T* __restrict__ out) {
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    T acc = static_cast<const T*>(src[0])[i];
    for (int r = 1; r < nr; ++r) {  // fixed rank order
      const T v = static_cast<const T*>(src[r])[i];
      acc = OP == 0 ? acc + v : (OP == 1 ? (v > acc ? v : acc) : (v < acc ? v : acc));
    }
    out[i] = acc;
  }
}

struct LocalGroup {
  int n;
  std::mutex m;
  std::condition_variable cv;
  int arrived = 0;
  long long gen = 0;
  std::vector<const void*> ptr;               // published per-rank buffers
  std::vector<std::vector<Comm::Msg>> mail;   // [src] -> outgoing messages
  explicit LocalGroup(int n_) : n(n_), ptr(n_), mail(n_) {}
  void barrier() {
    std::unique_lock<std::mutex> lk(m);
    const long long g = gen;
    if (++arrived == n) {
      arrived = 0;
      ++gen;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != g; });
    }
  }
};

struct LocalComm final : Comm {
  std::shared_ptr<LocalGroup> grp;
  void* tmp = nullptr;
  size_t tmp_bytes = 0;
  void** dsrc_own = nullptr;
  LocalComm(std::shared_ptr<LocalGroup> g, int r) : grp(std::move(g)) {
    rank = r;
    nranks = grp->n;
    if (cudaMalloc(reinterpret_cast<void**>(&dsrc_own), sizeof(void*) * nranks) != cudaSuccess)
      throw CommError("local comm: cudaMalloc failed");
  }
  ~LocalComm() override {
    if (tmp) cudaFree(tmp);
    if (dsrc_own) cudaFree(dsrc_own);
  }
  static void ck(cudaError_t e) {
    if (e != cudaSuccess) throw CommError(std::string("local comm: ") + cudaGetErrorString(e));
  }
  template <class T>
  void reduce_into(size_t n, RedOp o, cudaStream_t s) {
    const unsigned blocks = static_cast<unsigned>(std::min<size_t>(1184, (n + 255) / 256 + 1));
    T* out = static_cast<T*>(tmp);
    if (o == RedOp::Sum) k_reduce_ranks<T, 0><<<blocks, 256, 0, s>>>(nranks, dsrc_own, n, out);
    else if (o == RedOp::Max) k_reduce_ranks<T, 1><<<blocks, 256, 0, s>>>(nranks, dsrc_own, n, out);
    else k_reduce_ranks<T, 2><<<blocks, 256, 0, s>>>(nranks, dsrc_own, n, out);
    ck(cudaGetLastError());
  }
  void allreduce(void* d, size_t n, RedType t, RedOp o, cudaStream_t s) override {
    if (nranks == 1 || n == 0) return;
    const size_t es = t == RedType::I32 ? 4 : 8;
    if (tmp_bytes < n * es) {
      if (tmp) cudaFree(tmp);
      ck(cudaMalloc(&tmp, n * es));
      tmp_bytes = n * es;
    }
    ck(cudaStreamSynchronize(s));
    grp->ptr[rank] = d;
    grp->barrier();  // every rank's buffer is final and published
    ck(cudaMemcpyAsync(dsrc_own, grp->ptr.data(), sizeof(void*) * nranks, cudaMemcpyHostToDevice, s));
    if (t == RedType::F64) reduce_into<double>(n, o, s);
    else if (t == RedType::I64) reduce_into<long long>(n, o, s);
    else reduce_into<int>(n, o, s);
    ck(cudaStreamSynchronize(s));
    grp->barrier();  // nobody reads the published buffers any more
    ck(cudaMemcpyAsync(d, tmp, n * es, cudaMemcpyDeviceToDevice, s));
    ck(cudaStreamSynchronize(s));
  }
  void exchange(const std::vector<Msg>& sends, const std::vector<Msg>& recvs, cudaStream_t s) override {
    ck(cudaStreamSynchronize(s));
    grp->mail[rank] = sends;
    grp->barrier();
    for (const auto& rm : recvs) {
      if (!rm.bytes) continue;
      const Msg* found = nullptr;
      for (const auto& sm : grp->mail[rm.peer])
        if (sm.peer == rank) found = &sm;
      if (!found || found->bytes != rm.bytes)
        throw CommError("local comm: unmatched message from rank " + std::to_string(rm.peer));
      ck(cudaMemcpyAsync(rm.buf, found->buf, rm.bytes, cudaMemcpyDeviceToDevice, s));
    }
    ck(cudaStreamSynchronize(s));
    grp->barrier();  // senders may reuse their buffers
  }
  const char* kind() const override { return "local"; }
};

}  // namespace impm_gpu
