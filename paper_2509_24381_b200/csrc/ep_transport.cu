// rserve-b200 — EP transports: in-process loopback and NCCL point-to-point.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <thread>

#include "ep.cuh"

namespace rserve::ep {

void Transport::wait(Xfer& x) {
  while (!test(x)) std::this_thread::yield();
}

namespace {

/// Events for receive completions: each Xfer owns one until it is dropped.
class EventPool {
 public:
  ~EventPool() {
    for (cudaEvent_t e : free_) cudaEventDestroy(e);
  }
  cudaEvent_t get() {
    std::lock_guard<std::mutex> g(mu_);
    if (!free_.empty()) {
      cudaEvent_t e = free_.back();
      free_.pop_back();
      return e;
    }
    cudaEvent_t e;  // timing-enabled: P0 stamps completions with it
    RS_CUDA_CHECK(cudaEventCreate(&e));
    return e;
  }
  void put(cudaEvent_t e) {
    std::lock_guard<std::mutex> g(mu_);
    free_.push_back(e);
  }

 private:
  std::mutex mu_;
  std::vector<cudaEvent_t> free_;
};

/// Send-completion events: a ring per link. Reusing an event only ever makes
/// a later waiter wait for a later send on the same in-order link stream,
/// which is conservative.
struct EventRing {
  std::vector<cudaEvent_t> ev;
  std::size_t next = 0;
  void init(std::size_t n) {
    ev.resize(n);
    for (auto& e : ev) RS_CUDA_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  void destroy() {
    for (auto e : ev) cudaEventDestroy(e);
    ev.clear();
  }
  cudaEvent_t take() {
    cudaEvent_t e = ev[next];
    next = (next + 1) % ev.size();
    return e;
  }
};

std::shared_ptr<Xfer> new_xfer(EventPool& pool) {
  Xfer* x = new Xfer();
  x->done = pool.get();
  return std::shared_ptr<Xfer>(x, [&pool](Xfer* p) {
    pool.put(p->done);
    delete p;
  });
}

}  // namespace

// ---- loopback ----------------------------------------------------------------------------
LoopbackHub::~LoopbackHub() {
  cudaDeviceSynchronize();
  for (auto& q : queues_)
    for (Msg& m : q) {
      cudaFree(m.buf);
      cudaEventDestroy(m.ready);
    }
  for (Buf& b : pool_) {
    cudaFree(b.p);
    if (b.after) cudaEventDestroy(b.after);
  }
}

void LoopbackHub::push(int src, int dst, const Msg& m) {
  std::lock_guard<std::mutex> g(mu_);
  queues_[static_cast<std::size_t>(src * world_ + dst)].push_back(m);
}

bool LoopbackHub::pop(int src, int dst, Msg* out) {
  std::lock_guard<std::mutex> g(mu_);
  auto& q = queues_[static_cast<std::size_t>(src * world_ + dst)];
  if (q.empty()) return false;
  *out = q.front();
  q.pop_front();
  return true;
}

void* LoopbackHub::take_buffer(std::size_t bytes) {
  std::lock_guard<std::mutex> g(mu_);
  for (Buf& b : pool_) {
    if (b.in_use || b.bytes < bytes) continue;
    if (b.after != nullptr) {
      const cudaError_t q = cudaEventQuery(b.after);
      if (q == cudaErrorNotReady) continue;
      RS_CUDA_CHECK(q);
    }
    b.in_use = true;
    return b.p;
  }
  void* p = nullptr;
  RS_CUDA_CHECK(cudaMalloc(&p, bytes));
  pool_.push_back({p, bytes, true, nullptr});
  return p;
}

void LoopbackHub::give_buffer(void* p, cudaStream_t reader) {
  std::lock_guard<std::mutex> g(mu_);
  for (Buf& b : pool_) {
    if (b.p != p) continue;
    if (b.after == nullptr) RS_CUDA_CHECK(cudaEventCreateWithFlags(&b.after, cudaEventDisableTiming));
    RS_CUDA_CHECK(cudaEventRecord(b.after, reader));  // free once the reader's copy ran
    b.in_use = false;
    return;
  }
  throw DeviceError(RS_ERR_CUDA, "loopback: unknown buffer returned");
}

namespace {

class LoopbackTransport final : public Transport {
 public:
  LoopbackTransport(LoopbackHub& hub, int rank, int device) : hub_(hub), rank_(rank), dev_(device) {
    RS_CUDA_CHECK(cudaSetDevice(device));
    const int w = hub.world();
    send_st_.resize(static_cast<std::size_t>(w));
    recv_st_.resize(static_cast<std::size_t>(w));
    rings_.resize(static_cast<std::size_t>(w));
    pending_.resize(static_cast<std::size_t>(w));
    for (int p = 0; p < w; ++p) {
      RS_CUDA_CHECK(cudaStreamCreateWithFlags(&send_st_[static_cast<std::size_t>(p)], cudaStreamNonBlocking));
      RS_CUDA_CHECK(cudaStreamCreateWithFlags(&recv_st_[static_cast<std::size_t>(p)], cudaStreamNonBlocking));
      rings_[static_cast<std::size_t>(p)].init(64);
    }
  }
  ~LoopbackTransport() override {
    cudaDeviceSynchronize();
    for (auto s : send_st_) cudaStreamDestroy(s);
    for (auto s : recv_st_) cudaStreamDestroy(s);
    for (auto& r : rings_) r.destroy();
  }
  int rank() const override { return rank_; }
  int world() const override { return hub_.world(); }

  cudaEvent_t send(int peer, const void* src, std::size_t bytes, cudaEvent_t wait) override {
    cudaStream_t st = send_st_.at(static_cast<std::size_t>(peer));
    if (wait != nullptr) RS_CUDA_CHECK(cudaStreamWaitEvent(st, wait, 0));
    LoopbackHub::Msg m;
    m.bytes = bytes;
    m.buf = hub_.take_buffer(bytes);
    RS_CUDA_CHECK(cudaEventCreateWithFlags(&m.ready, cudaEventDisableTiming));
    RS_CUDA_CHECK(cudaMemcpyAsync(m.buf, src, bytes, cudaMemcpyDeviceToDevice, st));
    RS_CUDA_CHECK(cudaEventRecord(m.ready, st));
    cudaEvent_t done = rings_[static_cast<std::size_t>(peer)].take();
    RS_CUDA_CHECK(cudaEventRecord(done, st));
    hub_.push(rank_, peer, m);
    return done;
  }

  std::shared_ptr<Xfer> post_recv(int peer, void* dst, std::size_t bytes, cudaEvent_t wait) override {
    auto x = new_xfer(events_);
    x->peer = peer;
    x->dst = dst;
    x->bytes = bytes;
    x->wait = wait;
    pending_.at(static_cast<std::size_t>(peer)).push_back(x);
    progress(peer);
    return x;
  }

  void wait_posted(Xfer& x) override {
    while (!x.posted) {
      progress(x.peer);
      if (!x.posted) std::this_thread::yield();
    }
  }

  bool test(Xfer& x) override {
    if (!x.posted) progress(x.peer);
    if (!x.posted) return false;
    const cudaError_t q = cudaEventQuery(x.done);
    if (q == cudaErrorNotReady) return false;
    RS_CUDA_CHECK(q);
    return true;
  }

 private:
  // Matches queued messages from `peer` with posted receives, in order.
  void progress(int peer) {
    auto& pend = pending_[static_cast<std::size_t>(peer)];
    while (!pend.empty()) {
      std::shared_ptr<Xfer> x = pend.front().lock();
      if (!x) {  // receive dropped before completion: still consume its message
        LoopbackHub::Msg m;
        if (!hub_.pop(peer, rank_, &m)) return;
        cudaStream_t st = recv_st_[static_cast<std::size_t>(peer)];
        RS_CUDA_CHECK(cudaStreamWaitEvent(st, m.ready, 0));
        hub_.give_buffer(m.buf, st);
        cudaEventDestroy(m.ready);
        pend.pop_front();
        continue;
      }
      LoopbackHub::Msg m;
      if (!hub_.pop(peer, rank_, &m)) return;
      if (m.bytes != x->bytes)
        throw DeviceError(RS_ERR_CUDA, "loopback: message of " + std::to_string(m.bytes) +
                                           " bytes for a receive of " + std::to_string(x->bytes));
      cudaStream_t st = recv_st_[static_cast<std::size_t>(peer)];
      RS_CUDA_CHECK(cudaStreamWaitEvent(st, m.ready, 0));
      if (x->wait != nullptr) RS_CUDA_CHECK(cudaStreamWaitEvent(st, x->wait, 0));
      RS_CUDA_CHECK(cudaMemcpyAsync(x->dst, m.buf, m.bytes, cudaMemcpyDeviceToDevice, st));
      RS_CUDA_CHECK(cudaEventRecord(x->done, st));
      x->posted = true;
      hub_.give_buffer(m.buf, st);
      RS_CUDA_CHECK(cudaEventDestroy(m.ready));
      pend.pop_front();
    }
  }

  LoopbackHub& hub_;
  int rank_, dev_;
  std::vector<cudaStream_t> send_st_, recv_st_;
  std::vector<EventRing> rings_;
  EventPool events_;
  std::vector<std::deque<std::weak_ptr<Xfer>>> pending_;
};

}  // namespace

std::unique_ptr<Transport> make_loopback(LoopbackHub& hub, int rank, int device) {
  return std::make_unique<LoopbackTransport>(hub, rank, device);
}

// ---- NCCL ----------------------------------------------------------------------------------
namespace {

/// libnccl.so.2 resolved at run time: in a torch process this is the NCCL
/// torch already loaded, so both share one library instance.
struct NcclApi {
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;

  static NcclApi& get() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
      void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
      if (h == nullptr) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
      if (h == nullptr) return;
      api.get_unique_id = reinterpret_cast<decltype(api.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
      api.comm_init_rank = reinterpret_cast<decltype(api.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
      api.comm_destroy = reinterpret_cast<decltype(api.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
      api.send = reinterpret_cast<decltype(api.send)>(dlsym(h, "ncclSend"));
      api.recv = reinterpret_cast<decltype(api.recv)>(dlsym(h, "ncclRecv"));
      api.error_string = reinterpret_cast<decltype(api.error_string)>(dlsym(h, "ncclGetErrorString"));
    });
    if (api.send == nullptr || api.comm_init_rank == nullptr)
      throw DeviceError(RS_ERR_NCCL, "libnccl.so.2 not loadable (EP over NCCL needs it)");
    return api;
  }
};

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    throw DeviceError(RS_ERR_NCCL, std::string(what) + ": " + NcclApi::get().error_string(r));
}

class NcclTransport final : public Transport {
 public:
  NcclTransport(const Topology& topo, int rank, int device, const void* ids)
      : rank_(rank), world_(topo.world()) {
    RS_CUDA_CHECK(cudaSetDevice(device));
    NcclApi& api = NcclApi::get();
    const auto links = topo.links();
    const int W = world_;
    send_comm_.assign(static_cast<std::size_t>(W), nullptr);
    recv_comm_.assign(static_cast<std::size_t>(W), nullptr);
    send_st_.assign(static_cast<std::size_t>(W), nullptr);
    recv_st_.assign(static_cast<std::size_t>(W), nullptr);
    rings_.resize(static_cast<std::size_t>(W));
    // Every rank walks the links in the same order and joins the ones it is
    // an end of: a blocking 2-rank init per link cannot deadlock.
    for (std::size_t l = 0; l < links.size(); ++l) {
      const auto [src, dst] = links[l];
      if (src != rank && dst != rank) continue;
      ncclUniqueId id;
      std::memcpy(&id, static_cast<const char*>(ids) + l * sizeof(ncclUniqueId), sizeof(id));
      ncclComm_t comm = nullptr;
      nccl_check(api.comm_init_rank(&comm, 2, id, src == rank ? 0 : 1), "ncclCommInitRank");
      cudaStream_t st;
      RS_CUDA_CHECK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
      if (src == rank) {
        send_comm_[static_cast<std::size_t>(dst)] = comm;
        send_st_[static_cast<std::size_t>(dst)] = st;
        rings_[static_cast<std::size_t>(dst)].init(64);
      } else {
        recv_comm_[static_cast<std::size_t>(src)] = comm;
        recv_st_[static_cast<std::size_t>(src)] = st;
      }
    }
  }
  ~NcclTransport() override {
    cudaDeviceSynchronize();
    NcclApi& api = NcclApi::get();
    for (auto c : send_comm_)
      if (c) api.comm_destroy(c);
    for (auto c : recv_comm_)
      if (c) api.comm_destroy(c);
    for (auto s : send_st_)
      if (s) cudaStreamDestroy(s);
    for (auto s : recv_st_)
      if (s) cudaStreamDestroy(s);
    for (auto& r : rings_) r.destroy();
  }
  int rank() const override { return rank_; }
  int world() const override { return world_; }

  cudaEvent_t send(int peer, const void* src, std::size_t bytes, cudaEvent_t wait) override {
    ncclComm_t comm = send_comm_.at(static_cast<std::size_t>(peer));
    if (comm == nullptr) throw DeviceError(RS_ERR_NCCL, "no EP link " + std::to_string(rank_) + "->" + std::to_string(peer));
    cudaStream_t st = send_st_[static_cast<std::size_t>(peer)];
    if (wait != nullptr) RS_CUDA_CHECK(cudaStreamWaitEvent(st, wait, 0));
    nccl_check(NcclApi::get().send(src, bytes, ncclUint8, 1, comm, st), "ncclSend");
    cudaEvent_t done = rings_[static_cast<std::size_t>(peer)].take();
    RS_CUDA_CHECK(cudaEventRecord(done, st));
    return done;
  }

  std::shared_ptr<Xfer> post_recv(int peer, void* dst, std::size_t bytes, cudaEvent_t wait) override {
    ncclComm_t comm = recv_comm_.at(static_cast<std::size_t>(peer));
    if (comm == nullptr) throw DeviceError(RS_ERR_NCCL, "no EP link " + std::to_string(peer) + "->" + std::to_string(rank_));
    cudaStream_t st = recv_st_[static_cast<std::size_t>(peer)];
    if (wait != nullptr) RS_CUDA_CHECK(cudaStreamWaitEvent(st, wait, 0));
    auto x = new_xfer(events_);
    x->peer = peer;
    x->dst = dst;
    x->bytes = bytes;
    nccl_check(NcclApi::get().recv(dst, bytes, ncclUint8, 0, comm, st), "ncclRecv");
    RS_CUDA_CHECK(cudaEventRecord(x->done, st));
    x->posted = true;
    return x;
  }

  void wait_posted(Xfer&) override {}

  bool test(Xfer& x) override {
    const cudaError_t q = cudaEventQuery(x.done);
    if (q == cudaErrorNotReady) return false;
    RS_CUDA_CHECK(q);
    return true;
  }

 private:
  int rank_, world_;
  std::vector<ncclComm_t> send_comm_, recv_comm_;
  std::vector<cudaStream_t> send_st_, recv_st_;
  std::vector<EventRing> rings_;
  EventPool events_;
};

}  // namespace

std::unique_ptr<Transport> make_nccl(const Topology& topo, int rank, int device, const void* ids) {
  return std::make_unique<NcclTransport>(topo, rank, device, ids);
}

void nccl_unique_id(void* out128) {
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
  ncclUniqueId id;
  nccl_check(NcclApi::get().get_unique_id(&id), "ncclGetUniqueId");
  std::memcpy(out128, &id, sizeof(id));
}

}  // namespace rserve::ep
