// rserve-b200 — EP transport over CUDA IPC peer memory (one process per GPU,
// or several processes on one GPU).
//
// Every directed link src -> dst owns a mailbox in dst's HBM: kSlots slots of
// slot_bytes, exported with cudaIpcGetMemHandle and mapped by src. Message k
// of the link goes to slot k % kSlots:
//   sender   wait(slot free: consumed[l] > k - kSlots, then free_ev[slot])
//            peer copy src -> mailbox slot (NVLink when the GPUs differ)
//            record data_ev[slot]; publish sent[l] = k + 1
//   receiver wait(sent[l] > k), stream-wait data_ev[slot], copy slot -> dst,
//            record free_ev[slot]; publish consumed[l] = k + 1
// data_ev / free_ev are interprocess events created by the receiver. The
// sequence counters live in a POSIX shared-memory segment of the group, so a
// wait is only ever issued after the matching record was (program order
// through the counter), which is what makes reusing the per-slot events safe.
#include <fcntl.h>
#include <sys/mman.h>
#include <unistd.h>

#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <chrono>
#include <cstring>
#include <mutex>
#include <thread>

#include "ep.cuh"

namespace rserve::ep {

namespace {

constexpr int kSlots = 4;

bool trace_on() {
  static const bool on = [] {
    const char* v = std::getenv("RS_EP_TRACE");
    return v != nullptr && v[0] == '1';
  }();
  return on;
}
#define EP_TRACE(...)                         \
  do {                                        \
    if (trace_on()) {                         \
      std::fprintf(stderr, "[ep r%d] ", rank_); \
      std::fprintf(stderr, __VA_ARGS__);      \
      std::fprintf(stderr, "\n");             \
    }                                         \
  } while (0)

struct alignas(64) Counter {
  std::atomic<std::uint64_t> v;
  char pad[64 - sizeof(std::atomic<std::uint64_t>)];
};
struct ShmLink {
  Counter sent, consumed;
  std::uint64_t bytes[kSlots];  // message sizes (checked by the receiver)
};

/// Per-incoming-link export: mailbox + events (receiver side).
struct LinkExport {
  cudaIpcMemHandle_t mem;
  cudaIpcEventHandle_t data_ev[kSlots];
  cudaIpcEventHandle_t free_ev[kSlots];
};

class IpcTransport final : public Transport {
 public:
  IpcTransport(const Topology& topo, int rank, int device, std::size_t slot_bytes, const std::string& shm)
      : topo_(topo), rank_(rank), dev_(device), slot_bytes_(slot_bytes), shm_name_(shm) {
    RS_CUDA_CHECK(cudaSetDevice(device));
    links_ = topo.links();
    const std::size_t L = links_.size();
    // Shared counters: every rank maps the group's segment; rank 0 zeroes it
    // before the handle exchange, i.e. before anyone touches a counter.
    const std::size_t bytes = L * sizeof(ShmLink);
    int fd = shm_open(shm_name_.c_str(), O_RDWR | O_CREAT, 0600);
    if (fd < 0) throw DeviceError(RS_ERR_CUDA, "ipc: shm_open(" + shm_name_ + ") failed");
    if (ftruncate(fd, static_cast<off_t>(bytes)) != 0) {
      close(fd);
      throw DeviceError(RS_ERR_CUDA, "ipc: ftruncate failed");
    }
    void* p = mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
    close(fd);
    if (p == MAP_FAILED) throw DeviceError(RS_ERR_CUDA, "ipc: mmap failed");
    shm_ = static_cast<ShmLink*>(p);
    shm_bytes_ = bytes;
    if (rank == 0) std::memset(p, 0, bytes);

    ends_.resize(L);
    for (std::size_t l = 0; l < L; ++l) {
      auto [src, dst] = links_[l];
      End& e = ends_[l];
      if (dst == rank) {  // receiver: owns the mailbox and the events
        RS_CUDA_CHECK(cudaMalloc(&e.mailbox, slot_bytes_ * kSlots));
        for (int k = 0; k < kSlots; ++k) {
          RS_CUDA_CHECK(cudaEventCreateWithFlags(&e.data_ev[k], cudaEventDisableTiming | cudaEventInterprocess));
          RS_CUDA_CHECK(cudaEventCreateWithFlags(&e.free_ev[k], cudaEventDisableTiming | cudaEventInterprocess));
        }
        RS_CUDA_CHECK(cudaStreamCreateWithFlags(&e.stream, cudaStreamNonBlocking));
        e.role = End::kRecv;
      } else if (src == rank) {
        RS_CUDA_CHECK(cudaStreamCreateWithFlags(&e.stream, cudaStreamNonBlocking));
        e.ring.resize(64);
        for (auto& ev : e.ring) RS_CUDA_CHECK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
        e.role = End::kSend;
      }
    }
  }

  ~IpcTransport() override {
    stop_.store(true);
    if (progress_thread_.joinable()) progress_thread_.join();
    cudaDeviceSynchronize();
    for (End& e : ends_) {
      if (e.role == End::kRecv) {
        cudaFree(e.mailbox);
        for (int k = 0; k < kSlots; ++k) {
          cudaEventDestroy(e.data_ev[k]);
          cudaEventDestroy(e.free_ev[k]);
        }
      } else if (e.role == End::kSend) {
        if (e.mailbox) cudaIpcCloseMemHandle(e.mailbox);
        for (auto ev : e.ring) cudaEventDestroy(ev);
        // imported IPC events are released with the process's context
      }
      if (e.stream) cudaStreamDestroy(e.stream);
    }
    if (shm_) munmap(shm_, shm_bytes_);
    if (rank_ == 0) shm_unlink(shm_name_.c_str());
  }

  /// This rank's receive-side handles, in links() order of its incoming links.
  std::vector<char> export_blob() const {
    std::vector<char> out;
    for (std::size_t l = 0; l < links_.size(); ++l) {
      if (links_[l].second != rank_) continue;
      const End& e = ends_[l];
      LinkExport x{};
      RS_CUDA_CHECK(cudaIpcGetMemHandle(&x.mem, e.mailbox));
      for (int k = 0; k < kSlots; ++k) {
        RS_CUDA_CHECK(cudaIpcGetEventHandle(&x.data_ev[k], e.data_ev[k]));
        RS_CUDA_CHECK(cudaIpcGetEventHandle(&x.free_ev[k], e.free_ev[k]));
      }
      const char* b = reinterpret_cast<const char*>(&x);
      out.insert(out.end(), b, b + sizeof(x));
    }
    return out;
  }

  /// Maps the mailboxes / events of the links this rank sends on.
  void connect(const std::vector<std::vector<char>>& blobs) {
    if (static_cast<int>(blobs.size()) != topo_.world())
      throw lmmsim::InputError("ipc connect: need one export blob per rank");
    std::vector<std::size_t> cursor(blobs.size(), 0);
    for (std::size_t l = 0; l < links_.size(); ++l) {
      const auto [src, dst] = links_[l];
      const std::vector<char>& blob = blobs[static_cast<std::size_t>(dst)];
      std::size_t& at = cursor[static_cast<std::size_t>(dst)];
      if (at + sizeof(LinkExport) > blob.size()) throw lmmsim::DataError("ipc connect: export blob too short");
      LinkExport x;
      std::memcpy(&x, blob.data() + at, sizeof(x));
      at += sizeof(x);
      if (src != rank_) continue;
      End& e = ends_[l];
      RS_CUDA_CHECK(cudaIpcOpenMemHandle(&e.mailbox, x.mem, cudaIpcMemLazyEnablePeerAccess));
      for (int k = 0; k < kSlots; ++k) {
        RS_CUDA_CHECK(cudaIpcOpenEventHandle(&e.data_ev[k], x.data_ev[k]));
        RS_CUDA_CHECK(cudaIpcOpenEventHandle(&e.free_ev[k], x.free_ev[k]));
      }
    }
    connected_ = true;
    EP_TRACE("connected (%zu links)", links_.size());
    // Receives posted by this rank are drained even while its main thread
    // is blocked in send() on a full ring: that is what keeps a
    // P0 <-> worker pair from waiting on each other.
    progress_thread_ = std::thread([this] {
      try {
        RS_CUDA_CHECK(cudaSetDevice(dev_));
        while (!stop_.load()) {
          {
            std::lock_guard<std::mutex> g(mu_);
            for (std::size_t l = 0; l < ends_.size(); ++l)
              if (ends_[l].role == End::kRecv && !ends_[l].pending.empty()) progress(static_cast<int>(l));
          }
          std::this_thread::sleep_for(std::chrono::microseconds(20));
        }
      } catch (...) {
        std::lock_guard<std::mutex> g(mu_);
        thread_error_ = std::current_exception();
      }
    });
  }

  int rank() const override { return rank_; }
  int world() const override { return topo_.world(); }

  cudaEvent_t send(int peer, const void* src, std::size_t bytes, cudaEvent_t wait) override {
    const int l = link(rank_, peer);
    End& e = ends_[static_cast<std::size_t>(l)];
    if (bytes > slot_bytes_)
      throw DeviceError(RS_ERR_CUDA, "ipc: message of " + std::to_string(bytes) + " bytes > slot of " +
                                         std::to_string(slot_bytes_));
    const std::uint64_t k = e.seq++;  // the send side of a link is one thread's
    EP_TRACE("send l%d -> %d msg %llu bytes %zu", l, peer, static_cast<unsigned long long>(k), bytes);
    const int slot = static_cast<int>(k % kSlots);
    ShmLink& s = shm_[l];
    // Slot reuse: the receiver must have consumed message k - kSlots (spin
    // without the lock so this rank's own receives keep draining).
    if (k >= kSlots)
      while (s.consumed.v.load(std::memory_order_acquire) <= k - kSlots) std::this_thread::yield();
    std::lock_guard<std::mutex> g(mu_);
    if (k >= kSlots) RS_CUDA_CHECK(cudaStreamWaitEvent(e.stream, e.free_ev[slot], 0));
    if (wait != nullptr) RS_CUDA_CHECK(cudaStreamWaitEvent(e.stream, wait, 0));
    RS_CUDA_CHECK(cudaMemcpyAsync(static_cast<char*>(e.mailbox) + static_cast<std::size_t>(slot) * slot_bytes_,
                                  src, bytes, cudaMemcpyDefault, e.stream));
    RS_CUDA_CHECK(cudaEventRecord(e.data_ev[slot], e.stream));
    cudaEvent_t done = e.ring[e.ring_pos];
    e.ring_pos = (e.ring_pos + 1) % e.ring.size();
    RS_CUDA_CHECK(cudaEventRecord(done, e.stream));
    s.bytes[slot] = bytes;
    s.sent.v.store(k + 1, std::memory_order_release);
    return done;
  }

  std::shared_ptr<Xfer> post_recv(int peer, void* dst, std::size_t bytes, cudaEvent_t wait) override {
    const int l = link(peer, rank_);
    End& e = ends_[static_cast<std::size_t>(l)];
    Xfer* raw = new Xfer();
    RS_CUDA_CHECK(cudaEventCreate(&raw->done));  // timing-enabled: P0 stamps completions
    std::shared_ptr<Xfer> x(raw, [](Xfer* p) {
      cudaEventDestroy(p->done);
      delete p;
    });
    x->peer = peer;
    x->dst = dst;
    x->bytes = bytes;
    x->wait = wait;
    std::lock_guard<std::mutex> g(mu_);
    e.pending.push_back(x);
    progress(l);
    return x;
  }

  void wait_posted(Xfer& x) override {
    const int l = link(x.peer, rank_);
    for (;;) {
      {
        std::lock_guard<std::mutex> g(mu_);
        if (!x.posted) progress(l);
        if (x.posted) return;
      }
      std::this_thread::yield();
    }
  }

  bool test(Xfer& x) override {
    {
      std::lock_guard<std::mutex> g(mu_);
      if (!x.posted) progress(link(x.peer, rank_));
      if (!x.posted) return false;
    }
    const cudaError_t q = cudaEventQuery(x.done);
    if (q == cudaErrorNotReady) return false;
    RS_CUDA_CHECK(q);
    return true;
  }

 private:
  struct End {
    enum Role { kNone, kSend, kRecv } role = kNone;
    void* mailbox = nullptr;
    cudaEvent_t data_ev[kSlots] = {};
    cudaEvent_t free_ev[kSlots] = {};
    cudaStream_t stream = nullptr;
    std::uint64_t seq = 0;  // next message index (send) / next to consume (recv)
    std::vector<cudaEvent_t> ring;
    std::size_t ring_pos = 0;
    std::deque<std::shared_ptr<Xfer>> pending;
  };

  int link(int src, int dst) const {
    for (std::size_t l = 0; l < links_.size(); ++l)
      if (links_[l].first == src && links_[l].second == dst) return static_cast<int>(l);
    throw DeviceError(RS_ERR_CUDA, "no EP link " + std::to_string(src) + "->" + std::to_string(dst));
  }

  // Consumes arrived messages of link l into the posted receives, in order.
  void progress(int l) {  // caller holds mu_
    if (thread_error_) std::rethrow_exception(thread_error_);
    End& e = ends_[static_cast<std::size_t>(l)];
    ShmLink& s = shm_[l];
    while (!e.pending.empty()) {
      const std::uint64_t k = e.seq;
      if (s.sent.v.load(std::memory_order_acquire) <= k) return;
      std::shared_ptr<Xfer> x = e.pending.front();
      const int slot = static_cast<int>(k % kSlots);
      EP_TRACE("recv l%d <- %d msg %llu bytes %zu", l, x->peer, static_cast<unsigned long long>(k), x->bytes);
      if (s.bytes[slot] != x->bytes)
        throw DeviceError(RS_ERR_CUDA, "ipc: message of " + std::to_string(s.bytes[slot]) +
                                           " bytes for a receive of " + std::to_string(x->bytes));
      RS_CUDA_CHECK(cudaStreamWaitEvent(e.stream, e.data_ev[slot], 0));
      if (x->wait != nullptr) RS_CUDA_CHECK(cudaStreamWaitEvent(e.stream, x->wait, 0));
      RS_CUDA_CHECK(cudaMemcpyAsync(x->dst, static_cast<char*>(e.mailbox) + static_cast<std::size_t>(slot) * slot_bytes_,
                                    x->bytes, cudaMemcpyDeviceToDevice, e.stream));
      RS_CUDA_CHECK(cudaEventRecord(x->done, e.stream));
      RS_CUDA_CHECK(cudaEventRecord(e.free_ev[slot], e.stream));
      x->posted = true;
      e.seq = k + 1;
      s.consumed.v.store(k + 1, std::memory_order_release);
      e.pending.pop_front();
    }
  }

  Topology topo_;
  int rank_, dev_;
  std::size_t slot_bytes_;
  std::string shm_name_;
  std::vector<std::pair<int, int>> links_;
  std::vector<End> ends_;
  ShmLink* shm_ = nullptr;
  std::size_t shm_bytes_ = 0;
  bool connected_ = false;
  std::mutex mu_;  // receive state (pending, seq) and CUDA calls on link streams
  std::atomic<bool> stop_{false};
  std::thread progress_thread_;
  std::exception_ptr thread_error_;
};

}  // namespace

std::unique_ptr<Transport> make_ipc(const Topology& topo, int rank, int device, std::size_t slot_bytes,
                                    const std::string& shm_name) {
  return std::make_unique<IpcTransport>(topo, rank, device, slot_bytes, shm_name);
}

std::vector<char> ipc_export(Transport& t) {
  auto* x = dynamic_cast<IpcTransport*>(&t);
  if (x == nullptr) throw lmmsim::ConfigError("ipc export: not an IPC transport");
  return x->export_blob();
}

void ipc_connect(Transport& t, const std::vector<std::vector<char>>& blobs) {
  auto* x = dynamic_cast<IpcTransport*>(&t);
  if (x == nullptr) throw lmmsim::ConfigError("ipc connect: not an IPC transport");
  x->connect(blobs);
}

}  // namespace rserve::ep
