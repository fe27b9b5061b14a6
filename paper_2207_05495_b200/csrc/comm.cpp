#include "comm.hpp"

#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>
#include <stdexcept>
#include <string>

#include "../../include/synchro_b200.h"
#include "device/dev.hpp"

namespace synchro {

std::vector<u64> Comm::all_to_all_counts(dev::Context& c, const std::vector<u64>& send) {
  const int n = size();
  u64* d = static_cast<u64*>(c.alloc(2 * n * sizeof(u64)));
  c.memcpy_h2d(d, send.data(), n * sizeof(u64));
  const std::vector<u64> eight(n, sizeof(u64));
  const u64 saved = bytes_sent;
  all_to_allv(c, d, eight, d + n, eight);
  bytes_sent = saved;  // bookkeeping, not payload
  std::vector<u64> recv(n);
  c.memcpy_d2h(recv.data(), d + n, n * sizeof(u64));
  c.free(d);
  return recv;
}

std::vector<u64> Comm::all_gather_u64(dev::Context& c, u64 mine) {
  std::vector<u64> v(size(), 0);
  v[rank()] = mine;
  all_reduce(c, v.data(), v.size(), ReduceOp::Sum);
  return v;
}

namespace {

// ---------------------------------------------------------- host callbacks
class CallbackComm final : public Comm {
 public:
  explicit CallbackComm(const sw_comm& d) : d_(d) {
    if (!d.all_to_allv || !d.all_gather_v || !d.all_reduce_u64)
      throw std::invalid_argument("sw_comm: callback transport needs all three callbacks");
  }
  int rank() const override { return d_.rank; }
  int size() const override { return d_.nranks; }

  void all_to_allv(dev::Context& c, const void* send, const std::vector<u64>& send_bytes,
                   void* recv, const std::vector<u64>& recv_bytes) override {
    u64 st = 0, rt = 0;
    for (int r = 0; r < size(); ++r) {
      st += send_bytes[r];
      rt += recv_bytes[r];
      if (r != rank()) bytes_sent += send_bytes[r];
    }
    std::vector<unsigned char> hs(st ? st : 1), hr(rt ? rt : 1);
    c.memcpy_d2h(hs.data(), send, st);
    check(d_.all_to_allv(d_.user, hs.data(), send_bytes.data(), hr.data(), recv_bytes.data()),
          "all_to_allv");
    c.memcpy_h2d(recv, hr.data(), rt);
    c.sync();
  }

  void all_gather_v(dev::Context& c, const void* send, u64 bytes, void* recv,
                    const std::vector<u64>& recv_bytes) override {
    u64 rt = 0;
    for (u64 b : recv_bytes) rt += b;
    bytes_sent += bytes * (size() - 1);
    std::vector<unsigned char> hs(bytes ? bytes : 1), hr(rt ? rt : 1);
    c.memcpy_d2h(hs.data(), send, bytes);
    check(d_.all_gather_v(d_.user, hs.data(), bytes, hr.data(), recv_bytes.data()), "all_gather_v");
    c.memcpy_h2d(recv, hr.data(), rt);
    c.sync();
  }

  void all_reduce(dev::Context&, u64* values, size_t count, ReduceOp op) override {
    check(d_.all_reduce_u64(d_.user, values, count, static_cast<int32_t>(op)), "all_reduce");
  }

 private:
  static void check(int rc, const char* what) {
    if (rc != 0) throw DeviceError(std::string("sw_comm callback ") + what + " failed");
  }
  sw_comm d_;
};

// -------------------------------------------------------------------- NCCL
// libnccl.so.2 is loaded at run time: the library has no link-time NCCL
// dependency, and inside a process that already loaded torch's NCCL the same
// soname resolves to that copy.
struct NcclApi {
  decltype(&ncclGetUniqueId) get_unique_id = nullptr;
  decltype(&ncclCommInitRank) init_rank = nullptr;
  decltype(&ncclCommDestroy) destroy = nullptr;
  decltype(&ncclGroupStart) group_start = nullptr;
  decltype(&ncclGroupEnd) group_end = nullptr;
  decltype(&ncclSend) send = nullptr;
  decltype(&ncclRecv) recv = nullptr;
  decltype(&ncclAllReduce) all_reduce = nullptr;
  decltype(&ncclGetErrorString) error_string = nullptr;
};

const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    api.get_unique_id = reinterpret_cast<decltype(api.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
    api.init_rank = reinterpret_cast<decltype(api.init_rank)>(dlsym(h, "ncclCommInitRank"));
    api.destroy = reinterpret_cast<decltype(api.destroy)>(dlsym(h, "ncclCommDestroy"));
    api.group_start = reinterpret_cast<decltype(api.group_start)>(dlsym(h, "ncclGroupStart"));
    api.group_end = reinterpret_cast<decltype(api.group_end)>(dlsym(h, "ncclGroupEnd"));
    api.send = reinterpret_cast<decltype(api.send)>(dlsym(h, "ncclSend"));
    api.recv = reinterpret_cast<decltype(api.recv)>(dlsym(h, "ncclRecv"));
    api.all_reduce = reinterpret_cast<decltype(api.all_reduce)>(dlsym(h, "ncclAllReduce"));
    api.error_string =
        reinterpret_cast<decltype(api.error_string)>(dlsym(h, "ncclGetErrorString"));
  });
  if (!api.init_rank || !api.send || !api.recv || !api.all_reduce || !api.group_start)
    throw DeviceError("NCCL transport: libnccl.so.2 not loadable");
  return api;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    throw DeviceError(std::string("NCCL ") + what + ": " +
                      (nccl().error_string ? nccl().error_string(r) : "error"));
}

class NcclComm final : public Comm {
 public:
  explicit NcclComm(const sw_comm& d) : rank_(d.rank), size_(d.nranks) {
    ncclUniqueId id;
    static_assert(sizeof(id.internal) <= sizeof(d.nccl_id), "nccl id size");
    std::memcpy(id.internal, d.nccl_id, sizeof(id.internal));
    nccl_check(nccl().init_rank(&comm_, size_, id, rank_), "ncclCommInitRank");
  }
  ~NcclComm() override {
    if (comm_) nccl().destroy(comm_);
  }
  int rank() const override { return rank_; }
  int size() const override { return size_; }

  void all_to_allv(dev::Context& c, const void* send, const std::vector<u64>& send_bytes,
                   void* recv, const std::vector<u64>& recv_bytes) override {
    cudaStream_t s = static_cast<cudaStream_t>(c.stream());
    const auto* sp = static_cast<const unsigned char*>(send);
    auto* rp = static_cast<unsigned char*>(recv);
    nccl_check(nccl().group_start(), "group");
    for (int r = 0; r < size_; ++r) {
      if (send_bytes[r]) nccl_check(nccl().send(sp, send_bytes[r], ncclUint8, r, comm_, s), "send");
      if (recv_bytes[r]) nccl_check(nccl().recv(rp, recv_bytes[r], ncclUint8, r, comm_, s), "recv");
      if (r != rank_) bytes_sent += send_bytes[r];
      sp += send_bytes[r];
      rp += recv_bytes[r];
    }
    nccl_check(nccl().group_end(), "group");
    c.sync();
  }

  void all_gather_v(dev::Context& c, const void* send, u64 bytes, void* recv,
                    const std::vector<u64>& recv_bytes) override {
    cudaStream_t s = static_cast<cudaStream_t>(c.stream());
    auto* rp = static_cast<unsigned char*>(recv);
    nccl_check(nccl().group_start(), "group");
    for (int r = 0; r < size_; ++r) {
      if (bytes && r != rank_) {
        nccl_check(nccl().send(send, bytes, ncclUint8, r, comm_, s), "send");
        bytes_sent += bytes;
      }
      if (recv_bytes[r]) {
        if (r == rank_)
          c.memcpy_d2d(rp, send, bytes);
        else
          nccl_check(nccl().recv(rp, recv_bytes[r], ncclUint8, r, comm_, s), "recv");
      }
      rp += recv_bytes[r];
    }
    nccl_check(nccl().group_end(), "group");
    c.sync();
  }

  void all_reduce(dev::Context& c, u64* values, size_t count, ReduceOp op) override {
    u64* d = static_cast<u64*>(c.alloc(count * sizeof(u64)));
    c.memcpy_h2d(d, values, count * sizeof(u64));
    const ncclRedOp_t o = op == ReduceOp::Sum ? ncclSum : (op == ReduceOp::Min ? ncclMin : ncclMax);
    nccl_check(nccl().all_reduce(d, d, count, ncclUint64, o, comm_,
                                 static_cast<cudaStream_t>(c.stream())),
               "all_reduce");
    c.memcpy_d2h(values, d, count * sizeof(u64));
    c.free(d);
  }

 private:
  int rank_, size_;
  ncclComm_t comm_ = nullptr;
};

}  // namespace

std::unique_ptr<Comm> make_comm(const sw_comm& d) {
  if (d.nranks < 1 || d.rank < 0 || d.rank >= d.nranks)
    throw std::invalid_argument("sw_comm: rank must be in [0, nranks)");
  if (d.kind == SW_COMM_CALLBACK) return std::make_unique<CallbackComm>(d);
  if (d.kind == SW_COMM_NCCL) return std::make_unique<NcclComm>(d);
  throw std::invalid_argument("sw_comm: unknown transport kind");
}

void nccl_unique_id(uint8_t out[128]) {
  ncclUniqueId id;
  if (!nccl().get_unique_id) throw DeviceError("NCCL transport: libnccl.so.2 not loadable");
  nccl_check(nccl().get_unique_id(&id), "ncclGetUniqueId");
  std::memset(out, 0, 128);
  std::memcpy(out, id.internal, sizeof(id.internal));
}

}  // namespace synchro
