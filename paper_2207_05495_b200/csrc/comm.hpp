// Collectives between the ranks of one partitioned solve (one process per
// GPU).  The reference has no multi-process path; this is SURVEY §8(e)'s hash
// ownership: each rank owns the subsets whose hash maps to it, one
// all-to-all per level carries newly generated subsets to their owners,
// all-gathers replicate what containment needs (containment is not
// hash-local), all-reduces keep the cost model's statistics global so that
// every rank takes the same step sequence as the single-GPU solve.
//
// Two transports behind one interface:
//   * NcclComm     — NCCL on device buffers (NVLink / NVSwitch), loaded at
//                    run time (libnccl.so.2), communicator from a unique id
//                    the caller distributes;
//   * CallbackComm — caller-supplied host-buffer collectives (torch.distributed,
//                    MPI, gloo ...): device data is staged through host memory.
// Every call is collective and synchronous with respect to the engine stream.
#pragma once

#include <cstdint>
#include <memory>
#include <vector>

#include "common.hpp"

struct sw_comm;  // include/synchro_b200.h

namespace synchro {

namespace dev {
class Context;
}

enum class ReduceOp { Sum = 0, Min = 1, Max = 2 };

class Comm {
 public:
  virtual ~Comm() = default;
  virtual int rank() const = 0;
  virtual int size() const = 0;
  // send: device buffer holding, rank by rank, send_bytes[r] bytes for rank r;
  // recv: device buffer receiving recv_bytes[r] bytes from rank r, rank by rank.
  virtual void all_to_allv(dev::Context& c, const void* send, const std::vector<u64>& send_bytes,
                           void* recv, const std::vector<u64>& recv_bytes) = 0;
  // Every rank contributes `bytes` (device); recv (device) holds all
  // contributions in rank order, recv_bytes[r] from rank r.
  virtual void all_gather_v(dev::Context& c, const void* send, u64 bytes, void* recv,
                            const std::vector<u64>& recv_bytes) = 0;
  // In place on host values.
  virtual void all_reduce(dev::Context& c, u64* values, size_t count, ReduceOp op) = 0;
  // Bytes this rank sent to other ranks over the transport (all_to_allv and
  // all_gather_v payloads), for the NVLink accounting of the bench.
  u64 bytes_sent = 0;

  // Convenience: exchange one u64 per rank (counts).
  std::vector<u64> all_to_all_counts(dev::Context& c, const std::vector<u64>& send);
  std::vector<u64> all_gather_u64(dev::Context& c, u64 mine);
};

// Builds the transport an sw_comm descriptor asks for (SW_COMM_NCCL /
// SW_COMM_CALLBACK); throws on a malformed descriptor or a missing libnccl.
std::unique_ptr<Comm> make_comm(const sw_comm& desc);
// ncclGetUniqueId through the run-time loaded library (128 bytes).
void nccl_unique_id(uint8_t out[128]);

}  // namespace synchro
