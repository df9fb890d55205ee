// comm.hpp -- cross-rank reads between the ranks of one node (SURVEY.md 8(e),
// NEXT-2, StarPU-MPI "a task runs on the node that owns
// the data it writes; data it only reads is transferred there").
//
// Every rank submits the same task stream.  A task that writes data owned by
// rank b and reads data owned by rank a != b runs on b; at that task both
// ranks meet (a "rendezvous"), in submission order, which both see alike:
//
//   owner a:  flush; record READY[a->b] on its stream; signal b;
//             wait until b has enqueued its copy; order its stream after
//             DONE[b<-a] (so a's later writers of the data cannot overwrite
//             it before b's copy has read it -- WAR across ranks)
//   reader b: flush; wait for a's signal; order its stream after READY[a->b];
//             copy the range from a's device memory (CUDA IPC mapping: a peer
//             copy over NVLink between GPUs) into b's own replica of it;
//             record DONE[b<-a]; signal a; the task then reads the replica.
//
// Device protocol (default): no host waits at all.  Every rank owns a flag
// page in device memory (ready[16], done[16]: per-peer sequence numbers),
// mapped into every peer by CUDA IPC at bt_comm_init.  The k-th rendezvous of
// the ordered pair (a, b) -- both sides count it alike, in submission order --
// is, on the GPUs' streams:
//   owner a:  WRITE b.ready[a] = k  (a stream memory write into b's page, after
//             a's earlier work: a's writers of the data)
//             WAIT  a.done[b] >= k  (a's later work, e.g. the next writer of the
//             data, waits until b has copied it: WAR across ranks)
//   reader b: WAIT  b.ready[a] >= k (RAW across ranks); copy the range from a's
//             memory (IPC mapping; a peer copy over NVLink between GPUs);
//             WRITE a.done[b] = k
// Stream memory operations (cuStreamWaitValue32 / cuStreamWriteValue32, which
// fence before the write) when the driver has them, else one-thread flag
// kernels.  Host protocol (BT_COMM_HOST=1, the first implementation):
// sequence counters in a POSIX shared-memory segment and interprocess events
// (the owner's host waits until the reader has enqueued its copy).
// Either way only streams wait, never a kernel for another rank's kernel, so
// two ranks may also share one GPU (the tests do).  Internal to libbtask.so.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <map>
#include <string>
#include <utility>

namespace bt {

struct CommShm;

class Comm {
 public:
  // Collective over nranks processes (same name).  0 or a negative errno
  // (err gets a message).
  static int create(const char *name, int rank, int nranks, int device, Comm **out, std::string *err);
  ~Comm();

  // Owner side.  root: device address of the registered root (key: its
  // registration ordinal, equal on all ranks) and its size; the data to be
  // read is complete on `stream` (everything earlier on it).
  int send(cudaStream_t stream, int peer, uint64_t key, const void *root, uint64_t root_bytes, std::string *err);
  // Reader side: copy bytes [off, off + bytes) of the peer's root `key` into
  // dst, ordered on `stream`.
  int recv(cudaStream_t stream, int peer, uint64_t key, uint64_t off, void *dst, uint64_t bytes, std::string *err);

  bool device_protocol() const { return dev_; }
  int rank() const { return rank_; }
  int nranks() const { return nranks_; }

 private:
  Comm() = default;
  int export_root(uint64_t key, const void *root, uint64_t bytes, std::string *err);
  int open_root(int peer, uint64_t key, char **base, std::string *err);
  int wait_seq(const void *counter, uint64_t want, const char *what, std::string *err);
  int peer_event(int peer, bool ready, cudaEvent_t *ev, std::string *err);

  CommShm *seg_ = nullptr;
  size_t seg_bytes_ = 0;
  std::string name_;
  bool creator_ = false;
  int rank_ = 0, nranks_ = 1, device_ = 0;
  cudaEvent_t ev_ready_[16] = {};     // recorded here: "data for peer p is ready"
  cudaEvent_t ev_done_[16] = {};      // recorded here: "copy from peer p is done"
  cudaEvent_t peer_ready_[16] = {};   // opened: peer p's READY[p->me]
  cudaEvent_t peer_done_[16] = {};    // opened: peer p's DONE[p<-me]
  uint64_t sent_[16] = {}, recvd_[16] = {};
  bool dev_ = true;                   // device protocol (flag pages); false: host protocol
  uint32_t *flags_ = nullptr;         // this rank's flag page: ready[16] | done[16]
  uint32_t *peer_flags_[16] = {};     // the peers' pages, mapped here
  bool peer_local_[16] = {};          // the peer is a rank of this process (no IPC mapping)
  int flag_wait(cudaStream_t stream, const uint32_t *addr, uint32_t value, std::string *err);
  int flag_write(cudaStream_t stream, uint32_t *addr, uint32_t value, std::string *err);
  std::map<uint64_t, int> exported_;                   // key -> export slot
  std::map<std::pair<int, uint64_t>, char *> opened_;  // (peer, key) -> root address here
  std::map<std::pair<int, std::string>, char *> alloc_opened_;   // (peer, IPC handle bytes) -> mapping
};

}  // namespace bt
