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
// Host signalling goes through a POSIX shared-memory segment (sequence
// counters per ordered rank pair, exported IPC handles); device ordering
// through interprocess CUDA events.  No kernel ever waits for another rank:
// only streams wait for events, so two ranks may also share one GPU (the
// tests do).  Internal to libbtask.so.
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
  std::map<uint64_t, int> exported_;                   // key -> export slot
  std::map<std::pair<int, uint64_t>, char *> opened_;  // (peer, key) -> root address here
  std::map<std::pair<int, std::string>, char *> alloc_opened_;   // (peer, IPC handle bytes) -> mapping
};

}  // namespace bt
