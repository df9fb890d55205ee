// comm.cpp -- see comm.hpp.
#include "comm.hpp"

#include <errno.h>
#include <fcntl.h>
#include <sched.h>
#include <stdio.h>
#include <string.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <atomic>
#include <chrono>
#include <thread>

namespace bt {

cudaError_t launch_flag_wait(const uint32_t *addr, uint32_t value, uint64_t watchdog_ns, cudaStream_t stream);
cudaError_t launch_flag_write(uint32_t *addr, uint32_t value, cudaStream_t stream);

namespace {

constexpr int kMaxRanks = 16;
constexpr int kMaxExports = 1024;
constexpr uint32_t kMagic = 0x62746331u;   // "btc1"
constexpr double kTimeoutS = 60.0;

struct ShmExport {
  std::atomic<uint32_t> valid;   // 1 once the fields below are written
  uint32_t pad;
  uint64_t key;                  // registration ordinal of the root
  uint64_t offset;               // bytes from the allocation base to the root
  uint64_t bytes;
  uint64_t ptr;                  // the root's device address in the owner (same-process peers use it as is)
  cudaIpcMemHandle_t mem;        // handle of the allocation holding the root
};

struct ShmRank {
  std::atomic<uint32_t> attached;
  std::atomic<uint32_t> nexports;
  cudaIpcEventHandle_t ev_ready[kMaxRanks];
  cudaIpcEventHandle_t ev_done[kMaxRanks];
  cudaIpcMemHandle_t flag_mem;   // the rank's flag page (device protocol)
  uint64_t flag_ptr;             // ... its device address (same-process peers use it as is)
  int32_t pid;                   // ranks in one process (threads, one runtime each) share addresses
  ShmExport exports[kMaxExports];
};

double seconds() {
  using namespace std::chrono;
  return duration<double>(steady_clock::now().time_since_epoch()).count();
}

}  // namespace

struct CommShm {
  std::atomic<uint32_t> magic;
  uint32_t nranks;
  std::atomic<uint64_t> ready[kMaxRanks][kMaxRanks];   // [owner][reader]: rendezvous published by the owner
  std::atomic<uint64_t> done[kMaxRanks][kMaxRanks];    // [reader][owner]: copies enqueued by the reader
  ShmRank ranks[kMaxRanks];
};

namespace {

int set_err(std::string *err, int code, const char *fmt, const char *detail = "") {
  char buf[256];
  snprintf(buf, sizeof buf, fmt, detail);
  if (err) *err = buf;
  return code;
}

// cuMemGetAddressRange through the runtime's driver entry point (libbtask
// links the static CUDA runtime, not libcuda): the base of the allocation
// holding p, which is what an IPC handle refers to.
int alloc_base(const void *p, uint64_t *base) {
  typedef int (*Fn)(unsigned long long *, size_t *, unsigned long long);
  static Fn fn = nullptr;
  if (!fn) {
    void *sym = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &sym, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !sym)
      return -ENOSYS;
    fn = reinterpret_cast<Fn>(sym);
  }
  unsigned long long b = 0;
  size_t sz = 0;
  if (fn(&b, &sz, reinterpret_cast<unsigned long long>(p)) != 0) return -EINVAL;
  *base = b;
  return 0;
}

// Stream memory operations through the runtime's driver entry points.
// CUresult cuStreamWaitValue32(CUstream, CUdeviceptr, cuuint32_t, unsigned) (GEQ = 0);
// CUresult cuStreamWriteValue32(CUstream, CUdeviceptr, cuuint32_t, unsigned) (0 = fence before the write).
typedef int (*StreamValueFn)(cudaStream_t, unsigned long long, uint32_t, unsigned);
StreamValueFn driver_fn(const char *name) {
  if (getenv("BT_COMM_FLAG_KERNELS")) return nullptr;   // tests: the kernel fallback
  void *sym = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &sym, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  return reinterpret_cast<StreamValueFn>(sym);
}

}  // namespace

int Comm::flag_wait(cudaStream_t stream, const uint32_t *addr, uint32_t value, std::string *err) {
  static const StreamValueFn fn = driver_fn("cuStreamWaitValue32");
  if (fn && fn(stream, reinterpret_cast<unsigned long long>(addr), value, 0u) == 0) return 0;
  if (launch_flag_wait(addr, value, (uint64_t)(kTimeoutS * 1e9), stream) != cudaSuccess) {
    cudaGetLastError();
    return set_err(err, -EIO, "cross-rank flag wait failed");
  }
  return 0;
}

int Comm::flag_write(cudaStream_t stream, uint32_t *addr, uint32_t value, std::string *err) {
  static const StreamValueFn fn = driver_fn("cuStreamWriteValue32");
  if (fn && fn(stream, reinterpret_cast<unsigned long long>(addr), value, 0u) == 0) return 0;
  if (launch_flag_write(addr, value, stream) != cudaSuccess) {
    cudaGetLastError();
    return set_err(err, -EIO, "cross-rank flag write failed");
  }
  return 0;
}

int Comm::create(const char *name, int rank, int nranks, int device, Comm **out, std::string *err) {
  *out = nullptr;
  if (!name || name[0] != '/' || strlen(name) > 200) return set_err(err, -EINVAL, "bad shared-memory name");
  if (nranks < 2 || nranks > kMaxRanks || rank < 0 || rank >= nranks)
    return set_err(err, -EINVAL, "cross-rank reads need 2..16 ranks");
  Comm *c = new Comm();
  c->name_ = name;
  c->rank_ = rank;
  c->nranks_ = nranks;
  c->device_ = device;
  c->creator_ = rank == 0;
  c->seg_bytes_ = sizeof(CommShm);
  const double t0 = seconds();
  int fd = -1;
  if (c->creator_) {
    shm_unlink(name);   // a stale segment of an earlier job of the same name
    fd = shm_open(name, O_CREAT | O_EXCL | O_RDWR, 0600);
    if (fd < 0 || ftruncate(fd, (off_t)c->seg_bytes_) != 0) {
      if (fd >= 0) close(fd);
      delete c;
      return set_err(err, -EIO, "cannot create shared memory %s", name);
    }
  } else {
    for (;;) {   // wait for rank 0 to create and size it
      fd = shm_open(name, O_RDWR, 0600);
      if (fd >= 0) {
        struct stat st;
        if (fstat(fd, &st) == 0 && (size_t)st.st_size == c->seg_bytes_) break;
        close(fd);
        fd = -1;
      }
      if (seconds() - t0 > kTimeoutS) {
        delete c;
        return set_err(err, -ETIMEDOUT, "rank 0 did not create %s", name);
      }
      std::this_thread::sleep_for(std::chrono::milliseconds(1));
    }
  }
  void *m = mmap(nullptr, c->seg_bytes_, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
  close(fd);
  if (m == MAP_FAILED) {
    delete c;
    return set_err(err, -EIO, "cannot map shared memory %s", name);
  }
  c->seg_ = static_cast<CommShm *>(m);
  if (c->creator_) {
    c->seg_->nranks = (uint32_t)nranks;   // the rest is zero (a fresh segment)
    c->seg_->magic.store(kMagic, std::memory_order_release);
  } else {
    while (c->seg_->magic.load(std::memory_order_acquire) != kMagic) {
      if (seconds() - t0 > kTimeoutS) {
        delete c;
        return set_err(err, -ETIMEDOUT, "shared memory %s never initialised", name);
      }
      std::this_thread::sleep_for(std::chrono::milliseconds(1));
    }
    if ((int)c->seg_->nranks != nranks) {
      delete c;
      return set_err(err, -EINVAL, "ranks disagree on nranks (%s)", name);
    }
  }
  // this rank's interprocess events and flag page, published for the peers
  cudaSetDevice(device);
  ShmRank &me = c->seg_->ranks[rank];
  c->dev_ = getenv("BT_COMM_HOST") == nullptr;
  if (c->dev_) {
    if (cudaMalloc((void **)&c->flags_, 256) != cudaSuccess || cudaMemset(c->flags_, 0, 256) != cudaSuccess ||
        cudaDeviceSynchronize() != cudaSuccess || cudaIpcGetMemHandle(&me.flag_mem, c->flags_) != cudaSuccess) {
      cudaGetLastError();
      delete c;
      return set_err(err, -EIO, "cannot create the cross-rank flag page");
    }
  }
  for (int p = 0; p < nranks; ++p) {
    if (p == rank) continue;
    if (cudaEventCreateWithFlags(&c->ev_ready_[p], cudaEventDisableTiming | cudaEventInterprocess) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->ev_done_[p], cudaEventDisableTiming | cudaEventInterprocess) != cudaSuccess ||
        cudaIpcGetEventHandle(&me.ev_ready[p], c->ev_ready_[p]) != cudaSuccess ||
        cudaIpcGetEventHandle(&me.ev_done[p], c->ev_done_[p]) != cudaSuccess) {
      cudaGetLastError();
      delete c;
      return set_err(err, -EIO, "cannot create interprocess events");
    }
  }
  me.flag_ptr = reinterpret_cast<uint64_t>(c->flags_);
  me.pid = (int32_t)getpid();
  me.attached.store(1, std::memory_order_release);
  for (int p = 0; p < nranks; ++p)   // collective: every rank has published its events
    while (c->seg_->ranks[p].attached.load(std::memory_order_acquire) != 1) {
      if (seconds() - t0 > kTimeoutS) {
        delete c;
        return set_err(err, -ETIMEDOUT, "not every rank joined %s", name);
      }
      std::this_thread::sleep_for(std::chrono::microseconds(100));
    }
  if (c->dev_)
    for (int p = 0; p < nranks; ++p) {
      if (p == rank) continue;
      void *fp = nullptr;
      if (c->seg_->ranks[p].pid == (int32_t)getpid()) {   // a rank in this process: same address space
        c->peer_flags_[p] = reinterpret_cast<uint32_t *>(c->seg_->ranks[p].flag_ptr);
        c->peer_local_[p] = true;
        continue;
      }
      if (cudaIpcOpenMemHandle(&fp, c->seg_->ranks[p].flag_mem, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
        cudaGetLastError();
        delete c;
        return set_err(err, -EIO, "cannot map a peer's flag page");
      }
      c->peer_flags_[p] = static_cast<uint32_t *>(fp);
    }
  *out = c;
  return 0;
}

Comm::~Comm() {
  for (auto &kv : alloc_opened_) cudaIpcCloseMemHandle(kv.second);
  for (int p = 0; p < 16; ++p)
    if (peer_flags_[p] && !peer_local_[p]) cudaIpcCloseMemHandle(peer_flags_[p]);
  if (flags_) cudaFree(flags_);
  for (int p = 0; p < 16; ++p) {
    if (ev_ready_[p]) cudaEventDestroy(ev_ready_[p]);
    if (ev_done_[p]) cudaEventDestroy(ev_done_[p]);
    if (peer_ready_[p]) cudaEventDestroy(peer_ready_[p]);
    if (peer_done_[p]) cudaEventDestroy(peer_done_[p]);
  }
  if (seg_) munmap(seg_, seg_bytes_);
  if (creator_) shm_unlink(name_.c_str());
}

int Comm::wait_seq(const void *counter, uint64_t want, const char *what, std::string *err) {
  const auto *c = static_cast<const std::atomic<uint64_t> *>(counter);
  const double t0 = seconds();
  for (unsigned spin = 0; c->load(std::memory_order_acquire) < want; ++spin) {
    if (spin > 64) std::this_thread::yield();
    if ((spin & 1023) == 1023 && seconds() - t0 > kTimeoutS)
      return set_err(err, -ETIMEDOUT, "cross-rank rendezvous timed out (%s)", what);
  }
  return 0;
}

int Comm::peer_event(int peer, bool ready, cudaEvent_t *ev, std::string *err) {
  cudaEvent_t &e = ready ? peer_ready_[peer] : peer_done_[peer];
  if (!e) {
    const ShmRank &pr = seg_->ranks[peer];
    cudaIpcEventHandle_t h = ready ? pr.ev_ready[rank_] : pr.ev_done[rank_];
    if (cudaIpcOpenEventHandle(&e, h) != cudaSuccess) {
      cudaGetLastError();
      e = nullptr;
      return set_err(err, -EIO, "cannot open a peer's interprocess event");
    }
  }
  *ev = e;
  return 0;
}

int Comm::export_root(uint64_t key, const void *root, uint64_t bytes, std::string *err) {
  if (exported_.count(key)) return 0;
  ShmRank &me = seg_->ranks[rank_];
  const uint32_t i = me.nexports.load(std::memory_order_relaxed);
  if (i >= (uint32_t)kMaxExports) return set_err(err, -ENOSPC, "too many exported buffers");
  uint64_t base = 0;
  if (int r = alloc_base(root, &base)) return set_err(err, r, "cannot find the allocation of a buffer");
  ShmExport &x = me.exports[i];
  if (cudaIpcGetMemHandle(&x.mem, reinterpret_cast<void *>(base)) != cudaSuccess) {
    cudaGetLastError();
    return set_err(err, -EINVAL, "buffer memory cannot be shared between processes (%s)",
                   "register it after bt_comm_init, or pass cudaMalloc'ed device memory");
  }
  x.key = key;
  x.ptr = reinterpret_cast<uint64_t>(root);
  x.offset = reinterpret_cast<uint64_t>(root) - base;
  x.bytes = bytes;
  x.valid.store(1, std::memory_order_release);
  me.nexports.store(i + 1, std::memory_order_release);
  exported_[key] = (int)i;
  return 0;
}

int Comm::open_root(int peer, uint64_t key, char **out, std::string *err) {
  auto it = opened_.find({peer, key});
  if (it != opened_.end()) {
    *out = it->second;
    return 0;
  }
  // device protocol: the owner exports a root the first time it sends it,
  // possibly after we got here: wait for it (once per root and peer)
  const double t0 = seconds();
  for (;;) {
    const ShmRank &pr = seg_->ranks[peer];
    const uint32_t n = pr.nexports.load(std::memory_order_acquire);
    bool found = false;
    for (uint32_t i = 0; i < n && !found; ++i)
      found = pr.exports[i].valid.load(std::memory_order_acquire) == 1 && pr.exports[i].key == key;
    if (found || !dev_) break;
    if (seconds() - t0 > kTimeoutS) return set_err(err, -ETIMEDOUT, "the owner rank never exported the buffer");
    std::this_thread::yield();
  }
  // the owner exported the root before it published the rendezvous we waited for
  const ShmRank &pr = seg_->ranks[peer];
  const uint32_t n = pr.nexports.load(std::memory_order_acquire);
  for (uint32_t i = 0; i < n; ++i) {
    const ShmExport &x = pr.exports[i];
    if (x.valid.load(std::memory_order_acquire) != 1 || x.key != key) continue;
    if (pr.pid == (int32_t)getpid()) {   // a rank in this process: its address as is
      *out = opened_[{peer, key}] = reinterpret_cast<char *>(x.ptr);
      return 0;
    }
    std::string hk(reinterpret_cast<const char *>(&x.mem), sizeof x.mem);
    char *base = nullptr;
    auto a = alloc_opened_.find({peer, hk});
    if (a != alloc_opened_.end()) {
      base = a->second;
    } else {
      void *p = nullptr;
      if (cudaIpcOpenMemHandle(&p, x.mem, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
        cudaGetLastError();
        return set_err(err, -EIO, "cannot map a peer's buffer");
      }
      base = static_cast<char *>(p);
      alloc_opened_[{peer, hk}] = base;
    }
    *out = opened_[{peer, key}] = base + x.offset;
    return 0;
  }
  return set_err(err, -ENOENT, "the owner rank never exported the buffer");
}

int Comm::send(cudaStream_t stream, int peer, uint64_t key, const void *root, uint64_t root_bytes, std::string *err) {
  if (int r = export_root(key, root, root_bytes, err)) return r;
  if (dev_) {
    const uint32_t k = (uint32_t)++sent_[peer];
    if (int r = flag_write(stream, peer_flags_[peer] + rank_, k, err)) return r;        // peer's ready[me] = k
#ifndef BT_COMM_MUTANT_NO_WAR   // test-sensitivity check only: drop the WAR ordering
    if (int r = flag_wait(stream, flags_ + 16 + peer, k, err)) return r;                // my done[peer] >= k
#endif
    return 0;
  }
  if (cudaEventRecord(ev_ready_[peer], stream) != cudaSuccess) return set_err(err, -EIO, "event record failed");
  seg_->ready[rank_][peer].fetch_add(1, std::memory_order_acq_rel);
  // WAR across ranks: later work here (a writer of the data) waits for the
  // peer's copy; the peer enqueues it before it signals
  const uint64_t want = ++sent_[peer];
#ifdef BT_COMM_MUTANT_NO_WAR   // test-sensitivity check only: drop the WAR ordering
  (void)want;
  return 0;
#endif
  if (int r = wait_seq(&seg_->done[peer][rank_], want, "owner waits for the reader's copy", err)) return r;
  cudaEvent_t ev;
  if (int r = peer_event(peer, false, &ev, err)) return r;
  if (cudaStreamWaitEvent(stream, ev, 0) != cudaSuccess) return set_err(err, -EIO, "stream wait failed");
  return 0;
}

int Comm::recv(cudaStream_t stream, int peer, uint64_t key, uint64_t off, void *dst, uint64_t bytes,
               std::string *err) {
  if (dev_) {
    const uint32_t k = (uint32_t)++recvd_[peer];
#ifndef BT_COMM_MUTANT_NO_RAW   // test-sensitivity check only: drop the RAW ordering
    if (int r = flag_wait(stream, flags_ + peer, k, err)) return r;                     // my ready[peer] >= k
#endif
    char *src = nullptr;
    if (int r = open_root(peer, key, &src, err)) return r;
    if (bytes && cudaMemcpyAsync(dst, src + off, bytes, cudaMemcpyDeviceToDevice, stream) != cudaSuccess) {
      cudaGetLastError();
      return set_err(err, -EIO, "peer copy failed");
    }
    return flag_write(stream, peer_flags_[peer] + 16 + rank_, k, err);                  // peer's done[me] = k
  }
  const uint64_t want = ++recvd_[peer];
  if (int r = wait_seq(&seg_->ready[peer][rank_], want, "reader waits for the owner", err)) return r;
  cudaEvent_t ev;
  if (int r = peer_event(peer, true, &ev, err)) return r;
#ifndef BT_COMM_MUTANT_NO_RAW   // test-sensitivity check only: drop the RAW ordering
  if (cudaStreamWaitEvent(stream, ev, 0) != cudaSuccess) return set_err(err, -EIO, "stream wait failed");
#endif
  char *src = nullptr;
  if (int r = open_root(peer, key, &src, err)) return r;
  if (bytes && cudaMemcpyAsync(dst, src + off, bytes, cudaMemcpyDeviceToDevice, stream) != cudaSuccess) {
    cudaGetLastError();
    return set_err(err, -EIO, "peer copy failed");
  }
  if (cudaEventRecord(ev_done_[peer], stream) != cudaSuccess) return set_err(err, -EIO, "event record failed");
  seg_->done[rank_][peer].fetch_add(1, std::memory_order_acq_rel);
  return 0;
}

}  // namespace bt
