// nccl_fake.cu — TEST INFRASTRUCTURE ONLY: an in-process stand-in for the
// NCCL calls libpf makes, so the multi-rank data path (pack -> send/recv ->
// unpack, the window allreduce, the checkpoint agreement) can run with every
// rank as a host thread of ONE process on ONE GPU.  Linked instead of
// libnccl into a test copy of libpf (tests/test_gpu_fakenccl.py); the product
// library never contains it.
//
// No kernel waits on another: a "send" is an event recorded on the sender's
// stream after its pack kernel; the receiving thread blocks on the HOST until
// the peer has posted it, then orders a device-to-device copy after that event
// on its own stream; the sender's stream in turn waits for the copy before it
// may reuse its send buffer.  Allreduce synchronises each rank's stream and
// reduces on the host.  (Running real NCCL ranks as processes on one GPU is
// what B200_PROFILING.md forbids: their kernels wait on one another.)
#include <cuda_runtime.h>
#include <nccl.h>

#include <condition_variable>
#include <cstdint>
#include <cstring>
#include <deque>
#include <map>
#include <memory>
#include <mutex>
#include <random>
#include <vector>

namespace {

struct Msg {
  const void *ptr;
  size_t bytes;
  cudaEvent_t ready;   // recorded on the sender's stream after its pack
};
struct Ack {
  cudaEvent_t done;    // recorded on the receiver's stream after its copy
};

struct World {
  int n = 0;
  std::mutex m;
  std::condition_variable cv;
  std::map<std::pair<int, int>, std::deque<Msg>> msgs;   // (src, dst)
  std::map<std::pair<int, int>, std::deque<Ack>> acks;   // (dst, src)
  // allreduce rendezvous
  uint64_t red_gen = 0;
  int red_arrived = 0;
  std::vector<uint64_t> red_acc;
  std::vector<uint64_t> red_out;
  // comm splits: generation -> child world
  std::map<int, std::shared_ptr<World>> splits;
  std::map<int, int> split_arrived;
};

std::mutex g_m;
std::map<std::string, std::shared_ptr<World>> g_worlds;   // by unique id bytes

}  // namespace

struct ncclComm {
  std::shared_ptr<World> w;
  int rank, nranks;
  int nsplits = 0;
};

namespace {

struct Op {
  bool send;
  void *buf;
  size_t bytes;
  int peer;
  ncclComm_t comm;
  cudaStream_t stream;
};
thread_local std::vector<Op> t_group;
thread_local int t_depth = 0;

size_t type_size(ncclDataType_t t) {
  switch (t) {
    case ncclInt8: case ncclUint8: return 1;
    case ncclFloat16: case ncclBfloat16: return 2;
    case ncclInt32: case ncclUint32: case ncclFloat32: return 4;
    default: return 8;
  }
}

ncclResult_t run_ops(std::vector<Op> &ops) {
  // 1. post every send (non-blocking)
  for (auto &o : ops) {
    if (!o.send) continue;
    cudaEvent_t e;
    if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) return ncclUnhandledCudaError;
    cudaEventRecord(e, o.stream);
    World &w = *o.comm->w;
    std::lock_guard<std::mutex> lk(w.m);
    w.msgs[{o.comm->rank, o.peer}].push_back(Msg{o.buf, o.bytes, e});
    w.cv.notify_all();
  }
  // 2. serve every receive: wait for the peer's post, copy after its pack
  for (auto &o : ops) {
    if (o.send) continue;
    World &w = *o.comm->w;
    Msg msg;
    {
      std::unique_lock<std::mutex> lk(w.m);
      auto &q = w.msgs[{o.peer, o.comm->rank}];
      w.cv.wait(lk, [&] { return !q.empty(); });
      msg = q.front();
      q.pop_front();
    }
    if (msg.bytes != o.bytes) return ncclInvalidUsage;
    cudaStreamWaitEvent(o.stream, msg.ready, 0);
    cudaMemcpyAsync(o.buf, msg.ptr, o.bytes, cudaMemcpyDeviceToDevice, o.stream);
    cudaEventDestroy(msg.ready);
    cudaEvent_t done;
    cudaEventCreateWithFlags(&done, cudaEventDisableTiming);
    cudaEventRecord(done, o.stream);
    std::lock_guard<std::mutex> lk(w.m);
    w.acks[{o.comm->rank, o.peer}].push_back(Ack{done});
    w.cv.notify_all();
  }
  // 3. every send: the sender's stream waits until the receiver has copied
  for (auto &o : ops) {
    if (!o.send) continue;
    World &w = *o.comm->w;
    Ack a;
    {
      std::unique_lock<std::mutex> lk(w.m);
      auto &q = w.acks[{o.peer, o.comm->rank}];
      w.cv.wait(lk, [&] { return !q.empty(); });
      a = q.front();
      q.pop_front();
    }
    cudaStreamWaitEvent(o.stream, a.done, 0);
    cudaEventDestroy(a.done);
  }
  return cudaGetLastError() == cudaSuccess ? ncclSuccess : ncclUnhandledCudaError;
}

}  // namespace

extern "C" {

const char *ncclGetErrorString(ncclResult_t r) { return r == ncclSuccess ? "success (fake nccl)" : "error (fake nccl)"; }

ncclResult_t ncclGetUniqueId(ncclUniqueId *id) {
  static std::mt19937_64 rng(std::random_device{}());
  std::lock_guard<std::mutex> lk(g_m);
  memset(id, 0, sizeof(*id));
  const uint64_t v = rng();
  memcpy(id->internal, &v, sizeof(v));
  return ncclSuccess;
}

ncclResult_t ncclCommInitRank(ncclComm_t *comm, int nranks, ncclUniqueId id, int rank) {
  std::lock_guard<std::mutex> lk(g_m);
  auto &w = g_worlds[std::string(id.internal, sizeof(id.internal))];
  if (!w) { w = std::make_shared<World>(); w->n = nranks; }
  if (w->n != nranks || rank < 0 || rank >= nranks) return ncclInvalidArgument;
  *comm = new ncclComm{w, rank, nranks};
  return ncclSuccess;
}

ncclResult_t ncclCommSplit(ncclComm_t comm, int color, int key, ncclComm_t *newcomm, ncclConfig_t *) {
  // every rank splits with one color (libpf: the mu-halo communicator)
  World &w = *comm->w;
  std::unique_lock<std::mutex> lk(w.m);
  const int gen = comm->nsplits++;
  auto &child = w.splits[gen];
  if (!child) { child = std::make_shared<World>(); child->n = comm->nranks; }
  *newcomm = new ncclComm{child, key, comm->nranks};
  (void)color;
  return ncclSuccess;
}

ncclResult_t ncclCommDestroy(ncclComm_t comm) {
  delete comm;
  return ncclSuccess;
}

ncclResult_t ncclGroupStart() {
  ++t_depth;
  return ncclSuccess;
}

ncclResult_t ncclGroupEnd() {
  if (--t_depth > 0) return ncclSuccess;
  std::vector<Op> ops;
  ops.swap(t_group);
  return run_ops(ops);
}

ncclResult_t ncclSend(const void *buf, size_t count, ncclDataType_t t, int peer, ncclComm_t comm, cudaStream_t s) {
  Op o{true, const_cast<void *>(buf), count * type_size(t), peer, comm, s};
  if (t_depth > 0) { t_group.push_back(o); return ncclSuccess; }
  std::vector<Op> ops{o};
  return run_ops(ops);
}

ncclResult_t ncclRecv(void *buf, size_t count, ncclDataType_t t, int peer, ncclComm_t comm, cudaStream_t s) {
  Op o{false, buf, count * type_size(t), peer, comm, s};
  if (t_depth > 0) { t_group.push_back(o); return ncclSuccess; }
  std::vector<Op> ops{o};
  return run_ops(ops);
}

// max / sum of uint64 or int64 (what libpf reduces: window front, I/O flags)
ncclResult_t ncclAllReduce(const void *sb, void *rb, size_t count, ncclDataType_t t, ncclRedOp_t op, ncclComm_t comm,
                           cudaStream_t s) {
  if (type_size(t) != 8 || (t != ncclUint64 && t != ncclInt64) || (op != ncclMax && op != ncclSum))
    return ncclInvalidArgument;
  std::vector<uint64_t> v(count);
  if (cudaStreamSynchronize(s) != cudaSuccess) return ncclUnhandledCudaError;
  cudaMemcpy(v.data(), sb, count * 8, cudaMemcpyDeviceToHost);
  World &w = *comm->w;
  std::vector<uint64_t> out;
  {
    std::unique_lock<std::mutex> lk(w.m);
    const uint64_t gen = w.red_gen;
    if (w.red_arrived == 0) w.red_acc = v;
    else
      for (size_t i = 0; i < count; ++i) {
        if (op == ncclMax) w.red_acc[i] = t == ncclInt64 ? (uint64_t)std::max((int64_t)w.red_acc[i], (int64_t)v[i])
                                                         : std::max(w.red_acc[i], v[i]);
        else w.red_acc[i] += v[i];
      }
    if (++w.red_arrived == w.n) {
      w.red_out = w.red_acc;
      w.red_arrived = 0;
      ++w.red_gen;
      w.cv.notify_all();
    } else {
      w.cv.wait(lk, [&] { return w.red_gen != gen; });
    }
    out = w.red_out;
  }
  cudaMemcpy(rb, out.data(), count * 8, cudaMemcpyHostToDevice);
  return ncclSuccess;
}

}  // extern "C"
