// In-process NCCL emulation for testing the library's multi-rank code path
// (exchange(), the LLG all-reduces, the overlapped exchange communicator,
// the suspended-step continuation) on ONE GPU: every rank is a thread of one
// process driving its own handle, and this library, LD_PRELOADed, replaces
// the NCCL entry points the library imports.  Point-to-point operations are
// matched per (sender, receiver) pair in posting order, as NCCL does, and
// performed as stream-ordered device copies (the receiver's stream waits for
// the sender's data, the sender's stream for the copy); all-reduces
// rendezvous every rank of the communicator, gather all inputs, then reduce.
// Sizes and types are checked on both sides; a mismatch aborts.  Host-side
// waits stand in for NCCL's device-side ones, which is sound here because
// every rank issues the same calls in the same order.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -shared -Xcompiler -fPIC \
//        -o libnccl_emul.so nccl_emul.cu
#include <cuda_runtime.h>
#include <nccl.h>

#include <condition_variable>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

namespace {

void die(const char* msg) {
    fprintf(stderr, "nccl_emul: %s\n", msg);
    fflush(stderr);
    abort();
}
#define EM_CU(x) do { if ((x) != cudaSuccess) die(#x); } while (0)

size_t type_size(ncclDataType_t t) {
    switch (t) {
        case ncclInt8: case ncclUint8: return 1;
        case ncclFloat16: return 2;
        case ncclInt32: case ncclUint32: case ncclFloat32: return 4;
        case ncclInt64: case ncclUint64: case ncclFloat64: return 8;
        default: die("unsupported data type"); return 0;
    }
}

struct SendPost {
    const void* src = nullptr;
    size_t bytes = 0;
    cudaEvent_t ready = nullptr;     // sender's stream reached the send
    cudaEvent_t done = nullptr;      // receiver's copy finished
    bool acked = false;
};

struct ArSlot {
    const void* send = nullptr;
    void* recv = nullptr;
    size_t count = 0;
    ncclDataType_t type = ncclUint64;
    cudaEvent_t ready = nullptr, gathered = nullptr;
    bool posted = false, gathered_posted = false;
};

struct Group {
    int nranks = 0;
    std::mutex m;
    std::condition_variable cv;
    std::map<std::pair<int, int>, std::deque<std::shared_ptr<SendPost>>> mail;
    std::map<long long, std::vector<ArSlot>> ar;
    std::map<long long, int> ar_left;
    std::vector<long long> ar_next;
    std::vector<int> splits;          // per rank: ncclCommSplit calls so far
};

std::mutex g_m;
std::map<std::string, std::shared_ptr<Group>> g_groups;
unsigned long long g_id_counter = 0;

}  // namespace

struct ncclComm {
    std::shared_ptr<Group> g;
    std::string key;
    int rank = 0, nranks = 0;
};

namespace {

enum OpKind { kSend, kRecv, kAllReduce };
struct Op {
    OpKind kind;
    const void* send;
    void* recv;
    size_t count;
    ncclDataType_t type;
    ncclRedOp_t red;
    int peer;
    ncclComm_t comm;
    cudaStream_t stream;
};

thread_local int t_depth = 0;
thread_local std::vector<Op> t_pending;

template <typename T>
__global__ void k_max(const T* __restrict__ st, T* __restrict__ out, size_t count, int n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < count;
         i += (size_t)gridDim.x * blockDim.x) {
        T m = st[i];
        for (int r = 1; r < n; ++r) {
            const T v = st[r * count + i];
            m = v > m ? v : m;
        }
        out[i] = m;
    }
}

void reduce_max(const void* staging, void* out, size_t count, int n, ncclDataType_t t,
                cudaStream_t s) {
    const unsigned blocks = (unsigned)std::min<size_t>((count + 255) / 256, 1024);
    switch (t) {
        case ncclUint64: k_max<<<blocks, 256, 0, s>>>((const unsigned long long*)staging,
                                                      (unsigned long long*)out, count, n); break;
        case ncclInt32: k_max<<<blocks, 256, 0, s>>>((const int*)staging, (int*)out, count, n);
            break;
        case ncclFloat64: k_max<<<blocks, 256, 0, s>>>((const double*)staging, (double*)out,
                                                       count, n); break;
        default: die("all-reduce type not emulated");
    }
    EM_CU(cudaGetLastError());
}

cudaEvent_t record(cudaStream_t s) {
    cudaEvent_t e;
    EM_CU(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    EM_CU(cudaEventRecord(e, s));
    return e;
}

void run_batch(std::vector<Op>& ops) {
    // 1. post every send of the batch
    std::vector<std::shared_ptr<SendPost>> mine;
    for (Op& op : ops) {
        if (op.kind != kSend) continue;
        auto p = std::make_shared<SendPost>();
        p->src = op.send;
        p->bytes = op.count * type_size(op.type);
        p->ready = record(op.stream);
        Group& G = *op.comm->g;
        {
            std::lock_guard<std::mutex> lk(G.m);
            G.mail[{op.comm->rank, op.peer}].push_back(p);
        }
        G.cv.notify_all();
        mine.push_back(p);
    }
    // 2. receive (in order per sender)
    for (Op& op : ops) {
        if (op.kind != kRecv) continue;
        Group& G = *op.comm->g;
        std::shared_ptr<SendPost> p;
        {
            std::unique_lock<std::mutex> lk(G.m);
            auto& q = G.mail[{op.peer, op.comm->rank}];
            G.cv.wait(lk, [&] { return !q.empty(); });
            p = q.front();
            q.pop_front();
        }
        const size_t bytes = op.count * type_size(op.type);
        if (bytes != p->bytes) {
            char msg[160];
            snprintf(msg, sizeof msg, "size mismatch: rank %d receives %zu B from %d, which sent %zu B",
                     op.comm->rank, bytes, op.peer, p->bytes);
            die(msg);
        }
        EM_CU(cudaStreamWaitEvent(op.stream, p->ready, 0));
        EM_CU(cudaMemcpyAsync(op.recv, p->src, bytes, cudaMemcpyDeviceToDevice, op.stream));
        cudaEvent_t done = record(op.stream);
        {
            std::lock_guard<std::mutex> lk(G.m);
            p->done = done;
            p->acked = true;
        }
        G.cv.notify_all();
    }
    // 3. a send completes once its copy has run
    size_t si = 0;
    for (Op& op : ops) {
        if (op.kind != kSend) continue;
        Group& G = *op.comm->g;
        auto& p = mine[si++];
        {
            std::unique_lock<std::mutex> lk(G.m);
            G.cv.wait(lk, [&] { return p->acked; });
        }
        EM_CU(cudaStreamWaitEvent(op.stream, p->done, 0));
    }
    // 4. all-reduces, in call order
    for (Op& op : ops) {
        if (op.kind != kAllReduce) continue;
        if (op.red != ncclMax) die("only ncclMax is emulated");
        Group& G = *op.comm->g;
        const int me = op.comm->rank, n = G.nranks;
        long long seq;
        {
            std::unique_lock<std::mutex> lk(G.m);
            seq = G.ar_next[me]++;
            auto& slots = G.ar[seq];
            if (slots.empty()) { slots.resize(n); G.ar_left[seq] = n; }
            ArSlot& sl = slots[me];
            sl.send = op.send; sl.recv = op.recv; sl.count = op.count; sl.type = op.type;
            sl.ready = record(op.stream);
            sl.posted = true;
            G.cv.notify_all();
            G.cv.wait(lk, [&] {
                for (auto& x : G.ar[seq]) if (!x.posted) return false;
                return true;
            });
            for (auto& x : G.ar[seq])
                if (x.count != op.count || x.type != op.type) die("all-reduce size/type mismatch");
        }
        const size_t bytes = op.count * type_size(op.type);
        void* staging = nullptr;
        EM_CU(cudaMallocAsync(&staging, bytes * n, op.stream));
        std::vector<ArSlot> snap;
        {
            std::lock_guard<std::mutex> lk(G.m);
            snap = G.ar[seq];
        }
        for (int r = 0; r < n; ++r) {
            EM_CU(cudaStreamWaitEvent(op.stream, snap[r].ready, 0));
            EM_CU(cudaMemcpyAsync((char*)staging + r * bytes, snap[r].send, bytes,
                                  cudaMemcpyDeviceToDevice, op.stream));
        }
        {
            std::unique_lock<std::mutex> lk(G.m);
            G.ar[seq][me].gathered = record(op.stream);
            G.ar[seq][me].gathered_posted = true;
            G.cv.notify_all();
            G.cv.wait(lk, [&] {
                for (auto& x : G.ar[seq]) if (!x.gathered_posted) return false;
                return true;
            });
            snap = G.ar[seq];
        }
        for (int r = 0; r < n; ++r) EM_CU(cudaStreamWaitEvent(op.stream, snap[r].gathered, 0));
        reduce_max(staging, op.recv, op.count, n, op.type, op.stream);
        EM_CU(cudaFreeAsync(staging, op.stream));
        {
            std::lock_guard<std::mutex> lk(G.m);
            if (--G.ar_left[seq] == 0) { G.ar.erase(seq); G.ar_left.erase(seq); }
        }
    }
    ops.clear();
}

void submit(const Op& op) {
    t_pending.push_back(op);
    if (t_depth == 0) run_batch(t_pending);
}

}  // namespace

extern "C" {

ncclResult_t ncclGetVersion(int* version) { *version = 99999; return ncclSuccess; }

ncclResult_t ncclGetUniqueId(ncclUniqueId* id) {
    std::lock_guard<std::mutex> lk(g_m);
    memset(id, 0, sizeof *id);
    snprintf(id->internal, sizeof id->internal, "emul-%llu", ++g_id_counter);
    return ncclSuccess;
}

ncclResult_t ncclCommInitRank(ncclComm_t* comm, int nranks, ncclUniqueId id, int rank) {
    std::lock_guard<std::mutex> lk(g_m);
    const std::string key(id.internal, strnlen(id.internal, sizeof id.internal));
    auto& g = g_groups[key];
    if (!g) {
        g = std::make_shared<Group>();
        g->nranks = nranks;
        g->ar_next.assign(nranks, 0);
        g->splits.assign(nranks, 0);
    }
    if (g->nranks != nranks || rank < 0 || rank >= nranks) return ncclInvalidArgument;
    *comm = new ncclComm{g, key, rank, nranks};
    return ncclSuccess;
}

ncclResult_t ncclCommSplit(ncclComm_t comm, int color, int key, ncclComm_t* newcomm,
                           ncclConfig_t*) {
    std::lock_guard<std::mutex> lk(g_m);
    const int k = comm->g->splits[comm->rank]++;
    const std::string ck = comm->key + "/split" + std::to_string(k) + ":" + std::to_string(color);
    auto& g = g_groups[ck];
    if (!g) {
        g = std::make_shared<Group>();
        g->nranks = comm->nranks;
        g->ar_next.assign(comm->nranks, 0);
        g->splits.assign(comm->nranks, 0);
    }
    *newcomm = new ncclComm{g, ck, key, comm->nranks};   // key = rank in every use here
    return ncclSuccess;
}

ncclResult_t ncclCommDestroy(ncclComm_t comm) { delete comm; return ncclSuccess; }
ncclResult_t ncclCommCount(const ncclComm_t comm, int* count) { *count = comm->nranks; return ncclSuccess; }
ncclResult_t ncclCommUserRank(const ncclComm_t comm, int* rank) { *rank = comm->rank; return ncclSuccess; }
const char* ncclGetErrorString(ncclResult_t r) { return r == ncclSuccess ? "success" : "emulated error"; }

ncclResult_t ncclGroupStart() { ++t_depth; return ncclSuccess; }
ncclResult_t ncclGroupEnd() {
    if (--t_depth == 0) run_batch(t_pending);
    return ncclSuccess;
}

ncclResult_t ncclSend(const void* buf, size_t count, ncclDataType_t type, int peer,
                      ncclComm_t comm, cudaStream_t stream) {
    if (peer < 0 || peer >= comm->nranks || peer == comm->rank) die("bad send peer");
    submit(Op{kSend, buf, nullptr, count, type, ncclSum, peer, comm, stream});
    return ncclSuccess;
}

ncclResult_t ncclRecv(void* buf, size_t count, ncclDataType_t type, int peer,
                      ncclComm_t comm, cudaStream_t stream) {
    if (peer < 0 || peer >= comm->nranks || peer == comm->rank) die("bad recv peer");
    submit(Op{kRecv, nullptr, buf, count, type, ncclSum, peer, comm, stream});
    return ncclSuccess;
}

ncclResult_t ncclAllReduce(const void* send, void* recv, size_t count, ncclDataType_t type,
                           ncclRedOp_t op, ncclComm_t comm, cudaStream_t stream) {
    submit(Op{kAllReduce, send, recv, count, type, op, -1, comm, stream});
    return ncclSuccess;
}

}  // extern "C"
