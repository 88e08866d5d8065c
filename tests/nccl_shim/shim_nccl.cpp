// shim_nccl.cpp -- TEST INFRASTRUCTURE, not part of the product.
// A stand-in for the nine NCCL entry points libbdm.so resolves with dlopen (dist_abi.cu),
// so that the two-rank code path of bdm_aura_exchange -- the order of its sends and
// receives, the count exchange, the zero-size skips, the edge ranks -- runs on a box with
// ONE GPU: the ranks are separate processes sharing the device, and a message is a file
// in the directory $BDM_SHIM_DIR (device -> host -> file -> host -> device).  Only the host
// waits (a receive polls for its file); no kernel ever waits on another rank's kernel.
// Semantics kept from NCCL: operations between a pair of ranks match in issue order; inside
// ncclGroupStart/End nothing blocks until the group ends (sends are issued before receives).
// Selected with BDM_NCCL_LIB=<this .so> (tests/test_gpu_nccl_shim.py).
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <sys/stat.h>
#include <time.h>
#include <unistd.h>

#include <map>
#include <string>
#include <vector>

extern "C" {
typedef enum { ncclSuccess = 0, ncclUnhandledCudaError = 1, ncclSystemError = 2, ncclInternalError = 3,
               ncclInvalidArgument = 4 } ncclResult_t;
typedef struct { char internal[128]; } ncclUniqueId;
typedef struct ShimComm *ncclComm_t;
typedef int ncclDataType_t;  // 0,1: 1 byte; 2,3: 4; 4,5: 8; 6: 2; 7: 4; 8: 8
typedef int ncclRedOp_t;     // 0 sum, 1 prod, 2 max, 3 min
}

struct Op {
    bool send;
    void *buf;
    size_t bytes;
    int peer;
    cudaStream_t st;
};
struct ShimComm {
    int rank, nranks;
    std::string dir;
    std::map<std::pair<int, int>, long> seq;  // messages so far per (src, dst)
    long ar_seq = 0;
};
static int g_depth = 0;
static std::vector<std::pair<ShimComm *, Op>> g_queue;

static size_t dsize(ncclDataType_t t) {
    static const size_t s[] = {1, 1, 4, 4, 8, 8, 2, 4, 8};
    return t >= 0 && t <= 8 ? s[t] : 0;
}
static bool publish(const std::string &path, const void *data, size_t bytes) {
    const std::string tmp = path + ".tmp";
    FILE *f = fopen(tmp.c_str(), "wb");
    if (!f) return false;
    const bool ok = bytes == 0 || fwrite(data, 1, bytes, f) == bytes;
    fclose(f);
    return ok && rename(tmp.c_str(), path.c_str()) == 0;
}
static bool await(const std::string &path, std::vector<char> &out) {
    struct stat sb;
    for (int i = 0; i < 120000; ++i) {  // 120 s
        if (stat(path.c_str(), &sb) == 0) {
            out.resize((size_t)sb.st_size);
            FILE *f = fopen(path.c_str(), "rb");
            if (!f) return false;
            const bool ok = out.empty() || fread(out.data(), 1, out.size(), f) == out.size();
            fclose(f);
            return ok;
        }
        usleep(1000);
    }
    fprintf(stderr, "shim_nccl: timed out waiting for %s\n", path.c_str());
    return false;
}
static ncclResult_t run(ShimComm *c, const Op &o) {
    if (o.peer < 0 || o.peer >= c->nranks || o.peer == c->rank) return ncclInvalidArgument;
    if (o.send) {
        std::vector<char> h(o.bytes);
        if (cudaStreamSynchronize(o.st) != cudaSuccess) return ncclUnhandledCudaError;
        if (o.bytes && cudaMemcpy(h.data(), o.buf, o.bytes, cudaMemcpyDeviceToHost) != cudaSuccess)
            return ncclUnhandledCudaError;
        const long k = c->seq[{c->rank, o.peer}]++;
        const std::string p = c->dir + "/m_" + std::to_string(c->rank) + "_" + std::to_string(o.peer) + "_" +
                              std::to_string(k) + ".bin";
        return publish(p, h.data(), o.bytes) ? ncclSuccess : ncclSystemError;
    }
    const long k = c->seq[{o.peer, c->rank}]++;
    const std::string p = c->dir + "/m_" + std::to_string(o.peer) + "_" + std::to_string(c->rank) + "_" +
                          std::to_string(k) + ".bin";
    std::vector<char> h;
    if (!await(p, h)) return ncclSystemError;
    if (h.size() != o.bytes) {  // a size mismatch between the two ranks' views of one message
        fprintf(stderr, "shim_nccl: %s holds %zu bytes, the receive expects %zu\n", p.c_str(), h.size(), o.bytes);
        return ncclInvalidArgument;
    }
    if (o.bytes && cudaMemcpyAsync(o.buf, h.data(), o.bytes, cudaMemcpyHostToDevice, o.st) != cudaSuccess)
        return ncclUnhandledCudaError;
    if (cudaStreamSynchronize(o.st) != cudaSuccess) return ncclUnhandledCudaError;
    unlink(p.c_str());
    return ncclSuccess;
}
static ncclResult_t issue(ShimComm *c, const Op &o) {
    if (g_depth > 0) {
        g_queue.push_back({c, o});
        return ncclSuccess;
    }
    return run(c, o);
}

extern "C" {
ncclResult_t ncclGetUniqueId(ncclUniqueId *id) {
    memset(id, 0, sizeof(*id));
    snprintf(id->internal, sizeof(id->internal), "shim-%ld-%ld", (long)getpid(), (long)time(nullptr));
    return ncclSuccess;
}
ncclResult_t ncclCommInitRank(ncclComm_t *comm, int nranks, ncclUniqueId id, int rank) {
    const char *d = getenv("BDM_SHIM_DIR");
    if (!d || nranks < 1 || rank < 0 || rank >= nranks) return ncclInvalidArgument;
    ShimComm *c = new ShimComm();
    c->rank = rank;
    c->nranks = nranks;
    c->dir = d;
    (void)id;
    *comm = c;
    return ncclSuccess;
}
ncclResult_t ncclCommDestroy(ncclComm_t comm) {
    delete comm;
    return ncclSuccess;
}
ncclResult_t ncclSend(const void *buf, size_t count, ncclDataType_t t, int peer, ncclComm_t c, cudaStream_t st) {
    if (!dsize(t)) return ncclInvalidArgument;
    return issue(c, Op{true, const_cast<void *>(buf), count * dsize(t), peer, st});
}
ncclResult_t ncclRecv(void *buf, size_t count, ncclDataType_t t, int peer, ncclComm_t c, cudaStream_t st) {
    if (!dsize(t)) return ncclInvalidArgument;
    return issue(c, Op{false, buf, count * dsize(t), peer, st});
}
ncclResult_t ncclGroupStart() {
    ++g_depth;
    return ncclSuccess;
}
ncclResult_t ncclGroupEnd() {
    if (g_depth <= 0) return ncclInvalidArgument;
    if (--g_depth > 0) return ncclSuccess;
    std::vector<std::pair<ShimComm *, Op>> q;
    q.swap(g_queue);
    ncclResult_t r = ncclSuccess;
    for (int pass = 0; pass < 2 && r == ncclSuccess; ++pass)  // every send, then every receive
        for (auto &e : q)
            if (e.second.send == (pass == 0) && r == ncclSuccess) r = run(e.first, e.second);
    return r;
}
ncclResult_t ncclAllReduce(const void *send, void *recv, size_t count, ncclDataType_t t, ncclRedOp_t op,
                           ncclComm_t c, cudaStream_t st) {
    if (t != 8 || op != 3) return ncclInvalidArgument;  // MIN of doubles is all the library uses
    std::vector<double> mine(count), acc(count);
    if (cudaStreamSynchronize(st) != cudaSuccess) return ncclUnhandledCudaError;
    if (cudaMemcpy(mine.data(), send, count * 8, cudaMemcpyDeviceToHost) != cudaSuccess)
        return ncclUnhandledCudaError;
    const long k = c->ar_seq++;
    const std::string base = c->dir + "/ar_" + std::to_string(k) + "_";
    if (!publish(base + std::to_string(c->rank) + ".bin", mine.data(), count * 8)) return ncclSystemError;
    acc = mine;
    for (int r = 0; r < c->nranks; ++r) {
        if (r == c->rank) continue;
        std::vector<char> h;
        if (!await(base + std::to_string(r) + ".bin", h) || h.size() != count * 8) return ncclSystemError;
        const double *v = reinterpret_cast<const double *>(h.data());
        for (size_t i = 0; i < count; ++i) acc[i] = v[i] < acc[i] ? v[i] : acc[i];
    }
    if (cudaMemcpyAsync(recv, acc.data(), count * 8, cudaMemcpyHostToDevice, st) != cudaSuccess)
        return ncclUnhandledCudaError;
    return cudaStreamSynchronize(st) == cudaSuccess ? ncclSuccess : ncclUnhandledCudaError;
}
const char *ncclGetErrorString(ncclResult_t r) {
    switch (r) {
        case ncclSuccess: return "success";
        case ncclUnhandledCudaError: return "shim: CUDA error";
        case ncclSystemError: return "shim: file or timeout error";
        case ncclInvalidArgument: return "shim: invalid argument or message size mismatch";
        default: return "shim: internal error";
    }
}
}
