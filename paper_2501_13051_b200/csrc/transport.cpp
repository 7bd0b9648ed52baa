// Transports for the partitioned engine (see transport.h).
#include "transport.h"

#include <dlfcn.h>

#include <condition_variable>
#include <cstring>
#include <mutex>

namespace fv {

void Transport::exchange_counts_dev(Ctx* c, const u64* d_send, u64* send_counts, u64* recv_counts) {
    FV_CUDA(cudaMemcpyAsync(send_counts, d_send, sizeof(u64) * world(), cudaMemcpyDeviceToHost, c->stream));
    c->sync();
    exchange_counts(c, send_counts, recv_counts);
}


// ---- NCCL (resolved at run time) ---------------------------------------------

namespace {

typedef int nccl_result;
typedef void* nccl_comm;
struct nccl_id {
    char internal[128];
};
enum { kNcclUint8 = 1, kNcclUint64 = 5 };
enum { kNcclSum = 0 };

struct NcclApi {
    void* h = nullptr;
    nccl_result (*GetUniqueId)(nccl_id*) = nullptr;
    nccl_result (*CommInitRank)(nccl_comm*, int, nccl_id, int) = nullptr;
    nccl_result (*CommDestroy)(nccl_comm) = nullptr;
    nccl_result (*Send)(const void*, size_t, int, int, nccl_comm, cudaStream_t) = nullptr;
    nccl_result (*Recv)(void*, size_t, int, int, nccl_comm, cudaStream_t) = nullptr;
    nccl_result (*GroupStart)() = nullptr;
    nccl_result (*GroupEnd)() = nullptr;
    nccl_result (*AllReduce)(const void*, void*, size_t, int, int, nccl_comm, cudaStream_t) = nullptr;
    nccl_result (*AllGather)(const void*, void*, size_t, int, nccl_comm, cudaStream_t) = nullptr;
    const char* (*GetErrorString)(nccl_result) = nullptr;
};

NcclApi& nccl() {
    static NcclApi api;
    if (api.h) return api;
    // Prefer the NCCL already mapped into the process (torch's), else load one.
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) fail(FV_ERR_CUDA, "multi-GPU requested but libnccl.so.2 cannot be loaded");
    auto sym = [&](const char* n) {
        void* p = dlsym(h, n);
        if (!p) fail(FV_ERR_CUDA, std::string("libnccl lacks ") + n);
        return p;
    };
    api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(sym("ncclGetUniqueId"));
    api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(sym("ncclCommInitRank"));
    api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(sym("ncclCommDestroy"));
    api.Send = reinterpret_cast<decltype(api.Send)>(sym("ncclSend"));
    api.Recv = reinterpret_cast<decltype(api.Recv)>(sym("ncclRecv"));
    api.GroupStart = reinterpret_cast<decltype(api.GroupStart)>(sym("ncclGroupStart"));
    api.GroupEnd = reinterpret_cast<decltype(api.GroupEnd)>(sym("ncclGroupEnd"));
    api.AllReduce = reinterpret_cast<decltype(api.AllReduce)>(sym("ncclAllReduce"));
    api.AllGather = reinterpret_cast<decltype(api.AllGather)>(sym("ncclAllGather"));
    api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(sym("ncclGetErrorString"));
    api.h = h;
    return api;
}

void nccl_check(nccl_result r, const char* what) {
    if (r != 0) fail(FV_ERR_CUDA, std::string("NCCL ") + what + ": " + nccl().GetErrorString(r));
}

class NcclTransport final : public Transport {
public:
    NcclTransport(Ctx* c, int rank, int world, const void* id) : rank_(rank), world_(world) {
        nccl_id nid;
        std::memcpy(&nid, id, sizeof nid);
        c->activate();
        nccl_check(nccl().CommInitRank(&comm_, world, nid, rank), "CommInitRank");
    }
    ~NcclTransport() override {
        if (comm_) nccl().CommDestroy(comm_);
    }
    int rank() const override { return rank_; }
    int world() const override { return world_; }

    void exchange_counts(Ctx* c, const u64* send_counts, u64* recv_counts) override {
        DBuf<u64> mine(c, world_), all(c, u64(world_) * world_);
        mine.upload(send_counts, world_);
        nccl_check(nccl().AllGather(mine.get(), all.get(), world_, kNcclUint64, comm_, c->stream), "AllGather");
        std::vector<u64> h(u64(world_) * world_);
        all.download(h.data(), h.size());
        for (int p = 0; p < world_; ++p) recv_counts[p] = h[u64(p) * world_ + rank_];
    }

    void exchange_counts_dev(Ctx* c, const u64* d_send, u64* send_counts, u64* recv_counts) override {
        DBuf<u64> all(c, u64(world_) * world_);
        nccl_check(nccl().AllGather(d_send, all.get(), world_, kNcclUint64, comm_, c->stream), "AllGather");
        std::vector<u64> h(u64(world_) * world_);
        all.download(h.data(), h.size());  // the one host round trip of the exchange
        for (int p = 0; p < world_; ++p) {
            send_counts[p] = h[u64(rank_) * world_ + p];
            recv_counts[p] = h[u64(p) * world_ + rank_];
        }
    }

    void exchange_rows(Ctx* c, const std::vector<ExchangeCol>& cols, const u64* scnt, const u64* soff,
                       const u64* rcnt, const u64* roff) override {
        nccl_check(nccl().GroupStart(), "GroupStart");
        for (const auto& col : cols) {
            for (int p = 0; p < world_; ++p) {
                const char* s = static_cast<const char*>(col.send) + soff[p] * col.elem;
                char* r = static_cast<char*>(col.recv) + roff[p] * col.elem;
                if (p == rank_) {
                    if (scnt[p])
                        FV_CUDA(cudaMemcpyAsync(r, s, scnt[p] * col.elem, cudaMemcpyDeviceToDevice, c->stream));
                    continue;
                }
                if (scnt[p]) nccl_check(nccl().Send(s, scnt[p] * col.elem, kNcclUint8, p, comm_, c->stream), "Send");
                if (rcnt[p]) nccl_check(nccl().Recv(r, rcnt[p] * col.elem, kNcclUint8, p, comm_, c->stream), "Recv");
            }
        }
        nccl_check(nccl().GroupEnd(), "GroupEnd");
    }

    void allreduce_sum(Ctx* c, u64* vals, int n) override {
        DBuf<u64> d(c, n);
        d.upload(vals, n);
        nccl_check(nccl().AllReduce(d.get(), d.get(), n, kNcclUint64, kNcclSum, comm_, c->stream), "AllReduce");
        d.download(vals, n);
    }

private:
    int rank_, world_;
    nccl_comm comm_ = nullptr;
};

// ---- in-process group -----------------------------------------------------------

struct LocalShared {
    explicit LocalShared(int w) : world(w), counts(w), cols(w), scnt(w), soff(w), vals(w) {}
    int world;
    std::mutex mu;
    std::condition_variable cv;
    int arrived = 0;
    u64 generation = 0;
    // Set by the first rank that fails: every rank waiting in (or later
    // reaching) a barrier throws instead of waiting for it forever.
    bool aborted = false;
    int first_failed = -1;
    std::vector<const u64*> counts;
    std::vector<const std::vector<ExchangeCol>*> cols;
    std::vector<const u64*> scnt, soff;
    std::vector<u64*> vals;

    void barrier() {
        std::unique_lock<std::mutex> lk(mu);
        if (aborted) fail(FV_ERR_INVALID, "in-process group aborted by another rank");
        const u64 gen = generation;
        if (++arrived == world) {
            arrived = 0;
            ++generation;
            cv.notify_all();
        } else {
            cv.wait(lk, [&] { return generation != gen || aborted; });
            if (generation == gen) fail(FV_ERR_INVALID, "in-process group aborted by another rank");
        }
    }

    void abort(int rank) {
        std::lock_guard<std::mutex> lk(mu);
        if (first_failed < 0) first_failed = rank;
        aborted = true;
        cv.notify_all();
    }
};

class LocalTransport final : public Transport {
public:
    LocalTransport(std::shared_ptr<LocalShared> s, int rank) : s_(std::move(s)), rank_(rank) {}
    int rank() const override { return rank_; }
    int world() const override { return s_->world; }
    void abort() override { s_->abort(rank_); }
    int first_failed() const override { return s_->first_failed; }

    void exchange_counts(Ctx*, const u64* send_counts, u64* recv_counts) override {
        s_->counts[rank_] = send_counts;
        s_->barrier();
        for (int p = 0; p < s_->world; ++p) recv_counts[p] = s_->counts[p][rank_];
        s_->barrier();
    }

    void exchange_rows(Ctx* c, const std::vector<ExchangeCol>& cols, const u64* scnt, const u64* soff,
                       const u64* rcnt, const u64* roff) override {
        c->sync();  // our send buffers are complete before peers read them
        s_->cols[rank_] = &cols;
        s_->scnt[rank_] = scnt;
        s_->soff[rank_] = soff;
        s_->barrier();
        // Validate before touching any peer buffer, and report a mismatch
        // only after the closing barrier: a rank must not unwind (and free
        // the send buffers its peers are reading) while the exchange runs.
        bool ok = true;
        for (int p = 0; p < s_->world; ++p) ok = ok && s_->scnt[p][rank_] == rcnt[p];
        if (ok) {
            for (size_t j = 0; j < cols.size(); ++j) {
                for (int p = 0; p < s_->world; ++p) {
                    const ExchangeCol& src = (*s_->cols[p])[j];
                    const u64 n = s_->scnt[p][rank_];
                    if (!n) continue;
                    const char* from = static_cast<const char*>(src.send) + s_->soff[p][rank_] * src.elem;
                    char* to = static_cast<char*>(cols[j].recv) + roff[p] * cols[j].elem;
                    FV_CUDA(cudaMemcpyAsync(to, from, n * src.elem, cudaMemcpyDeviceToDevice, c->stream));
                }
            }
            c->sync();
        }
        s_->barrier();  // peers may release their send buffers now
        if (!ok) fail(FV_ERR_INVALID, "local exchange: count mismatch");
    }

    void allreduce_sum(Ctx*, u64* vals, int n) override {
        s_->vals[rank_] = vals;
        s_->barrier();
        std::vector<u64> sum(n, 0);
        for (int p = 0; p < s_->world; ++p)
            for (int i = 0; i < n; ++i) sum[i] += s_->vals[p][i];
        s_->barrier();
        for (int i = 0; i < n; ++i) vals[i] = sum[i];
        s_->barrier();
    }

private:
    std::shared_ptr<LocalShared> s_;
    int rank_;
};

}  // namespace

std::unique_ptr<Transport> make_nccl_transport(Ctx* c, int rank, int world, const void* id) {
    return std::make_unique<NcclTransport>(c, rank, world, id);
}

void nccl_unique_id(void* out128) {
    nccl_id id;
    nccl_check(nccl().GetUniqueId(&id), "GetUniqueId");
    std::memcpy(out128, &id, sizeof id);
}

std::vector<std::unique_ptr<Transport>> make_local_group(int world) {
    auto shared = std::make_shared<LocalShared>(world);
    std::vector<std::unique_ptr<Transport>> out;
    for (int r = 0; r < world; ++r) out.push_back(std::make_unique<LocalTransport>(shared, r));
    return out;
}

}  // namespace fv
