// Row exchange between ranks for the hash-partitioned engine.
//
// Two implementations behind one interface:
//   NcclTransport  one process per GPU, NCCL grouped send/recv over NVLink /
//                  NVSwitch (libnccl is dlopen'ed so the process shares the
//                  NCCL that torch.distributed already loaded);
//   LocalGroup     W virtual ranks as threads of one process on one GPU,
//                  exchanging through device-to-device copies. It runs the
//                  exact distributed engine code path (partitioning, bucket
//                  routing, count exchange, Δ forwarding, all-reduced stats)
//                  so multi-rank correctness is testable on a single B200.
#pragma once

#include <memory>
#include <vector>

#include "fv_common.cuh"

namespace fv {

struct ExchangeCol {
    const void* send = nullptr;  // rows grouped by destination rank
    void* recv = nullptr;        // rows grouped by source rank
    u32 elem = 4;                // bytes per row
};

class Transport {
public:
    virtual ~Transport() = default;
    virtual int rank() const = 0;
    virtual int world() const = 0;
    // send_counts[p] rows go to peer p; recv_counts[p] rows arrive from p.
    virtual void exchange_counts(Ctx* c, const u64* send_counts, u64* recv_counts) = 0;
    // The same from send counts already on the device (written by the route
    // kernel): fills both host arrays with one host round trip where the
    // transport can (NCCL: an all-gather of the device counts, then one read).
    virtual void exchange_counts_dev(Ctx* c, const u64* d_send_counts, u64* send_counts, u64* recv_counts);
    // Move every column's per-peer segments (offsets/counts in rows).
    virtual void exchange_rows(Ctx* c, const std::vector<ExchangeCol>& cols, const u64* scnt, const u64* soff,
                               const u64* rcnt, const u64* roff) = 0;
    // Element-wise sum over ranks of n host values (in place).
    virtual void allreduce_sum(Ctx* c, u64* vals, int n) = 0;
    // In-process groups: a failing rank releases its peers (their pending
    // and later collectives throw) and the group remembers who failed first.
    virtual void abort() {}
    virtual int first_failed() const { return -1; }
};

// NCCL (one process per GPU). `id` is a 128-byte ncclUniqueId.
std::unique_ptr<Transport> make_nccl_transport(Ctx* c, int rank, int world, const void* id);
void nccl_unique_id(void* out128);

// In-process group of `world` ranks (all on the same device).
std::vector<std::unique_ptr<Transport>> make_local_group(int world);

// owner(v) = floor(hash32(v) * world / 2^32)
inline u32 owner_of(u32 v, u32 world) {
    u32 k = v;
    k ^= k >> 16;
    k *= 0x85ebca6bu;
    k ^= k >> 13;
    k *= 0xc2b2ae35u;
    k ^= k >> 16;
    return static_cast<u32>((static_cast<u64>(k) * world) >> 32);
}

}  // namespace fv
