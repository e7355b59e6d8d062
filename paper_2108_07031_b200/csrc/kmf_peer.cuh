// kmf_peer.cuh -- the peer transport of a partitioned solve: halo q and
// residue limbs moved by the GPUs themselves over peer memory (NVLink /
// NVSwitch P2P, CUDA IPC between processes), no NCCL on the data path.
//
// Every rank's device memory holds its q array and one PeerFlags block;
// each rank maps its peers' q and PeerFlags (cudaIpcOpenMemHandle, or plain
// pointers between contexts of one process).  Per RK stage:
//
//   band pass (stream s3)   k_peer_wait_data: every peer this rank
//                           receives from has pushed the halo of the last
//                           update (data[r] >= own pushes)
//   after the band pass     k_peer_band_done: bands += 1, tell every peer
//                           this rank receives from (read[me] = bands), then
//                           wait until every peer this rank SENDS to has
//                           finished its own band pass (read[r] >= bands):
//                           their halo slots may be overwritten
//   k_update<STAGE>         computes U, q of its owned points AND stores the
//                           new q of every send point straight into the
//                           peers' halo slots (PeerPush: compute and transfer
//                           in one kernel)
//   k_peer_pushed           pushes += 1, data[me] = pushes at every peer this
//                           rank sends to (system-scope release)
//   stage 4                 k_peer_limbs: the exact residue limbs are
//                           written into every rank's gather row, then summed
//                           after the flags (an all-gather over peer memory;
//                           integer sums, so every rank holds the same total)
//                           -> k_close
//
// Each captured graph ends with k_peer_wait_data on the solver stream (no
// run returns with a peer's push into this rank still in flight); a
// continued run's seed waits for the peers to have read this rank's last
// push (k_peer_wait_read), pushes the refreshed q (k_peer_push_all) and
// publishes it (k_peer_pushed).
//
// The counters only grow and every rank runs the same sequence of stages,
// so "peer r has done as many pushes / band passes as I have" is the whole
// protocol.  Waits spin on system-scope acquire loads with a deadline
// (kPeerTimeoutNs): a peer that never arrives turns into a KMF_EPEER error
// on every rank instead of a hang.  The signalling kernels ignore the
// positivity / convergence skip (a failed rank keeps the protocol going so
// its peers finish the replay too).
#pragma once
#include "kmf_kernels.cuh"

namespace kmf {

constexpr unsigned long long kPeerTimeoutNs = 30ull * 1000000000ull;

struct PeerFlags {
    unsigned long long data[kMaxRanks];   // pushes peer r made into this rank's halo
    unsigned long long read[kMaxRanks];   // band passes peer r finished (done reading what this rank pushed)
    unsigned long long limb_seq[kMaxRanks];
    // peer r's residue limbs, by iteration parity: a rank writes parity p
    // again only after every rank signalled the iteration in between, which
    // each does after summing the rows of parity p
    unsigned long long gather[2][kMaxRanks][kLimbs];
    unsigned long long pushes, bands, iters;      // this rank's own counters
    unsigned long long failed;                    // a wait timed out: stop waiting
};

// the ranks of one partition as seen from rank `rank`
struct PeerSet {
    PeerFlags *me;
    PeerFlags *peer[kMaxRanks];  // every other rank (the limb all-gather spans all ranks)
    unsigned send_mask, recv_mask;
    int rank, nranks;
    unsigned long long timeout_ns;  // deadline of one wait (kPeerTimeoutNs; KMF_PEER_TIMEOUT_S overrides)
};

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long *p)
{
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_sys(unsigned long long *p, unsigned long long v)
{
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_volatile(const unsigned long long *p)
{
    return *(volatile const unsigned long long *)p;
}
__device__ __forceinline__ unsigned long long global_ns()
{
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// wait until flag[r] >= target for every rank r in mask (one thread)
__device__ bool peer_wait(PeerSet &ps, unsigned long long *flags, unsigned mask, unsigned long long target, Ctrl *c)
{
    const unsigned long long t0 = global_ns();
    for (int r = 0; r < ps.nranks; r++) {
        if (!((mask >> r) & 1u)) continue;
        while (ld_acquire_sys(&flags[r]) < target) {
            if (ld_volatile(&ps.me->failed) || global_ns() - t0 > ps.timeout_ns) {
                ps.me->failed = 1ull;
                c->peer_fail = 1ull;
                return false;
            }
            __nanosleep(64);
        }
    }
    return true;
}

// DATA: the halo of the last update has landed from every peer this rank
// receives from
__global__ void k_peer_wait_data(PeerSet ps, Ctrl *c)
{
    if (threadIdx.x == 0) peer_wait(ps, ps.me->data, ps.recv_mask, ld_volatile(&ps.me->pushes), c);
}

// a continued run's seed: the peers this rank pushes into have finished
// reading its last push (their band passes caught up with this rank's)
__global__ void k_peer_wait_read(PeerSet ps, Ctrl *c)
{
    if (threadIdx.x == 0) peer_wait(ps, ps.me->read, ps.send_mask, ld_volatile(&ps.me->bands), c);
}

// this rank's band pass is over: tell the peers that push into it, then wait
// for the peers it pushes into
__global__ void k_peer_band_done(PeerSet ps, Ctrl *c)
{
    if (threadIdx.x != 0) return;
    const unsigned long long b = ps.me->bands + 1;
    ps.me->bands = b;
    for (int r = 0; r < ps.nranks; r++)
        if ((ps.recv_mask >> r) & 1u) st_release_sys(&ps.peer[r]->read[ps.rank], b);
    peer_wait(ps, ps.me->read, ps.send_mask, b, c);
}

// the update's pushes are complete (stream order + each pushing thread's
// system fence): publish them
__global__ void k_peer_pushed(PeerSet ps)
{
    if (threadIdx.x != 0) return;
    const unsigned long long p = ps.me->pushes + 1;
    ps.me->pushes = p;
    __threadfence_system();
    for (int r = 0; r < ps.nranks; r++)
        if ((ps.send_mask >> r) & 1u) st_release_sys(&ps.peer[r]->data[ps.rank], p);
}

// push q of every send point (a continued run's seed, after k_refresh)
__global__ void k_peer_push_all(int n_owned, PeerPush pp, const double *__restrict__ q)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_owned) return;
    const int b = pp.ptr[i], e = pp.ptr[i + 1];
    if (b == e) return;
    const Q4 v = qload(q, i);
    for (int t = b; t < e; t++) {
        const unsigned d = pp.dst[t];
        reinterpret_cast<Q4 *>(pp.q[d >> kPeerSlotBits])[d & ((1u << kPeerSlotBits) - 1)] = v;
    }
    __threadfence_system();
}

// exact residue across ranks: all-gather of the limb rows over peer memory,
// then every rank sums the same rows (integer adds: order-free) into its
// Ctrl limbs for k_close
__global__ void k_peer_limbs(PeerSet ps, Ctrl *c)
{
    __shared__ unsigned long long it;
    __shared__ int ok;
    if (threadIdx.x == 0) it = ps.me->iters + 1;
    __syncthreads();
    for (int r = 0; r < ps.nranks; r++) {
        if (r == ps.rank) continue;
        for (int t = threadIdx.x; t < kLimbs; t += blockDim.x) ps.peer[r]->gather[it & 1][ps.rank][t] = c->limbs[t];
    }
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0) {
        ps.me->iters = it;
        for (int r = 0; r < ps.nranks; r++)
            if (r != ps.rank) st_release_sys(&ps.peer[r]->limb_seq[ps.rank], it);
        const unsigned all = ((ps.nranks >= 32) ? ~0u : ((1u << ps.nranks) - 1u)) & ~(1u << ps.rank);
        ok = peer_wait(ps, ps.me->limb_seq, all, it, c);
    }
    __syncthreads();
    if (!ok) return;
    for (int t = threadIdx.x; t < kLimbs; t += blockDim.x) {
        unsigned long long s = c->limbs[t];
        for (int r = 0; r < ps.nranks; r++)
            if (r != ps.rank) s += ld_volatile(&ps.me->gather[it & 1][r][t]);
        c->limbs[t] = s;
    }
}

}  // namespace kmf
