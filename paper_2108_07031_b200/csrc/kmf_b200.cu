// kmf_b200.cu -- context, CUDA-graph outer loop and C ABI (include/kmf_b200.h).
//
// Build: paper_2108_07031_b200/csrc/Makefile (nvcc -gencode
// arch=compute_100a,code=sm_100a -O3 -lineinfo -fmad=false).
#include "../../include/kmf_b200.h"
#include "kmf_kernels.cuh"
#include "kmf_flux.cuh"
#include "kmf_peer.cuh"

#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>  // types only: the library dlopens libnccl at run time

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>



using namespace kmf;

namespace {

thread_local std::string g_last_error;

void set_msg(const char *fmt, ...)
{
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_last_error = buf;
}

#define CK(expr)                                                                                  \
    do {                                                                                          \
        cudaError_t e_ = (expr);                                                                  \
        if (e_ != cudaSuccess) {                                                                  \
            set_msg("%s:%d %s: %s", __FILE__, __LINE__, #expr, cudaGetErrorString(e_));           \
            return KMF_ECUDA;                                                                     \
        }                                                                                         \
    } while (0)

inline int nblk(long long n, int tb = kTB) { return (int)((n + tb - 1) / tb); }

template <typename T>
struct DBuf {
    T *p = nullptr;
    size_t n = 0;
    ~DBuf() { release(); }
    void release()
    {
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
    }
    cudaError_t alloc(size_t count)
    {
        release();
        n = count;
        if (!count) return cudaSuccess;
        return cudaMalloc((void **)&p, sizeof(T) * count);
    }
    cudaError_t upload(const T *h, size_t count)
    {
        cudaError_t e = alloc(count);
        if (e != cudaSuccess || !count) return e;
        return cudaMemcpy(p, h, sizeof(T) * count, cudaMemcpyHostToDevice);
    }
};

struct GraphKey {
    double gamma, cfl, fs[4], tol;
    int n_inner, mode, unroll, how;
    bool operator==(const GraphKey &o) const { return std::memcmp(this, &o, sizeof o) == 0; }
};

// Timed launch groups inside a captured iteration graph: external event
// record nodes around each group, read back after the replay.
enum {
    KC_QGRAD = 0,   // instrument: q_derivatives (first order + sweeps)
    KC_FLUXBND,     // instrument: flux_residual (interior flux + boundary closure)
    KC_UPDATE,      // instrument: state_update (+ fused q_variables, timestep, residue)
    KC_FLUX,        // bench: interior flux kernel launches
    KC_FO,          // bench: first-order q-gradient launches
    KC_SWEEP,       // bench: Jacobi sweep launches
    KC_N
};

struct EvPair {
    int cls;
    cudaEvent_t a, b;
};

// One instantiated iteration graph (`unroll` outer iterations) and the
// event pairs captured into it.
struct Graph {
    cudaGraphExec_t exec = nullptr;
    GraphKey key{};
    std::vector<EvPair> ev;
    int launches = 0;  // kernels of this library per captured iteration
    void reset()
    {
        if (exec) cudaGraphExecDestroy(exec);
        exec = nullptr;
        for (auto &e : ev) {
            cudaEventDestroy(e.a);
            cudaEventDestroy(e.b);
        }
        ev.clear();
    }
    ~Graph() { reset(); }
};

}  // namespace

struct kmf_ctx {
    int device = 0;
    int n = 0, ld = 0;
    bool xy = true;  // offsets recomputed from coordinates
    int qg_nc = 2;   // q-gradient components per thread (4 above 100K points)
    bool has_perm = false;
    // solver, boundary branch, halo exchange, band pass (partitions)
    cudaStream_t s0 = nullptr, s1 = nullptr, s2 = nullptr, s3 = nullptr;
    // kmf_run_cases: upload / download streams and their buffer events
    // (per half of the double-buffered P0 / stage_buf)
    cudaStream_t sh = nullptr, sd = nullptr;
    cudaEvent_t cs_up[2] = {}, cs_free[2] = {}, cs_got[2] = {}, cs_down[2] = {};
    cudaEvent_t fork = nullptr, join = nullptr, xfork = nullptr, xjoin = nullptr;
    // band pass: stage start on s0 / halo unpacked (group runner) / done
    cudaEvent_t bfork = nullptr, bready = nullptr, bjoin = nullptr;
    static constexpr int kMaxEv = 10;
    cudaEvent_t lev[kMaxEv] = {};                  // interior pass: level k written

    // geometry
    DBuf<double> x, y, pxy, dmin, fsum, fcoef, edx, edy;
    DBuf<unsigned char> flag;
    DBuf<int> eoff, deg, eidx;
    DBuf<long long> perm, cptr;
    long long n_edges = 0;
    // boundary
    int nb = 0, nb_wall = 0;
    DBuf<int> bpoint, bptr[3], bidx[3];
    DBuf<unsigned char> btype;
    DBuf<double> bframe, bcoef, bdt[3], bdn[3];
    long long bedges[3] = {0, 0, 0};

    // state
    DBuf<double> Uo, Us, q, GA, GB, R, dt, stage_buf, stage_buf2;
    DBuf<Ctrl> ctrl;
    DBuf<double> history;
    DBuf<unsigned char> diag;
    DBuf<double> P0;  // initial primitives (caller order) pending the next run
    bool have_state = false, pending_init = false;
    double state_gamma = 1.4;

    // graphs: 1 iteration, 8 iterations, bench (1 iteration with kernel events)
    Graph g1, gU, gB;
    std::vector<EvPair> *cap_ev = nullptr;  // event list of the graph being captured
    int nlaunch = 0;                        // kernel launches enqueued (counted while capturing)
    int cap_how = 0;

    // instrumentation
    double stage_sec[6] = {0, 0, 0, 0, 0, 0};
    cudaEvent_t evs[2] = {};  // bench: around one step
    DBuf<unsigned char> flush;

    // last error
    kmf_error_info err{};
    std::vector<long long> err_idx;
    const double *G_last = nullptr;  // final gradients of the last stage enqueued (diagnostics)

    // partition (multi-GPU, partition.py): owned points first, ordered by
    // depth (hop distance to the nearest halo slot, deepest first), then the
    // halo layers 1..depth
    bool dist_on = false;
    int n_owned = 0, rank = 0, nranks = 1, depth = 0;
    long long n_global = 0;
    std::vector<int> layer_end;     // [k]: n_owned + |L1..Lk|, k = 0..depth
    std::vector<int> interior_end;  // [k]: owned slots at depth >= k, k = 0..depth+1
    std::vector<int> peer_rank;
    std::vector<long long> send_off, send_cnt, recv_off, recv_cnt;  // points, per peer
    long long send_total = 0, recv_total = 0;
    DBuf<int> ps_slot, ps_base, ps_stride, pr_slot, pr_base, pr_stride;
    DBuf<double> sendbuf, recvbuf;
    // one gradient buffer per level (first order, sweep 1..): the band pass
    // reads lower levels at slots the interior pass already advanced, so the
    // single-domain ping-pong (GA, GB) would have been overwritten
    static constexpr int kMaxLevels = 8;
    static_assert(kMaxLevels < kMaxEv, "one interior-level event per gradient level");
    DBuf<double> Glev[kMaxLevels];
    void *nccl = nullptr;  // ncclComm_t when the NCCL transport is initialised
    void (*nccl_destroy)(void *) = nullptr;
    // peer transport (kmf_peer.cuh): flag block in this device's memory, the
    // peers' q / flag blocks mapped here, the push map of the update
    bool peer_on = false;
    bool peer_local = false;  // linked to contexts of this process: runs only through kmf_run_linked
    bool peer_broken = false; // a peer wait timed out: the counters no longer agree across ranks
    DBuf<PeerFlags> pflags;
    PeerSet pset{};
    PeerPush ppush{};
    DBuf<int> push_ptr;
    DBuf<unsigned> push_dst;
    std::vector<void *> ipc_opened;             // cudaIpcOpenMemHandle mappings (closed at teardown)
    std::vector<int> send_slot_h, recv_slot_h;  // host copies of the partition's lists
    bool transport() const { return nccl != nullptr || peer_on; }

    DG dg() const
    {
        DG g;
        g.n = n;
        g.ld = ld;
        g.n_norm = dist_on ? (int)n_global : n;
        g.x = x.p;
        g.y = y.p;
        g.pxy = reinterpret_cast<const double2 *>(pxy.p);
        g.flag = flag.p;
        g.dmin = dmin.p;
        g.eoff = eoff.p;
        g.deg = deg.p;
        g.eidx = eidx.p;
        g.edx = edx.p;
        g.edy = edy.p;
        g.fsum = fsum.p;
        g.fcoef = fcoef.p;
        g.cptr = cptr.p;
        return g;
    }
    DB db() const
    {
        DB b;
        b.nb = nb;
        b.point = bpoint.p;
        b.type = btype.p;
        b.frame = bframe.p;
        b.coef = bcoef.p;
        for (int f = 0; f < 3; f++) {
            b.ptr[f] = bptr[f].p;
            b.idx[f] = bidx[f].p;
            b.dt[f] = bdt[f].p;
            b.dn[f] = bdn[f].p;
        }
        return b;
    }
    int n_act() const { return dist_on ? n_owned : n; }
    // gradient buffer of level k (0 first order, s = sweep s)
    double *gbuf(int k) { return dist_on ? Glev[k].p : ((k & 1) ? GB.p : GA.p); }
    void drop_graphs()
    {
        g1.reset();
        gU.reset();
        gB.reset();
    }
    ~kmf_ctx()
    {
        drop_graphs();  // the graphs hold NCCL kernel nodes: before the communicator goes
        if (nccl && nccl_destroy) nccl_destroy(nccl);
        for (void *m : ipc_opened) cudaIpcCloseMemHandle(m);
        for (auto &e : evs)
            if (e) cudaEventDestroy(e);
        for (cudaEvent_t e : {fork, join, xfork, xjoin, bfork, bready, bjoin})
            if (e) cudaEventDestroy(e);
        for (cudaEvent_t e : lev)
            if (e) cudaEventDestroy(e);
        for (cudaEvent_t *arr : {cs_up, cs_free, cs_got, cs_down})
            for (int b = 0; b < 2; b++)
                if (arr[b]) cudaEventDestroy(arr[b]);
        for (cudaStream_t s : {s0, s1, s2, s3, sh, sd})
            if (s) cudaStreamDestroy(s);
    }
};

namespace {

// ------------------------------------------------------------------ create

int build_context(kmf_ctx *c, const kmf_geometry *g)
{
    const long long n = g->n;
    if (n <= 0 || n > (1ll << 30)) {
        set_msg("kmf_create: bad point count %lld", n);
        return KMF_EINVAL;
    }
    const kmf_stencil &F = g->full;
    if (F.n_owners != n || !F.ptr || !F.idx || !F.sxx || !F.sxy || !F.syy || !F.det) {
        set_msg("kmf_create: full stencil missing or owner count mismatch");
        return KMF_EINVAL;
    }
    const long long E = F.ptr[n];
    if (E != F.n_edges || E >= (1ll << 31)) {
        set_msg("kmf_create: edge count mismatch (%lld vs %lld)", E, (long long)F.n_edges);
        return KMF_EINVAL;
    }
    c->n = (int)n;
    c->ld = (int)((n + 31) / 32 * 32);
    c->n_edges = E;
    const int ld = c->ld;

    // permutation: slot k holds caller point perm[k]
    std::vector<long long> perm(n), inv(n);
    c->has_perm = g->perm != nullptr;
    for (long long k = 0; k < n; k++) perm[k] = c->has_perm ? g->perm[k] : k;
    {
        std::vector<char> seen(n, 0);
        for (long long k = 0; k < n; k++) {
            long long p = perm[k];
            if (p < 0 || p >= n || seen[p]) {
                set_msg("kmf_create: perm is not a permutation of 0..n-1");
                return KMF_EINVAL;
            }
            seen[p] = 1;
            inv[p] = k;
        }
    }

    // offsets derivable from coordinates? (geometry.py:382-383)
    bool xy = g->x && g->y;
    if (xy && F.dx && F.dy) {
        for (long long i = 0; i < n && xy; i++)
            for (long long e = F.ptr[i]; e < F.ptr[i + 1]; e++) {
                long long j = F.idx[e];
                if (j < 0 || j >= n) {
                    set_msg("kmf_create: neighbour index %lld out of range", j);
                    return KMF_EINVAL;
                }
                double dx = g->x[j] - g->x[i], dy = g->y[j] - g->y[i];
                if (std::memcmp(&dx, &F.dx[e], 8) || std::memcmp(&dy, &F.dy[e], 8)) {
                    xy = false;
                    break;
                }
            }
    } else if (!F.dx || !F.dy) {
        if (!xy) {
            set_msg("kmf_create: need either x/y or full.dx/dy");
            return KMF_EINVAL;
        }
    }
    c->xy = xy;

    auto pad = [&](const double *src, double fill) {
        std::vector<double> v(ld, fill);
        for (long long k = 0; k < n; k++) v[k] = src ? src[perm[k]] : fill;
        return v;
    };
    std::vector<double> hx = pad(g->x, 0.0), hy = pad(g->y, 0.0), hd = pad(g->d_min, 1.0);
    CK(c->x.upload(hx.data(), ld));
    CK(c->y.upload(hy.data(), ld));
    {
        std::vector<double> hxy(2 * (size_t)ld);
        for (long long k = 0; k < ld; k++) hxy[2 * k] = hx[k], hxy[2 * k + 1] = hy[k];
        CK(c->pxy.upload(hxy.data(), hxy.size()));
    }
    CK(c->dmin.upload(hd.data(), ld));
    {
        std::vector<unsigned char> fl(ld, 0);
        for (long long k = 0; k < n; k++) fl[k] = (unsigned char)g->flag[perm[k]];
        CK(c->flag.upload(fl.data(), ld));
    }
    // full-stencil sums [4][ld]
    {
        std::vector<double> fs(4 * (size_t)ld, 0.0);
        for (long long k = 0; k < n; k++) {
            long long p = perm[k];
            fs[k] = F.sxx[p];
            fs[ld + k] = F.sxy[p];
            fs[2 * ld + k] = F.syy[p];
            fs[3 * ld + k] = F.det[p];
        }
        for (long long k = n; k < ld; k++) fs[3 * ld + k] = 1.0;
        CK(c->fsum.upload(fs.data(), fs.size()));
    }
    // split-family weight coefficients [8][ld]: x-family w = (syy dx - sxy dy)/det,
    // y-family w = (sxx dy - sxy dx)/det  (solver.py:192-195, det = det_safe)
    {
        std::vector<double> cf(8 * (size_t)ld, 0.0);
        for (int f = 0; f < 4; f++) {
            if (!g->split_sxx[f] || !g->split_sxy[f] || !g->split_syy[f] || !g->det_safe[f]) {
                set_msg("kmf_create: split family %d sums missing", f);
                return KMF_EINVAL;
            }
        }
        for (long long k = 0; k < n; k++) {
            long long p = perm[k];
            for (int f = 0; f < 4; f++) {
                double det = g->det_safe[f][p];
                double sxx = g->split_sxx[f][p], sxy = g->split_sxy[f][p], syy = g->split_syy[f][p];
                double cx, cy;
                if (f < 2) {
                    cx = syy / det;
                    cy = -sxy / det;
                } else {
                    cx = -sxy / det;
                    cy = sxx / det;
                }
                cf[(2 * f) * (size_t)ld + k] = cx;
                cf[(2 * f + 1) * (size_t)ld + k] = cy;
            }
        }
        CK(c->fcoef.upload(cf.data(), cf.size()));
    }
    // sliced ELL of the full stencil, slots in caller CSR order
    {
        const long long ns = (n + 31) / 32;
        std::vector<int> off(ns + 1, 0), dg(ld, 0);
        long long total = 0;
        for (long long s = 0; s < ns; s++) {
            int w = 0;
            for (long long k = s * 32; k < std::min(n, s * 32 + 32); k++) {
                long long p = perm[k];
                int d = (int)(F.ptr[p + 1] - F.ptr[p]);
                dg[k] = d;
                w = std::max(w, d);
            }
            if (total > (1ll << 31) - 1) {
                set_msg("kmf_create: ELL too large");
                return KMF_EINVAL;
            }
            off[s] = (int)total;
            total += (long long)w * 32;
        }
        off[ns] = (int)total;
        std::vector<int> ei(total > 0 ? total : 1, 0);
        std::vector<double> ex, ey;
        if (!xy) {
            ex.assign(ei.size(), 0.0);
            ey.assign(ei.size(), 0.0);
        }
        std::vector<long long> cp(ld, 0);
        for (long long k = 0; k < n; k++) {
            long long p = perm[k];
            long long base = off[k / 32] + (k % 32);
            cp[k] = F.ptr[p];
            for (long long e = F.ptr[p], s = 0; e < F.ptr[p + 1]; e++, s++) {
                ei[base + s * 32] = (int)inv[F.idx[e]];
                if (!xy) {
                    ex[base + s * 32] = F.dx[e];
                    ey[base + s * 32] = F.dy[e];
                }
            }
            // padding slots point at the owner itself (never read: s < deg)
            for (long long s = F.ptr[p + 1] - F.ptr[p]; s < (off[k / 32 + 1] - off[k / 32]) / 32; s++)
                ei[base + s * 32] = (int)k;
        }
        CK(c->eoff.upload(off.data(), off.size()));
        CK(c->deg.upload(dg.data(), dg.size()));
        CK(c->eidx.upload(ei.data(), ei.size()));
        CK(c->cptr.upload(cp.data(), cp.size()));
        if (!xy) {
            CK(c->edx.upload(ex.data(), ex.size()));
            CK(c->edy.upload(ey.data(), ey.size()));
        }
    }
    if (c->has_perm) CK(c->perm.upload(perm.data(), n));

    // boundary table: wall entries then outer entries
    {
        std::vector<const kmf_frame *> frames;
        if (g->has_wall) frames.push_back(&g->wall);
        if (g->has_outer) frames.push_back(&g->outer);
        int nb = 0;
        for (auto *fr : frames) nb += (int)fr->b;
        c->nb = nb;
        c->nb_wall = g->has_wall ? (int)g->wall.b : 0;
        std::vector<int> bp(std::max(nb, 1)), bpt[3];
        std::vector<unsigned char> bt(std::max(nb, 1));
        std::vector<double> bfr(4 * (size_t)std::max(nb, 1)), bco(6 * (size_t)std::max(nb, 1));
        std::vector<int> bi[3];
        std::vector<double> bd[3], bn[3];
        for (int f = 0; f < 3; f++) bpt[f].push_back(0);
        int row = 0;
        for (size_t fi = 0; fi < frames.size(); fi++) {
            const kmf_frame *fr = frames[fi];
            const bool is_wall = g->has_wall && fi == 0;
            const kmf_stencil *fam[3] = {&fr->tplus, &fr->tminus, &fr->normal};
            for (int f = 0; f < 3; f++) {
                if (fam[f]->n_owners != fr->b || !fam[f]->ptr) {
                    set_msg("kmf_create: frame family %d owner mismatch", f);
                    return KMF_EINVAL;
                }
            }
            for (long long l = 0; l < fr->b; l++, row++) {
                long long gp = fr->points[l];
                if (gp < 0 || gp >= n) {
                    set_msg("kmf_create: frame point out of range");
                    return KMF_EINVAL;
                }
                bp[row] = (int)inv[gp];
                bt[row] = is_wall ? 1 : 2;
                bfr[row] = fr->tx[l];
                bfr[(size_t)nb + row] = fr->ty[l];
                bfr[2 * (size_t)nb + row] = fr->nx[l];
                bfr[3 * (size_t)nb + row] = fr->ny[l];
                for (int f = 0; f < 3; f++) {
                    const kmf_stencil *s = fam[f];
                    double det = s->det[l];
                    double ct, cn;
                    if (f < 2) {  // d/dt row: (syy st - sxy sn)/det
                        ct = s->syy[l] / det;
                        cn = -s->sxy[l] / det;
                    } else {  // d/dn row: (sxx sn - sxy st)/det
                        ct = -s->sxy[l] / det;
                        cn = s->sxx[l] / det;
                    }
                    bco[(2 * f) * (size_t)nb + row] = ct;
                    bco[(2 * f + 1) * (size_t)nb + row] = cn;
                    for (long long e = s->ptr[l]; e < s->ptr[l + 1]; e++) {
                        bi[f].push_back((int)inv[s->idx[e]]);
                        bd[f].push_back(s->dx[e]);
                        bn[f].push_back(s->dy[e]);
                    }
                    bpt[f].push_back((int)bi[f].size());
                }
            }
        }
        if (nb > 0) {
            CK(c->bpoint.upload(bp.data(), nb));
            CK(c->btype.upload(bt.data(), nb));
            CK(c->bframe.upload(bfr.data(), 4 * (size_t)nb));
            CK(c->bcoef.upload(bco.data(), 6 * (size_t)nb));
            for (int f = 0; f < 3; f++) {
                c->bedges[f] = (long long)bi[f].size();
                if (bi[f].empty()) {
                    bi[f].push_back(0);
                    bd[f].push_back(0);
                    bn[f].push_back(0);
                }
                CK(c->bptr[f].upload(bpt[f].data(), bpt[f].size()));
                CK(c->bidx[f].upload(bi[f].data(), bi[f].size()));
                CK(c->bdt[f].upload(bd[f].data(), bd[f].size()));
                CK(c->bdn[f].upload(bn[f].data(), bn[f].size()));
            }
        }
    }

    // state buffers
    CK(c->Uo.alloc(4 * (size_t)ld));
    CK(c->Us.alloc(4 * (size_t)ld));
    CK(c->q.alloc(4 * (size_t)ld));
    CK(c->GA.alloc(8 * (size_t)ld));
    CK(c->GB.alloc(8 * (size_t)ld));
    CK(c->R.alloc(4 * (size_t)ld));
    CK(c->dt.alloc(ld));
    CK(c->stage_buf.alloc(8 * (size_t)n));
    CK(c->stage_buf2.alloc(8 * (size_t)n));
    CK(c->ctrl.alloc(1));
    CK(cudaMemset(c->ctrl.p, 0, sizeof(Ctrl)));
    CK(cudaMemset(c->R.p, 0, sizeof(double) * 4 * ld));
    CK(c->diag.alloc(std::max<long long>(E, std::max(std::max(c->bedges[0], c->bedges[1]), c->bedges[2])) + 1));
    for (cudaStream_t *s : {&c->s0, &c->s1, &c->s2, &c->s3, &c->sh, &c->sd})
        CK(cudaStreamCreateWithFlags(s, cudaStreamNonBlocking));
    for (cudaEvent_t *arr : {c->cs_up, c->cs_free, c->cs_got, c->cs_down})
        for (int b = 0; b < 2; b++) CK(cudaEventCreateWithFlags(&arr[b], cudaEventDisableTiming));
    for (cudaEvent_t &e : c->lev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    for (cudaEvent_t *e : {&c->fork, &c->join, &c->xfork, &c->xjoin, &c->bfork, &c->bready, &c->bjoin})
        CK(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
    for (auto &e : c->evs) CK(cudaEventCreate(&e));
    // one thread per point (all 4 components) from 160K points up: -6 %
    // q-gradient time at 160K / 2.5M / 10M against 2 threads per point;
    // small clouds keep 2 threads per point (more threads in flight)
    c->qg_nc = n > 100000 ? 4 : 2;
    return KMF_OK;
}


// ------------------------------------------------------------ stage launch

// Kernel `k` of a stage (0 first order, 1..n_inner the sweeps; the flux is
// k = n_inner + 1 in the second-order scheme and k = 0 in the first-order
// one, where it reads q only) over the slots of one pass.  Single domain:
// one pass over every slot.  Partition: kernel k at
// slot i reads data produced k+1 hops away, so it runs in the INTERIOR pass
// -- before this stage's halo exchange has arrived -- on the owned slots at
// depth >= k + 2 (a prefix: owned slots are ordered by depth), and in the
// BAND pass, after the exchange, on the rest of the slots where it is exact
// (owned slots for the flux, halo layers <= depth - 1 - k otherwise).
void stage_range(const kmf_ctx *c, int k, bool flux, bool band, int &lo, int &hi)
{
    if (!c->dist_on) {
        lo = 0;
        hi = band ? 0 : c->n;
        return;
    }
    const int cut = c->interior_end[std::min(k + 2, c->depth + 1)];
    const int end = flux ? c->n_owned : c->layer_end[std::max(0, c->depth - 1 - k)];
    lo = band ? cut : 0;
    hi = band ? std::max(cut, end) : cut;
}

// Event pair around a launch group while capturing a timed graph.
struct Mark {
    kmf_ctx *c;
    int cls;
    bool on;
    cudaStream_t st;
    cudaEvent_t a = nullptr;
    Mark(kmf_ctx *c_, int cls_, bool on_, cudaStream_t st_ = nullptr)
        : c(c_), cls(cls_), on(on_ && c_->cap_ev), st(st_ ? st_ : c_->s0)
    {
        if (!on) return;
        cudaEventCreate(&a);
        cudaEventRecordWithFlags(a, st, cudaEventRecordExternal);
    }
    ~Mark()
    {
        if (!on) return;
        cudaEvent_t b;
        cudaEventCreate(&b);
        cudaEventRecordWithFlags(b, st, cudaEventRecordExternal);
        c->cap_ev->push_back(EvPair{cls, a, b});
    }
};

enum { ITER_PLAIN = 0, ITER_INSTRUMENT = 1, ITER_BENCH = 2 };

template <bool XY, int NC>
void launch_fo_t(kmf_ctx *c, cudaStream_t s, int lo, int hi, double *G, Ctrl *ctl, int stage)
{
    if (hi <= lo) return;
    c->nlaunch++;
    k_first_order<XY, NC><<<nblk(hi - range_base(lo), qg_points_per_block<NC>()), kTB, 0, s>>>(
        c->dg(), lo, hi, (const double *)c->q.p, G, ctl, stage);
}

template <bool XY, int NC>
void launch_sw_t(kmf_ctx *c, cudaStream_t s, int lo, int hi, const double *Gin, double *Gout, Ctrl *ctl, int stage,
                 int slot, int want_res, bool outp)
{
    if (hi <= lo) return;
    c->nlaunch++;
    const int nb = nblk(hi - range_base(lo), qg_points_per_block<NC>());
    if (outp)
        k_sweep<XY, NC, true><<<nb, kTB, 0, s>>>(c->dg(), lo, hi, (const double *)c->q.p, Gin, Gout, ctl, stage, slot,
                                                 want_res);
    else
        k_sweep<XY, NC, false><<<nb, kTB, 0, s>>>(c->dg(), lo, hi, (const double *)c->q.p, Gin, Gout, ctl, stage,
                                                  slot, want_res);
}

// q-gradient launch shape: offsets from coordinates (XY) or stored in the
// ELL table; 4 or 2 components per thread
#define KMF_QG_DISPATCH(CALL, ...)                                  \
    do {                                                            \
        if (!c->xy)                                                 \
            CALL<false, 2>(__VA_ARGS__);                            \
        else if (c->qg_nc == 4)                                     \
            CALL<true, 4>(__VA_ARGS__);                             \
        else                                                        \
            CALL<true, 2>(__VA_ARGS__);                             \
    } while (0)

void launch_first_order(kmf_ctx *c, cudaStream_t s, int lo, int hi, double *G, Ctrl *ctl, int stage)
{
    KMF_QG_DISPATCH(launch_fo_t, c, s, lo, hi, G, ctl, stage);
}

// outp: write the plane gradient layout the flux / boundary kernels read
// (the last sweep of a stage)
void launch_sweep(kmf_ctx *c, cudaStream_t s, int lo, int hi, const double *Gin, double *Gout, Ctrl *ctl, int stage,
                  int slot, int want_res, bool outp)
{
    KMF_QG_DISPATCH(launch_sw_t, c, s, lo, hi, Gin, Gout, ctl, stage, slot, want_res, outp);
}

// q-derivatives of one stage over one pass: level 0 (first order), then
// the n_inner sweeps, level k reading level k-1; returns the final level.
// Partitions: the interior pass records lev[k] after writing level k; the
// band pass (its own stream) waits for lev[k-1] before level k, since a band
// slot reads level k-1 at interior neighbours.
double *launch_qgrad(kmf_ctx *c, cudaStream_t s, int stage, int n_inner, Ctrl *ctl, bool band, bool timed)
{
    const bool ev = c->dist_on;  // n_inner + 2 <= depth <= kMaxLevels < kMaxEv (check_params)
    int lo, hi;
    {
        Mark m(c, KC_FO, timed, s);
        stage_range(c, 0, false, band, lo, hi);
        launch_first_order(c, s, lo, hi, c->gbuf(0), ctl, stage);
        if (ev && !band) cudaEventRecord(c->lev[0], s);
    }
    Mark m(c, KC_SWEEP, timed, s);
    for (int it = 0; it < n_inner; it++) {
        if (ev && band) cudaStreamWaitEvent(s, c->lev[it], 0);
        stage_range(c, 1 + it, false, band, lo, hi);
        launch_sweep(c, s, lo, hi, c->gbuf(it), c->gbuf(it + 1), ctl, stage, 1 + it, 0, it + 1 == n_inner);
        if (ev && !band) cudaEventRecord(c->lev[it + 1], s);
    }
    return c->gbuf(n_inner);
}

// beta^(-1/(gamma-1)) evaluation of the decode (kmf_flux.cuh fdecode):
// 1 for gamma = 7/5, 2 for gamma = 5/3, 0 otherwise (log/exp)
inline int gamma_kind(double gamma)
{
    if (gamma == 1.4) return 1;
    if (gamma == 5.0 / 3.0) return 2;
    return 0;
}

template <bool XY, int GK>
void launch_flux_t(kmf_ctx *c, cudaStream_t s, int lo, int hi, const double *G, int mode, double gamma, int zero_bnd,
                   Ctrl *ctl, int stage)
{
    if (hi <= lo) return;
    DG g = c->dg();
    const double inv_gm1 = 1.0 / (gamma - 1.0), c_i0 = (2.0 - gamma) / (gamma - 1.0);
    double *R = c->R.p;
    const double *q = c->q.p;
    const int nb = nblk(hi - range_base(lo));
    c->nlaunch += mode == 0 ? 1 : 4;
    if (mode == 0) {
        k_flux<XY, -1, GK><<<nb, kTB, 0, s>>>(g, lo, hi, q, G, R, inv_gm1, c_i0, zero_bnd, ctl, stage);
    } else {
        // split4 (the paper's "optimised" variant): one kernel per family,
        // R accumulated x+, x-, y+, y- (solver.py:218-229)
        k_flux<XY, 0, GK><<<nb, kTB, 0, s>>>(g, lo, hi, q, G, R, inv_gm1, c_i0, zero_bnd, ctl, stage);
        k_flux<XY, 1, GK><<<nb, kTB, 0, s>>>(g, lo, hi, q, G, R, inv_gm1, c_i0, zero_bnd, ctl, stage);
        k_flux<XY, 2, GK><<<nb, kTB, 0, s>>>(g, lo, hi, q, G, R, inv_gm1, c_i0, zero_bnd, ctl, stage);
        k_flux<XY, 3, GK><<<nb, kTB, 0, s>>>(g, lo, hi, q, G, R, inv_gm1, c_i0, zero_bnd, ctl, stage);
    }
}

void launch_flux(kmf_ctx *c, cudaStream_t s, int lo, int hi, const double *G, int mode, double gamma, int zero_bnd,
                 Ctrl *ctl, int stage)
{
    const int gk = gamma_kind(gamma);
#define KMF_FLUX_ARGS c, s, lo, hi, G, mode, gamma, zero_bnd, ctl, stage
    if (!c->xy) {
        if (gk == 1) launch_flux_t<false, 1>(KMF_FLUX_ARGS);
        else if (gk == 2) launch_flux_t<false, 2>(KMF_FLUX_ARGS);
        else launch_flux_t<false, 0>(KMF_FLUX_ARGS);
    } else {
        if (gk == 1) launch_flux_t<true, 1>(KMF_FLUX_ARGS);
        else if (gk == 2) launch_flux_t<true, 2>(KMF_FLUX_ARGS);
        else launch_flux_t<true, 0>(KMF_FLUX_ARGS);
    }
#undef KMF_FLUX_ARGS
}

void launch_boundary(kmf_ctx *c, cudaStream_t s, const double *G, const double fs[4], double gamma, Ctrl *ctl,
                     int stage)
{
    if (c->nb == 0) return;
    c->nlaunch++;
    const double inv_gm1 = 1.0 / (gamma - 1.0), c_i0 = (2.0 - gamma) / (gamma - 1.0);
    const int warps_per_block = kTB / 32;
    const int nbk = (c->nb + warps_per_block - 1) / warps_per_block;
#define KMF_BND(GK)                                                                                                \
    k_boundary<GK><<<nbk, kTB, 0, s>>>(c->dg(), c->db(), c->q.p, G, c->R.p, inv_gm1, c_i0, fs[0], fs[1], fs[2], \
                                       fs[3], ctl, stage)
    switch (gamma_kind(gamma)) {
    case 1: KMF_BND(1); break;
    case 2: KMF_BND(2); break;
    default: KMF_BND(0);
    }
#undef KMF_BND
}

void launch_update(kmf_ctx *c, cudaStream_t s, int stage, double gamma, double cfl, IterOut io)
{
    DG g = c->dg();
    const int hi = c->n_act(), nb = nblk(hi);
    Ctrl *ctl = c->ctrl.p;
    double *Uo = c->Uo.p, *Us = c->Us.p, *dt = c->dt.p, *q = c->q.p;
    const double *R = c->R.p;
    const PeerPush pp = c->peer_on ? c->ppush : PeerPush{};
    c->nlaunch++;
    switch (stage) {
    case 1: k_update<1><<<nb, kTB, 0, s>>>(g, 0, hi, Uo, Us, R, dt, q, gamma, cfl, ctl, io, pp); break;
    case 2: k_update<2><<<nb, kTB, 0, s>>>(g, 0, hi, Uo, Us, R, dt, q, gamma, cfl, ctl, io, pp); break;
    case 3: k_update<3><<<nb, kTB, 0, s>>>(g, 0, hi, Uo, Us, R, dt, q, gamma, cfl, ctl, io, pp); break;
    default: k_update<4><<<nb, kTB, 0, s>>>(g, 0, hi, Uo, Us, R, dt, q, gamma, cfl, ctl, io, pp); break;
    }
}

// ------------------------------------------------------------- NCCL (dlopen)
// The library does not link NCCL: the multi-process transport resolves it at
// run time (libnccl.so.2, torch's or the system's), so single-GPU use never
// needs it.
struct NcclApi {
    bool ok = false;
    ncclResult_t (*GetUniqueId)(ncclUniqueId *) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*CommAbort)(ncclComm_t) = nullptr;
    ncclResult_t (*Send)(const void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*AllReduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char *(*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi &nccl_api()
{
    static NcclApi api;
    static bool tried = false;
    if (tried) return api;
    tried = true;
    void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return api;
#define KMF_SYM(field, name) api.field = reinterpret_cast<decltype(api.field)>(dlsym(h, name))
    KMF_SYM(GetUniqueId, "ncclGetUniqueId");
    KMF_SYM(CommInitRank, "ncclCommInitRank");
    KMF_SYM(CommDestroy, "ncclCommDestroy");
    KMF_SYM(CommAbort, "ncclCommAbort");
    KMF_SYM(Send, "ncclSend");
    KMF_SYM(Recv, "ncclRecv");
    KMF_SYM(AllReduce, "ncclAllReduce");
    KMF_SYM(GroupStart, "ncclGroupStart");
    KMF_SYM(GroupEnd, "ncclGroupEnd");
    KMF_SYM(GetErrorString, "ncclGetErrorString");
#undef KMF_SYM
    api.ok = api.GetUniqueId && api.CommInitRank && api.Send && api.Recv && api.AllReduce && api.GroupStart &&
             api.GroupEnd;
    return api;
}

// halo pack on the owner side: q of the points each peer needs
void enqueue_pack(kmf_ctx *c, cudaStream_t s)
{
    if (c->send_total && ++c->nlaunch)
        k_halo_pack<<<nblk(c->send_total), kTB, 0, s>>>((int)c->send_total, c->ps_slot.p, c->ps_base.p,
                                                        c->ps_stride.p, c->q.p, c->ld, c->sendbuf.p);
}

void enqueue_unpack(kmf_ctx *c, cudaStream_t s)
{
    if (c->recv_total && ++c->nlaunch)
        k_halo_unpack<<<nblk(c->recv_total), kTB, 0, s>>>((int)c->recv_total, c->pr_slot.p, c->pr_base.p,
                                                          c->pr_stride.p, c->recvbuf.p, c->q.p, c->ld);
}

// NCCL halo exchange on stream s: pack, one grouped send/recv per peer, unpack
ncclResult_t enqueue_exchange_nccl(kmf_ctx *c, cudaStream_t s)
{
    NcclApi &api = nccl_api();
    ncclComm_t comm = (ncclComm_t)c->nccl;
    enqueue_pack(c, s);
    api.GroupStart();
    for (size_t k = 0; k < c->peer_rank.size(); k++) {
        if (c->send_cnt[k])
            api.Send(c->sendbuf.p + 4 * c->send_off[k], 4 * c->send_cnt[k], ncclDouble, c->peer_rank[k], comm, s);
        if (c->recv_cnt[k])
            api.Recv(c->recvbuf.p + 4 * c->recv_off[k], 4 * c->recv_cnt[k], ncclDouble, c->peer_rank[k], comm, s);
    }
    ncclResult_t r = api.GroupEnd();
    enqueue_unpack(c, s);
    return r;
}

// ---------------------------------------------------------- one RK stage
// Per stage (solver.py:524-549) on s0:
//   interior pass: q-gradients, interior flux            (no halo data read)
//   band pass (partition, stream s3): after the halo q exchanged after the
//     previous update, level k once the interior pass wrote level k-1;
//     boundary closure, band flux
//   update (+ stage 4: residue limbs; partition: limb all-reduce, close)
//   [NCCL partition: fork the halo exchange of the new q onto s2; the next
//    stage's interior pass overlaps it]
// Single domain: the band pass is empty and the boundary branch runs beside
// the interior flux.  `xchg_pending` tracks a forked exchange inside the
// graph being captured (joined by the next stage's band pass or at the end
// of the capture).
struct StageCtx {
    const kmf_params *p;
    IterOut io;
    int how;
    bool xchg_pending;
};

void enqueue_head(kmf_ctx *c, StageCtx &sc, int stage, double *&G)
{
    const kmf_params *p = sc.p;
    Ctrl *ctl = c->ctrl.p;
    const bool inst = sc.how == ITER_INSTRUMENT, bench = sc.how == ITER_BENCH;
    if (c->dist_on) cudaEventRecord(c->bfork, c->s0);  // the band pass starts from here (enqueue_tail)
    {
        Mark m(c, KC_QGRAD, inst);
        if (p->n_inner > 0) {
            G = launch_qgrad(c, c->s0, stage, p->n_inner, ctl, false, bench);
        } else {  // n_inner = 0: the first-order scheme (qx = qy = 0 -> q~ = q bitwise)
            G = c->gbuf(0);
            cudaMemsetAsync(G, 0, sizeof(double) * 8 * (size_t)c->ld, c->s0);
        }
    }
    Mark m(c, KC_FLUXBND, inst);
    if (!c->dist_on) {
        cudaEventRecord(c->fork, c->s0);
        cudaStreamWaitEvent(c->s1, c->fork, 0);
        launch_boundary(c, c->s1, G, p->fs, p->gamma, ctl, stage);
        cudaEventRecord(c->join, c->s1);
    }
    int lo, hi;
    stage_range(c, p->n_inner > 0 ? p->n_inner + 1 : 0, true, false, lo, hi);
    Mark mf(c, KC_FLUX, bench);
    launch_flux(c, c->s0, lo, hi, G, p->mode, p->gamma, 0, ctl, stage);
}

void enqueue_tail(kmf_ctx *c, StageCtx &sc, int stage, const double *G)
{
    const kmf_params *p = sc.p;
    Ctrl *ctl = c->ctrl.p;
    const bool inst = sc.how == ITER_INSTRUMENT, bench = sc.how == ITER_BENCH;
    if (c->dist_on) {
        // band pass on s3, concurrent with the rest of the interior pass: it
        // needs the halo (the exchange joined, or the group runner's unpack
        // marked by bready) and, per level, the interior level below it
        cudaStream_t sb = c->s3;
        cudaStreamWaitEvent(sb, c->bfork, 0);  // the previous update
        if (sc.xchg_pending) {
            cudaStreamWaitEvent(sb, c->xjoin, 0);
            sc.xchg_pending = false;
        }
        if (c->peer_on) {  // the peers' pushes of the previous update have landed
            k_peer_wait_data<<<1, 32, 0, sb>>>(c->pset, ctl);
            c->nlaunch++;
        } else if (!c->nccl) {
            cudaStreamWaitEvent(sb, c->bready, 0);
        }
        if (p->n_inner > 0) {
            launch_qgrad(c, sb, stage, p->n_inner, ctl, true, false);
            // boundary and band flux read the final level at interior slots
            cudaStreamWaitEvent(sb, c->lev[p->n_inner], 0);
        } else {
            cudaEventRecord(c->fork, c->s0);  // the zeroed gradients
            cudaStreamWaitEvent(sb, c->fork, 0);
        }
        launch_boundary(c, sb, G, p->fs, p->gamma, ctl, stage);
        int lo, hi;
        stage_range(c, p->n_inner > 0 ? p->n_inner + 1 : 0, true, true, lo, hi);
        launch_flux(c, sb, lo, hi, G, p->mode, p->gamma, 0, ctl, stage);
        cudaEventRecord(c->bjoin, sb);
        Mark m(c, KC_FLUXBND, inst);
        cudaStreamWaitEvent(c->s0, c->bjoin, 0);
        if (c->peer_on) {  // halo read: release it to the pushing peers, wait for the ones this rank pushes into
            k_peer_band_done<<<1, 32, 0, c->s0>>>(c->pset, ctl);
            c->nlaunch++;
        }
    } else {
        Mark m(c, KC_FLUXBND, inst);
        cudaStreamWaitEvent(c->s0, c->join, 0);
    }
    c->G_last = G;
    Mark m(c, KC_UPDATE, inst);
    IterOut io = sc.io;
    // The stage-4 update closes the iteration itself (last block: residue,
    // history, counters) on small clouds, where one more launch would cost
    // more than the per-block fence; from 1M points a one-block k_close
    // after it is cheaper (the update runs fence-free: -0.7 ms at 40M).
    // Partitions close after the limb all-reduce (enqueue_after_update_nccl).
    const bool own_close = !c->dist_on && c->n >= (1 << 20);
    io.close_in_kernel = (c->dist_on || own_close) ? 0 : 1;
    launch_update(c, c->s0, stage, p->gamma, p->cfl, io);
    if (stage == 4 && own_close) {
        k_close<<<1, kTB, 0, c->s0>>>(c->ctrl.p, c->n, io);
        c->nlaunch++;
    }
    if (c->peer_on) {
        // publish the pushes fused into the update; at stage 4 the residue
        // limbs are all-gathered over peer memory, then the iteration closes
        k_peer_pushed<<<1, 32, 0, c->s0>>>(c->pset);
        c->nlaunch++;
        if (stage == 4) {
            k_peer_limbs<<<1, kTB, 0, c->s0>>>(c->pset, ctl);
            k_close<<<1, kTB, 0, c->s0>>>(ctl, (int)c->n_global, io);
            c->nlaunch += 2;
        }
    }
}

// NCCL partition: the iteration close after the stage-4 update (exact limb
// all-reduce, then k_close) and the halo exchange forked onto s2.
void enqueue_after_update_nccl(kmf_ctx *c, StageCtx &sc, int stage)
{
    NcclApi &api = nccl_api();
    if (stage == 4) {
        api.AllReduce(c->ctrl.p->limbs, c->ctrl.p->limbs, kLimbs, ncclUint64, ncclSum, (ncclComm_t)c->nccl, c->s0);
        k_close<<<1, kTB, 0, c->s0>>>(c->ctrl.p, (int)c->n_global, sc.io);
        c->nlaunch++;
    }
    cudaEventRecord(c->xfork, c->s0);
    cudaStreamWaitEvent(c->s2, c->xfork, 0);
    enqueue_exchange_nccl(c, c->s2);
    cudaEventRecord(c->xjoin, c->s2);
    sc.xchg_pending = true;
}

void enqueue_iteration(kmf_ctx *c, StageCtx &sc)
{
    const bool nccl = c->dist_on && c->nccl;
    for (int stage = 1; stage <= 4; stage++) {
        double *G = nullptr;
        enqueue_head(c, sc, stage, G);
        enqueue_tail(c, sc, stage, G);
        if (nccl) enqueue_after_update_nccl(c, sc, stage);
    }
}

int get_graph(kmf_ctx *c, const kmf_params *p, int unroll, Graph &gr, int how = ITER_PLAIN)
{
    GraphKey k;
    std::memset(&k, 0, sizeof k);
    k.gamma = p->gamma;
    k.cfl = p->cfl;
    for (int i = 0; i < 4; i++) k.fs[i] = p->fs[i];
    k.tol = p->convergence_tol;
    k.n_inner = p->n_inner;
    k.mode = p->mode;
    k.unroll = unroll;
    k.how = how;
    if (gr.exec && gr.key == k) return KMF_OK;
    if (gr.exec) CK(cudaStreamSynchronize(c->s0));  // a replay of the old graph may still be in flight
    gr.reset();
    cudaGraph_t graph;
    c->cap_ev = how == ITER_PLAIN ? nullptr : &gr.ev;
    StageCtx sc{p, IterOut{p->convergence_tol, 1}, how, false};
    c->nlaunch = 0;
    CK(cudaStreamBeginCapture(c->s0, cudaStreamCaptureModeThreadLocal));
    for (int u = 0; u < unroll; u++) enqueue_iteration(c, sc);
    if (sc.xchg_pending) cudaStreamWaitEvent(c->s0, c->xjoin, 0);  // join the last exchange
    if (c->peer_on) {  // ... and the peers' last pushes into this rank's halo
        k_peer_wait_data<<<1, 32, 0, c->s0>>>(c->pset, c->ctrl.p);
        c->nlaunch++;
    }
    cudaError_t ce = cudaStreamEndCapture(c->s0, &graph);
    c->cap_ev = nullptr;
    CK(ce);
    cudaError_t e = cudaGraphInstantiate(&gr.exec, graph, 0);
    cudaGraphDestroy(graph);
    CK(e);
    gr.key = k;
    gr.launches = c->nlaunch / unroll;
    return KMF_OK;
}

// per-class milliseconds of the last replay of a timed graph
int graph_times(const Graph &gr, double out[KC_N])
{
    for (int k = 0; k < KC_N; k++) out[k] = 0.0;
    for (const EvPair &e : gr.ev) {
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, e.a, e.b));
        out[e.cls] += ms;
    }
    return KMF_OK;
}

void record_error(kmf_ctx *c, int code, int iteration, int stage, int context, long long count, const char *msg)
{
    if (!c) return;
    c->err.code = code;
    c->err.iteration = iteration;
    c->err.stage = stage;
    c->err.context = context;
    c->err.count = count;
    c->err.n_indices = (long long)c->err_idx.size();
    std::snprintf(c->err.message, sizeof c->err.message, "%s", msg);
}

// first raise site of a failing stage in reference order: interior flux
// (solver.py:540) < boundary (:541) < decode (:547)
int first_context(unsigned mask)
{
    const int order[] = {KMF_CTX_FLUX_XP, KMF_CTX_WALL_TANGENT, KMF_CTX_WALL_NORMAL, KMF_CTX_OUTER_TANGENT,
                         KMF_CTX_OUTER_NORMAL, KMF_CTX_C2P_DENSITY, KMF_CTX_C2P_PRESSURE};
    for (int o : order)
        if (mask & (1u << o)) return o;
    return 0;
}

int check_params(const kmf_ctx *c, const kmf_params *p)
{
    if (p->n_inner < 0 || !(p->gamma > 1.0 && p->gamma < 2.0) || !(p->cfl > 0.0 && p->cfl <= 1.0) ||
        (p->mode != 0 && p->mode != 1)) {
        set_msg("kmf_run: invalid parameters");
        return KMF_EINVAL;
    }
    if (c->dist_on && p->n_inner + 2 > c->depth) {
        set_msg("kmf_run: n_inner %d needs a halo of depth %d, the partition has %d", p->n_inner, p->n_inner + 2,
                c->depth);
        return KMF_EINVAL;
    }
    return KMF_OK;
}

// U, q, dt of the first iteration (solver.py:502-506, :520) from the pending
// initial primitives (every local slot, halo included), or q, dt refreshed
// from U when continuing -- then, under a partition, the halo q refreshed
// from its owners (halo slots are never updated locally).
int seed_state(kmf_ctx *c, double gamma, double cfl)
{
    DG g = c->dg();
    if (c->pending_init) {
        k_init<<<nblk(c->n), kTB, 0, c->s0>>>(g, c->P0.p, c->has_perm ? c->perm.p : nullptr, c->Uo.p, c->q.p,
                                              c->dt.p, gamma, cfl);
        c->pending_init = false;
    } else {
        k_refresh<<<nblk(c->n_act()), kTB, 0, c->s0>>>(g, c->n_act(), c->Uo.p, c->q.p, c->dt.p, gamma, cfl);
        if (c->dist_on && c->peer_on) {
            // continued run: once the peers finished reading what this rank
            // pushed last, push the refreshed q of the send points
            k_peer_wait_read<<<1, 32, 0, c->s0>>>(c->pset, c->ctrl.p);
            if (c->n_owned) k_peer_push_all<<<nblk(c->n_owned), kTB, 0, c->s0>>>(c->n_owned, c->ppush, c->q.p);
            k_peer_pushed<<<1, 32, 0, c->s0>>>(c->pset);
        } else if (c->dist_on && c->nccl) {
            if (enqueue_exchange_nccl(c, c->s0) != ncclSuccess) {
                set_msg("seed_state: NCCL halo exchange failed");
                return KMF_ENCCL;
            }
        }
    }
    CK(cudaGetLastError());
    c->state_gamma = gamma;
    return KMF_OK;
}

// `count` outer iterations on s0: graphs of U iterations (U = 8, then 1 for
// the rest).  ITER_INSTRUMENT replays are read after each replay (event
// nodes around each stage's launch groups) into stage_sec.
int replay(kmf_ctx *c, const kmf_params *p, int count, int how)
{
    const int U = 8;
    int full = count / U, rest = count % U;
    for (int pass = 0; pass < 2; pass++) {
        const int reps = pass ? rest : full, unroll = pass ? 1 : U;
        if (!reps) continue;
        Graph &gr = pass ? c->g1 : c->gU;
        if (int rc = get_graph(c, p, unroll, gr, how)) return rc;
        for (int k = 0; k < reps; k++) {
            CK(cudaGraphLaunch(gr.exec, c->s0));
            if (how == ITER_INSTRUMENT) {
                CK(cudaStreamSynchronize(c->s0));
                double t[KC_N];
                if (int rc = graph_times(gr, t)) return rc;
                // STAGE_NAMES: timestep, q_variables, q_derivatives, flux_residual,
                // state_update, residue -- timestep, q_variables and residue run
                // fused inside the update kernels and are reported there
                c->stage_sec[2] += t[KC_QGRAD] * 1e-3;
                c->stage_sec[3] += t[KC_FLUXBND] * 1e-3;
                c->stage_sec[4] += t[KC_UPDATE] * 1e-3;
            }
        }
    }
    return KMF_OK;
}

int reset_run_ctrl(kmf_ctx *c, int hist_cap)
{
    Ctrl init;
    std::memset(&init, 0, sizeof init);
    init.iter = 1;
    init.epoch = 1;
    init.history = c->history.p;
    init.hist_cap = hist_cap;
    CK(cudaMemcpyAsync(c->ctrl.p, &init, sizeof init, cudaMemcpyHostToDevice, c->s0));
    CK(cudaStreamSynchronize(c->s0));  // `init` is a stack temporary
    return KMF_OK;
}

}  // namespace

// ====================================================================== ABI

extern "C" {

int kmf_abi_version(void) { return KMF_ABI_VERSION; }

int kmf_device_count(void)
{
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

const char *kmf_strerror(void) { return g_last_error.c_str(); }

int kmf_create(kmf_ctx **out, const kmf_geometry *g, int device)
{
    if (!out || !g) return KMF_EINVAL;
    *out = nullptr;
    CK(cudaSetDevice(device));
    kmf_ctx *c = new kmf_ctx();
    c->device = device;
    int rc = build_context(c, g);
    if (rc != KMF_OK) {
        delete c;
        return rc;
    }
    *out = c;
    return KMF_OK;
}

void kmf_destroy(kmf_ctx *c)
{
    if (!c) return;
    cudaSetDevice(c->device);
    cudaDeviceSynchronize();
    delete c;
}

int kmf_set_state(kmf_ctx *c, const double *prims)
{
    if (!c || !prims) return KMF_EINVAL;
    CK(cudaSetDevice(c->device));
    if (!c->P0.p) CK(c->P0.alloc(4 * (size_t)c->n));
    CK(cudaMemcpyAsync(c->P0.p, prims, sizeof(double) * 4 * (size_t)c->n, cudaMemcpyHostToDevice, c->s0));
    CK(cudaStreamSynchronize(c->s0));
    c->have_state = true;
    c->pending_init = true;
    return KMF_OK;
}

}  // extern "C"

namespace {

int run_check(kmf_ctx *c, const kmf_params *p, int n_iter, bool linked = false)
{
    if (!c || !p || n_iter < 0) return KMF_EINVAL;
    if (c->peer_broken) {
        set_msg("peer transport: this context saw a peer deadline (KMF_EPEER); its ranks' counters no longer "
                "agree -- re-create the partition's contexts");
        return KMF_EPEER;
    }
    if (c->peer_local && !linked) {
        // its peers are contexts of this process: run alone, it would wait
        // on ranks that never start
        set_msg("this context is peer-linked in-process: run all ranks with kmf_run_linked");
        return KMF_EINVAL;
    }
    if (!c->have_state) {
        set_msg("kmf_run: no state (call kmf_set_state first)");
        return KMF_EINVAL;
    }
    if (int rc = check_params(c, p)) return rc;
    if (c->dist_on && !c->transport()) {
        set_msg("kmf_run: partitioned context without a transport (kmf_nccl_init, kmf_peer_open / kmf_peer_link, "
                "or kmf_run_group)");
        return KMF_EINVAL;
    }
    return KMF_OK;
}

// kmf_run's enqueue half: seed, Ctrl reset, the graph replays (the
// instrumented replays synchronise after each to read their event nodes)
int run_begin(kmf_ctx *c, const kmf_params *p, int n_iter)
{
    CK(cudaSetDevice(c->device));
    c->err = kmf_error_info{};
    c->err_idx.clear();
    if (int rc = seed_state(c, p->gamma, p->cfl)) return rc;
    if ((int)c->history.n < n_iter) CK(c->history.alloc(n_iter));
    if (int rc = reset_run_ctrl(c, n_iter)) return rc;
    for (double &s : c->stage_sec) s = 0.0;
    const int skip = p->instrument ? std::max(0, std::min(p->timing_skip, n_iter)) : n_iter;
    if (int rc = replay(c, p, skip, ITER_PLAIN)) return rc;
    if (int rc = replay(c, p, n_iter - skip, ITER_INSTRUMENT)) return rc;
    CK(cudaGetLastError());
    return KMF_OK;
}

// ... and its completion half: wait, read the control block
int run_finish(kmf_ctx *c, int n_iter, double *history, int *iters_done, int *converged)
{
    CK(cudaSetDevice(c->device));
    CK(cudaStreamSynchronize(c->s0));
    Ctrl fin;
    CK(cudaMemcpy(&fin, c->ctrl.p, sizeof fin, cudaMemcpyDeviceToHost));
    const int status = (int)(fin.state & 3ull);
    int completed = fin.iter - 1;
    if (completed > n_iter) completed = n_iter;
    if (history && completed > 0)
        CK(cudaMemcpy(history, c->history.p, sizeof(double) * completed, cudaMemcpyDeviceToHost));
    if (iters_done) *iters_done = completed;
    if (converged) *converged = status == 2;
    if (fin.peer_fail) {
        c->peer_broken = true;
        record_error(c, KMF_EPEER, fin.iter, 0, 0, 0, "peer transport: a peer rank did not arrive in time");
        set_msg("peer transport: a peer rank did not arrive in time (rank %d)", c->rank);
        return KMF_EPEER;
    }
    if (status == 1) {
        record_error(c, KMF_EPOSITIVITY, fin.err_iter, fin.err_stage, first_context(fin.ctx_mask), 0, "positivity");
        return KMF_EPOSITIVITY;
    }
    return KMF_OK;
}

}  // namespace

extern "C" {

int kmf_run(kmf_ctx *c, const kmf_params *p, int n_iter, double *history, int *iters_done, int *converged)
{
    if (int rc = run_check(c, p, n_iter)) return rc;
    if (iters_done) *iters_done = 0;
    if (converged) *converged = 0;
    if (n_iter == 0) return KMF_OK;
    if (int rc = run_begin(c, p, n_iter)) return rc;
    return run_finish(c, n_iter, history, iters_done, converged);
}

int kmf_prepare(kmf_ctx *c, const kmf_params *p)
{
    if (!c || !p) return KMF_EINVAL;
    if (int rc = check_params(c, p)) return rc;
    if (c->dist_on && !c->transport()) {
        set_msg("kmf_prepare: partitioned context without a transport");
        return KMF_EINVAL;
    }
    CK(cudaSetDevice(c->device));
    const int how = p->instrument ? ITER_INSTRUMENT : ITER_PLAIN;
    if (int rc = get_graph(c, p, 8, c->gU, how)) return rc;
    return get_graph(c, p, 1, c->g1, how);
}

// Streaming cases (include/kmf_b200.h).  Per case k, buffer half b = k & 1:
//   sh: [wait free[b]] upload in[k] -> P0 half b, record up[b]
//   s0: [wait up[b]] k_init, record free[b]; Ctrl reset; n_iter iterations;
//       Ctrl snapshot; [wait down[b]] k_get_state -> stage_buf half b, record got[b]
//   sd: [wait got[b]] download -> out[k], record down[b]
// so case k+1's upload and case k-1's download run on the copy engines
// while case k iterates.  Every case runs exactly kmf_set_state + kmf_run
// (PLAIN) + kmf_get_state's arithmetic.
// Ctrl block copies on the solver stream as a kernel: a cudaMemcpyAsync
// would queue on the copy engine behind the next case's upload.
__global__ void k_ctrl_copy(Ctrl *dst, const Ctrl *src)
{
    static_assert(sizeof(Ctrl) % 8 == 0, "Ctrl is copied in 8-byte words");
    const unsigned long long *s = reinterpret_cast<const unsigned long long *>(src);
    unsigned long long *d = reinterpret_cast<unsigned long long *>(dst);
    for (int w = threadIdx.x; w < (int)(sizeof(Ctrl) / 8); w += blockDim.x) d[w] = s[w];
}

int kmf_run_cases(kmf_ctx *c, const kmf_params *params, int n_iter, int n_cases, const double *const *prims_in,
                  double *const *prims_out, double *const *conserved_out, double *history, int *iters_done,
                  int *converged, int *status)
{
    if (!c || !params || n_iter < 1 || n_cases < 1 || !prims_in || !prims_out) return KMF_EINVAL;
    for (int k = 0; k < n_cases; k++) {
        if (!prims_in[k] || !prims_out[k]) return KMF_EINVAL;
        if (int rc = check_params(c, &params[k])) return rc;
    }
    if (c->peer_local) {
        set_msg("kmf_run_cases: peer-linked in-process contexts run through kmf_run_linked");
        return KMF_EINVAL;
    }
    if (c->peer_broken) {
        set_msg("kmf_run_cases: this context saw a peer deadline; re-create the partition's contexts");
        return KMF_EPEER;
    }
    if (c->dist_on && !c->transport()) {
        set_msg("kmf_run_cases: partitioned context without a transport");
        return KMF_EINVAL;
    }
    CK(cudaSetDevice(c->device));
    c->err = kmf_error_info{};
    c->err_idx.clear();
    const size_t n4 = 4 * (size_t)c->n, bytes = sizeof(double) * n4;
    if (c->P0.n < 2 * n4) CK(c->P0.alloc(2 * n4));
    DBuf<double> hist;
    DBuf<Ctrl> snap, dinit;
    CK(hist.alloc((size_t)n_cases * n_iter));
    CK(snap.alloc(n_cases));
    std::vector<Ctrl> init(n_cases);
    for (int k = 0; k < n_cases; k++) {
        std::memset(&init[k], 0, sizeof(Ctrl));
        init[k].iter = 1;
        init[k].epoch = 1;
        init[k].history = hist.p + (size_t)k * n_iter;
        init[k].hist_cap = n_iter;
    }
    CK(dinit.upload(init.data(), n_cases));
    const DG g = c->dg();
    const long long *perm = c->has_perm ? c->perm.p : nullptr;
    CK(cudaDeviceSynchronize());  // earlier work on any stream of this context
    for (int k = 0; k < n_cases; k++) {
        const kmf_params *p = &params[k];
        const int b = k & 1;
        double *P = c->P0.p + b * n4, *S = c->stage_buf.p + b * n4;
        double *SU = conserved_out && conserved_out[k] ? c->stage_buf2.p + b * n4 : nullptr;
        CK(cudaStreamWaitEvent(c->sh, c->cs_free[b], 0));
        CK(cudaMemcpyAsync(P, prims_in[k], bytes, cudaMemcpyHostToDevice, c->sh));
        CK(cudaEventRecord(c->cs_up[b], c->sh));
        CK(cudaStreamWaitEvent(c->s0, c->cs_up[b], 0));
        k_init<<<nblk(c->n), kTB, 0, c->s0>>>(g, P, perm, c->Uo.p, c->q.p, c->dt.p, p->gamma, p->cfl);
        CK(cudaGetLastError());
        CK(cudaEventRecord(c->cs_free[b], c->s0));
        k_ctrl_copy<<<1, 32, 0, c->s0>>>(c->ctrl.p, dinit.p + k);
        if (int rc = replay(c, p, n_iter, ITER_PLAIN)) return rc;
        k_ctrl_copy<<<1, 32, 0, c->s0>>>(snap.p + k, c->ctrl.p);
        CK(cudaStreamWaitEvent(c->s0, c->cs_down[b], 0));
        k_get_state<<<nblk(c->n), kTB, 0, c->s0>>>(g, c->Uo.p, perm, p->gamma, S, SU);
        CK(cudaGetLastError());
        CK(cudaEventRecord(c->cs_got[b], c->s0));
        CK(cudaStreamWaitEvent(c->sd, c->cs_got[b], 0));
        CK(cudaMemcpyAsync(prims_out[k], S, bytes, cudaMemcpyDeviceToHost, c->sd));
        if (SU) CK(cudaMemcpyAsync(conserved_out[k], SU, bytes, cudaMemcpyDeviceToHost, c->sd));
        CK(cudaEventRecord(c->cs_down[b], c->sd));
    }
    CK(cudaDeviceSynchronize());
    c->have_state = true;  // the last case's final state
    c->pending_init = false;
    c->state_gamma = params[n_cases - 1].gamma;
    CK(cudaMemcpy(init.data(), snap.p, sizeof(Ctrl) * n_cases, cudaMemcpyDeviceToHost));
    if (history) CK(cudaMemcpy(history, hist.p, sizeof(double) * n_cases * n_iter, cudaMemcpyDeviceToHost));
    int rc = KMF_OK;
    for (int k = 0; k < n_cases; k++) {
        const Ctrl &f = init[k];
        const int st = (int)(f.state & 3ull);
        const int done = std::min(f.iter - 1, n_iter);
        if (history)
            for (int i = done; i < n_iter; i++) history[(size_t)k * n_iter + i] = 0.0;
        if (iters_done) iters_done[k] = done;
        if (converged) converged[k] = st == 2;
        if (status) status[k] = f.peer_fail ? KMF_EPEER : st == 1 ? KMF_EPOSITIVITY : KMF_OK;
        if (f.peer_fail) c->peer_broken = true;
        if (f.peer_fail && rc == KMF_OK) {
            set_msg("peer transport: a peer rank did not arrive in time (case %d)", k);
            rc = KMF_EPEER;
        }
        if (st == 1 && rc == KMF_OK) {
            char msg[64];
            std::snprintf(msg, sizeof msg, "positivity (case %d)", k);
            record_error(c, KMF_EPOSITIVITY, f.err_iter, f.err_stage, first_context(f.ctx_mask), 0, msg);
            rc = KMF_EPOSITIVITY;
        }
    }
    return rc;
}

int kmf_get_state(kmf_ctx *c, double *prims, double *U)
{
    if (!c) return KMF_EINVAL;
    CK(cudaSetDevice(c->device));
    if (!c->have_state) {
        set_msg("kmf_get_state: no state");
        return KMF_EINVAL;
    }
    if (c->pending_init)
        if (int rc = seed_state(c, c->state_gamma, 1.0)) return rc;
    double *dp = prims ? c->stage_buf.p : nullptr;
    double *du = U ? c->stage_buf2.p : nullptr;
    k_get_state<<<nblk(c->n), kTB, 0, c->s0>>>(c->dg(), c->Uo.p, c->has_perm ? c->perm.p : nullptr, c->state_gamma,
                                               dp, du);
    CK(cudaGetLastError());
    if (prims) CK(cudaMemcpyAsync(prims, dp, sizeof(double) * 4 * (size_t)c->n, cudaMemcpyDeviceToHost, c->s0));
    if (U) CK(cudaMemcpyAsync(U, du, sizeof(double) * 4 * (size_t)c->n, cudaMemcpyDeviceToHost, c->s0));
    CK(cudaStreamSynchronize(c->s0));
    return KMF_OK;
}

int kmf_stage_seconds(kmf_ctx *c, double out[6])
{
    if (!c || !out) return KMF_EINVAL;
    for (int i = 0; i < 6; i++) out[i] = c->stage_sec[i];
    return KMF_OK;
}

int kmf_last_error(kmf_ctx *c, kmf_error_info *info)
{
    if (!c || !info) return KMF_EINVAL;
    *info = c->err;
    return KMF_OK;
}

int kmf_last_indices(kmf_ctx *c, int64_t *idx, int64_t cap)
{
    if (!c) return KMF_EINVAL;
    int64_t k = 0;
    for (; k < cap && k < (int64_t)c->err_idx.size(); k++) idx[k] = c->err_idx[k];
    return (int)k;
}

// ------------------------------------------------------- context operators

namespace {
// SoA by default; ps = 2: one derivative (dev = G or G + 1) of the
// component-major gradients; ps = 4, fs = 1: the per-point q records;
// ps = 4, fs = 2: two components of one derivative in a gradient plane
int upload_fields(kmf_ctx *c, const double *h, int nc, double *dev, int ps = 1, long long fs = -1)
{
    CK(cudaMemcpyAsync(c->stage_buf.p, h, sizeof(double) * nc * (size_t)c->n, cudaMemcpyHostToDevice, c->s0));
    k_to_dev<<<nblk(c->n), kTB, 0, c->s0>>>(c->n, fs < 0 ? (long long)ps * c->ld : fs, ps, nc, c->stage_buf.p,
                                            c->has_perm ? c->perm.p : nullptr, dev);
    CK(cudaGetLastError());
    return KMF_OK;
}
int download_fields(kmf_ctx *c, const double *dev, int nc, double *h, int ps = 1, long long fs = -1)
{
    k_from_dev<<<nblk(c->n), kTB, 0, c->s0>>>(c->n, fs < 0 ? (long long)ps * c->ld : fs, ps, nc, dev,
                                              c->has_perm ? c->perm.p : nullptr, c->stage_buf.p);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(h, c->stage_buf.p, sizeof(double) * nc * (size_t)c->n, cudaMemcpyDeviceToHost, c->s0));
    CK(cudaStreamSynchronize(c->s0));
    return KMF_OK;
}
// one derivative (d = 0: qx, 1: qy; host (4, n)) in the plane gradient layout
int upload_grad(kmf_ctx *c, const double *h, int d, double *G)
{
    for (int p = 0; p < 2; p++)
        if (int rc = upload_fields(c, h + 2 * (size_t)p * c->n, 2, G + 4 * (size_t)p * c->ld + d, 4, 2)) return rc;
    return KMF_OK;
}
int download_grad(kmf_ctx *c, const double *G, int d, double *h)
{
    for (int p = 0; p < 2; p++)
        if (int rc = download_fields(c, G + 4 * (size_t)p * c->ld + d, 2, h + 2 * (size_t)p * c->n, 4, 2)) return rc;
    return KMF_OK;
}
int reset_ctrl(kmf_ctx *c)
{
    CK(cudaMemsetAsync(c->ctrl.p, 0, sizeof(Ctrl), c->s0));
    return KMF_OK;
}
int read_ctrl(kmf_ctx *c, Ctrl *out)
{
    CK(cudaMemcpyAsync(out, c->ctrl.p, sizeof(Ctrl), cudaMemcpyDeviceToHost, c->s0));
    CK(cudaStreamSynchronize(c->s0));
    return KMF_OK;
}
}  // namespace

int kmf_op_timestep(kmf_ctx *c, const double *prims, double cfl, double gamma, double *dt)
{
    if (!c || !prims || !dt) return KMF_EINVAL;
    if (!(cfl > 0.0 && cfl <= 1.0)) {
        set_msg("cfl must lie in (0, 1]");
        return KMF_EINVAL;
    }
    CK(cudaSetDevice(c->device));
    int rc = upload_fields(c, prims, 4, c->R.p);
    if (rc) return rc;
    k_op_timestep<<<nblk(c->n), kTB, 0, c->s0>>>(c->dg(), c->R.p, cfl, gamma, c->dt.p);
    CK(cudaGetLastError());
    return download_fields(c, c->dt.p, 1, dt);
}

int kmf_op_first_order(kmf_ctx *c, const double *q, double *qx, double *qy)
{
    if (!c || !q || !qx || !qy) return KMF_EINVAL;
    CK(cudaSetDevice(c->device));
    int rc = upload_fields(c, q, 4, c->q.p, 4, 1);
    if (rc) return rc;
    if ((rc = reset_ctrl(c))) return rc;
    launch_first_order(c, c->s0, 0, c->n, c->GA.p, c->ctrl.p, 0);
    CK(cudaGetLastError());
    if ((rc = download_fields(c, c->GA.p, 4, qx, 2))) return rc;
    return download_fields(c, c->GA.p + 1, 4, qy, 2);
}

int kmf_op_q_derivatives(kmf_ctx *c, const double *q, int n_inner, const double *pqx, const double *pqy,
                         double *qx, double *qy, double *inner_residuals)
{
    if (!c || !q || !qx || !qy) return KMF_EINVAL;
    if (n_inner < 1) {
        set_msg("n_inner must be at least 1");
        return KMF_EINVAL;
    }
    CK(cudaSetDevice(c->device));
    int rc = upload_fields(c, q, 4, c->q.p, 4, 1);
    if (rc) return rc;
    if ((rc = reset_ctrl(c))) return rc;
    const int nb = nblk(c->n);
    DG g = c->dg();
    if (pqx && pqy) {
        if ((rc = upload_fields(c, pqx, 4, c->GA.p, 2))) return rc;
        if ((rc = upload_fields(c, pqy, 4, c->GA.p + 1, 2))) return rc;
    } else {
        launch_first_order(c, c->s0, 0, c->n, c->GA.p, c->ctrl.p, 0);
    }
    double *cur = c->GA.p, *nxt = c->GB.p;
    for (int it = 0; it < n_inner; it++) {
        CK(cudaMemsetAsync(&c->ctrl.p->resmax, 0, sizeof(unsigned long long), c->s0));
        launch_sweep(c, c->s0, 0, c->n, cur, nxt, c->ctrl.p, 0, 1 + it, 1, it + 1 == n_inner);
        CK(cudaGetLastError());
        if (inner_residuals) {
            unsigned long long b = 0;
            CK(cudaMemcpyAsync(&b, &c->ctrl.p->resmax, sizeof b, cudaMemcpyDeviceToHost, c->s0));
            CK(cudaStreamSynchronize(c->s0));
            std::memcpy(&inner_residuals[it], &b, 8);
        }
        std::swap(cur, nxt);
    }
    if ((rc = download_grad(c, cur, 0, qx))) return rc;  // plane layout (last sweep)
    return download_grad(c, cur, 1, qy);
}

namespace {
int upload_flow(kmf_ctx *c, const double *q, const double *qx, const double *qy)
{
    int rc = upload_fields(c, q, 4, c->q.p, 4, 1);
    if (rc) return rc;
    if ((rc = upload_grad(c, qx, 0, c->GA.p))) return rc;  // plane layout (flux / boundary input)
    return upload_grad(c, qy, 1, c->GA.p);
}
}  // namespace

int kmf_op_flux_residual(kmf_ctx *c, const double *q, const double *qx, const double *qy, int mode, double gamma,
                         double *R)
{
    if (!c || !q || !qx || !qy || !R) return KMF_EINVAL;
    if (mode != 0 && mode != 1) {
        set_msg("mode must be one of ('fused', 'split4')");
        return KMF_EINVAL;
    }
    CK(cudaSetDevice(c->device));
    int rc = upload_flow(c, q, qx, qy);
    if (rc) return rc;
    if ((rc = reset_ctrl(c))) return rc;
    c->err = kmf_error_info{};
    c->err_idx.clear();
    launch_flux(c, c->s0, 0, c->n, c->GA.p, mode, gamma, 1, c->ctrl.p, 0);
    CK(cudaGetLastError());
    Ctrl fin;
    if ((rc = read_ctrl(c, &fin))) return rc;
    if (fin.state & 1ull) {
        c->G_last = c->GA.p;
        record_error(c, KMF_EPOSITIVITY, 0, 0, KMF_CTX_FLUX_XP, 0, "positivity");
        return KMF_EPOSITIVITY;
    }
    return download_fields(c, c->R.p, 4, R);
}

int kmf_op_boundary(kmf_ctx *c, const double *q, const double *qx, const double *qy, const double fs[4],
                    double gamma, double *R)
{
    if (!c || !q || !qx || !qy || !R || !fs) return KMF_EINVAL;
    CK(cudaSetDevice(c->device));
    int rc = upload_flow(c, q, qx, qy);
    if (rc) return rc;
    if ((rc = upload_fields(c, R, 4, c->R.p))) return rc;
    if ((rc = reset_ctrl(c))) return rc;
    c->err = kmf_error_info{};
    c->err_idx.clear();
    launch_boundary(c, c->s0, c->GA.p, fs, gamma, c->ctrl.p, 0);
    CK(cudaGetLastError());
    Ctrl fin;
    if ((rc = read_ctrl(c, &fin))) return rc;
    if (fin.state & 1ull) {
        const int ctx = first_context(fin.ctx_mask & ~(1u << KMF_CTX_FLUX_XP));
        c->G_last = c->GA.p;
        record_error(c, KMF_EPOSITIVITY, 0, 0, ctx ? ctx : KMF_CTX_WALL_TANGENT, 0, "positivity");
        return KMF_EPOSITIVITY;
    }
    return download_fields(c, c->R.p, 4, R);
}

// the gradient buffer a positivity diagnostic reads: 0 GA, 1 GB, 2 the
// final gradients of the last stage enqueued (run / run_group failures)
static const double *diag_grad(kmf_ctx *c, int which)
{
    if (which == 2 && c->G_last) return c->G_last;
    return which == 1 ? c->GB.p : c->GA.p;
}

// flags for every caller-CSR edge of the full stencil computed from the
// device's current q and the gradient buffer `which` (diag_grad)
int kmf_diag_flux(kmf_ctx *c, int which, uint8_t *flags)
{
    if (!c || !flags) return KMF_EINVAL;
    CK(cudaSetDevice(c->device));
    const double *G = diag_grad(c, which);
    if (c->xy)
        k_diag_flux<true><<<nblk(c->n), kTB, 0, c->s0>>>(c->dg(), c->q.p, G, c->diag.p);
    else
        k_diag_flux<false><<<nblk(c->n), kTB, 0, c->s0>>>(c->dg(), c->q.p, G, c->diag.p);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(flags, c->diag.p, (size_t)c->n_edges, cudaMemcpyDeviceToHost, c->s0));
    CK(cudaStreamSynchronize(c->s0));
    return KMF_OK;
}

// flags per frame edge of family fam (0 tplus, 1 tminus, 2 normal) over the
// concatenated boundary table (wall rows first, then outer)
int kmf_diag_frame(kmf_ctx *c, int which, int fam, uint8_t *flags)
{
    if (!c || !flags || fam < 0 || fam > 2) return KMF_EINVAL;
    if (c->nb == 0) return KMF_OK;
    CK(cudaSetDevice(c->device));
    const double *G = diag_grad(c, which);
    k_diag_frame<<<nblk(c->nb), kTB, 0, c->s0>>>(c->dg(), c->db(), fam, c->q.p, G, c->diag.p);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(flags, c->diag.p, (size_t)c->bedges[fam], cudaMemcpyDeviceToHost, c->s0));
    CK(cudaStreamSynchronize(c->s0));
    return KMF_OK;
}

// the stage-state U written by the last update launch ((4,n), caller order):
// U_stage for stages 1-3, U_outer for stage 4
int kmf_diag_stage_state(kmf_ctx *c, int stage, double *U)
{
    if (!c || !U) return KMF_EINVAL;
    CK(cudaSetDevice(c->device));
    return download_fields(c, stage == 4 ? c->Uo.p : c->Us.p, 4, U);
}


// ------------------------------------------------------ point operators

}  // extern "C"

namespace {
struct Tmp {
    std::vector<void *> ptrs;
    ~Tmp()
    {
        for (void *p : ptrs) cudaFree(p);
    }
    template <typename T>
    T *get(size_t count)
    {
        void *p = nullptr;
        if (cudaMalloc(&p, sizeof(T) * (count ? count : 1)) != cudaSuccess) return nullptr;
        ptrs.push_back(p);
        return (T *)p;
    }
};

#define TMP_OR_FAIL(var, T, count)                    \
    T *var = tmp.get<T>(count);                       \
    if (!var) {                                       \
        set_msg("cudaMalloc failed (%zu)", (size_t)(count)); \
        return KMF_ECUDA;                             \
    }

int ensure_device()
{
    int n = kmf_device_count();
    if (n <= 0) {
        set_msg("no CUDA device visible");
        return KMF_ECUDA;
    }
    return KMF_OK;
}
}  // namespace

extern "C" {

int kmf_op_primitives_to_q(int64_t n, const double *prims, double gamma, double *q, uint8_t *flags)
{
    if (n <= 0 || !prims || !q || !flags) return KMF_EINVAL;
    if (int rc = ensure_device()) return rc;
    Tmp tmp;
    TMP_OR_FAIL(dp, double, 4 * n);
    TMP_OR_FAIL(dq, double, 4 * n);
    TMP_OR_FAIL(df, unsigned char, n);
    CK(cudaMemcpy(dp, prims, sizeof(double) * 4 * n, cudaMemcpyHostToDevice));
    k_op_p2q<<<nblk(n), kTB>>>((int)n, dp, gamma, dq, df);
    CK(cudaGetLastError());
    CK(cudaMemcpy(q, dq, sizeof(double) * 4 * n, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(flags, df, n, cudaMemcpyDeviceToHost));
    return KMF_OK;
}

int kmf_op_q_to_primitives(int64_t n, const double *q, double gamma, double *prims, uint8_t *flags)
{
    if (n <= 0 || !prims || !q || !flags) return KMF_EINVAL;
    if (int rc = ensure_device()) return rc;
    Tmp tmp;
    TMP_OR_FAIL(dq, double, 4 * n);
    TMP_OR_FAIL(dp, double, 4 * n);
    TMP_OR_FAIL(df, unsigned char, n);
    CK(cudaMemcpy(dq, q, sizeof(double) * 4 * n, cudaMemcpyHostToDevice));
    k_op_q2p<<<nblk(n), kTB>>>((int)n, dq, gamma, dp, df);
    CK(cudaGetLastError());
    CK(cudaMemcpy(prims, dp, sizeof(double) * 4 * n, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(flags, df, n, cudaMemcpyDeviceToHost));
    return KMF_OK;
}

int kmf_op_primitives_to_conserved(int64_t n, const double *prims, double gamma, double *U, uint8_t *flags)
{
    if (n <= 0 || !prims || !U || !flags) return KMF_EINVAL;
    if (int rc = ensure_device()) return rc;
    Tmp tmp;
    TMP_OR_FAIL(dp, double, 4 * n);
    TMP_OR_FAIL(du, double, 4 * n);
    TMP_OR_FAIL(df, unsigned char, n);
    CK(cudaMemcpy(dp, prims, sizeof(double) * 4 * n, cudaMemcpyHostToDevice));
    k_op_p2u<<<nblk(n), kTB>>>((int)n, dp, gamma, du, df);
    CK(cudaGetLastError());
    CK(cudaMemcpy(U, du, sizeof(double) * 4 * n, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(flags, df, n, cudaMemcpyDeviceToHost));
    return KMF_OK;
}

int kmf_op_conserved_to_primitives(int64_t n, const double *U, double gamma, double *prims, uint8_t *flags)
{
    if (n <= 0 || !prims || !U || !flags) return KMF_EINVAL;
    if (int rc = ensure_device()) return rc;
    Tmp tmp;
    TMP_OR_FAIL(du, double, 4 * n);
    TMP_OR_FAIL(dp, double, 4 * n);
    TMP_OR_FAIL(df, unsigned char, n);
    CK(cudaMemcpy(du, U, sizeof(double) * 4 * n, cudaMemcpyHostToDevice));
    k_op_u2p<<<nblk(n), kTB>>>((int)n, du, gamma, dp, df);
    CK(cudaGetLastError());
    CK(cudaMemcpy(prims, dp, sizeof(double) * 4 * n, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(flags, df, n, cudaMemcpyDeviceToHost));
    return KMF_OK;
}

int kmf_op_split_flux(int64_t n, const double *prims, int axis, int sign, double gamma, double *G)
{
    if (n <= 0 || !prims || !G || (axis != 0 && axis != 1) || (sign != 1 && sign != -1)) return KMF_EINVAL;
    if (int rc = ensure_device()) return rc;
    Tmp tmp;
    TMP_OR_FAIL(dp, double, 4 * n);
    TMP_OR_FAIL(dg, double, 4 * n);
    CK(cudaMemcpy(dp, prims, sizeof(double) * 4 * n, cudaMemcpyHostToDevice));
    k_op_split_flux<<<nblk(n), kTB>>>((int)n, dp, axis, (double)sign, (2.0 - gamma) / (gamma - 1.0), dg);
    CK(cudaGetLastError());
    CK(cudaMemcpy(G, dg, sizeof(double) * 4 * n, cudaMemcpyDeviceToHost));
    return KMF_OK;
}

int kmf_op_full_flux(int64_t n, const double *prims, int axis, double gamma, double *F)
{
    if (n <= 0 || !prims || !F || (axis != 0 && axis != 1)) return KMF_EINVAL;
    if (int rc = ensure_device()) return rc;
    Tmp tmp;
    TMP_OR_FAIL(dp, double, 4 * n);
    TMP_OR_FAIL(df, double, 4 * n);
    CK(cudaMemcpy(dp, prims, sizeof(double) * 4 * n, cudaMemcpyHostToDevice));
    k_op_full_flux<<<nblk(n), kTB>>>((int)n, dp, axis, gamma, df);
    CK(cudaGetLastError());
    CK(cudaMemcpy(F, df, sizeof(double) * 4 * n, cudaMemcpyDeviceToHost));
    return KMF_OK;
}

int kmf_op_state_update(int64_t n, const double *Uo, const double *Us, int stage, const double *dt,
                        const double *R, double *Un)
{
    if (n <= 0 || !Uo || !Us || !dt || !R || !Un) return KMF_EINVAL;
    if (stage < 1 || stage > 4) {
        set_msg("stage must be 1..4");
        return KMF_EINVAL;
    }
    if (int rc = ensure_device()) return rc;
    Tmp tmp;
    TMP_OR_FAIL(a, double, 4 * n);
    TMP_OR_FAIL(b, double, 4 * n);
    TMP_OR_FAIL(r, double, 4 * n);
    TMP_OR_FAIL(d, double, n);
    TMP_OR_FAIL(o, double, 4 * n);
    CK(cudaMemcpy(a, Uo, sizeof(double) * 4 * n, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(b, Us, sizeof(double) * 4 * n, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(r, R, sizeof(double) * 4 * n, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d, dt, sizeof(double) * n, cudaMemcpyHostToDevice));
    k_op_update<<<nblk(n), kTB>>>((int)n, a, b, stage, d, r, o);
    CK(cudaGetLastError());
    CK(cudaMemcpy(Un, o, sizeof(double) * 4 * n, cudaMemcpyDeviceToHost));
    return KMF_OK;
}

int kmf_op_residue(int64_t n, const double *Un, const double *Uold, double *out)
{
    if (n <= 0 || !Un || !Uold || !out) return KMF_EINVAL;
    if (int rc = ensure_device()) return rc;
    Tmp tmp;
    TMP_OR_FAIL(a, double, n);
    TMP_OR_FAIL(b, double, n);
    TMP_OR_FAIL(l, unsigned long long, kLimbs);
    TMP_OR_FAIL(o, double, 1);
    CK(cudaMemcpy(a, Un, sizeof(double) * n, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(b, Uold, sizeof(double) * n, cudaMemcpyHostToDevice));
    CK(cudaMemset(l, 0, sizeof(unsigned long long) * kLimbs));
    k_op_residue<<<nblk(n), kTB>>>((int)n, a, b, l);
    k_op_residue_fin<<<1, 1>>>((int)n, l, o);
    CK(cudaGetLastError());
    CK(cudaMemcpy(out, o, sizeof(double), cudaMemcpyDeviceToHost));
    return KMF_OK;
}

}  // extern "C"

// ================================================================ bench ABI

extern "C" {

// Timed outer iterations for bench.py.  Pass 1: n_steps plain iteration
// graphs (no timing nodes inside), each bracketed by CUDA events on the
// context stream -> step_ms[i]; between steps a `flush_bytes` memset on the
// same stream evicts L2 outside the timed events.  Pass 2: n_steps more with
// the kernel-timing graph (event nodes around the launch groups, on their
// own stream) -> kernel_ms[KMF_BENCH_KERNELS * i + k] = step i's summed
// launches of kernel class k (0 interior flux, 1 first-order q-gradients,
// 2 Jacobi sweeps); the event nodes never perturb step_ms.
int kmf_bench_steps(kmf_ctx *c, const kmf_params *p, int n_steps, int64_t flush_bytes, double *step_ms,
                    double *kernel_ms, int *launches_per_step)
{
    if (!c || !p || n_steps < 1 || !step_ms || !kernel_ms) return KMF_EINVAL;
    if (!c->have_state) {
        set_msg("kmf_bench_steps: no state");
        return KMF_EINVAL;
    }
    if (c->peer_local || (c->dist_on && !c->transport())) {
        set_msg("kmf_bench_steps: a partitioned context needs its own transport (NCCL or IPC peers)");
        return KMF_EINVAL;
    }
    if (c->peer_broken) {
        set_msg("kmf_bench_steps: this context saw a peer deadline; re-create the partition's contexts");
        return KMF_EPEER;
    }
    if (int rc = check_params(c, p)) return rc;
    CK(cudaSetDevice(c->device));
    if (int rc = seed_state(c, p->gamma, p->cfl)) return rc;
    if ((int)c->history.n < 2 * n_steps) CK(c->history.alloc(2 * n_steps));
    if (flush_bytes > 0 && (int64_t)c->flush.n < flush_bytes) CK(c->flush.alloc((size_t)flush_bytes));
    if (int rc = reset_run_ctrl(c, 2 * n_steps)) return rc;
    kmf_params q = *p;
    q.convergence_tol = 0.0;
    for (int pass = 0; pass < 2; pass++) {
        Graph &gr = pass ? c->gB : c->g1;
        if (int rc = get_graph(c, &q, 1, gr, pass ? ITER_BENCH : ITER_PLAIN))
            return rc;
        for (int i = 0; i < n_steps; i++) {
            if (flush_bytes > 0) CK(cudaMemsetAsync(c->flush.p, i & 0xff, (size_t)flush_bytes, c->s0));
            CK(cudaEventRecord(c->evs[0], c->s0));
            CK(cudaGraphLaunch(gr.exec, c->s0));
            CK(cudaEventRecord(c->evs[1], c->s0));
            CK(cudaEventSynchronize(c->evs[1]));
            if (pass == 0) {
                float ms = 0;
                CK(cudaEventElapsedTime(&ms, c->evs[0], c->evs[1]));
                step_ms[i] = ms;
                continue;
            }
            double t[KC_N];
            if (int rc = graph_times(gr, t)) return rc;
            kernel_ms[KMF_BENCH_KERNELS * i + 0] = t[KC_FLUX];
            kernel_ms[KMF_BENCH_KERNELS * i + 1] = t[KC_FO];
            kernel_ms[KMF_BENCH_KERNELS * i + 2] = t[KC_SWEEP];
        }
    }
    Ctrl fin;
    CK(cudaMemcpy(&fin, c->ctrl.p, sizeof fin, cudaMemcpyDeviceToHost));
    if (launches_per_step) *launches_per_step = c->g1.launches;
    if (fin.peer_fail) {
        c->peer_broken = true;
        set_msg("kmf_bench_steps: peer transport deadline (a peer rank did not arrive)");
        return KMF_EPEER;
    }
    if ((fin.state & 3ull) == 1ull) {
        set_msg("kmf_bench_steps: positivity failure at iteration %d", fin.err_iter);
        return KMF_EPOSITIVITY;
    }
    return KMF_OK;
}

// FP64 pipe peak of this device (DFMA chains on every SM), TFLOP/s.
int kmf_fp64_peak(double *tflops)
{
    if (!tflops) return KMF_EINVAL;
    if (int rc = ensure_device()) return rc;
    int dev = 0, sms = 0;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    Tmp tmp;
    TMP_OR_FAIL(o, double, 1);
    const int blocks = sms * 8, threads = 256, iters = 16384;
    k_fp64_peak<<<blocks, threads>>>(64, 1.0, o);  // warm-up
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    double best = 0.0;
    for (int rep = 0; rep < 3; rep++) {
        CK(cudaEventRecord(a));
        k_fp64_peak<<<blocks, threads>>>(iters, 1.0, o);
        CK(cudaEventRecord(b));
        CK(cudaEventSynchronize(b));
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, a, b));
        double fl = 2.0 * 8.0 * iters * (double)blocks * threads;
        best = std::max(best, fl / (ms * 1e-3) / 1e12);
    }
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    *tflops = best;
    return KMF_OK;
}

// pinned host buffers for the end-to-end (host-buffer) measurement
void *kmf_host_alloc(int64_t bytes)
{
    void *p = nullptr;
    if (cudaMallocHost(&p, (size_t)bytes) != cudaSuccess) return nullptr;
    return p;
}

void kmf_host_free(void *p)
{
    if (p) cudaFreeHost(p);
}

int kmf_fastmath_probe(int64_t n, const double *x, int which, double *out)
{
    if (n <= 0 || !x || !out || which < 0 || which > 5) return KMF_EINVAL;
    if (int rc = ensure_device()) return rc;
    Tmp tmp;
    TMP_OR_FAIL(dx, double, n);
    TMP_OR_FAIL(dout, double, n);
    CK(cudaMemcpy(dx, x, sizeof(double) * n, cudaMemcpyHostToDevice));
    k_fastmath_probe<<<nblk(n), kTB>>>((int)n, dx, which, dout);
    CK(cudaGetLastError());
    CK(cudaMemcpy(out, dout, sizeof(double) * n, cudaMemcpyDeviceToHost));
    return KMF_OK;
}

int kmf_probe_edge_state(int64_t n, const double *q, double gamma, double *prims, double *flux)
{
    if (n <= 0 || !q || !prims || !flux || !(gamma > 1.0 && gamma < 2.0)) return KMF_EINVAL;
    if (int rc = ensure_device()) return rc;
    Tmp tmp;
    TMP_OR_FAIL(dq, double, 4 * n);
    TMP_OR_FAIL(dp, double, 4 * n);
    TMP_OR_FAIL(df, double, 16 * n);
    CK(cudaMemcpy(dq, q, sizeof(double) * 4 * n, cudaMemcpyHostToDevice));
    const double inv_gm1 = 1.0 / (gamma - 1.0), c_i0 = (2.0 - gamma) / (gamma - 1.0);
    switch (gamma_kind(gamma)) {
    case 1: k_probe_edge_state<1><<<nblk(n), kTB>>>((int)n, dq, inv_gm1, c_i0, dp, df); break;
    case 2: k_probe_edge_state<2><<<nblk(n), kTB>>>((int)n, dq, inv_gm1, c_i0, dp, df); break;
    default: k_probe_edge_state<0><<<nblk(n), kTB>>>((int)n, dq, inv_gm1, c_i0, dp, df);
    }
    CK(cudaGetLastError());
    CK(cudaMemcpy(prims, dp, sizeof(double) * 4 * n, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(flux, df, sizeof(double) * 16 * n, cudaMemcpyDeviceToHost));
    return KMF_OK;
}

}  // extern "C"

// ============================================================ multi-GPU ABI

extern "C" int kmf_set_partition(kmf_ctx *c, int64_t n_owned, int64_t n_global, int rank, int nranks, int depth,
                                 const int64_t *layer_end, const int64_t *interior_end, int npeers,
                                 const int *peer_ranks, const int64_t *send_counts, const int64_t *send_slots,
                                 const int64_t *recv_counts, const int64_t *recv_slots)
{
    if (!c || n_owned <= 0 || n_owned > c->n || n_global < n_owned || npeers < 0 || rank < 0 || rank >= nranks ||
        depth < 1 || !layer_end || !interior_end)
        return KMF_EINVAL;
    if (c->has_perm) {
        set_msg("kmf_set_partition: partitioned contexts use the partition's local order");
        return KMF_EINVAL;
    }
    // layer_end[k] = n_owned + |L1..Lk| (k = 0..depth, ending at n);
    // interior_end[k] = owned slots at depth >= k (k = 0..depth+1), non-increasing
    if (layer_end[0] != n_owned || layer_end[depth] != c->n || interior_end[0] != n_owned) {
        set_msg("kmf_set_partition: layer / interior counts inconsistent with the context");
        return KMF_EINVAL;
    }
    for (int k = 0; k < depth; k++)
        if (layer_end[k + 1] < layer_end[k]) return KMF_EINVAL;
    for (int k = 0; k <= depth; k++)
        if (interior_end[k + 1] > interior_end[k] || interior_end[k + 1] < 0) return KMF_EINVAL;
    CK(cudaSetDevice(c->device));
    c->n_owned = (int)n_owned;
    c->n_global = n_global;
    c->rank = rank;
    c->nranks = nranks;
    c->depth = depth;
    c->layer_end.assign(layer_end, layer_end + depth + 1);
    c->interior_end.assign(interior_end, interior_end + depth + 2);
    c->peer_rank.assign(peer_ranks, peer_ranks + npeers);
    c->send_off.assign(npeers, 0);
    c->send_cnt.assign(npeers, 0);
    c->recv_off.assign(npeers, 0);
    c->recv_cnt.assign(npeers, 0);
    long long so = 0, ro = 0;
    for (int k = 0; k < npeers; k++) {
        c->send_off[k] = so;
        c->send_cnt[k] = send_counts[k];
        so += send_counts[k];
        c->recv_off[k] = ro;
        c->recv_cnt[k] = recv_counts[k];
        ro += recv_counts[k];
    }
    c->send_total = so;
    c->recv_total = ro;
    auto build = [&](const int64_t *slots, const std::vector<long long> &off, const std::vector<long long> &cnt,
                     long long total, DBuf<int> &sl, DBuf<int> &ba, DBuf<int> &st, bool owned_side) -> int {
        std::vector<int> s(std::max<long long>(total, 1)), b(s.size()), t(s.size());
        for (int k = 0; k < npeers; k++)
            for (long long e = 0; e < cnt[k]; e++) {
                const long long idx = off[k] + e;
                const long long slot = slots[idx];
                if (slot < 0 || slot >= c->n || (owned_side && slot >= n_owned) || (!owned_side && slot < n_owned)) {
                    set_msg("kmf_set_partition: slot %lld out of range", slot);
                    return KMF_EINVAL;
                }
                s[idx] = (int)slot;
                b[idx] = (int)(4 * off[k] + e);
                t[idx] = (int)cnt[k];
            }
        CK(sl.upload(s.data(), s.size()));
        CK(ba.upload(b.data(), b.size()));
        CK(st.upload(t.data(), t.size()));
        return KMF_OK;
    };
    if (int rc = build(send_slots, c->send_off, c->send_cnt, so, c->ps_slot, c->ps_base, c->ps_stride, true)) return rc;
    c->send_slot_h.assign(send_slots, send_slots + so);
    c->recv_slot_h.assign(recv_slots, recv_slots + ro);
    if (int rc = build(recv_slots, c->recv_off, c->recv_cnt, ro, c->pr_slot, c->pr_base, c->pr_stride, false))
        return rc;
    CK(c->sendbuf.alloc(4 * (size_t)std::max<long long>(so, 1)));
    CK(c->recvbuf.alloc(4 * (size_t)std::max<long long>(ro, 1)));
    if (depth - 1 > kmf_ctx::kMaxLevels) {
        set_msg("kmf_set_partition: depth %d exceeds %d", depth, kmf_ctx::kMaxLevels + 1);
        return KMF_EINVAL;
    }
    for (int k = 0; k < depth - 1; k++) CK(c->Glev[k].alloc(8 * (size_t)c->ld));  // levels 0..n_inner, n_inner <= depth - 2
    c->dist_on = true;
    c->drop_graphs();  // graphs captured before the partition are stale
    return KMF_OK;
}

extern "C" int kmf_nccl_get_unique_id(void *out128)
{
    if (!out128) return KMF_EINVAL;
    NcclApi &api = nccl_api();
    if (!api.ok) {
        set_msg("libnccl.so.2 not loadable");
        return KMF_ENCCL;
    }
    ncclUniqueId id;
    if (api.GetUniqueId(&id) != ncclSuccess) return KMF_ENCCL;
    std::memcpy(out128, &id, sizeof id);
    return KMF_OK;
}

extern "C" int kmf_nccl_init(kmf_ctx *c, const void *id128, int rank, int nranks)
{
    if (!c || !id128 || rank < 0 || rank >= nranks) return KMF_EINVAL;
    NcclApi &api = nccl_api();
    if (!api.ok) {
        set_msg("libnccl.so.2 not loadable");
        return KMF_ENCCL;
    }
    CK(cudaSetDevice(c->device));
    ncclUniqueId id;
    std::memcpy(&id, id128, sizeof id);
    ncclComm_t comm;
    ncclResult_t r = api.CommInitRank(&comm, nranks, id, rank);
    if (r != ncclSuccess) {
        set_msg("ncclCommInitRank: %s", api.GetErrorString ? api.GetErrorString(r) : "error");
        return KMF_ENCCL;
    }
    c->nccl = comm;
    // Teardown runs after the context's streams are idle (kmf_destroy
    // synchronises), so nothing is in flight: ncclCommAbort releases the
    // communicator locally, whereas ncclCommDestroy's finalize waits on its
    // peers' proxies and hung at interpreter exit with the socket transport.
    c->nccl_destroy = [](void *p) {
        NcclApi &a = nccl_api();
        if (a.CommAbort)
            a.CommAbort((ncclComm_t)p);
        else if (a.CommDestroy)
            a.CommDestroy((ncclComm_t)p);
    };
    c->drop_graphs();
    // One eager round of the exact send/recv pattern (on both streams the
    // graphs use) and of the limb all-reduce before any graph capture: NCCL
    // sets its P2P connections up lazily at first use, which must not happen
    // inside stream capture.  Nothing is unpacked and the all-reduce runs on
    // scratch memory, so the solver state is untouched.
    if (c->dist_on) {
        for (cudaStream_t s : {c->s0, c->s2}) {
            api.GroupStart();
            for (size_t k = 0; k < c->peer_rank.size(); k++) {
                if (c->send_cnt[k])
                    api.Send(c->sendbuf.p + 4 * c->send_off[k], 4 * c->send_cnt[k], ncclDouble, c->peer_rank[k],
                             comm, s);
                if (c->recv_cnt[k])
                    api.Recv(c->recvbuf.p + 4 * c->recv_off[k], 4 * c->recv_cnt[k], ncclDouble, c->peer_rank[k],
                             comm, s);
            }
            r = api.GroupEnd();
            if (r != ncclSuccess) break;
            CK(cudaStreamSynchronize(s));
        }
        DBuf<unsigned long long> scratch;
        CK(scratch.alloc(kLimbs));
        CK(cudaMemsetAsync(scratch.p, 0, sizeof(unsigned long long) * kLimbs, c->s0));
        if (r == ncclSuccess) r = api.AllReduce(scratch.p, scratch.p, kLimbs, ncclUint64, ncclSum, comm, c->s0);
        if (r != ncclSuccess) {
            set_msg("NCCL warm-up exchange: %s", api.GetErrorString ? api.GetErrorString(r) : "error");
            return KMF_ENCCL;
        }
        CK(cudaStreamSynchronize(c->s0));
    }
    return KMF_OK;
}

// Single-process driver for several partitioned contexts (one per rank, on
// the same or different GPUs) with the multi-process schedule: per stage
// every context runs its interior pass, then the halo q packed after the
// previous update moves by device / peer copies, then every context runs
// its band pass and update and packs its new halo q.  The residue limbs are
// summed on the host (exact integers) and every context closes the
// iteration with the same total.  Used by the multi-rank parity tests on a
// single GPU (the interior / band split is exercised exactly as under NCCL)
// and as a one-process multi-GPU mode.
extern "C" int kmf_run_group(kmf_ctx **ctxs, int nctx, const kmf_params *p, int n_iter, double *history,
                             int *iters_done, int *converged)
{
    if (!ctxs || nctx < 1 || !p || n_iter < 0) return KMF_EINVAL;
    std::vector<kmf_ctx *> byrank(nctx, nullptr);
    for (int k = 0; k < nctx; k++) {
        kmf_ctx *c = ctxs[k];
        if (!c || !c->dist_on || c->nranks != nctx || byrank[c->rank] || !c->have_state || c->peer_on) {
            set_msg("kmf_run_group: contexts must be partitioned ranks 0..n-1 with state (peer-linked "
                    "contexts run with kmf_run_linked)");
            return KMF_EINVAL;
        }
        if (int rc = check_params(c, p)) return rc;
        byrank[c->rank] = c;
    }
    if (iters_done) *iters_done = 0;
    if (converged) *converged = 0;
    if (n_iter == 0) return KMF_OK;
    for (kmf_ctx *c : byrank) {
        CK(cudaSetDevice(c->device));
        c->err = kmf_error_info{};
        if (int rc = seed_state(c, p->gamma, p->cfl)) return rc;
        if ((int)c->history.n < n_iter) CK(c->history.alloc(n_iter));
        if (int rc = reset_run_ctrl(c, n_iter)) return rc;
        enqueue_pack(c, c->s0);  // the halo q the first band pass reads (and a continuation needs)
    }
    auto sync_all = [&]() -> int {
        for (kmf_ctx *c : byrank) {
            CK(cudaSetDevice(c->device));
            CK(cudaStreamSynchronize(c->s0));
        }
        return KMF_OK;
    };
    auto exchange = [&]() -> int {
        if (int rc = sync_all()) return rc;
        for (kmf_ctx *dst : byrank)
            for (size_t k = 0; k < dst->peer_rank.size(); k++) {
                kmf_ctx *src = byrank[dst->peer_rank[k]];
                size_t j = 0;
                while (j < src->peer_rank.size() && src->peer_rank[j] != dst->rank) j++;
                if (j == src->peer_rank.size() || src->send_cnt[j] != dst->recv_cnt[k]) {
                    set_msg("kmf_run_group: send/recv lists of ranks %d and %d disagree", src->rank, dst->rank);
                    return KMF_EINVAL;
                }
                // on the receiver's solver stream, ahead of its unpack (the
                // context streams are non-blocking: a legacy-stream copy would
                // not be ordered before the unpack kernel)
                if (dst->recv_cnt[k]) {
                    CK(cudaSetDevice(dst->device));
                    CK(cudaMemcpyPeerAsync(dst->recvbuf.p + 4 * dst->recv_off[k], dst->device,
                                           src->sendbuf.p + 4 * src->send_off[j], src->device,
                                           sizeof(double) * 4 * dst->recv_cnt[k], dst->s0));
                }
            }
        for (kmf_ctx *c : byrank) {
            CK(cudaSetDevice(c->device));
            enqueue_unpack(c, c->s0);
            CK(cudaEventRecord(c->bready, c->s0));
        }
        return KMF_OK;
    };
    for (int it = 0; it < n_iter; it++) {
        for (int stage = 1; stage <= 4; stage++) {
            std::vector<double *> Gs(nctx, nullptr);
            std::vector<StageCtx> sc;
            for (kmf_ctx *c : byrank)
                sc.push_back(StageCtx{p, IterOut{p->convergence_tol, 0}, ITER_PLAIN, false});
            for (int r = 0; r < nctx; r++) {
                CK(cudaSetDevice(byrank[r]->device));
                enqueue_head(byrank[r], sc[r], stage, Gs[r]);  // interior pass: no halo data read
            }
            if (int rc = exchange()) return rc;
            for (int r = 0; r < nctx; r++) {
                kmf_ctx *c = byrank[r];
                CK(cudaSetDevice(c->device));
                enqueue_tail(c, sc[r], stage, Gs[r]);
                enqueue_pack(c, c->s0);
                CK(cudaGetLastError());
            }
        }
        // exact residue across ranks: integer limb sums
        std::vector<unsigned long long> tot(kLimbs, 0ull), part(kLimbs);
        if (int rc = sync_all()) return rc;
        for (kmf_ctx *c : byrank) {
            CK(cudaSetDevice(c->device));
            CK(cudaMemcpy(part.data(), c->ctrl.p->limbs, sizeof(unsigned long long) * kLimbs, cudaMemcpyDeviceToHost));
            for (int l = 0; l < kLimbs; l++) tot[l] += part[l];
        }
        for (kmf_ctx *c : byrank) {
            CK(cudaSetDevice(c->device));
            CK(cudaMemcpy(c->ctrl.p->limbs, tot.data(), sizeof(unsigned long long) * kLimbs, cudaMemcpyHostToDevice));
            IterOut io{p->convergence_tol, 0};
            k_close<<<1, kTB, 0, c->s0>>>(c->ctrl.p, (int)c->n_global, io);
            CK(cudaGetLastError());
        }
        if (int rc = sync_all()) return rc;
        // stop early on convergence or an error on any rank
        int stop = 0;
        for (kmf_ctx *c : byrank) {
            unsigned long long st = 0;
            CK(cudaMemcpy(&st, &c->ctrl.p->state, sizeof st, cudaMemcpyDeviceToHost));
            if (st) stop = 1;
        }
        if (stop) break;
    }
    // outputs from rank 0 (all ranks agree on history and convergence);
    // errors: the earliest failing rank
    Ctrl fin;
    int err_rank = -1, err_it = 1 << 30, err_stage = 99;
    for (kmf_ctx *c : byrank) {
        Ctrl f;
        CK(cudaMemcpy(&f, c->ctrl.p, sizeof f, cudaMemcpyDeviceToHost));
        if ((f.state & 3ull) == 1ull && (f.err_iter < err_it || (f.err_iter == err_it && f.err_stage < err_stage))) {
            err_rank = c->rank;
            err_it = f.err_iter;
            err_stage = f.err_stage;
        }
        if ((f.state & 3ull) == 1ull)
            record_error(c, KMF_EPOSITIVITY, f.err_iter, f.err_stage, first_context(f.ctx_mask), c->rank,
                         "positivity");
        if (c->rank == 0) fin = f;
    }
    int completed = std::min(fin.iter - 1, n_iter);
    if (history && completed > 0)
        CK(cudaMemcpy(history, byrank[0]->history.p, sizeof(double) * completed, cudaMemcpyDeviceToHost));
    if (iters_done) *iters_done = completed;
    if (converged) *converged = (fin.state & 3ull) == 2ull;
    if (err_rank >= 0) {
        set_msg("positivity failure on rank %d", err_rank);
        return KMF_EPOSITIVITY;
    }
    return KMF_OK;
}

// ------------------------------------------------------- peer transport
namespace {

// PeerSet / PeerPush of context c from its peers' mapped q arrays and flag
// blocks and, per peer it sends to (partition peer order), the peer's
// local slots receiving c's send list
int peer_setup(kmf_ctx *c, double *const *peer_q, PeerFlags *const *peer_flags,
               const std::vector<std::vector<long long>> &dst)
{
    if (c->nranks > kMaxRanks) {
        set_msg("peer transport: %d ranks exceed %d", c->nranks, kMaxRanks);
        return KMF_EINVAL;
    }
    PeerSet ps{};
    PeerPush pp{};
    ps.me = c->pflags.p;
    ps.rank = c->rank;
    ps.nranks = c->nranks;
    ps.timeout_ns = kPeerTimeoutNs;
    if (const char *t = std::getenv("KMF_PEER_TIMEOUT_S"))
        if (std::atof(t) > 0) ps.timeout_ns = (unsigned long long)(std::atof(t) * 1e9);
    for (int r = 0; r < c->nranks; r++) {
        ps.peer[r] = r == c->rank ? c->pflags.p : peer_flags[r];
        pp.q[r] = r == c->rank ? c->q.p : peer_q[r];
    }
    std::vector<int> cnt((size_t)c->n_owned + 1, 0);
    for (size_t k = 0; k < c->peer_rank.size(); k++) {
        const int r = c->peer_rank[k];
        if (r < 0 || r >= c->nranks || r == c->rank) return KMF_EINVAL;
        if (c->send_cnt[k]) ps.send_mask |= 1u << r;
        if (c->recv_cnt[k]) ps.recv_mask |= 1u << r;
        if ((long long)dst[k].size() != c->send_cnt[k]) {
            set_msg("peer transport: rank %d expects %lld halo slots from rank %d, rank %d sends %lld", r,
                    (long long)dst[k].size(), c->rank, c->rank, c->send_cnt[k]);
            return KMF_EINVAL;
        }
        for (long long e = 0; e < c->send_cnt[k]; e++) cnt[c->send_slot_h[c->send_off[k] + e] + 1]++;
    }
    for (int i = 0; i < c->n_owned; i++) cnt[i + 1] += cnt[i];
    std::vector<int> fill(cnt.begin(), cnt.end() - 1);
    std::vector<unsigned> out(std::max<long long>(c->send_total, 1));
    for (size_t k = 0; k < c->peer_rank.size(); k++)
        for (long long e = 0; e < c->send_cnt[k]; e++) {
            const long long d = dst[k][e];
            if (d < 0 || d >= (1ll << kPeerSlotBits)) return KMF_EINVAL;
            out[fill[c->send_slot_h[c->send_off[k] + e]]++] =
                ((unsigned)c->peer_rank[k] << kPeerSlotBits) | (unsigned)d;
        }
    CK(c->push_ptr.upload(cnt.data(), cnt.size()));
    CK(c->push_dst.upload(out.data(), out.size()));
    // load the transport's kernels now: with lazy module loading a kernel's
    // first launch may wait for the device to go idle, which a rank already
    // spinning on its peers never does
    cudaFuncAttributes fa;
    for (const void *f : {(const void *)k_peer_wait_data, (const void *)k_peer_wait_read, (const void *)k_peer_band_done,
                          (const void *)k_peer_pushed, (const void *)k_peer_push_all, (const void *)k_peer_limbs})
        CK(cudaFuncGetAttributes(&fa, f));
    pp.ptr = c->push_ptr.p;
    pp.dst = c->push_dst.p;
    c->pset = ps;
    c->ppush = pp;
    c->peer_on = true;
    c->drop_graphs();
    return KMF_OK;
}

int peer_flags_alloc(kmf_ctx *c)
{
    if (!c->pflags.p) {
        CK(c->pflags.alloc(1));
        CK(cudaMemset(c->pflags.p, 0, sizeof(PeerFlags)));
        CK(cudaDeviceSynchronize());  // the legacy-stream memset before any peer or stream touches the block
    }
    return KMF_OK;
}

}  // namespace

extern "C" int kmf_peer_handle(kmf_ctx *c, void *out)
{
    if (!c || !out || !c->dist_on) return KMF_EINVAL;
    CK(cudaSetDevice(c->device));
    if (int rc = peer_flags_alloc(c)) return rc;
    cudaIpcMemHandle_t h[2];
    CK(cudaIpcGetMemHandle(&h[0], c->q.p));
    CK(cudaIpcGetMemHandle(&h[1], c->pflags.p));
    std::memcpy(out, h, sizeof h);
    static_assert(sizeof h == KMF_PEER_HANDLE_BYTES, "two IPC handles");
    return KMF_OK;
}

extern "C" int kmf_peer_open(kmf_ctx *c, const void *handles, const int64_t *dst_counts, const int64_t *dst_slots)
{
    if (!c || !handles || !c->dist_on || c->nccl || c->peer_on) return KMF_EINVAL;
    CK(cudaSetDevice(c->device));
    if (int rc = peer_flags_alloc(c)) return rc;
    std::vector<double *> q(c->nranks, nullptr);
    std::vector<PeerFlags *> f(c->nranks, nullptr);
    const cudaIpcMemHandle_t *h = static_cast<const cudaIpcMemHandle_t *>(handles);
    for (int r = 0; r < c->nranks; r++) {
        if (r == c->rank) continue;
        void *a = nullptr, *b = nullptr;
        CK(cudaIpcOpenMemHandle(&a, h[2 * r], cudaIpcMemLazyEnablePeerAccess));
        c->ipc_opened.push_back(a);
        CK(cudaIpcOpenMemHandle(&b, h[2 * r + 1], cudaIpcMemLazyEnablePeerAccess));
        c->ipc_opened.push_back(b);
        q[r] = static_cast<double *>(a);
        f[r] = static_cast<PeerFlags *>(b);
    }
    std::vector<std::vector<long long>> dst(c->peer_rank.size());
    long long off = 0;
    for (size_t k = 0; k < c->peer_rank.size(); k++) {
        const long long n = dst_counts ? dst_counts[k] : 0;
        dst[k].assign(dst_slots + off, dst_slots + off + n);
        off += n;
    }
    return peer_setup(c, q.data(), f.data(), dst);
}

extern "C" int kmf_peer_link(kmf_ctx **ctxs, int nctx)
{
    if (!ctxs || nctx < 1) return KMF_EINVAL;
    std::vector<kmf_ctx *> byrank(nctx, nullptr);
    for (int k = 0; k < nctx; k++) {
        kmf_ctx *c = ctxs[k];
        if (!c || !c->dist_on || c->nranks != nctx || byrank[c->rank] || c->nccl || c->peer_on) {
            set_msg("kmf_peer_link: contexts must be partitioned ranks 0..n-1 without a transport");
            return KMF_EINVAL;
        }
        byrank[c->rank] = c;
    }
    // Ranks sharing a device share its hardware work queues (one per
    // stream up to CUDA_DEVICE_MAX_CONNECTIONS, default 8); a rank spinning
    // on its peers at the head of a queue another rank's stream maps to would
    // block that rank for good.  Each rank runs two streams (solver, band
    // pass): refuse what cannot be scheduled.
    int conns = 8;
    if (const char *e = std::getenv("CUDA_DEVICE_MAX_CONNECTIONS")) conns = std::max(1, std::atoi(e));
    for (kmf_ctx *c : byrank) {
        int same = 0;
        for (kmf_ctx *o : byrank) same += o->device == c->device;
        if (same > 1 && 2 * same > conns) {
            set_msg("kmf_peer_link: %d ranks on device %d need CUDA_DEVICE_MAX_CONNECTIONS >= %d (set before CUDA "
                    "initialises; it is %d)", same, c->device, 2 * same, conns);
            return KMF_EINVAL;
        }
    }
    for (kmf_ctx *c : byrank) {
        CK(cudaSetDevice(c->device));
        if (int rc = peer_flags_alloc(c)) return rc;
    }
    std::vector<double *> q(nctx);
    std::vector<PeerFlags *> f(nctx);
    for (int r = 0; r < nctx; r++) {
        q[r] = byrank[r]->q.p;
        f[r] = byrank[r]->pflags.p;
    }
    for (kmf_ctx *c : byrank) {
        for (kmf_ctx *o : byrank)  // peer access between distinct devices (NVLink); same device: nothing to do
            if (o->device != c->device) {
                CK(cudaSetDevice(c->device));
                cudaError_t e = cudaDeviceEnablePeerAccess(o->device, 0);
                if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) CK(e);
                cudaGetLastError();
            }
        std::vector<std::vector<long long>> dst(c->peer_rank.size());
        for (size_t k = 0; k < c->peer_rank.size(); k++) {
            const kmf_ctx *o = byrank[c->peer_rank[k]];
            size_t j = 0;
            while (j < o->peer_rank.size() && o->peer_rank[j] != c->rank) j++;
            if (j < o->peer_rank.size())
                dst[k].assign(o->recv_slot_h.begin() + o->recv_off[j],
                              o->recv_slot_h.begin() + o->recv_off[j] + o->recv_cnt[j]);
        }
        CK(cudaSetDevice(c->device));
        if (int rc = peer_setup(c, q.data(), f.data(), dst)) return rc;
        c->peer_local = true;
    }
    return KMF_OK;
}

extern "C" int kmf_run_linked(kmf_ctx **ctxs, int nctx, const kmf_params *p, int n_iter, double *history,
                              int *iters_done, int *converged)
{
    if (!ctxs || nctx < 1 || !p) return KMF_EINVAL;
    std::vector<kmf_ctx *> byrank(nctx, nullptr);
    for (int k = 0; k < nctx; k++) {
        kmf_ctx *c = ctxs[k];
        if (!c || !c->peer_on || c->nranks != nctx || byrank[c->rank]) {
            set_msg("kmf_run_linked: contexts must be peer-linked ranks 0..n-1 (kmf_peer_link)");
            return KMF_EINVAL;
        }
        if (int rc = run_check(c, p, n_iter, true)) return rc;
        byrank[c->rank] = c;
    }
    if (iters_done) *iters_done = 0;
    if (converged) *converged = 0;
    if (n_iter == 0) return KMF_OK;
    kmf_params q = *p;
    q.instrument = 0;  // the ranks run concurrently: no per-replay host reads
    // every graph is captured and instantiated, every buffer sized, before
    // any rank starts (an instantiation or a cudaFree may wait for the
    // device to go idle, which it does not while a rank spins on its
    // peers); then every rank's whole run is
    // enqueued before any is awaited (the ranks wait on each other on the
    // device)
    for (kmf_ctx *c : byrank) {
        CK(cudaSetDevice(c->device));
        // (re)allocations before any launch too: cudaFree waits for the device
        if ((int)c->history.n < n_iter) CK(c->history.alloc(n_iter));
        if (n_iter >= 8)
            if (int rc = get_graph(c, &q, 8, c->gU, ITER_PLAIN)) return rc;
        if (n_iter % 8)
            if (int rc = get_graph(c, &q, 1, c->g1, ITER_PLAIN)) return rc;
    }
    for (kmf_ctx *c : byrank)
        if (int rc = run_begin(c, &q, n_iter)) {
            // ranks already started spin on this one: release them, then wait
            for (kmf_ctx *o : byrank) {
                cudaSetDevice(o->device);
                const unsigned long long one = 1ull;
                cudaMemcpy(&o->pflags.p->failed, &one, sizeof one, cudaMemcpyHostToDevice);
                o->peer_broken = true;
            }
            for (kmf_ctx *o : byrank) {
                cudaSetDevice(o->device);
                cudaDeviceSynchronize();
            }
            return rc;
        }
    std::vector<int> rcs(nctx);
    for (int r = 0; r < nctx; r++) {
        int done = 0, conv = 0;
        rcs[r] = run_finish(byrank[r], n_iter, r == 0 ? history : nullptr, &done, &conv);
        if (r == 0) {
            if (iters_done) *iters_done = done;
            if (converged) *converged = conv;
        }
    }
    // a transport / CUDA failure first; positivity failures stay recorded on
    // each failing context (kmf_last_error), as with kmf_run_group
    for (int r = 0; r < nctx; r++)
        if (rcs[r] != KMF_OK && rcs[r] != KMF_EPOSITIVITY) return rcs[r];
    for (int r = 0; r < nctx; r++)
        if (rcs[r] == KMF_EPOSITIVITY) return KMF_EPOSITIVITY;
    return KMF_OK;
}

// diagnostics: this rank's peer counters -- out[0..2] pushes, bands,
// iterations; then data[r], read[r], limb_seq[r] for r < nranks
extern "C" int kmf_peer_counters(kmf_ctx *c, uint64_t *out)
{
    if (!c || !out || !c->pflags.p) return KMF_EINVAL;
    CK(cudaSetDevice(c->device));
    PeerFlags f;
    CK(cudaMemcpy(&f, c->pflags.p, sizeof f, cudaMemcpyDeviceToHost));
    out[0] = f.pushes;
    out[1] = f.bands;
    out[2] = f.iters;
    for (int r = 0; r < c->nranks; r++) {
        out[3 + r] = f.data[r];
        out[3 + c->nranks + r] = f.read[r];
        out[3 + 2 * c->nranks + r] = f.limb_seq[r];
    }
    return KMF_OK;
}
