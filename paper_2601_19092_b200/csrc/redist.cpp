// redist.cpp -- axe_redistribute: layout-driven resharding across the device
// axis "gpuid" (P:173-199 distributed layouts; P:399-403 DTensor signatures;
// P:408 "a copy might involve an all-gather ... under the hood").
//
// Planning (host, identical on every rank):
//   1. compose both layouts with their local storages, keeping the gpuid
//      pieces (compose_linear keep_dev) and refine them jointly;
//   2. joint digits touching gpuid on either side index "blocks" (one
//      (source rank, destination rank) pair each); the remaining digits form
//      one memory-only sub-box shared by every block;
//   3. every block gets one sender: the destination rank itself when it owns
//      the element (local copy), else a source replica balanced by egress
//      (reading R5);
//   4. per rank: pack plans (src_local -> send staging), NCCL send/recv per
//      block, unpack plans (recv staging -> dst_local), local copy plans;
//      pack/unpack are elided when a block is contiguous on that side, and an
//      all-gather pattern is lowered to ncclAllGather.
#include <cuda.h>
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <numeric>
#include <unordered_map>
#include <chrono>
#include <thread>

#include <nvtx3/nvToolsExt.h>

#include "handles.hpp"

using namespace axe;

namespace axe {
void stream_forget(cudaStream_t st);
}

struct axe_comm {
  ncclComm_t comm = nullptr;
  int nranks = 0, rank = 0, device = 0;
  std::mutex mu;         // NCCL enqueues on one communicator are not concurrent-safe: one call at a time
  bool aborted = false;  // axe_comm_wait aborted it (timeout or asynchronous error)
};

namespace {
// NVTX range for the timeline (nsys / ncu --nvtx): plan, pack, wire, unpack phases
struct Nvtx {
  explicit Nvtx(const char *name) { nvtxRangePushA(name); }
  ~Nvtx() { nvtxRangePop(); }
};
}  // namespace

namespace {

struct Xfer {
  int peer = -1;
  int64_t ms = 0, md = 0;          // element offsets (source local, destination local)
  bool elided = false;             // send straight from src / receive straight into dst
  int64_t stage = 0;               // element offset in the staging buffer when not elided
  std::shared_ptr<CopyPlan> plan;  // local copy
  std::vector<std::shared_ptr<CopyPlan>> cp;  // per wire chunk: pack (send) or unpack (recv)
};

}  // namespace

struct axe_redist_plan {
  int nranks = 0, rank = 0, es = 0;
  std::vector<Joint> M;            // memory-only digits, packed order (outermost first)
  std::vector<int64_t> packed;     // packed (compact) element strides of M
  int64_t n = 1;                   // elements per block
  int nchunk = 1;                  // wire chunks per block (cut along the outermost packed digit)
  int64_t cn = 1;                  // elements per chunk
  std::vector<Xfer> sends, recvs, locals;
  int64_t send_elems = 0, recv_elems = 0;
  int64_t src_cells = 0, dst_cells = 0;
  bool allgather = false;
  int64_t ag_src = 0, ag_dst = 0;  // element offsets of the all-gather
  std::string desc;
  int64_t dst_rep = 1;             // destination memory replicas per element (distinct cells)
  // reduction (axe_redist_reduce_plan_create): `inner` moves the partials into the stage
  // buffer (K slabs shaped like this rank's dst storage), `red` sums the slabs into dst_local
  std::shared_ptr<axe_redist_plan> inner;
  ReducePlan red;
  int64_t stage_bytes = 0;
  // two-phase reduction (destination replicated over >= 3 ranks): phase_a reduce-scatters into an
  // evenly sharded temporary, phase_b redistributes (all-gathers) it into the destination
  std::shared_ptr<axe_redist_plan> phase_a, phase_b;
  int64_t tmp_bytes = 0;
  // one-sided pull form of a reduction (axe_redist_plan_execute_peers_reduce): per destination
  // region, one K4 launch summing the K partials straight from the senders' src buffers
  struct Pull {
    K4Params k;
    std::vector<int> senders;  // rank owning summand k
  };
  std::vector<Pull> pulls;
  bool multicast_ok = false;  // every region: one partial per rank at the same offset (NVLS form)
  int pull_vb = 0;
  unsigned pull_blocks = 1;
  std::string pull_why;
  // scratch owned by the plan (allocated on first execute, on the current device)
  mutable std::mutex mu;
  mutable void *send_buf = nullptr, *recv_buf = nullptr, *stage = nullptr, *tmp = nullptr;
  mutable cudaStream_t side = nullptr;
  mutable cudaEvent_t ev_fork = nullptr, ev_join = nullptr, ev_join2 = nullptr;
  mutable cudaStream_t pk = nullptr, up = nullptr;  // pack / unpack streams
  mutable std::vector<cudaEvent_t> ev_pack, ev_recv;
  // executes of one plan are serialised: the host enqueue under exec_mu, and on the device every
  // execute waits for the previous one (ev_done) -- they share the staging buffers and side streams
  mutable std::mutex exec_mu;
  mutable cudaEvent_t ev_done = nullptr;
  mutable bool done_valid = false;
  ~axe_redist_plan() {
    if (send_buf) cudaFree(send_buf);
    if (recv_buf) cudaFree(recv_buf);
    if (stage) cudaFree(stage);
    if (tmp) cudaFree(tmp);
    for (cudaStream_t x : {side, pk, up})
      if (x) cudaStreamDestroy(x);
    for (cudaEvent_t x : {ev_fork, ev_join, ev_join2, ev_done})
      if (x) cudaEventDestroy(x);
    for (auto &v : {ev_pack, ev_recv})
      for (cudaEvent_t x : v)
        if (x) cudaEventDestroy(x);
  }
};

namespace {

Layout mlayout(const std::vector<std::pair<int64_t, int64_t>> &D, const std::vector<LinIter> &R, int64_t off) {
  std::vector<Iter> d, r;
  for (auto &p : D) d.push_back(Iter{p.first, p.second, axis_m()});
  if (d.empty()) d.push_back(Iter{1, 1, axis_m()});
  for (auto &q : R) r.push_back(Iter{q.e, q.s, axis_m()});
  std::vector<std::pair<int, int64_t>> o;
  if (off) o.push_back({axis_m(), off});
  Layout L;
  make_layout(d, r, o, &L);
  return L;
}

Storage mstorage(int64_t cells, const Storage *swz_from) {
  Storage s;
  s.d.push_back(SDigit{axis_m(), cells, 1, 1});
  s.cells = cells;
  if (swz_from) {
    s.swz_b = swz_from->swz_b;
    s.swz_m = swz_from->swz_m;
    s.swz_s = swz_from->swz_s;
  }
  return s;
}

axe_status subplan(const Layout &src, const Storage &sst, const Layout &dst, const Storage &dstst, int es,
                   std::shared_ptr<CopyPlan> *out) {
  auto p = std::make_shared<CopyPlan>();
  PlanRequest rq{&src, &dst, &sst, &dstst, es, AXE_KERNEL_AUTO, 16, -1};
  AXE_TRY(plan_copy(rq, p.get()));
  *out = p;
  return AXE_OK;
}

}  // namespace

static axe_status plan_redist(const Layout &S, const Storage &sst, const Layout &T, const Storage &dstst, int es,
                              int nranks, int rank, axe_redist_plan *P) {
  const int g = axis_gpuid();
  if (es != 1 && es != 2 && es != 4 && es != 8 && es != 16)
    AXE_FAIL(AXE_ERR_ALIGNMENT, "elem_size %d not in {1,2,4,8,16}", es);
  if (nranks < 1 || rank < 0 || rank >= nranks) AXE_FAIL(AXE_ERR_INVALID_ARG, "bad rank %d of %d", rank, nranks);
  if (S.ED != T.ED) AXE_FAIL(AXE_ERR_SIZE_MISMATCH, "E_D(src) = %lld != E_D(dst) = %lld", (long long)S.ED, (long long)T.ED);
  AXE_TRY(check_side(S, sst, g, "source"));
  AXE_TRY(check_side(T, dstst, g, "destination"));
  for (const Layout *L : {&S, &T}) {
    int64_t mn, mx;
    axis_bounds(*L, g, &mn, &mx);
    if (mn < 0 || mx >= nranks)
      AXE_FAIL(AXE_ERR_BOUNDS, "%s layout reaches gpuid in [%lld, %lld] with %d ranks", L == &S ? "source" : "destination",
               (long long)mn, (long long)mx, nranks);
  }
  Linear ls, ld;
  if (!compose_linear(S, sst, g, &ls, true) || !compose_linear(T, dstst, g, &ld, true))
    AXE_FAIL(AXE_ERR_UNSUPPORTED, "redistribute needs affine storage compositions");
  std::vector<Joint> J;
  if (!joint_refine(ls.D, ld.D, &J))
    AXE_FAIL(AXE_ERR_UNSUPPORTED, "redistribute: the two digit systems are not nested");

  // destination injectivity over (rank, cell): cumulative separation on the combined index
  {
    std::vector<LinIter> all;
    for (auto *v : {&ld.D, &ld.R})
      for (auto &it : *v) all.push_back(LinIter{it.e, it.dev ? it.s * dstst.cells : it.s, 0});
    std::sort(all.begin(), all.end(), [](const LinIter &a, const LinIter &b) { return std::llabs(a.s) < std::llabs(b.s); });
    int64_t reach = 0;
    for (auto &it : all) {
      if (std::llabs(it.s) <= reach)
        AXE_FAIL(AXE_ERR_NONINJECTIVE, "redistribute: destination layout is not injective over (rank, cell)");
      reach += (it.e - 1) * std::llabs(it.s);
    }
  }

  // replicas: device-axis replica offsets (owners / receivers) and memory replicas of the destination
  std::vector<int64_t> own{0}, recvr{0};
  std::vector<LinIter> dst_mem_R;
  for (auto &r : ls.R)
    if (r.dev) {
      std::vector<int64_t> nx;
      for (int64_t b : own)
        for (int64_t d = 0; d < r.e; d++) nx.push_back(b + d * r.s);
      own.swap(nx);
    }
  for (auto &r : ld.R) {
    if (!r.dev) {
      dst_mem_R.push_back(r);
      continue;
    }
    std::vector<int64_t> nx;
    for (int64_t b : recvr)
      for (int64_t d = 0; d < r.e; d++) nx.push_back(b + d * r.s);
    recvr.swap(nx);
  }

  std::vector<Joint> G;
  for (auto &j : J) (j.sdev || j.ddev ? G : P->M).push_back(j);
  // packed order: destination order (largest |dst stride| outermost)
  std::stable_sort(P->M.begin(), P->M.end(), [](const Joint &a, const Joint &b) { return std::llabs(a.ds) > std::llabs(b.ds); });
  P->n = 1;
  for (auto &m : P->M) P->n *= m.e;
  P->packed.assign(P->M.size(), 1);
  for (int k = (int)P->M.size() - 2; k >= 0; k--) P->packed[k] = P->packed[k + 1] * P->M[k + 1].e;
  // wire chunks: cutting the outermost packed digit lets packing chunk c+1 overlap sending chunk c
  // (every chunk is a contiguous slice of the packed block on both sides of the wire)
  P->nchunk = 1;
  // (AXE_REDIST_CHUNK_BYTES lowers the 8 MiB minimum chunk, for tests)
  const char *cb = getenv("AXE_REDIST_CHUNK_BYTES");
  const int64_t min_chunk = (cb && *cb) ? atoll(cb) : (int64_t(8) << 20);
  if (!P->M.empty() && P->n * es >= 2 * min_chunk)
    for (int c : {4, 2})
      if (P->M[0].e % c == 0 && P->n * es / c >= min_chunk) {
        P->nchunk = c;
        break;
      }
  P->cn = P->n / P->nchunk;

  int64_t nblk = (int64_t)recvr.size();
  for (auto &j : G) nblk *= j.e;
  if (nblk > (1 << 20)) AXE_FAIL(AXE_ERR_UNSUPPORTED, "redistribute: %lld blocks", (long long)nblk);

  struct Blk {
    int snd, rcv;
    int64_t ms, md;
  };
  std::vector<Blk> blocks;
  std::vector<int64_t> egress(nranks, 0);
  std::vector<int64_t> dig(G.size(), 0);
  for (int64_t b = 0; b < (int64_t)(nblk / recvr.size()); b++) {
    int64_t rem = b, gs = ls.dev_base, ms = ls.base, gd0 = ld.dev_base, md = ld.base;
    for (int k = (int)G.size() - 1; k >= 0; k--) {
      int64_t d = rem % G[k].e;
      rem /= G[k].e;
      (G[k].sdev ? gs : ms) += d * G[k].ss;
      (G[k].ddev ? gd0 : md) += d * G[k].ds;
    }
    std::vector<int> owners;
    for (int64_t o : own) owners.push_back((int)(gs + o));
    std::sort(owners.begin(), owners.end());
    owners.erase(std::unique(owners.begin(), owners.end()), owners.end());
    for (int64_t r : recvr) {
      int gd = (int)(gd0 + r);
      int snd;
      if (std::find(owners.begin(), owners.end(), gd) != owners.end()) {
        snd = gd;
      } else {
        int dflt = owners[(size_t)gd % owners.size()];
        int best = dflt;
        for (int o : owners)
          if (egress[o] < egress[best]) best = o;
        snd = egress[best] + P->n <= egress[dflt] ? best : dflt;  // keep the default unless clearly unbalanced
        egress[snd] += P->n;
      }
      blocks.push_back(Blk{snd, gd, ms, md});
    }
  }

  P->nranks = nranks;
  P->rank = rank;
  P->es = es;
  for (auto &r : dst_mem_R) P->dst_rep *= r.e;
  P->src_cells = sst.cells;
  P->dst_cells = dstst.cells;
  // contiguity of a block on each side in packed order
  bool src_contig = !sst.swz_b, dst_contig = !dstst.swz_b && dst_mem_R.empty();
  for (size_t k = 0; k < P->M.size(); k++) {
    if (P->M[k].ss != P->packed[k]) src_contig = false;
    if (P->M[k].ds != P->packed[k]) dst_contig = false;
  }
  std::vector<std::pair<int64_t, int64_t>> Dsrc, Ddst, Dpk;
  for (size_t k = 0; k < P->M.size(); k++) {
    Dsrc.push_back({P->M[k].e, P->M[k].ss});
    Ddst.push_back({P->M[k].e, P->M[k].ds});
    Dpk.push_back({P->M[k].e, P->packed[k]});
  }
  // this rank's lists (block order within each peer is the global block order)
  for (auto &b : blocks) {
    Xfer x;
    x.ms = b.ms;
    x.md = b.md;
    if (b.snd == rank && b.rcv == rank) {
      x.peer = rank;
      P->locals.push_back(x);
    } else if (b.snd == rank) {
      x.peer = b.rcv;
      x.elided = src_contig;
      P->sends.push_back(x);
    } else if (b.rcv == rank) {
      x.peer = b.snd;
      x.elided = dst_contig;
      P->recvs.push_back(x);
    }
  }
  auto by_peer = [](const Xfer &a, const Xfer &b) { return a.peer < b.peer; };
  std::stable_sort(P->sends.begin(), P->sends.end(), by_peer);
  std::stable_sort(P->recvs.begin(), P->recvs.end(), by_peer);
  for (auto &x : P->sends)
    if (!x.elided) {
      x.stage = P->send_elems;
      P->send_elems += P->n;
    }
  for (auto &x : P->recvs)
    if (!x.elided) {
      x.stage = P->recv_elems;
      P->recv_elems += P->n;
    }
  Storage s_src = mstorage(sst.cells, &sst), s_dst = mstorage(dstst.cells, &dstst);
  Storage s_send = mstorage(std::max<int64_t>(1, P->send_elems), nullptr);
  Storage s_recv = mstorage(std::max<int64_t>(1, P->recv_elems), nullptr);
  // per-chunk pack / unpack plans: the outermost packed digit shrinks to e0 / nchunk
  std::vector<std::pair<int64_t, int64_t>> cDsrc = Dsrc, cDdst = Ddst, cDpk = Dpk;
  const int64_t ce0 = P->M.empty() ? 1 : P->M[0].e / P->nchunk;
  if (!P->M.empty()) cDsrc[0].first = cDdst[0].first = cDpk[0].first = ce0;
  for (auto &x : P->sends)
    if (!x.elided)
      for (int c = 0; c < P->nchunk; c++) {
        std::shared_ptr<CopyPlan> q;
        AXE_TRY(subplan(mlayout(cDsrc, {}, x.ms + (P->M.empty() ? 0 : c * ce0 * P->M[0].ss)), s_src,
                        mlayout(cDpk, {}, x.stage + c * P->cn), s_send, es, &q));
        x.cp.push_back(q);
      }
  for (auto &x : P->recvs)
    if (!x.elided)
      for (int c = 0; c < P->nchunk; c++) {
        std::shared_ptr<CopyPlan> q;
        AXE_TRY(subplan(mlayout(cDpk, {}, x.stage + c * P->cn), s_recv,
                        mlayout(cDdst, dst_mem_R, x.md + (P->M.empty() ? 0 : c * ce0 * P->M[0].ds)), s_dst, es, &q));
        x.cp.push_back(q);
      }
  for (auto &x : P->locals)
    AXE_TRY(subplan(mlayout(Dsrc, {}, x.ms), s_src, mlayout(Ddst, dst_mem_R, x.md), s_dst, es, &x.plan));
  // one-sided form (axe_redist_plan_execute_peers): every outgoing block is one copy kernel from
  // src_local straight into the receiver's dst_local (peer memory over NVLink) -- pack, wire and
  // unpack fused, no staging
  for (auto &x : P->sends)
    AXE_TRY(subplan(mlayout(Dsrc, {}, x.ms), s_src, mlayout(Ddst, dst_mem_R, x.md), s_dst, es, &x.plan));

  // all-gather pattern (decided from the global block list, so every rank agrees):
  // each rank r sends one contiguous block at the same offset to every other rank and
  // holds it locally; rank r's block lands contiguous at dst offset base + r * n everywhere.
  {
    bool ag = nranks > 1 && src_contig && dst_contig && (int64_t)blocks.size() == (int64_t)nranks * nranks;
    int64_t base = 0, soff = -1;
    if (ag) {
      std::map<std::pair<int, int>, const Blk *> m;
      for (auto &b : blocks) m[{b.snd, b.rcv}] = &b;
      if ((int)m.size() != nranks * nranks) ag = false;
      for (int r = 0; ag && r < nranks; r++)
        for (int q = 0; ag && q < nranks; q++) {
          const Blk *b = m[{r, q}];
          if (!b) {
            ag = false;
            break;
          }
          if (r == 0 && q == 0) {
            base = b->md;
            soff = b->ms;
          }
          if (b->ms != soff || b->md != base + (int64_t)r * P->n) ag = false;
        }
    }
    if (ag) {
      P->allgather = true;
      P->ag_src = soff;
      P->ag_dst = base;
    }
  }
  char buf[512];
  int64_t sc = 0, rc = 0;
  for (auto &x : P->sends) sc += P->n;
  for (auto &x : P->recvs) rc += P->n;
  int ps = 0, pu = 0;
  for (auto &x : P->sends) ps += !x.elided;
  for (auto &x : P->recvs) pu += !x.elided;
  snprintf(buf, sizeof buf,
           "{\"pattern\":\"%s\",\"nranks\":%d,\"rank\":%d,\"block_elems\":%lld,\"blocks\":%lld,\"sends\":%zu,"
           "\"recvs\":%zu,\"locals\":%zu,\"send_elems\":%lld,\"recv_elems\":%lld,\"packs\":%d,\"unpacks\":%d,"
           "\"owner_replicas\":%zu,\"receiver_replicas\":%zu,\"wire_chunks\":%d}",
           P->allgather ? "allgather" : (P->sends.empty() && P->recvs.empty() ? "local" : "exchange"), nranks, rank,
           (long long)P->n, (long long)blocks.size(), P->sends.size(), P->recvs.size(), P->locals.size(), (long long)sc,
           (long long)rc, ps, pu, own.size(), recvr.size(), P->nchunk);
  P->desc = buf;
  return AXE_OK;
}

// The pull form of a single-phase reduction: every block this rank's stage receives (or copies
// locally) is summand k = md / C of the destination cells md mod C.  Blocks sharing those cells
// form one region; a region with exactly one block per k becomes one K4 launch whose summand k is
// read at senders[k]'s src buffer (peer memory) -- exchange, staging and sum fused in one kernel.
static void build_pull(const axe_redist_plan &in, int64_t K, int64_t C, const Storage &sst, const Storage &dstst,
                       int dtype, int es, axe_redist_plan *P) {
  auto no = [&](const char *w) {
    P->pulls.clear();
    P->pull_why = w;
  };
  if (K > K4_MAXK) return no("more than 256 summands");
  if (in.dst_rep != 1) return no("destination memory replicas");
  int64_t lo = 0, hi = 0;  // stage offsets reached by the sub-box
  for (auto &m : in.M) (m.ds < 0 ? lo : hi) += (m.e - 1) * m.ds;
  struct Ent {
    int64_t k;
    int q;
    int64_t ms;
  };
  std::map<int64_t, std::vector<Ent>> groups;
  for (int pass = 0; pass < 2; pass++)
    for (auto &x : pass == 0 ? in.locals : in.recvs) {
      const int64_t k = x.md / C, r0 = x.md % C;
      if (r0 + lo < 0 || r0 + hi >= C) return no("a block straddles two stage slabs");
      groups[r0].push_back(Ent{k, pass == 0 ? in.rank : x.peer, x.ms});
    }
  // vector width over the sub-box (as K4: innermost digit contiguous on both sides)
  std::vector<Joint> Y;
  for (auto &m : in.M)
    if (m.e > 1) Y.push_back(m);
  int64_t V = 1;
  if (!Y.empty() && Y.back().ss == 1 && Y.back().ds == 1) {
    std::vector<int64_t> all;
    for (size_t k = 0; k + 1 < Y.size(); k++) {
      all.push_back(Y[k].ss);
      all.push_back(Y[k].ds);
    }
    for (auto &g : groups) {
      all.push_back(g.first);
      for (auto &e : g.second) all.push_back(e.ms);
    }
    int64_t cap = 16 / es;
    if (sst.swz_b > 0) cap = std::min<int64_t>(cap, std::max<int64_t>(1, (int64_t(1) << sst.swz_m) / es));
    if (dstst.swz_b > 0) cap = std::min<int64_t>(cap, std::max<int64_t>(1, (int64_t(1) << dstst.swz_m) / es));
    for (int64_t v = 2; v <= cap; v *= 2) {
      bool ok = Y.back().e % v == 0;
      for (int64_t a : all) ok = ok && a % v == 0;
      if (ok) V = v;
    }
  }
  if (V > 1) {
    Joint last = Y.back();
    Y.pop_back();
    if (last.e / V > 1) Y.push_back(Joint{last.e / V, V, V});
  }
  if ((int)Y.size() > K4_MAXD) return no("too many sub-box digits");
  int64_t total = 1;
  for (auto &j : Y) total *= j.e;
  if (total >= (int64_t(1) << 31)) return no("2^31 or more vectors per region");
  for (auto &g : groups) {
    std::vector<Ent> v = g.second;
    std::sort(v.begin(), v.end(), [](const Ent &a, const Ent &b) { return a.k < b.k; });
    if ((int64_t)v.size() != K) return no("a region does not receive exactly K summands");
    for (int64_t k = 0; k < K; k++)
      if (v[k].k != k) return no("a region receives a summand twice");
    axe_redist_plan::Pull pl;
    K4Params &kp = pl.k;
    memset(&kp, 0, sizeof(kp));
    kp.total = (uint32_t)total;
    kp.nd = (int)Y.size();
    for (int i = 0; i < kp.nd; i++) {
      kp.fd[i] = make_fastdiv((uint32_t)Y[i].e);
      kp.ss[i] = Y[i].ss * es;
      kp.ds[i] = Y[i].ds * es;
    }
    kp.nk = (int)K;
    for (int64_t k = 0; k < K; k++) {
      kp.koff[k] = v[k].ms * es;
      pl.senders.push_back(v[k].q);
    }
    kp.sbase = 0;
    kp.dbase = g.first * es;
    kp.nrep = 1;
    kp.rep[0] = 0;
    kp.ssw = make_swz(sst);
    kp.dsw = make_swz(dstst);
    P->pulls.push_back(pl);
  }
  P->pull_vb = (int)(V * es);
  // NVLS: a multicast load at one offset reduces over every rank's buffer, so each region must take
  // exactly one partial from every rank, all at the same source offset; 16-byte float vectors
  P->multicast_ok = (dtype == DT_F32 || dtype == DT_BF16 || dtype == DT_F16) && V * es == 16 &&
                    K == in.nranks && !sst.swz_b;
  for (auto &pl : P->pulls) {
    std::vector<int> seen(in.nranks, 0);
    for (size_t k = 0; k < pl.senders.size(); k++) {
      seen[pl.senders[k]]++;
      if (pl.k.koff[k] != pl.k.koff[0]) P->multicast_ok = false;
    }
    for (int c : seen)
      if (c != 1) P->multicast_ok = false;
  }
  const int64_t blocks = (total + 255) / 256, cap = (int64_t)num_sms() * 8;
  P->pull_blocks = (unsigned)std::max<int64_t>(1, std::min(blocks, cap));
}

// Reduce-redistribute (reading R24): dst(y) = sum_k src(k E_D(dst) + y).
// Phase 1 redistributes the source (its K partials) into a stage layout -- the destination
// layout with the summed dimension prepended on a private storage axis, so rank g's stage
// buffer holds K slabs shaped exactly like its dst storage.  Phase 2 sums the slabs cell by
// cell in k order (K4).  A swizzle permutes every slab identically (the slab is a whole number
// of swizzle blocks), so phase 2 is a flat elementwise sum.  Every rank's destination image
// must be its whole dst storage (checked), or phase 2 would write cells outside the image.
static axe_status plan_redist_reduce_1(const Layout &S, const Storage &sst, const Layout &T, const Storage &dstst,
                                       int dtype, int nranks, int rank, axe_redist_plan *P) {
  const int es = dtype_size(dtype);
  if (!es) AXE_FAIL(AXE_ERR_INVALID_ARG, "unknown dtype %d", dtype);
  if (S.ED % T.ED)
    AXE_FAIL(AXE_ERR_SIZE_MISMATCH, "E_D(src) = %lld is not a multiple of E_D(dst) = %lld", (long long)S.ED,
             (long long)T.ED);
  const int64_t K = S.ED / T.ED;
  const int ak = intern_axis("axe_reduce_k");
  if (T.names_axis(ak) || S.names_axis(ak)) AXE_FAIL(AXE_ERR_INVALID_ARG, "axis name axe_reduce_k is reserved");
  if (dstst.swz_b > 0 && (dstst.cells * es) % (int64_t(1) << (dstst.swz_b + dstst.swz_m + dstst.swz_s)))
    AXE_FAIL(AXE_ERR_BOUNDS, "swizzled destination storage is not a whole number of swizzle blocks");
  Layout T2;
  std::vector<Iter> d2 = T.D;
  d2.insert(d2.begin(), Iter{K, 1, ak});
  AXE_TRY(make_layout(d2, T.R, T.O, &T2));
  Storage st2 = dstst;
  st2.d.insert(st2.d.begin(), SDigit{ak, K, 1, dstst.cells});
  st2.cells = K * dstst.cells;
  auto in = std::make_shared<axe_redist_plan>();
  AXE_TRY(plan_redist(S, sst, T2, st2, es, nranks, rank, in.get()));
  const int64_t covered = (int64_t)(in->locals.size() + in->recvs.size()) * in->n * in->dst_rep;
  if (covered != st2.cells)
    AXE_FAIL(AXE_ERR_UNSUPPORTED,
             "reduce-redistribute: rank %d's destination image (%lld of %lld cells) must be its whole storage", rank,
             (long long)(covered / std::max<int64_t>(1, K)), (long long)dstst.cells);
  // phase 2: (K, C):(C, 1) -> (C):(1) on flat storages
  const int64_t C = dstst.cells;
  Layout a, b;
  std::vector<Iter> da{Iter{C, 1, axis_m()}};
  if (K > 1) da.insert(da.begin(), Iter{K, C, axis_m()});
  AXE_TRY(make_layout(da, {}, {}, &a));
  AXE_TRY(make_layout({Iter{C, 1, axis_m()}}, {}, {}, &b));
  AXE_TRY(plan_reduce(a, mstorage(K * C, nullptr), b, mstorage(C, nullptr), dtype, 16, &P->red));
  P->inner = in;
  P->nranks = nranks;
  P->rank = rank;
  P->es = es;
  P->src_cells = sst.cells;
  P->dst_cells = dstst.cells;
  P->stage_bytes = K * C * es;
  build_pull(*in, K, C, sst, dstst, dtype, es, P);
  P->desc = "{\"pattern\":\"reduce\",\"K\":" + std::to_string(K) + ",\"exchange\":" + in->desc +
            ",\"reduce\":" + P->red.desc + ",\"pull_regions\":" + std::to_string(P->pulls.size()) +
            ",\"pull_vec_bytes\":" + std::to_string(P->pull_vb) + ",\"multicast\":" +
            (P->multicast_ok ? "true" : "false") + "}";
  return AXE_OK;
}

// A destination replicated over R >= 3 ranks would receive every partial on every replica
// ((P-1) partials of wire per GPU); instead reduce-scatter into an even shard of the logical
// range, (P, E_D/P):(1@gpuid, 1@m), and redistribute that (an all-gather for a row-major
// replicated destination): 2(P-1)/P of a partial per GPU, as a ring all-reduce.
static axe_status plan_redist_reduce(const Layout &S, const Storage &sst, const Layout &T, const Storage &dstst,
                                     int dtype, int nranks, int rank, axe_redist_plan *P) {
  const int g = axis_gpuid();
  int64_t reps = 1;
  for (auto &it : T.R)
    if (it.a == g) reps *= it.e;
  const int es = dtype_size(dtype);
  if (reps < 3 || nranks < 3 || T.ED % nranks || !es)
    return plan_redist_reduce_1(S, sst, T, dstst, dtype, nranks, rank, P);
  Layout Tt;
  AXE_TRY(make_layout({Iter{nranks, 1, g}, Iter{T.ED / nranks, 1, axis_m()}}, {}, {}, &Tt));
  const Storage tst = mstorage(T.ED / nranks, nullptr);
  auto A = std::make_shared<axe_redist_plan>(), B = std::make_shared<axe_redist_plan>();
  AXE_TRY(plan_redist_reduce_1(S, sst, Tt, tst, dtype, nranks, rank, A.get()));
  AXE_TRY(plan_redist(Tt, tst, T, dstst, es, nranks, rank, B.get()));
  P->phase_a = A;
  P->phase_b = B;
  P->nranks = nranks;
  P->rank = rank;
  P->es = es;
  P->src_cells = sst.cells;
  P->dst_cells = dstst.cells;
  P->tmp_bytes = tst.cells * es;
  P->desc = "{\"pattern\":\"reduce_scatter_allgather\",\"K\":" + std::to_string(S.ED / T.ED) +
            ",\"phase_a\":" + A->desc + ",\"phase_b\":" + B->desc + "}";
  return AXE_OK;
}

static axe_status ensure_stage(const axe_redist_plan *P) {
  std::lock_guard<std::mutex> lk(P->mu);
  cudaError_t e = cudaSuccess;
  if (!P->stage && P->stage_bytes) e = cudaMalloc(&P->stage, (size_t)P->stage_bytes);
  if (e == cudaSuccess && !P->tmp && P->tmp_bytes) e = cudaMalloc(&P->tmp, (size_t)P->tmp_bytes);
  if (e != cudaSuccess) AXE_FAIL(AXE_ERR_CUDA, "reduce staging: %s", cudaGetErrorString(e));
  return AXE_OK;
}

static axe_status ensure_scratch(const axe_redist_plan *P) {
  std::lock_guard<std::mutex> lk(P->mu);
  cudaError_t e = cudaSuccess;
  if (!P->send_buf && P->send_elems) e = cudaMalloc(&P->send_buf, (size_t)(P->send_elems * P->es));
  if (e == cudaSuccess && !P->recv_buf && P->recv_elems) e = cudaMalloc(&P->recv_buf, (size_t)(P->recv_elems * P->es));
  if (e == cudaSuccess && !P->side) e = cudaStreamCreateWithFlags(&P->side, cudaStreamNonBlocking);
  if (e == cudaSuccess && !P->ev_fork) e = cudaEventCreateWithFlags(&P->ev_fork, cudaEventDisableTiming);
  if (e == cudaSuccess && !P->ev_join) e = cudaEventCreateWithFlags(&P->ev_join, cudaEventDisableTiming);
  if (e == cudaSuccess && !P->ev_join2) e = cudaEventCreateWithFlags(&P->ev_join2, cudaEventDisableTiming);
  if (e == cudaSuccess && !P->pk) e = cudaStreamCreateWithFlags(&P->pk, cudaStreamNonBlocking);
  if (e == cudaSuccess && !P->up) e = cudaStreamCreateWithFlags(&P->up, cudaStreamNonBlocking);
  while (e == cudaSuccess && (int)P->ev_pack.size() < P->nchunk) {
    cudaEvent_t a = nullptr, b = nullptr;
    e = cudaEventCreateWithFlags(&a, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&b, cudaEventDisableTiming);
    P->ev_pack.push_back(a);
    P->ev_recv.push_back(b);
  }
  if (e != cudaSuccess) AXE_FAIL(AXE_ERR_CUDA, "redistribute scratch: %s", cudaGetErrorString(e));
  return AXE_OK;
}

#define NCCL_TRY(call)                                                                  \
  do {                                                                                  \
    ncclResult_t _r = (call);                                                           \
    if (_r != ncclSuccess) AXE_FAIL(AXE_ERR_NCCL, "%s: %s", #call, ncclGetErrorString(_r)); \
  } while (0)

static axe_status exec_redist(const axe_redist_plan *P, axe_comm *C, const void *src, void *dst, cudaStream_t st) {
  if (!C || !C->comm) AXE_FAIL(AXE_ERR_INVALID_ARG, "no communicator");
  if (P->phase_a) {  // two-phase reduction: reduce-scatter into tmp, then redistribute tmp
    AXE_TRY(ensure_stage(P));
    AXE_TRY(exec_redist(P->phase_a.get(), C, src, P->tmp, st));
    return exec_redist(P->phase_b.get(), C, P->tmp, dst, st);
  }
  if (P->inner) {  // reduce-redistribute: partials -> stage (exchange), then the slab sum
    AXE_TRY(ensure_stage(P));
    AXE_TRY(exec_redist(P->inner.get(), C, src, P->stage, st));
    return run_reduce(P->red, P->stage, dst, st);
  }
  if (C->nranks != P->nranks || C->rank != P->rank)
    AXE_FAIL(AXE_ERR_INVALID_ARG, "plan for rank %d/%d used on comm rank %d/%d", P->rank, P->nranks, C->rank, C->nranks);
  const uint8_t *s = (const uint8_t *)src;
  uint8_t *d = (uint8_t *)dst;
  const size_t bytes = (size_t)(P->n * P->es);
  if (P->allgather) {
    Nvtx r("axe.redist.allgather");
    NCCL_TRY(ncclAllGather(s + P->ag_src * P->es, d + P->ag_dst * P->es, bytes, ncclUint8, C->comm, st));
    stream_forget(st);
    return AXE_OK;
  }
  AXE_TRY(ensure_scratch(P));
  cudaError_t e = cudaSuccess;
#define CU_TRY(x)                                                                        \
  do {                                                                                   \
    e = (x);                                                                             \
    if (e != cudaSuccess) AXE_FAIL(AXE_ERR_CUDA, "%s: %s", #x, cudaGetErrorString(e));   \
  } while (0)
  bool packs = false, unpacks = false;
  for (auto &x : P->sends) packs |= !x.elided;
  for (auto &x : P->recvs) unpacks |= !x.elided;
  CU_TRY(cudaEventRecord(P->ev_fork, st));
  // local copies on a side stream, overlapping pack + exchange
  if (!P->locals.empty()) {
    Nvtx r("axe.redist.local");
    CU_TRY(cudaStreamWaitEvent(P->side, P->ev_fork, 0));
    stream_forget(P->side);
    for (auto &x : P->locals) AXE_TRY(run_copy(*x.plan, src, dst, P->side));
  }
  // packs, chunk by chunk, on the pack stream
  if (packs) {
    Nvtx r("axe.redist.pack");
    CU_TRY(cudaStreamWaitEvent(P->pk, P->ev_fork, 0));
    stream_forget(P->pk);
    for (int c = 0; c < P->nchunk; c++) {
      for (auto &x : P->sends)
        if (!x.elided) AXE_TRY(run_copy(*x.cp[c], src, P->send_buf, P->pk));
      CU_TRY(cudaEventRecord(P->ev_pack[c], P->pk));
    }
  }
  if (unpacks) {
    CU_TRY(cudaStreamWaitEvent(P->up, P->ev_fork, 0));
  }
  // the wire: one NCCL group per chunk (chunk c of every block), after that chunk is packed
  const size_t cbytes = (size_t)(P->cn * P->es);
  Nvtx wire("axe.redist.wire+unpack");
  for (int c = 0; c < P->nchunk; c++) {
    if (packs) CU_TRY(cudaStreamWaitEvent(st, P->ev_pack[c], 0));
    NCCL_TRY(ncclGroupStart());
    for (auto &x : P->sends) {
      const uint8_t *ptr = x.elided ? s + (x.ms + (P->M.empty() ? 0 : c * (P->M[0].e / P->nchunk) * P->M[0].ss)) * P->es
                                    : (const uint8_t *)P->send_buf + (x.stage + c * P->cn) * P->es;
      NCCL_TRY(ncclSend(ptr, cbytes, ncclUint8, x.peer, C->comm, st));
    }
    for (auto &x : P->recvs) {
      uint8_t *ptr = x.elided ? d + (x.md + (P->M.empty() ? 0 : c * (P->M[0].e / P->nchunk) * P->M[0].ds)) * P->es
                              : (uint8_t *)P->recv_buf + (x.stage + c * P->cn) * P->es;
      NCCL_TRY(ncclRecv(ptr, cbytes, ncclUint8, x.peer, C->comm, st));
    }
    NCCL_TRY(ncclGroupEnd());
    if (unpacks) {
      CU_TRY(cudaEventRecord(P->ev_recv[c], st));
      CU_TRY(cudaStreamWaitEvent(P->up, P->ev_recv[c], 0));
      stream_forget(P->up);  // full dependency on the NCCL kernels that filled this chunk
      for (auto &x : P->recvs)
        if (!x.elided) AXE_TRY(run_copy(*x.cp[c], P->recv_buf, dst, P->up));
    }
  }
  stream_forget(st);
  if (!P->locals.empty()) {
    CU_TRY(cudaEventRecord(P->ev_join, P->side));
    CU_TRY(cudaStreamWaitEvent(st, P->ev_join, 0));
  }
  if (unpacks) {
    CU_TRY(cudaEventRecord(P->ev_join2, P->up));
    CU_TRY(cudaStreamWaitEvent(st, P->ev_join2, 0));
  }
#undef CU_TRY
  return AXE_OK;
}

// NCCL reports errors of kernels already enqueued (a peer that died, a network failure) only
// asynchronously: checked before and after every enqueue on the communicator.
static axe_status comm_check(axe_comm *C) {
  if (!C) return AXE_OK;
  if (C->aborted || !C->comm) AXE_FAIL(AXE_ERR_NCCL, "communicator was aborted (axe_comm_wait)");
  ncclResult_t ar = ncclSuccess;
  const ncclResult_t r = ncclCommGetAsyncError(C->comm, &ar);
  if (r != ncclSuccess) AXE_FAIL(AXE_ERR_NCCL, "ncclCommGetAsyncError: %s", ncclGetErrorString(r));
  if (ar != ncclSuccess && ar != ncclInProgress)
    AXE_FAIL(AXE_ERR_NCCL, "asynchronous NCCL error: %s", ncclGetErrorString(ar));
  return AXE_OK;
}

// Every public execute of a plan: one at a time on the host (exec_mu, and the communicator's lock when
// it enqueues NCCL work), and on the device after the previous execute of the same plan (ev_done) --
// executes on different streams would otherwise share the plan's staging buffers and side streams.
template <class F>
static axe_status serialized(const axe_redist_plan *P, axe_comm *C, cudaStream_t st, F &&fn) {
  std::lock_guard<std::mutex> lk(P->exec_mu);
  std::unique_lock<std::mutex> ck;
  if (C) ck = std::unique_lock<std::mutex>(C->mu);
  AXE_TRY(comm_check(C));
  if (P->done_valid) {
    const cudaError_t e = cudaStreamWaitEvent(st, P->ev_done, 0);
    if (e != cudaSuccess) AXE_FAIL(AXE_ERR_CUDA, "cudaStreamWaitEvent: %s", cudaGetErrorString(e));
    stream_forget(st);
  }
  AXE_TRY(fn());
  if (!P->ev_done) {
    const cudaError_t e = cudaEventCreateWithFlags(&P->ev_done, cudaEventDisableTiming);
    if (e != cudaSuccess) AXE_FAIL(AXE_ERR_CUDA, "cudaEventCreate: %s", cudaGetErrorString(e));
  }
  const cudaError_t e = cudaEventRecord(P->ev_done, st);
  if (e != cudaSuccess) AXE_FAIL(AXE_ERR_CUDA, "cudaEventRecord: %s", cudaGetErrorString(e));
  P->done_valid = true;
  return comm_check(C);
}

extern "C" {

axe_status axe_get_unique_id(uint8_t out[128]) {
  if (!out) AXE_FAIL(AXE_ERR_INVALID_ARG, "out is NULL");
  static_assert(sizeof(ncclUniqueId) == 128, "NCCL unique id size");
  ncclUniqueId id;
  NCCL_TRY(ncclGetUniqueId(&id));
  memcpy(out, &id, 128);
  return AXE_OK;
}

axe_status axe_comm_create(const uint8_t id[128], int nranks, int rank, int cuda_device, axe_comm **out) {
  if (!id || !out) AXE_FAIL(AXE_ERR_INVALID_ARG, "NULL argument");
  *out = nullptr;
  if (nranks < 1 || rank < 0 || rank >= nranks) AXE_FAIL(AXE_ERR_INVALID_ARG, "bad rank %d of %d", rank, nranks);
  cudaError_t e = cudaSetDevice(cuda_device);
  if (e != cudaSuccess) AXE_FAIL(AXE_ERR_CUDA, "cudaSetDevice(%d): %s", cuda_device, cudaGetErrorString(e));
  ncclUniqueId uid;
  memcpy(&uid, id, 128);
  auto *c = new axe_comm;
  ncclResult_t r = ncclCommInitRank(&c->comm, nranks, uid, rank);
  if (r != ncclSuccess) {
    delete c;
    AXE_FAIL(AXE_ERR_NCCL, "ncclCommInitRank: %s", ncclGetErrorString(r));
  }
  c->nranks = nranks;
  c->rank = rank;
  c->device = cuda_device;
  *out = c;
  return AXE_OK;
}

void axe_comm_destroy(axe_comm *c) {
  if (!c) return;
  if (c->comm) {
    if (c->aborted) ncclCommAbort(c->comm);
    else ncclCommDestroy(c->comm);
  }
  delete c;
}

axe_status axe_comm_wait(axe_comm *c, void *stream, int timeout_ms) {
  if (!c) AXE_FAIL(AXE_ERR_INVALID_ARG, "comm is NULL");
  cudaStream_t st = (cudaStream_t)stream;
  const auto t0 = std::chrono::steady_clock::now();
  for (;;) {
    const cudaError_t q = cudaStreamQuery(st);
    if (q != cudaSuccess && q != cudaErrorNotReady) AXE_FAIL(AXE_ERR_CUDA, "cudaStreamQuery: %s", cudaGetErrorString(q));
    {
      std::lock_guard<std::mutex> lk(c->mu);
      const axe_status a = comm_check(c);
      if (a != AXE_OK) {
        if (c->comm && !c->aborted) {
          ncclCommAbort(c->comm);  // unblocks the NCCL kernels waiting on the failed peer
          c->comm = nullptr;
          c->aborted = true;
        }
        return a;
      }
    }
    if (q == cudaSuccess) return AXE_OK;
    const auto ms = std::chrono::duration_cast<std::chrono::milliseconds>(std::chrono::steady_clock::now() - t0);
    if (timeout_ms >= 0 && ms.count() >= timeout_ms) {
      std::lock_guard<std::mutex> lk(c->mu);
      if (c->comm && !c->aborted) {
        ncclCommAbort(c->comm);
        c->comm = nullptr;
        c->aborted = true;
      }
      AXE_FAIL(AXE_ERR_TIMEOUT, "stream not done after %d ms: communicator aborted", timeout_ms);
    }
    std::this_thread::sleep_for(std::chrono::microseconds(50));
  }
}

// ---------------------------------------------------------------- CUDA IPC (one-sided forms)
// A handle = cudaIpcMemHandle_t of the allocation holding the pointer (64 bytes) + the pointer's
// byte offset inside that allocation (the caching allocators of frameworks sub-allocate).
typedef CUresult (*PFN_getAddressRange)(CUdeviceptr *, size_t *, CUdeviceptr);
static std::mutex g_ipc_mu;
static std::map<void *, void *> g_ipc_open;  // imported pointer -> mapped allocation base

axe_status axe_ipc_export(const void *dev_ptr, uint8_t handle[128]) {
  if (!dev_ptr || !handle) AXE_FAIL(AXE_ERR_INVALID_ARG, "NULL argument");
  static PFN_getAddressRange range = [] {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return (PFN_getAddressRange)p;
  }();
  if (!range) AXE_FAIL(AXE_ERR_CUDA, "cuMemGetAddressRange unavailable");
  CUdeviceptr base = 0;
  size_t size = 0;
  if (range(&base, &size, (CUdeviceptr)(uintptr_t)dev_ptr) != CUDA_SUCCESS)
    AXE_FAIL(AXE_ERR_INVALID_ARG, "not a device allocation");
  cudaIpcMemHandle_t h;
  const cudaError_t e = cudaIpcGetMemHandle(&h, (void *)(uintptr_t)base);
  if (e != cudaSuccess) AXE_FAIL(AXE_ERR_CUDA, "cudaIpcGetMemHandle: %s", cudaGetErrorString(e));
  static_assert(sizeof(h) == 64, "IPC handle size");
  memset(handle, 0, 128);
  memcpy(handle, &h, 64);
  const int64_t off = (int64_t)((uintptr_t)dev_ptr - (uintptr_t)base);
  memcpy(handle + 64, &off, 8);
  return AXE_OK;
}

axe_status axe_ipc_import(const uint8_t handle[128], void **dev_ptr) {
  if (!handle || !dev_ptr) AXE_FAIL(AXE_ERR_INVALID_ARG, "NULL argument");
  *dev_ptr = nullptr;
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, 64);
  int64_t off = 0;
  memcpy(&off, handle + 64, 8);
  void *base = nullptr;
  const cudaError_t e = cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess);
  if (e != cudaSuccess) AXE_FAIL(AXE_ERR_CUDA, "cudaIpcOpenMemHandle: %s", cudaGetErrorString(e));
  void *p = (uint8_t *)base + off;
  std::lock_guard<std::mutex> lk(g_ipc_mu);
  g_ipc_open[p] = base;
  *dev_ptr = p;
  return AXE_OK;
}

axe_status axe_ipc_close(void *dev_ptr) {
  std::lock_guard<std::mutex> lk(g_ipc_mu);
  auto it = g_ipc_open.find(dev_ptr);
  if (it == g_ipc_open.end()) AXE_FAIL(AXE_ERR_INVALID_ARG, "pointer was not imported by axe_ipc_import");
  const cudaError_t e = cudaIpcCloseMemHandle(it->second);
  g_ipc_open.erase(it);
  if (e != cudaSuccess) AXE_FAIL(AXE_ERR_CUDA, "cudaIpcCloseMemHandle: %s", cudaGetErrorString(e));
  return AXE_OK;
}

axe_status axe_redist_plan_create(const axe_layout *src, const axe_storage *src_st, const axe_layout *dst,
                                  const axe_storage *dst_st, int elem_size, int nranks, int rank,
                                  axe_redist_plan **out) {
  if (!src || !dst || !out) AXE_FAIL(AXE_ERR_INVALID_ARG, "NULL argument");
  *out = nullptr;
  Storage ss, ds;
  AXE_TRY(make_storage(src_st, &ss));
  AXE_TRY(make_storage(dst_st, &ds));
  auto *p = new axe_redist_plan;
  axe_status st = plan_redist(src->L, ss, dst->L, ds, elem_size, nranks, rank, p);
  if (st != AXE_OK) {
    delete p;
    return st;
  }
  *out = p;
  return AXE_OK;
}

axe_status axe_redist_reduce_plan_create(const axe_layout *src, const axe_storage *src_st, const axe_layout *dst,
                                         const axe_storage *dst_st, int dtype, int nranks, int rank,
                                         axe_redist_plan **out) {
  if (!src || !dst || !out) AXE_FAIL(AXE_ERR_INVALID_ARG, "NULL argument");
  *out = nullptr;
  Storage ss, ds;
  AXE_TRY(make_storage(src_st, &ss));
  AXE_TRY(make_storage(dst_st, &ds));
  auto *p = new axe_redist_plan;
  axe_status st = plan_redist_reduce(src->L, ss, dst->L, ds, dtype, nranks, rank, p);
  if (st != AXE_OK) {
    delete p;
    return st;
  }
  *out = p;
  return AXE_OK;
}

axe_status axe_redistribute_reduce(const axe_layout *src, const axe_storage *src_st, const void *src_local,
                                   const axe_layout *dst, const axe_storage *dst_st, void *dst_local, int dtype,
                                   axe_comm *comm, void *stream) {
  if (!comm) AXE_FAIL(AXE_ERR_INVALID_ARG, "comm is NULL");
  if (!src || !dst) AXE_FAIL(AXE_ERR_INVALID_ARG, "NULL layout");
  static std::mutex mu;
  static std::unordered_map<std::string, std::shared_ptr<axe_redist_plan>> cache;
  Storage ss, ds;
  AXE_TRY(make_storage(src_st, &ss));
  AXE_TRY(make_storage(dst_st, &ds));
  const std::string key = layout_key(src->L) + "#" + storage_key(ss) + "#" + layout_key(dst->L) + "#" +
                          storage_key(ds) + "#" + std::to_string(dtype) + "#" + std::to_string(comm->nranks) + "#" +
                          std::to_string(comm->rank) + "#" + std::to_string((uintptr_t)comm);
  std::shared_ptr<axe_redist_plan> p;
  {
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find(key);
    if (it != cache.end()) p = it->second;
  }
  if (!p) {
    p = std::make_shared<axe_redist_plan>();
    AXE_TRY(plan_redist_reduce(src->L, ss, dst->L, ds, dtype, comm->nranks, comm->rank, p.get()));
    std::lock_guard<std::mutex> lk(mu);
    if (cache.size() >= 256) cache.clear();  // (plans hold staging memory; callers keep their own copies)
    cache[key] = p;
  }
  return serialized(p.get(), comm, (cudaStream_t)stream,
                    [&] { return exec_redist(p.get(), comm, src_local, dst_local, (cudaStream_t)stream); });
}

axe_status axe_redist_plan_execute(const axe_redist_plan *plan, axe_comm *comm, const void *src_local, void *dst_local,
                                   void *stream) {
  if (!plan) AXE_FAIL(AXE_ERR_INVALID_ARG, "plan is NULL");
  return serialized(plan, comm, (cudaStream_t)stream,
                    [&] { return exec_redist(plan, comm, src_local, dst_local, (cudaStream_t)stream); });
}

axe_status axe_redist_plan_execute_peers(const axe_redist_plan *plan, const void *src_local, void *const *dst_peers,
                                         void *stream) {
  if (!plan || !src_local || !dst_peers) AXE_FAIL(AXE_ERR_INVALID_ARG, "NULL argument");
  if (plan->inner || plan->phase_a)
    AXE_FAIL(AXE_ERR_UNSUPPORTED, "execute_peers: reduce plans stage through library memory");
  for (int r = 0; r < plan->nranks; r++)
    if (!dst_peers[r]) AXE_FAIL(AXE_ERR_INVALID_ARG, "dst_peers[%d] is NULL", r);
  cudaStream_t st = (cudaStream_t)stream;
  // remote blocks first (they cross NVLink), then the local ones
  for (auto &x : plan->sends) AXE_TRY(run_copy(*x.plan, src_local, dst_peers[x.peer], st));
  for (auto &x : plan->locals) AXE_TRY(run_copy(*x.plan, src_local, dst_peers[plan->rank], st));
  return AXE_OK;
}

axe_status axe_redist_plan_execute_peers_reduce(const axe_redist_plan *plan, const void *const *src_peers,
                                                void *dst_local, void *stream) {
  if (!plan || !src_peers || !dst_local) AXE_FAIL(AXE_ERR_INVALID_ARG, "NULL argument");
  if (!plan->inner) AXE_FAIL(AXE_ERR_UNSUPPORTED, "execute_peers_reduce: not a single-phase reduction plan");
  if (plan->pulls.empty()) AXE_FAIL(AXE_ERR_UNSUPPORTED, "execute_peers_reduce: %s", plan->pull_why.c_str());
  for (int r = 0; r < plan->nranks; r++)
    if (!src_peers[r]) AXE_FAIL(AXE_ERR_INVALID_ARG, "src_peers[%d] is NULL", r);
  if ((uintptr_t)dst_local % plan->pull_vb) AXE_FAIL(AXE_ERR_ALIGNMENT, "dst_local is not %d-byte aligned", plan->pull_vb);
  cudaStream_t st = (cudaStream_t)stream;
  stream_forget(st);  // peer buffers: no byte-range bookkeeping, full dependency
  for (auto &pl : plan->pulls) {
    K4Ptrs q;
    for (size_t k = 0; k < pl.senders.size(); k++) {
      q.p[k] = (uint64_t)(uintptr_t)src_peers[pl.senders[k]];
      if (q.p[k] % plan->pull_vb) AXE_FAIL(AXE_ERR_ALIGNMENT, "src_peers[%d] is not %d-byte aligned", pl.senders[k], plan->pull_vb);
    }
    K4Params k = pl.k;
    k.dep = 1;
    cudaError_t e = launch_k4_peer(k, q, plan->red.dtype, plan->pull_vb, plan->pull_blocks, dst_local, st);
    if (e != cudaSuccess) AXE_FAIL(AXE_ERR_CUDA, "pull reduce launch: %s", cudaGetErrorString(e));
  }
  stream_forget(st);
  return AXE_OK;
}

axe_status axe_redist_plan_execute_multicast_reduce(const axe_redist_plan *plan, const void *src_multicast,
                                                    void *dst_local, void *stream) {
  if (!plan || !src_multicast || !dst_local) AXE_FAIL(AXE_ERR_INVALID_ARG, "NULL argument");
  if (!plan->inner || plan->pulls.empty() || !plan->multicast_ok)
    AXE_FAIL(AXE_ERR_UNSUPPORTED, "multicast reduce: needs one partial per rank at one offset, 16-byte f32/bf16/f16");
  if ((uintptr_t)src_multicast % 16 || (uintptr_t)dst_local % 16) AXE_FAIL(AXE_ERR_ALIGNMENT, "16-byte alignment");
  cudaStream_t st = (cudaStream_t)stream;
  stream_forget(st);
  for (auto &pl : plan->pulls) {
    K4Params k = pl.k;
    k.dep = 1;
    cudaError_t e = launch_k4_multimem(k, plan->red.dtype, plan->pull_blocks, src_multicast, dst_local, st);
    if (e != cudaSuccess) AXE_FAIL(AXE_ERR_CUDA, "multimem reduce launch: %s", cudaGetErrorString(e));
  }
  stream_forget(st);
  return AXE_OK;
}

axe_status axe_redist_plan_describe(const axe_redist_plan *plan, char *buf, int capacity) {
  if (!plan || !buf) AXE_FAIL(AXE_ERR_INVALID_ARG, "NULL argument");
  if ((int)plan->desc.size() + 1 > capacity) AXE_FAIL(AXE_ERR_CAPACITY, "need %d bytes", (int)plan->desc.size() + 1);
  memcpy(buf, plan->desc.c_str(), plan->desc.size() + 1);
  return AXE_OK;
}

axe_status axe_redist_plan_counts(const axe_redist_plan *plan, int peer, int64_t *send, int64_t *recv) {
  if (!plan || !send || !recv) AXE_FAIL(AXE_ERR_INVALID_ARG, "NULL argument");
  if (peer < 0 || peer >= plan->nranks) AXE_FAIL(AXE_ERR_DOMAIN, "peer %d out of range", peer);
  if (plan->phase_a) AXE_FAIL(AXE_ERR_UNSUPPORTED, "two-phase plan: query axe_redist_plan_phase(plan, 0 / 1)");
  if (plan->inner) return axe_redist_plan_counts(plan->inner.get(), peer, send, recv);
  *send = *recv = 0;
  if (peer == plan->rank) {
    *send = *recv = (int64_t)plan->locals.size() * plan->n;
    return AXE_OK;
  }
  for (auto &x : plan->sends) *send += x.peer == peer ? plan->n : 0;
  for (auto &x : plan->recvs) *recv += x.peer == peer ? plan->n : 0;
  return AXE_OK;
}

axe_status axe_redist_plan_map(const axe_redist_plan *plan, int kind, int peer, int64_t k, int64_t *a, int64_t *b) {
  if (!plan || !a || !b) AXE_FAIL(AXE_ERR_INVALID_ARG, "NULL argument");
  if (kind < 0 || kind > 2) AXE_FAIL(AXE_ERR_INVALID_ARG, "kind must be 0, 1 or 2");
  if (plan->phase_a) AXE_FAIL(AXE_ERR_UNSUPPORTED, "two-phase plan: query axe_redist_plan_phase(plan, 0 / 1)");
  if (plan->inner) return axe_redist_plan_map(plan->inner.get(), kind, peer, k, a, b);
  const std::vector<Xfer> &lst = kind == 0 ? plan->sends : kind == 1 ? plan->recvs : plan->locals;
  std::vector<const Xfer *> mine;
  for (auto &e : lst)
    if (kind == 2 || e.peer == peer) mine.push_back(&e);
  const int64_t nb = (int64_t)mine.size();
  if (k < 0 || k >= nb * plan->n) AXE_FAIL(AXE_ERR_DOMAIN, "element %lld out of range", (long long)k);
  int64_t bi, j;
  if (kind == 2) {  // local copies: block-major
    bi = k / plan->n;
    j = k % plan->n;
  } else {          // the wire is chunk-major: chunk c of every block, then chunk c+1
    const int64_t c = k / (nb * plan->cn), w = k % (nb * plan->cn);
    bi = w / plan->cn;
    j = c * plan->cn + w % plan->cn;
  }
  const Xfer *x = mine[bi];
  int64_t so = x->ms, dof = x->md;
  for (int m = (int)plan->M.size() - 1; m >= 0; m--) {
    int64_t dg = j % plan->M[m].e;
    j /= plan->M[m].e;
    so += dg * plan->M[m].ss;
    dof += dg * plan->M[m].ds;
  }
  *a = kind == 1 ? dof : so;
  *b = kind == 2 ? dof : -1;
  return AXE_OK;
}

axe_status axe_redist_plan_phase(const axe_redist_plan *plan, int i, const axe_redist_plan **out) {
  if (!plan || !out) AXE_FAIL(AXE_ERR_INVALID_ARG, "NULL argument");
  *out = nullptr;
  if (!plan->phase_a) AXE_FAIL(AXE_ERR_UNSUPPORTED, "not a two-phase plan");
  if (i != 0 && i != 1) AXE_FAIL(AXE_ERR_DOMAIN, "phase %d: 0 (reduce-scatter) or 1 (gather)", i);
  *out = i == 0 ? plan->phase_a.get() : plan->phase_b.get();
  return AXE_OK;
}

void axe_redist_plan_destroy(axe_redist_plan *p) { delete p; }

axe_status axe_redistribute(const axe_layout *src, const axe_storage *src_st, const void *src_local,
                            const axe_layout *dst, const axe_storage *dst_st, void *dst_local, int elem_size,
                            axe_comm *comm, void *stream) {
  if (!comm) AXE_FAIL(AXE_ERR_INVALID_ARG, "comm is NULL");
  static std::mutex mu;
  static std::unordered_map<std::string, std::shared_ptr<axe_redist_plan>> cache;
  if (!src || !dst) AXE_FAIL(AXE_ERR_INVALID_ARG, "NULL layout");
  Storage ss, ds;
  AXE_TRY(make_storage(src_st, &ss));
  AXE_TRY(make_storage(dst_st, &ds));
  std::string key = layout_key(src->L) + "#" + storage_key(ss) + "#" + layout_key(dst->L) + "#" + storage_key(ds) +
                    "#" + std::to_string(elem_size) + "#" + std::to_string(comm->nranks) + "#" +
                    std::to_string(comm->rank) + "#" + std::to_string((uintptr_t)comm);
  std::shared_ptr<axe_redist_plan> p;
  {
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find(key);
    if (it != cache.end()) p = it->second;
  }
  if (!p) {
    p = std::make_shared<axe_redist_plan>();
    AXE_TRY(plan_redist(src->L, ss, dst->L, ds, elem_size, comm->nranks, comm->rank, p.get()));
    std::lock_guard<std::mutex> lk(mu);
    if (cache.size() >= 256) cache.clear();  // (plans hold staging memory; callers keep their own copies)
    cache[key] = p;
  }
  return serialized(p.get(), comm, (cudaStream_t)stream,
                    [&] { return exec_redist(p.get(), comm, src_local, dst_local, (cudaStream_t)stream); });
}

axe_status axe_redist_emulate(const axe_redist_plan *const *plans, int nranks, const void *const *src_locals,
                              void *const *dst_locals, void *stream) {
  if (!plans || !src_locals || !dst_locals || nranks < 1) AXE_FAIL(AXE_ERR_INVALID_ARG, "NULL argument");
  cudaStream_t st = (cudaStream_t)stream;
  for (int r = 0; r < nranks; r++)
    if (!plans[r] || plans[r]->rank != r || plans[r]->nranks != nranks)
      AXE_FAIL(AXE_ERR_INVALID_ARG, "plans[%d] is not rank %d of %d", r, r, nranks);
  if (plans[0]->phase_a) {  // two-phase reduction: emulate phase a into the temporaries, then phase b
    std::vector<const axe_redist_plan *> pa(nranks), pb(nranks);
    std::vector<void *> tmps(nranks);
    for (int r = 0; r < nranks; r++) {
      if (!plans[r]->phase_a) AXE_FAIL(AXE_ERR_INVALID_ARG, "plans mix two-phase and other plans");
      AXE_TRY(ensure_stage(plans[r]));
      pa[r] = plans[r]->phase_a.get();
      pb[r] = plans[r]->phase_b.get();
      tmps[r] = plans[r]->tmp;
    }
    AXE_TRY(axe_redist_emulate(pa.data(), nranks, src_locals, tmps.data(), stream));
    return axe_redist_emulate(pb.data(), nranks, tmps.data(), dst_locals, stream);
  }
  if (plans[0]->inner) {  // reduce plans: emulate the exchange into the stages, then sum per rank
    std::vector<const axe_redist_plan *> in(nranks);
    std::vector<void *> stages(nranks);
    for (int r = 0; r < nranks; r++) {
      if (!plans[r]->inner) AXE_FAIL(AXE_ERR_INVALID_ARG, "plans mix reduce and plain redistribution");
      AXE_TRY(ensure_stage(plans[r]));
      in[r] = plans[r]->inner.get();
      stages[r] = plans[r]->stage;
    }
    AXE_TRY(axe_redist_emulate(in.data(), nranks, src_locals, stages.data(), stream));
    for (int r = 0; r < nranks; r++) AXE_TRY(run_reduce(plans[r]->red, plans[r]->stage, dst_locals[r], st));
    return AXE_OK;
  }
  for (int r = 0; r < nranks; r++) AXE_TRY(ensure_scratch(plans[r]));
  const int nch = plans[0]->nchunk;
  for (int r = 0; r < nranks; r++)
    if (plans[r]->nchunk != nch) AXE_FAIL(AXE_ERR_INVALID_ARG, "plans disagree on wire chunks");
  for (int c = 0; c < nch; c++) {
    for (int r = 0; r < nranks; r++)
      for (auto &x : plans[r]->sends)
        if (!x.elided) AXE_TRY(run_copy(*x.cp[c], src_locals[r], plans[r]->send_buf, st));
    // the wire: chunk c of the k-th block rank r sends to p is chunk c of the k-th block p receives from r
    for (int r = 0; r < nranks; r++)
      for (int p = 0; p < nranks; p++) {
        if (p == r) continue;
        std::vector<const Xfer *> out, in;
        for (auto &x : plans[r]->sends)
          if (x.peer == p) out.push_back(&x);
        for (auto &x : plans[p]->recvs)
          if (x.peer == r) in.push_back(&x);
        if (out.size() != in.size())
          AXE_FAIL(AXE_ERR_INVALID_ARG, "plans disagree: rank %d sends %zu blocks to %d, which expects %zu", r,
                   out.size(), p, in.size());
        const axe_redist_plan *R = plans[r], *Q = plans[p];
        const size_t bytes = (size_t)(R->cn * R->es);
        const int64_t ce0 = R->M.empty() ? 0 : R->M[0].e / nch;
        for (size_t i = 0; i < out.size(); i++) {
          const uint8_t *sp = out[i]->elided
                                  ? (const uint8_t *)src_locals[r] + (out[i]->ms + (R->M.empty() ? 0 : c * ce0 * R->M[0].ss)) * R->es
                                  : (const uint8_t *)R->send_buf + (out[i]->stage + c * R->cn) * R->es;
          uint8_t *dp = in[i]->elided
                            ? (uint8_t *)dst_locals[p] + (in[i]->md + (Q->M.empty() ? 0 : c * ce0 * Q->M[0].ds)) * Q->es
                            : (uint8_t *)Q->recv_buf + (in[i]->stage + c * Q->cn) * Q->es;
          cudaError_t e = cudaMemcpyAsync(dp, sp, bytes, cudaMemcpyDeviceToDevice, st);
          if (e != cudaSuccess) AXE_FAIL(AXE_ERR_CUDA, "emulated exchange: %s", cudaGetErrorString(e));
        }
      }
    stream_forget(st);
    for (int r = 0; r < nranks; r++)
      for (auto &x : plans[r]->recvs)
        if (!x.elided) AXE_TRY(run_copy(*x.cp[c], plans[r]->recv_buf, dst_locals[r], st));
  }
  for (int r = 0; r < nranks; r++)
    for (auto &x : plans[r]->locals) AXE_TRY(run_copy(*x.plan, src_locals[r], dst_locals[r], st));
  return AXE_OK;
}

}  // extern "C"
