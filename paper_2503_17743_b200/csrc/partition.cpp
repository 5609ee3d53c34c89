// partition.cpp — multi-GPU decomposition of the sweep.
//
// 3D tracks are independent within a sweep given Jacobi boundary fluxes, so the
// stacks are split across ranks.  Order: polar pair {n, N-1-n} (outer), 2D cycle, then
// position of the 2D track along its cycle; both polars of a pair are adjacent.  Radial
// reflective links go to the cycle neighbour in the same polar pair and axial reflective
// links to the complementary polar of the same 2D track, so with contiguous pieces of
// this order only the P-1 cuts (and cycle wrap-arounds) cross ranks.  Pieces are cut on
// the prefix sum of a per-stack cost (raw piece count) for balance.
#include <omp.h>

#include <algorithm>
#include <numeric>

#include "host.h"

namespace moc {

void partition_stacks(const Laydown& L, int world, std::vector<int32_t>& owner, std::vector<double>* cost) {
  const int64_t T2 = L.T2(), S = L.S();
  const int N = L.N;
  if (world < 1) throw Error(MOC_E_INVALID_ARG, "world must be >= 1");
  // tracks ordered by (cycle, arc length of the track's first point in cycle order)
  std::vector<int64_t> tord(T2);
  std::iota(tord.begin(), tord.end(), 0);
  auto start = [&](int64_t t) { return L.t_sig[t] > 0 ? L.t_lt[t] : L.t_lt[t] - L.t_len[t]; };
  std::stable_sort(tord.begin(), tord.end(), [&](int64_t a, int64_t b) {
    if (L.t_cyc[a] != L.t_cyc[b]) return L.t_cyc[a] < L.t_cyc[b];
    return start(a) < start(b);
  });
  std::vector<int64_t> order;
  order.reserve(S);
  for (int p = 0; p < N / 2; ++p)
    for (int64_t t : tord) {
      order.push_back(t * N + p);
      order.push_back(t * N + (N - 1 - p));
    }
  double total = 0;
  for (int64_t s = 0; s < S; ++s) total += (double)L.st_raw[s];
  owner.assign(S, 0);
  if (cost) cost->assign(world, 0.0);
  double cum = 0;
  for (int64_t q = 0; q < S; ++q) {
    const int64_t s = order[q];
    // rank r takes the stacks whose cost midpoint falls in [r, r+1) * total / world
    const double mid = cum + 0.5 * (double)L.st_raw[s];
    int r = total > 0 ? (int)(mid * world / total) : 0;
    r = std::min(std::max(r, 0), world - 1);
    owner[s] = r;
    if (cost) (*cost)[r] += (double)L.st_raw[s];
    cum += (double)L.st_raw[s];
  }
}

// One pass over all links: send[p] = target slots written by `rank` that rank p owns,
// recv[p] = target slots owned by `rank` that rank p writes — both in source-slot order,
// so rank p's send[rank] list and this rank's recv[p] list are identical.
void halo_plans(const Laydown& L, const int64_t* link, const std::vector<int32_t>& owner, int rank, int world,
                std::vector<std::vector<int64_t>>& send, std::vector<std::vector<int64_t>>& recv) {
  const int64_t S = L.S();
  const int nth = omp_get_max_threads();
  std::vector<std::vector<std::vector<int64_t>>> ps(nth, std::vector<std::vector<int64_t>>(world)),
      pr(nth, std::vector<std::vector<int64_t>>(world));
#pragma omp parallel num_threads(nth)
  {
    const int th = omp_get_thread_num();
    const int64_t s0 = S * th / nth, s1 = S * (th + 1) / nth;
    for (int64_t s = s0; s < s1; ++s) {
      const int rs = owner[s];
      for (int64_t id = L.st_first[s]; id < L.st_first[s + 1]; ++id)
        for (int d = 0; d < 2; ++d) {
          const int64_t tgt = link[2 * id + d];
          if (tgt < 0) continue;
          const int64_t ts =
              std::upper_bound(L.st_first.begin(), L.st_first.end(), tgt / 2) - L.st_first.begin() - 1;
          const int rt = owner[ts];
          if (rs == rt) continue;
          if (rs == rank) ps[th][rt].push_back(tgt);
          if (rt == rank) pr[th][rs].push_back(tgt);
        }
    }
  }
  send.assign(world, {});
  recv.assign(world, {});
  for (int th = 0; th < nth; ++th)
    for (int p = 0; p < world; ++p) {
      send[p].insert(send[p].end(), ps[th][p].begin(), ps[th][p].end());
      recv[p].insert(recv[p].end(), pr[th][p].begin(), pr[th][p].end());
    }
}

// This rank's track numbering and link table (boundary psi owned by the sweeping rank,
// SURVEY §8(e)): its stacks' members in stack order get local ids 0..T3_local-1; a link to
// an owned target becomes that target's local slot, a link to another rank's target the
// next slot of that peer's block in the halo-send tail [2 T3_local, 2 T3_local + n_send)
// (source-slot order, the order of halo_plans and of the peer's receive list); received
// psi is scattered into recv_slots (local slots, peer-major).
void rank_layout(const Laydown& L, const int64_t* link, const std::vector<int32_t>& owner, int rank, int world,
                 RankLayout& out) {
  const int64_t S = L.S();
  out.slot_first.assign(S + 1, 0);
  int64_t run = 0;
  for (int64_t q = 0; q < S; ++q) {
    out.slot_first[q] = run;
    if (owner[q] == rank) run += L.st_cnt[q];
  }
  out.slot_first[S] = run;
  out.T3_local = run;
  auto stack_of = [&](int64_t gid) {
    return (int64_t)(std::upper_bound(L.st_first.begin(), L.st_first.end(), gid) - L.st_first.begin() - 1);
  };
  auto local_slot = [&](int64_t gslot) {
    const int64_t gid = gslot / 2, ts = stack_of(gid);
    return 2 * (out.slot_first[ts] + (gid - L.st_first[ts])) + (gslot & 1);
  };
  std::vector<std::vector<int64_t>> send, recv;
  halo_plans(L, link, owner, rank, world, send, recv);
  std::vector<int64_t> soff(world + 1, 0);
  out.send_counts.assign(world, 0);
  out.recv_counts.assign(world, 0);
  for (int p = 0; p < world; ++p) {
    out.send_counts[p] = (int64_t)send[p].size();
    out.recv_counts[p] = (int64_t)recv[p].size();
    soff[p + 1] = soff[p] + out.send_counts[p];
  }
  out.n_send = soff[world];
  out.link.assign(2 * out.T3_local, -1);
  std::vector<int64_t> cnt(world, 0);
  for (int64_t q = 0; q < S; ++q) {
    if (owner[q] != rank) continue;
    for (int64_t gid = L.st_first[q]; gid < L.st_first[q + 1]; ++gid)
      for (int d = 0; d < 2; ++d) {
        const int64_t tgt = link[2 * gid + d];
        if (tgt < 0) continue;
        const int rt = owner[stack_of(tgt / 2)];
        out.link[2 * (out.slot_first[q] + (gid - L.st_first[q])) + d] =
            rt == rank ? local_slot(tgt) : 2 * out.T3_local + soff[rt] + cnt[rt]++;
      }
  }
  out.recv_slots.clear();
  for (int p = 0; p < world; ++p)
    for (int64_t x : recv[p]) out.recv_slots.push_back(local_slot(x));
}

void halo_plan(const Laydown& L, const int64_t* link, const std::vector<int32_t>& owner, int rank, int peer,
               std::vector<int64_t>& slots) {
  int world = 1 + std::max(rank, peer);
  for (int32_t o : owner) world = std::max(world, o + 1);
  std::vector<std::vector<int64_t>> send, recv;
  halo_plans(L, link, owner, rank, world, send, recv);
  slots = send[peer];
}

}  // namespace moc
