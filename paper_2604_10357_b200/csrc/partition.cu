// partition.cu — element-block partition across GPUs (DESIGN.md
// reading Q20). A coefficient (node) is owned by the lowest rank among the
// partitions of its incident elements; each rank assembles its elements, keeps
// the rows it owns and sends partial 3x3 H blocks / nodal forces of the rows
// it does not own to their owner. The owner adds the received partials in
// ascending peer order, so the result is deterministic for a fixed partition.
// The transport (NCCL send/recv over NVLink) is done by the caller on the
// packed buffers; this file holds the host planner and the pack/unpack kernels.
#include <algorithm>
#include <tuple>

#include "common.cuh"

namespace tlfea {

struct BlkKey {
  int32_t peer;
  int32_t I, J;
  bool operator<(const BlkKey& o) const { return std::tie(peer, I, J) < std::tie(o.peer, o.I, o.J); }
  bool operator==(const BlkKey& o) const { return peer == o.peer && I == o.I && J == o.J; }
};

struct Plan {
  std::vector<int32_t> owner;
  std::vector<BlkKey> send_blk, recv_blk;  // (peer, I, J) sorted
  std::vector<BlkKey> send_node, recv_node;  // (peer, I, -1) sorted
};

static void make_plan(int64_t NE, int nen, const int32_t* cc, int64_t n_coef, const int32_t* part,
                      int32_t nranks, int32_t rank, Plan& pl) {
  pl.owner.assign((size_t)n_coef, nranks);
  for (int64_t e = 0; e < NE; ++e)
    for (int a = 0; a < nen; ++a) {
      int32_t& o = pl.owner[cc[e * nen + a]];
      o = std::min(o, part[e]);
    }
  for (auto& o : pl.owner)
    if (o == nranks) o = 0;
  for (int64_t e = 0; e < NE; ++e) {
    const int32_t* c = cc + e * nen;
    bool mixed = false;
    for (int a = 0; a < nen && !mixed; ++a) mixed = pl.owner[c[a]] != part[e];
    if (!mixed) continue;  // interior element: all its rows are owned by its own rank
    for (int a = 0; a < nen; ++a) {
      const int32_t I = c[a], oI = pl.owner[I];
      if (part[e] == rank && oI != rank) {
        pl.send_node.push_back({oI, I, -1});
        for (int b = 0; b < nen; ++b) pl.send_blk.push_back({oI, I, c[b]});
      }
      if (part[e] != rank && oI == rank) {
        pl.recv_node.push_back({part[e], I, -1});
        for (int b = 0; b < nen; ++b) pl.recv_blk.push_back({part[e], I, c[b]});
      }
    }
  }
  for (auto* v : {&pl.send_blk, &pl.recv_blk, &pl.send_node, &pl.recv_node}) {
    std::sort(v->begin(), v->end());
    v->erase(std::unique(v->begin(), v->end()), v->end());
  }
}

// ------------------------------------------------------------------ kernels
__device__ __forceinline__ int ublk_p(int n, int a, int b) { return a * n - (a * (a - 1)) / 2 + (b - a); }

// Kscr is element-major, or gather-sorted when dest is given: block (e, ub)
// at position dest >> 1, stored transposed (relative to a <= b) when dest & 1.
__global__ void k_pack_blocks(int64_t n, int nen, int nub, const int32_t* __restrict__ ptr,
                              const uint32_t* __restrict__ ent, const int64_t* __restrict__ off,
                              const double* __restrict__ Kscr, const int32_t* __restrict__ dest,
                              double* __restrict__ out) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= n) return;
  double acc[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
  for (int32_t t = ptr[k]; t < ptr[k + 1]; ++t) {
    const uint32_t en = ent[t];
    const int64_t e = en >> 8;
    const int a = (en >> 4) & 15, b = en & 15;
    const int64_t ub = e * nub + (a <= b ? ublk_p(nen, a, b) : ublk_p(nen, b, a));
    bool tr = a > b;
    const double* s = Kscr + ub * 9;
    if (dest) {
      const int32_t dd = dest[ub];
      s = Kscr + (int64_t)(dd >> 1) * 9;
      tr = tr != ((dd & 1) != 0);
    }
    if (!tr) {
      for (int r = 0; r < 9; ++r) acc[r] += s[r];
    } else {
      for (int i = 0; i < 3; ++i)
        for (int kk = 0; kk < 3; ++kk) acc[3 * i + kk] += s[3 * kk + i];
    }
  }
  for (int r = 0; r < 9; ++r) out[off[k] + r] = acc[r];
}

__global__ void k_pack_nodes(int64_t n, int nen, const int32_t* __restrict__ ptr,
                             const uint32_t* __restrict__ ent, const int64_t* __restrict__ off,
                             const double* __restrict__ fscr, const int32_t* __restrict__ fdest,
                             double* __restrict__ out) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= n) return;
  double f0 = 0, f1 = 0, f2 = 0;
  for (int32_t t = ptr[k]; t < ptr[k + 1]; ++t) {
    const uint32_t en = ent[t];
    const int64_t ea = (int64_t)(en >> 4) * nen + (en & 15);
    const double* s = fscr + (fdest ? (int64_t)fdest[ea] : ea) * 3;
    f0 += s[0];
    f1 += s[1];
    f2 += s[2];
  }
  out[off[k]] = f0;
  out[off[k] + 1] = f1;
  out[off[k] + 2] = f2;
}

__global__ void k_find_slots(int64_t n, const int32_t* __restrict__ rowJ, const int32_t* __restrict__ rowptr_c,
                             const int32_t* __restrict__ cols_c, int32_t* __restrict__ slot) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= n) return;
  const int32_t r = rowJ[2 * k], J = rowJ[2 * k + 1];
  int32_t lo = rowptr_c[r], hi = rowptr_c[r + 1];
  while (lo < hi) {
    const int32_t mid = (lo + hi) >> 1;
    if (cols_c[mid] < J)
      lo = mid + 1;
    else
      hi = mid;
  }
  slot[k] = lo;
}

// One launch per peer (ascending) keeps the accumulation order fixed.
__global__ void k_unpack_blocks(int64_t n, const int32_t* __restrict__ slot, const int32_t* __restrict__ blk_row,
                                const int32_t* __restrict__ rowptr_c, const double* __restrict__ in, double h,
                                double* __restrict__ H) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= n) return;
  const int32_t p = slot[k], i = blk_row[p], b0 = rowptr_c[i], deg = rowptr_c[i + 1] - b0, kk = p - b0;
  double* out = H + 9 * (int64_t)b0 + 3 * kk;
  for (int d = 0; d < 3; ++d)
    for (int f = 0; f < 3; ++f) out[3 * d * deg + f] += h * in[9 * k + 3 * d + f];
}

__global__ void k_unpack_nodes(int64_t n, const int32_t* __restrict__ row, const double* __restrict__ in,
                               double* __restrict__ fpart) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= n) return;
  const int64_t r = row[k];
  fpart[3 * r] += in[3 * k];
  fpart[3 * r + 1] += in[3 * k + 1];
  fpart[3 * r + 2] += in[3 * k + 2];
}

static inline unsigned gridn(int64_t n, int b) { return (unsigned)std::max<int64_t>(1, (n + b - 1) / b); }

// ------------------------------------------------------------ setup / eval

tlfea_status setup_exchange(Context* c, const std::vector<int32_t>& cc, const std::vector<int32_t>& part,
                            const std::vector<int32_t>& owner, const std::vector<int64_t>& local) {
  (void)owner;
  const int nen = c->nen, P = c->nranks;
  Plan pl;
  make_plan(c->n_el_global, nen, cc.data(), c->n_coef, part.data(), P, c->rank, pl);
  // local element index of each global element (-1 if not local)
  std::vector<int32_t> lidx((size_t)c->n_el_global, -1);
  for (size_t i = 0; i < local.size(); ++i) lidx[local[i]] = (int32_t)i;

  c->send_blk_count.assign(P, 0);
  c->send_node_count.assign(P, 0);
  c->recv_blk_count.assign(P, 0);
  c->recv_node_count.assign(P, 0);
  for (auto& k : pl.send_blk) c->send_blk_count[k.peer]++;
  for (auto& k : pl.send_node) c->send_node_count[k.peer]++;
  for (auto& k : pl.recv_blk) c->recv_blk_count[k.peer]++;
  for (auto& k : pl.recv_node) c->recv_node_count[k.peer]++;
  c->send_counts.assign(P, 0);
  c->recv_counts.assign(P, 0);
  for (int s = 0; s < P; ++s) {
    c->send_counts[s] = 9 * c->send_blk_count[s] + 3 * c->send_node_count[s];
    c->recv_counts[s] = 9 * c->recv_blk_count[s] + 3 * c->recv_node_count[s];
  }
  std::vector<int64_t> soff(P + 1, 0);
  for (int s = 0; s < P; ++s) soff[s + 1] = soff[s] + c->send_counts[s];
  c->n_send_blk = (int64_t)pl.send_blk.size();
  c->n_send_node = (int64_t)pl.send_node.size();
  c->n_recv_blk = (int64_t)pl.recv_blk.size();
  c->n_recv_node = (int64_t)pl.recv_node.size();

  // output offsets of every sent block / node in the send buffer
  std::vector<int64_t> blk_off(c->n_send_blk), node_off(c->n_send_node);
  {
    std::vector<int64_t> cursor(soff.begin(), soff.end() - 1);
    for (int64_t k = 0; k < c->n_send_blk; ++k) {
      blk_off[k] = cursor[pl.send_blk[k].peer];
      cursor[pl.send_blk[k].peer] += 9;
    }
    for (int64_t k = 0; k < c->n_send_node; ++k) {
      node_off[k] = cursor[pl.send_node[k].peer];
      cursor[pl.send_node[k].peer] += 3;
    }
  }
  // contribution lists (ascending local element)
  std::vector<std::pair<int64_t, uint32_t>> bc, nc;
  for (int64_t i = 0; i < c->n_el; ++i) {
    const int32_t* ce = cc.data() + local[i] * nen;
    for (int a = 0; a < nen; ++a) {
      const int32_t I = ce[a], oI = pl.owner[I];
      if (oI == c->rank) continue;
      const auto it = std::lower_bound(pl.send_node.begin(), pl.send_node.end(), BlkKey{oI, I, -1});
      nc.push_back({it - pl.send_node.begin(), ((uint32_t)i << 4) | (uint32_t)a});
      for (int b = 0; b < nen; ++b) {
        const auto jt = std::lower_bound(pl.send_blk.begin(), pl.send_blk.end(), BlkKey{oI, I, ce[b]});
        bc.push_back({jt - pl.send_blk.begin(), pack_eab((uint32_t)i, (uint32_t)a, (uint32_t)b)});
      }
    }
  }
  std::stable_sort(bc.begin(), bc.end(), [](auto& x, auto& y) { return x.first < y.first; });
  std::stable_sort(nc.begin(), nc.end(), [](auto& x, auto& y) { return x.first < y.first; });
  auto to_csr = [](const std::vector<std::pair<int64_t, uint32_t>>& v, int64_t n, std::vector<int32_t>& ptr,
                   std::vector<uint32_t>& ent) {
    ptr.assign(n + 1, 0);
    ent.resize(v.size());
    for (size_t t = 0; t < v.size(); ++t) {
      ptr[v[t].first + 1]++;
      ent[t] = v[t].second;
    }
    for (int64_t k = 0; k < n; ++k) ptr[k + 1] += ptr[k];
  };
  std::vector<int32_t> bptr, nptr;
  std::vector<uint32_t> bent, nent;
  to_csr(bc, c->n_send_blk, bptr, bent);
  to_csr(nc, c->n_send_node, nptr, nent);
  int64_t* dboff = nullptr;
  int64_t* dnoff = nullptr;
  {
    tlfea_status st;
    if ((st = c->alloc(&c->sblk_ptr, bptr.size())) != TLFEA_OK) return st;
    if ((st = c->alloc(&c->sblk_ent, bent.size())) != TLFEA_OK) return st;
    if ((st = c->alloc(&c->snode_ptr, nptr.size())) != TLFEA_OK) return st;
    if ((st = c->alloc(&c->snode_ent, nent.size())) != TLFEA_OK) return st;
    if ((st = c->alloc(&dboff, blk_off.size())) != TLFEA_OK) return st;
    if ((st = c->alloc(&dnoff, node_off.size())) != TLFEA_OK) return st;
    if ((st = c->alloc(&c->rblk_slot, pl.recv_blk.size())) != TLFEA_OK) return st;
    if ((st = c->alloc(&c->rnode_row, pl.recv_node.size())) != TLFEA_OK) return st;
  }
  TL_CUDA(cudaMemcpy(c->sblk_ptr, bptr.data(), bptr.size() * 4, cudaMemcpyHostToDevice));
  if (!bent.empty()) TL_CUDA(cudaMemcpy(c->sblk_ent, bent.data(), bent.size() * 4, cudaMemcpyHostToDevice));
  TL_CUDA(cudaMemcpy(c->snode_ptr, nptr.data(), nptr.size() * 4, cudaMemcpyHostToDevice));
  if (!nent.empty()) TL_CUDA(cudaMemcpy(c->snode_ent, nent.data(), nent.size() * 4, cudaMemcpyHostToDevice));
  if (!blk_off.empty()) TL_CUDA(cudaMemcpy(dboff, blk_off.data(), blk_off.size() * 8, cudaMemcpyHostToDevice));
  if (!node_off.empty()) TL_CUDA(cudaMemcpy(dnoff, node_off.data(), node_off.size() * 8, cudaMemcpyHostToDevice));
  c->send_blk_off = dboff;
  c->send_node_off = dnoff;

  // receive maps: (row, J) -> owned coefficient block; node -> owned row
  std::vector<int32_t> own_idx(c->n_coef, -1);
  TL_CUDA(cudaMemcpy(own_idx.data(), c->own_idx, sizeof(int32_t) * c->n_coef, cudaMemcpyDeviceToHost));
  if (c->n_recv_blk > 0) {
    std::vector<int32_t> rowJ(2 * c->n_recv_blk);
    for (int64_t k = 0; k < c->n_recv_blk; ++k) {
      rowJ[2 * k] = own_idx[pl.recv_blk[k].I];
      rowJ[2 * k + 1] = pl.recv_blk[k].J;
    }
    int32_t* drj = nullptr;
    TL_CUDA(cudaMalloc(&drj, rowJ.size() * 4));
    TL_CUDA(cudaMemcpy(drj, rowJ.data(), rowJ.size() * 4, cudaMemcpyHostToDevice));
    k_find_slots<<<gridn(c->n_recv_blk, 256), 256>>>(c->n_recv_blk, drj, c->rowptr_c, c->cols_c, c->rblk_slot);
    count_launch();
    TL_CUDA(cudaDeviceSynchronize());
    cudaFree(drj);
  }
  if (c->n_recv_node > 0) {
    std::vector<int32_t> rows(c->n_recv_node);
    for (int64_t k = 0; k < c->n_recv_node; ++k) rows[k] = own_idx[pl.recv_node[k].I];
    TL_CUDA(cudaMemcpy(c->rnode_row, rows.data(), rows.size() * 4, cudaMemcpyHostToDevice));
  }
  return TLFEA_OK;
}

tlfea_status launch_pack_send(Context* c, double* send, bool force_only, cudaStream_t s) {
  if (!force_only && c->n_send_blk > 0) {
    k_pack_blocks<<<gridn(c->n_send_blk, 256), 256, 0, s>>>(c->n_send_blk, c->nen, n_ublk_of(c->nen), c->sblk_ptr,
                                                            c->sblk_ent, c->send_blk_off, c->Kscr, c->dest, send);
    TL_CHECK_LAUNCH();
  }
  if (c->n_send_node > 0) {
    k_pack_nodes<<<gridn(c->n_send_node, 256), 256, 0, s>>>(c->n_send_node, c->nen, c->snode_ptr, c->snode_ent,
                                                            c->send_node_off, c->fscr, c->fdest, send);
    TL_CHECK_LAUNCH();
  }
  return TLFEA_OK;
}

tlfea_status launch_unpack_recv(Context* c, const double* recv, double h, double* H, bool force_only,
                                cudaStream_t s) {
  int64_t off = 0, bk = 0, nk = 0;
  for (int p = 0; p < c->nranks; ++p) {
    const int64_t nb = c->recv_blk_count[p], nn = c->recv_node_count[p];
    if (!force_only && nb > 0 && H) {
      k_unpack_blocks<<<gridn(nb, 256), 256, 0, s>>>(nb, c->rblk_slot + bk, c->blk_row, c->rowptr_c, recv + off, h, H);
      TL_CHECK_LAUNCH();
    }
    if (nn > 0) {
      k_unpack_nodes<<<gridn(nn, 256), 256, 0, s>>>(nn, c->rnode_row + nk, recv + off + 9 * nb, c->fpart);
      TL_CHECK_LAUNCH();
    }
    off += 9 * nb + 3 * nn;
    bk += nb;
    nk += nn;
  }
  return TLFEA_OK;
}

}  // namespace tlfea

// --------------------------------------------------------- host planner ABI
extern "C" tlfea_status tlfea_plan_partition(int64_t n_elements, int32_t n_en, const int32_t* conn_coef,
                                             int64_t n_coef, const int32_t* elem_part, int32_t nranks,
                                             int32_t rank, int32_t* owner_out, int64_t* n_send_blocks,
                                             int64_t* send_blocks, int64_t* send_block_peer,
                                             int64_t* n_send_nodes, int64_t* send_nodes,
                                             int64_t* send_node_peer) {
  using namespace tlfea;
  if (n_elements <= 0 || n_en <= 0 || n_en > 16 || !conn_coef || n_coef <= 0 || nranks < 1 || rank < 0 ||
      rank >= nranks || !n_send_blocks || !n_send_nodes)
    return fail(TLFEA_E_INVALID, "tlfea_plan_partition: bad arguments");
  std::vector<int32_t> part((size_t)n_elements);
  for (int64_t e = 0; e < n_elements; ++e) {
    part[e] = elem_part ? elem_part[e] : (int32_t)((e * nranks) / n_elements);
    if (part[e] < 0 || part[e] >= nranks) return fail(TLFEA_E_INVALID, "elem_part out of range");
  }
  for (int64_t t = 0; t < n_elements * n_en; ++t)
    if (conn_coef[t] < 0 || conn_coef[t] >= n_coef) return fail(TLFEA_E_INVALID, "conn id out of range");
  Plan pl;
  make_plan(n_elements, n_en, conn_coef, n_coef, part.data(), nranks, rank, pl);
  if (owner_out) std::copy(pl.owner.begin(), pl.owner.end(), owner_out);
  *n_send_blocks = (int64_t)pl.send_blk.size();
  *n_send_nodes = (int64_t)pl.send_node.size();
  if (send_blocks)
    for (size_t k = 0; k < pl.send_blk.size(); ++k) {
      send_blocks[2 * k] = pl.send_blk[k].I;
      send_blocks[2 * k + 1] = pl.send_blk[k].J;
      if (send_block_peer) send_block_peer[k] = pl.send_blk[k].peer;
    }
  if (send_nodes)
    for (size_t k = 0; k < pl.send_node.size(); ++k) {
      send_nodes[k] = pl.send_node[k].I;
      if (send_node_peer) send_node_peer[k] = pl.send_node[k].peer;
    }
  return TLFEA_OK;
}
