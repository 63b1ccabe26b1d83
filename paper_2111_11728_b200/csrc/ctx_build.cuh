// ctx_build.cuh -- operator construction on the device: ND Schur tree (K1/K2),
// slot frontals -> local operators (K3), FETI-DP coarse inverse, and their launch helpers.
// Part of the libfetigpu unity build (fetigpu.cu includes it); namespace fg.
#pragma once
#include "ctx.cuh"

namespace fg {

// ------------------------------------------------------- small kernels ----
__global__ void k_kcc_assemble(const int* optr, const int* osub, const int* oloc, const long long* kco,
                               const int* ncs, const double* kccs, int Nc, double* K) {
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < (long long)Nc * Nc;
       idx += (long long)gridDim.x * blockDim.x) {
    const int j = (int)(idx / Nc), i = (int)(idx - (long long)j * Nc);
    double v = 0.0;
    int a = optr[i], b = optr[j];
    const int ae = optr[i + 1], be = optr[j + 1];
    while (a < ae && b < be) {
      const int sa = osub[a], sb = osub[b];
      if (sa == sb) {
        const int nc = ncs[sa];
        v += kccs[kco[sa] + (long long)oloc[a] * nc + oloc[b]];
        ++a; ++b;
      } else if (sa < sb) ++a;
      else ++b;
    }
    K[idx] = v;
  }
}
__global__ void k_identity(double* X, int n) {
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < (long long)n * n;
       idx += (long long)gridDim.x * blockDim.x)
    X[idx] = (idx / n == idx % n) ? 1.0 : 0.0;
}
__global__ void k_symmetrize(double* A, int n) {
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < (long long)n * n;
       idx += (long long)gridDim.x * blockDim.x) {
    const int j = (int)(idx / n), i = (int)(idx % n);
    if (i < j) A[idx] = A[(long long)i * n + j];
  }
}
void Ctx::launch_kcc_assemble(const int* optr, const int* osub, const int* oloc, const long long* kco,
                              const int* ncs, const double* kccs, int Nc, double* K) {
  k_kcc_assemble<<<grid_for((long long)Nc * Nc), kThreads, 0, st>>>(optr, osub, oloc, kco, ncs, kccs, Nc, K);
  LAUNCH_CHECK();
}
void Ctx::launch_identity(double* X, int n) {
  k_identity<<<grid_for((long long)n * n), kThreads, 0, st>>>(X, n);
  LAUNCH_CHECK();
}
void Ctx::mirror_slots(const std::vector<long long>& moff, const std::vector<int>& ns, const std::vector<int>& ld,
                       double* mats) {
  if (moff.empty()) return;
  DBuf<long long> dm;
  DBuf<int> dn, dl;
  dm.upload(moff, st); dn.upload(ns, st); dl.upload(ld, st);
  k_mirror_slots<<<dim3(64, (unsigned)moff.size()), kThreads, 0, st>>>(dm.p, dn.p, dl.p, mats);
  LAUNCH_CHECK();
  CK(cudaStreamSynchronize(st));
}
void Ctx::launch_symmetrize(double* A, int n) {
  k_symmetrize<<<grid_for((long long)n * n), kThreads, 0, st>>>(A, n);
  LAUNCH_CHECK();
}

void Ctx::eliminate(const std::vector<FrontDesc>& fds, double* base) {
  std::vector<FrontDesc> small, large;
  int nfmax = 0;
  for (auto& f : fds) {
    if (f.nf <= kSmallFront && f.ld == f.nf) { small.push_back(f); nfmax = std::max(nfmax, f.nf); }
    else large.push_back(f);
  }
  if (!small.empty()) {
    FrontDesc* ds = scratch.upload(kScDescA, small, st);
    const int thr = nfmax <= 64 ? 64 : (nfmax <= 96 ? 128 : kThreads);
    k_front_elim_small<<<(int)small.size(), thr, nfmax * nfmax * 8, st>>>(ds, base, d_status.p);
    LAUNCH_CHECK();
  }
  if (!large.empty()) {
    FrontDesc* dl = scratch.upload(kScDescB, large, st);
    bpc(dl, large, base);
  }
}

void Ctx::bpc(const FrontDesc* d, const std::vector<FrontDesc>& fs, double* base) {
  const char* legacy = getenv("FETIGPU_LEGACY_ELIM");
  if (legacy && legacy[0] == '1') {
    k_front_elim_large<<<(int)fs.size(), kThreads, 0, st>>>(d, base, d_status.p);
    LAUNCH_CHECK();
    return;
  }
  int ne_max = 0, nf_max = 0;
  for (auto& f : fs) { ne_max = std::max(ne_max, f.ne); nf_max = std::max(nf_max, f.nf); }
  const int B = (int)fs.size();
  raise_smem_limit(k_bpc_update, kBpcUpdateSmem);
  for (int k0 = 0; k0 < ne_max; k0 += kBpcNB) {
    k_bpc_diag<<<B, kThreads, 0, st>>>(d, base, k0, d_status.p);
    const int rows = std::max(1, nf_max - k0 - 1);
    k_bpc_trsm<<<dim3((rows + kThreads - 1) / kThreads, B), kThreads, 0, st>>>(d, base, k0);
    const int nt = (rows + kTile - 1) / kTile;
    k_bpc_update<<<dim3(nt * (nt + 1) / 2, B), kThreads, kBpcUpdateSmem, st>>>(d, base, k0);
    LAUNCH_CHECK();
  }
}

void Ctx::build_nd() {
  const NdPlan& P = su.nd;
  const int nb = su.nb, n = su.n, D = su.n_designs;
  std::vector<NdDev> nodes(P.nodes.size());
  std::vector<int> elem_ids, emap, cmaps, dofs;
  for (size_t i = 0; i < P.nodes.size(); ++i) {
    const NdNode& s = P.nodes[i];
    NdDev& d = nodes[i];
    d.nf = s.nf; d.ne = s.ne; d.leaf = s.leaf; d.height = s.height;
    d.off = s.off; d.foff = s.foff;
    d.elem_off = (int)elem_ids.size();
    d.elem_cnt = (int)s.elems.size();
    elem_ids.insert(elem_ids.end(), s.elems.begin(), s.elems.end());
    emap.insert(emap.end(), s.emap.begin(), s.emap.end());
    for (int c = 0; c < 2; ++c) {
      d.child[c] = s.child[c];
      d.cmap_off[c] = (int)cmaps.size();
      cmaps.insert(cmaps.end(), s.cmap[c].begin(), s.cmap[c].end());
    }
    d.dof_off = (int)dofs.size();
    dofs.insert(dofs.end(), s.dofs.begin(), s.dofs.end());
  }
  d_nodes.upload(nodes, st);
  d_elem_ids.upload(elem_ids, st);
  d_emap.upload(emap, st);
  d_cmaps.upload(cmaps, st);
  d_nd_dofs.upload(dofs, st);
  d_topdown.upload(P.topdown, st);
  d_dens.upload(su.densities, st);
  d_S.alloc((size_t)D * nb * nb);
  if (keep_factors) d_ndfac.alloc((size_t)D * P.factor_stride);

  long long per_design = 0;
  for (long long s : P.height_stride) per_design += s;
  const size_t free_b = dev_free_bytes();
  // workspace capped at 8 GB: more, smaller chunks beat one huge cold cudaMalloc
  const long long budget = std::max<long long>(256ll << 20, std::min<long long>(8ll << 30, (long long)(free_b * 0.3)));
  const int chunk = (int)std::max<long long>(1, std::min<long long>(D, budget / (per_design * 8)));
  double* ws_p = static_cast<double*>(scratch.get(kScWs, (size_t)chunk * per_design * 8));
  // per-height node lists split by size
  std::vector<std::vector<int>> hsmall(P.max_height + 1), hlarge(P.max_height + 1);
  std::vector<int> hnfmax(P.max_height + 1, 0);
  for (int h = 0; h <= P.max_height; ++h)
    for (int t : P.by_height[h]) {
      if (P.nodes[t].nf <= kSmallFront) { hsmall[h].push_back(t); hnfmax[h] = std::max(hnfmax[h], P.nodes[t].nf); }
      else hlarge[h].push_back(t);
    }
  std::vector<DBuf<int>> dsm(P.max_height + 1), dlg(P.max_height + 1);
  for (int h = 0; h <= P.max_height; ++h) {
    dsm[h].upload(hsmall[h], st);
    dlg[h].upload(hlarge[h], st);
  }
  DBuf<long long> d_hbase, d_hstride;
  d_hstride.upload(P.height_stride, st);
  for (int d0 = 0; d0 < D; d0 += chunk) {
    const int dc = std::min(chunk, D - d0);
    std::vector<long long> hbase(P.max_height + 1, 0);
    long long acc = 0;
    for (int h = 0; h <= P.max_height; ++h) { hbase[h] = acc; acc += (long long)dc * P.height_stride[h]; }
    d_hbase.upload(hbase, st);
    NdArgs a{d_nodes.p, nullptr, d_hbase.p, d_hstride.p, ws_p, d_elem_ids.p, d_emap.p, d_cmaps.p,
             d_dens.p, n, d0, su.E0, su.Emin, su.p, keep_factors ? d_ndfac.p : nullptr,
             P.factor_stride, d_status.p};
    for (int h = 0; h <= P.max_height; ++h) {
      if (!hsmall[h].empty()) {
        a.level_nodes = dsm[h].p;
        dim3 grid((unsigned)hsmall[h].size(), dc);
        const int thr = hnfmax[h] <= 64 ? 64 : (hnfmax[h] <= 96 ? 128 : kThreads);
        k_nd_small<<<grid, thr, hnfmax[h] * (hnfmax[h] + 1) / 2 * 8, st>>>(a);
        LAUNCH_CHECK();
      }
      if (!hlarge[h].empty()) {
        a.level_nodes = dlg[h].p;
        dim3 grid((unsigned)hlarge[h].size(), dc);
        k_nd_assemble<<<grid, kThreads, 0, st>>>(a);
        LAUNCH_CHECK();
        std::vector<FrontDesc> fds;
        for (int dl = 0; dl < dc; ++dl)
          for (int t : hlarge[h]) {
            const NdNode& nd = P.nodes[t];
            fds.push_back({hbase[h] + (long long)dl * P.height_stride[h] + nd.off, nd.nf, nd.ne, nd.nf,
                           FETIGPU_E_SINGULAR_INTERIOR});
          }
        FrontDesc* dfd = scratch.upload(kScDescB, fds, st);
        bpc(dfd, fds, ws_p);
        if (keep_factors) {
          k_nd_copy_factors<<<grid, kThreads, 0, st>>>(a);
          LAUNCH_CHECK();
        }
      }
    }
    k_nd_extract_root<<<dim3(grid_for((long long)nb * nb), dc), kThreads, 0, st>>>(
        d_nodes.p, P.root, d_hbase.p, d_hstride.p, ws_p, d_S.p, nb, d0);
    LAUNCH_CHECK();
    CK(cudaStreamSynchronize(st));
  }
  check_status();
}

void Ctx::run_slots(const std::vector<SlotFront>& slots, const SlotOut& out, double* mats, double sign,
               bool nc_first, double* abc, double* kcc, double* fac, int errcode) {
  std::vector<int> src_all, ext_all;
  std::vector<SlotDev> sd(slots.size());
  for (size_t i = 0; i < slots.size(); ++i) {
    sd[i].design = slots[i].design;
    sd[i].nsrc = (int)slots[i].src.size();
    sd[i].ne = slots[i].ne;
    sd[i].next = (int)slots[i].ext.size();
    sd[i].src_off = (int)src_all.size();
    sd[i].ext_off = (int)ext_all.size();
    src_all.insert(src_all.end(), slots[i].src.begin(), slots[i].src.end());
    ext_all.insert(ext_all.end(), slots[i].ext.begin(), slots[i].ext.end());
  }
  DBuf<int> dsrc, dext;
  dsrc.upload(src_all, st);
  dext.upload(ext_all, st);
  const size_t free_b = dev_free_bytes();
  const long long budget =
      std::max<long long>(256ll << 20, std::min<long long>(8ll << 30, (long long)(free_b * 0.3))) / 8;
  size_t i0 = 0;
  while (i0 < slots.size()) {
    long long used = 0;
    size_t i1 = i0;
    std::vector<SlotDev> chunk;
    while (i1 < slots.size()) {
      const long long nf = slots[i1].nf();
      if (!chunk.empty() && used + nf * nf > budget) break;
      SlotDev d = sd[i1];
      d.woff = used;
      used += nf * nf;
      chunk.push_back(d);
      ++i1;
    }
    double* ws = static_cast<double*>(scratch.get(kScWs, (size_t)used * 8));
    SlotDev* dchunk = scratch.upload(kScSlots, chunk, st);
    const int nch = (int)chunk.size();
    k_slot_assemble<<<dim3(64, nch), kThreads, 0, st>>>(dchunk, dsrc.p, dext.p, d_S.p, su.nb, ws);
    LAUNCH_CHECK();
    std::vector<FrontDesc> fds;
    for (auto& c : chunk) fds.push_back({c.woff, c.nsrc + c.next, c.ne, c.nsrc + c.next, errcode});
    eliminate(fds, ws);
    auto sub = [&](const std::vector<long long>& v) {
      return std::vector<long long>(v.begin() + i0, v.begin() + i1);
    };
    long long* dmo = scratch.upload(kScMo, sub(out.mat_off), st);
    int* dml = scratch.upload(kScMl, std::vector<int>(out.mat_ld.begin() + i0, out.mat_ld.begin() + i1), st);
    long long* dao = abc ? scratch.upload(kScAo, sub(out.abc_off), st) : nullptr;
    long long* dko = abc ? scratch.upload(kScKo, sub(out.kcc_off), st) : nullptr;
    k_slot_extract<<<dim3(32, nch), kThreads, 0, st>>>(dchunk, ws, dmo, dml, mats, nc_first ? 1 : 0, sign, dao,
                                                       abc, dko, kcc);
    LAUNCH_CHECK();
    if (fac) {
      long long* dfo = scratch.upload(kScFo, sub(out.fac_off), st);
      k_slot_factor<<<dim3(32, nch), kThreads, 0, st>>>(dchunk, ws, dfo, fac);
      LAUNCH_CHECK();
    }
    if (i1 < slots.size()) CK(cudaStreamSynchronize(st));  // host vectors reused next chunk
    i0 = i1;
  }
  check_status();
}

void Ctx::plan_op_slots(SlotOut& so) {
  const int nslot = (int)su.op_slots.size();
  KR = su.method == FETIGPU_FETIDP ? 1 : 3;
  KRp = KR;
  long long mo = 0, ao = 0, ko = 0, fo = 0;
  op_ns.resize(nslot); op_ld.resize(nslot); op_moff.resize(nslot); op_foff.resize(nslot);
  for (int i = 0; i < nslot; ++i) {
    const SlotFront& s = su.op_slots[i];
    const int ns = (int)s.ext.size(), ld = round_up(ns, 4), nc = (int)s.src.size() - s.ne;
    op_ns[i] = ns; op_ld[i] = ld; op_moff[i] = mo;
    so.mat_off.push_back(mo); so.mat_ld.push_back(ld);
    so.abc_off.push_back(ao); so.kcc_off.push_back(ko); so.fac_off.push_back(fo);
    op_foff[i] = fo;
    mo += (long long)ns * ld; ao += (long long)ns * nc; ko += (long long)nc * nc;
    fo += (long long)s.ne * s.ne;
    max_ld = std::max(max_ld, ld);
    max_ne = std::max(max_ne, s.ne);
  }
  so.mat_total = mo; so.abc_total = ao; so.kcc_total = ko; so.fac_total = fo;
}

// Host-only index maps of the operators, preconditioner, projector, rhs /
// recovery and coarse problem.  They depend on the setup and the slot plan
// only, so build() computes them on a worker thread while the device runs
// the ND tree, and build_ops uploads them.
// threads for the maps: they run beside the thread driving the ND launches,
// so leave it (and the driver's threads) a share of the cores
static int map_threads() {
  return std::max(1, (int)std::thread::hardware_concurrency() / 2 - 1);
}

HostMaps Ctx::host_maps(const SlotOut& so) const {
  const int Ns = su.Ns, nb = su.nb;
  const bool dp = su.method == FETIGPU_FETIDP;
  HostMaps h;
  // ---- slot src/ext lists for rhs / recovery
  for (auto& s : su.op_slots) {
    h.src_off.push_back((int)h.src.size());
    h.ext_off.push_back((int)h.ext.size());
    h.src.insert(h.src.end(), s.src.begin(), s.src.end());
    h.ext.insert(h.ext.end(), s.ext.begin(), s.ext.end());
    h.fac_ne.push_back(s.ne);
  }
  // ---- per-subdomain operator maps
  // flat (subdomain, perimeter position) -> up to 3 (row, sign, weight) entries
  struct Ent { int row; double coef; double w; };
  // entries are read only below ecnt[k]: no zero fill (Ns x nb x KR of them)
  std::unique_ptr<Ent[]> ent(new Ent[(size_t)Ns * nb * KR]);
  std::vector<unsigned char> ecnt((size_t)Ns * nb, 0);
  auto add_ent = [&](int s, int pos, Ent e) {
    const size_t k = (size_t)s * nb + pos;
    if (ecnt[k] >= KR) fail(FETIGPU_E_STATE, "too many dual rows per DOF");
    ent[k * KR + ecnt[k]++] = e;
  };
  for (int i = 0; i < su.m; ++i) {
    const Row& r = su.rows[i];
    add_ent(r.sp, su.dpos[r.dp], {i, 1.0, su.wplus[i]});
    if (r.kind == 0) add_ent(r.sm, su.dpos[r.dm], {i, -1.0, su.wminus[i]});
  }
  h.ops.resize(Ns); h.pcs.resize(Ns); h.pjs.resize(Ns);
  h.slot_of.resize(Ns); h.top_off.resize(Ns); h.design.resize(Ns); h.rt_off.resize(Ns);
  h.ip_off.resize(Ns);
  size_t ntop = 0, nT = 0;
  for (int s = 0; s < Ns; ++s) {  // output offsets first, so subdomains can be filled in parallel
    h.top_off[s] = (int)ntop;
    h.ip_off[s] = nT;
    ntop += su.subs[s].Top.size();
    nT += su.subs[s].T.size();
  }
  h.rows.resize(ntop * KR); h.prow.resize(nT * KRp); h.top_pos.resize(ntop);
  h.coef.resize(ntop * KR); h.pcoef.resize(nT * KRp); h.pjcoef.resize(nT * KRp); h.RT.resize(nT * 3);
  h.sub_maxrow.assign(Ns, -1);
  parallel_for(Ns, [&](int s) {
    const SubPlan& S = su.subs[s];
    const int sl = S.op_slot;
    size_t io = (size_t)h.top_off[s], ip = h.ip_off[s];
    h.slot_of[s] = sl;
    h.design[s] = S.design;
    h.ops[s] = {op_moff[sl], op_ns[sl], op_ld[sl], (int)(io * KR), 0};
    int mx = -1;
    for (int t : S.Top) {
      const size_t k = (size_t)s * nb + t;
      h.top_pos[io] = t;
      for (int q = 0; q < KR; ++q) {
        const bool has = q < ecnt[k];
        h.rows[io * KR + q] = has ? ent[k * KR + q].row : -1;
        h.coef[io * KR + q] = has ? ent[k * KR + q].coef : 0.0;
        mx = std::max(mx, h.rows[io * KR + q]);
      }
      ++io;
    }
    h.sub_maxrow[s] = mx;
    // preconditioner / projector maps over T
    h.pcs[s] = {0, (int)S.T.size(), 0, (int)(ip * KRp), 0};
    h.pjs[s] = h.pcs[s];
    h.rt_off[s] = (int)(ip * 3);
    for (int t : S.T) {
      const size_t k = (size_t)s * nb + t;
      for (int q = 0; q < KRp; ++q) {
        const bool has = q < ecnt[k];
        h.prow[ip * KRp + q] = has ? ent[k * KR + q].row : -1;
        h.pcoef[ip * KRp + q] = has ? ent[k * KR + q].coef * ent[k * KR + q].w : 0.0;
        h.pjcoef[ip * KRp + q] = has ? ent[k * KR + q].coef : 0.0;
      }
      for (int q = 0; q < 3; ++q) h.RT[ip * 3 + q] = su.Rb[(size_t)q * nb + t];
      ++ip;
    }
  }, map_threads());
  // ---- T-FETI projector: per dual row its <= 2 (subdomain, RT offset) entries, and e
  if (!dp) {
    h.pj_sr.assign((size_t)2 * std::max(1, su.m), make_int2(-1, 0));
    h.pj_c.assign((size_t)std::max(1, su.m), make_double2(0.0, 0.0));
    for (int s = 0; s < Ns; ++s)
      for (size_t j = 0; j < su.subs[s].T.size(); ++j)
        for (int q = 0; q < KRp; ++q) {
          const size_t e = (h.ip_off[s] + j) * KRp + q;
          const int r = h.prow[e];
          if (r < 0) continue;
          const int slot = h.pj_sr[2 * (size_t)r].x < 0 ? 0 : 1;
          if (slot == 1 && h.pj_sr[2 * (size_t)r + 1].x >= 0)
            fail(FETIGPU_E_STATE, "projector: more than two entries in a dual row");
          h.pj_sr[2 * (size_t)r + slot] = make_int2(s, h.rt_off[s] + (int)j * 3);
          (slot == 0 ? h.pj_c[r].x : h.pj_c[r].y) = h.pjcoef[e];
        }
    h.e.assign(3 * Ns, 0.0);  // e = -R^T f (decomposition.hpp:127)
    for (int s = 0; s < Ns; ++s)
      for (int k = 0; k < 3; ++k) {
        double v = 0.0;
        for (int i = 0; i < nb; ++i) v += su.Rb[(size_t)k * nb + i] * su.subs[s].f[i];
        h.e[3 * s + k] = -v;
      }
  }
  // ---- boundary data for rhs / recovery
  h.xo = 0;
  for (int s = 0; s < Ns; ++s) {
    const SubPlan& S = su.subs[s];
    h.fb.insert(h.fb.end(), S.f.begin(), S.f.end());
    h.Doff.push_back((int)h.Dl.size());
    h.Dcnt.push_back((int)S.D.size());
    h.Dl.insert(h.Dl.end(), S.D.begin(), S.D.end());
    h.gD.insert(h.gD.end(), S.gD.begin(), S.gD.end());
    h.coff.push_back((int)h.cpos.size());
    h.cpos.insert(h.cpos.end(), S.c.begin(), S.c.end());
    h.xoff.push_back(h.xo);
    h.xo += su.op_slots[S.op_slot].ne;
  }
  // ---- FETI-DP coarse index lists
  if (dp) {
    h.dps.resize(Ns);
    h.optr.push_back(0);
    std::vector<int> toff(Ns);
    h.vo = 0;
    h.to = 0;
    for (int s = 0; s < Ns; ++s) {
      const SubPlan& S = su.subs[s];
      const int sl = S.op_slot;
      h.dps[s].abc_off = so.abc_off[sl];
      h.dps[s].nc = (int)S.c.size();
      if (h.dps[s].nc > 8) fail(FETIGPU_E_STATE, "more than 8 primal DOFs per subdomain");
      h.dps[s].cmap_off = (int)h.cmap.size();
      h.cmap.insert(h.cmap.end(), S.cg.begin(), S.cg.end());
      h.dps[s].v_off = h.vo;
      h.voff.push_back(h.vo);
      h.vo += (int)S.Top.size();
      h.dps[s].t_off = h.to;
      toff[s] = h.to;
      h.to += (int)S.c.size();
    }
    for (int i = 0; i < su.Nc; ++i) {
      for (auto& o : su.c_owners[i]) {
        h.oidx.push_back(toff[o.first] + o.second);
        h.osub.push_back(o.first);
        h.oloc.push_back(o.second);
      }
      h.optr.push_back((int)h.oidx.size());
    }
  }
  return h;
}

void Ctx::build_ops(const SlotOut& so, std::future<HostMaps>& maps) {
  const int Ns = su.Ns, nb = su.nb;
  const bool dp = su.method == FETIGPU_FETIDP;
  ptimer.mark("build_ops start", st);
  // ---- operator slots
  d_opmat.alloc(so.mat_total);
  d_opfac.alloc(so.fac_total);
  if (dp) { d_abc.alloc(so.abc_total); d_kccs.alloc(so.kcc_total); }
  ptimer.mark("op slot allocation", st);
  run_slots(su.op_slots, so, d_opmat.p, -1.0, dp, dp ? d_abc.p : nullptr, dp ? d_kccs.p : nullptr,
            d_opfac.p, dp ? FETIGPU_E_SINGULAR_REMAINDER : FETIGPU_E_NOT_POSITIVE_DEFINITE);
  mirror_slots(op_moff, op_ns, op_ld, d_opmat.p);
  ptimer.mark("op slots (device)", st);
  HostMaps h = maps.get();  // normally finished long before (overlapped with the ND tree)
  ptimer.mark("host maps (join)", st);
  d_op_src.upload(h.src, st); d_op_ext.upload(h.ext, st);
  d_op_src_off.upload(h.src_off, st); d_op_ext_off.upload(h.ext_off, st);
  d_fac_ne.upload(h.fac_ne, st);
  d_fac_off.upload(so.fac_off, st);
  sub_maxrow = h.sub_maxrow;
  d_oprows.upload(h.rows, st); d_opcoef.upload(h.coef, st);
  d_slot_of.upload(h.slot_of, st); d_design.upload(h.design, st);
  d_top_pos.upload(h.top_pos, st); d_top_off.upload(h.top_off, st);
  d_pcrows.upload(h.prow, st); d_pccoef.upload(h.pcoef, st);
  ptimer.mark("per-subdomain maps (upload)", st);
  // ---- preconditioner matrices
  std::vector<long long> pc_moff;
  std::vector<int> pc_ld;
  long long pm = 0;
  const int npc = su.precond == FETIGPU_DIRICHLET ? (int)su.pc_slots.size() : (int)su.pc_lumped_T.size();
  for (int i = 0; i < npc; ++i) {
    const int nt = su.precond == FETIGPU_DIRICHLET ? (int)(su.pc_slots[i].src.size() - su.pc_slots[i].ne)
                                                  : (int)su.pc_lumped_T[i].size();
    const int ld = round_up(nt, 4);
    pc_moff.push_back(pm); pc_ld.push_back(ld);
    pm += (long long)nt * ld;
    max_pc_ld = std::max(max_pc_ld, ld);
  }
  d_pcmat.alloc(pm);
  if (su.precond == FETIGPU_DIRICHLET) {
    SlotOut po;
    po.mat_off = pc_moff; po.mat_ld = pc_ld;
    run_slots(su.pc_slots, po, d_pcmat.p, 1.0, false, nullptr, nullptr, nullptr, FETIGPU_E_SINGULAR_INTERIOR);
    std::vector<int> pc_ns(npc);
    for (int i = 0; i < npc; ++i) pc_ns[i] = (int)(su.pc_slots[i].src.size() - su.pc_slots[i].ne);
    mirror_slots(pc_moff, pc_ns, pc_ld, d_pcmat.p);
  } else {
    // K_bb per design from element contributions
    std::vector<int> pne(su.nb / 2 * 4, -1);
    const int n = su.n, nn = n + 1;
    for (int q = 0; q < su.nb / 2; ++q) {
      const int v = su.perim_dof[2 * q] / 2, vx = v % nn, vy = v / nn;
      int cnt = 0;
      std::vector<std::pair<int, int>> el;
      for (int ey = std::max(0, vy - 1); ey <= std::min(n - 1, vy); ++ey)
        for (int ex = std::max(0, vx - 1); ex <= std::min(n - 1, vx); ++ex) {
          const int n0 = ey * nn + ex;
          const int en[4] = {n0, n0 + 1, n0 + nn + 1, n0 + nn};
          for (int a = 0; a < 4; ++a)
            if (en[a] == v) el.push_back({ey * n + ex, a});
        }
      std::sort(el.begin(), el.end());
      for (auto& e : el) {
        if (cnt < 2) { pne[q * 4 + 2 * cnt] = e.first; pne[q * 4 + 2 * cnt + 1] = e.second; }
        ++cnt;
      }
      if (cnt > 2) fail(FETIGPU_E_STATE, "perimeter node with > 2 elements");
    }
    DBuf<int> dpne, dpd;
    dpne.upload(pne, st);
    dpd.upload(su.perim_dof, st);
    DBuf<double> kbb;
    kbb.alloc((size_t)su.n_designs * nb * nb);
    k_kbb<<<dim3(grid_for((long long)nb * nb), su.n_designs), kThreads, 0, st>>>(
        d_dens.p, n, su.E0, su.Emin, su.p, dpne.p, dpd.p, nb, kbb.p);
    LAUNCH_CHECK();
    std::vector<int> tall, toff, tcnt;
    for (auto& T : su.pc_lumped_T) {
      toff.push_back((int)tall.size());
      tcnt.push_back((int)T.size());
      tall.insert(tall.end(), T.begin(), T.end());
    }
    DBuf<int> dt, dto, dtc, dsd, dld;
    DBuf<long long> dmo;
    dt.upload(tall, st); dto.upload(toff, st); dtc.upload(tcnt, st);
    dsd.upload(su.pc_lumped_design, st);
    dmo.upload(pc_moff, st); dld.upload(pc_ld, st);
    k_pc_lumped<<<dim3(16, npc), kThreads, 0, st>>>(dsd.p, dto.p, dtc.p, dt.p, kbb.p, nb, dmo.p, dld.p,
                                                   d_pcmat.p, su.precond == FETIGPU_SUPERLUMPED);
    LAUNCH_CHECK();
    CK(cudaStreamSynchronize(st));
  }
  ptimer.mark("preconditioner slots", st);
  pc_nsld.assign(Ns, 0);
  for (int s = 0; s < Ns; ++s) {
    const int sl = su.subs[s].pc_slot;
    h.pcs[s].moff = pc_moff[sl];
    h.pcs[s].ld = pc_ld[sl];
    pc_nsld[s] = h.pcs[s].ns * h.pcs[s].ld;
  }
  d_pc.upload(h.pcs, st);
  d_op.upload(h.ops, st);

  // ---- T-FETI projector data
  if (!dp) {
    d_pj.upload(h.pjs, st);
    d_pjcoef.upload(h.pjcoef, st);
    d_RT.upload(h.RT, st);
    d_rt_off.upload(h.rt_off, st);
    d_pjrow_sr.upload(h.pj_sr, st);
    d_pjrow_c.upload(h.pj_c, st);
    d_H.upload(su.H, st);
    d_e.upload(h.e, st);
  }
  // ---- boundary data for rhs / recovery
  d_fb.upload(h.fb, st); d_gD.upload(h.gD, st);
  d_D.upload(h.Dl, st); d_D_off.upload(h.Doff, st); d_D_cnt.upload(h.Dcnt, st);
  d_c_pos.upload(h.cpos, st); d_c_off.upload(h.coff, st);
  d_xoff.upload(h.xoff, st);
  d_xb.alloc(h.xo);
  // ---- FETI-DP coarse problem
  if (dp) {
    d_dp.upload(h.dps, st);
    d_cmap.upload(h.cmap, st);
    d_voff.upload(h.voff, st);
    d_optr.upload(h.optr, st);
    d_oidx.upload(h.oidx, st);
    d_vbuf.alloc(h.vo);
    d_tbuf.alloc(std::max(1, h.to));
    d_fbar_loc.alloc(std::max(1, h.to));
    d_fbar.alloc(std::max(1, su.Nc));
    build_coarse(so, h.osub, h.oloc);
  }
  ptimer.mark("projector/boundary data", st);
  // ---- fold the +-1 signs of the FETI-DP constraint rows into F_s and A_bc
  d_opcoef_apply.upload(h.coef, st);
  if (dp) {
    const int nsl = (int)su.op_slots.size();
    slot_sign.assign(nsl, {});
    bool ok = true;
    for (int s = 0; s < Ns && ok; ++s) {
      const int sl = su.subs[s].op_slot;
      std::vector<double> sg(op_ns[sl]);
      for (int a = 0; a < op_ns[sl]; ++a) sg[a] = h.coef[h.ops[s].map_off + a];
      if (slot_sign[sl].empty()) slot_sign[sl] = sg;
      else if (slot_sign[sl] != sg) ok = false;
    }
    if (ok) {
      std::vector<long long> ao(nsl);
      std::vector<int> ncv(nsl), soff(nsl), nsv(nsl);
      std::vector<double> sgn;
      for (int i = 0; i < nsl; ++i) {
        ao[i] = so.abc_off[i];
        ncv[i] = (int)su.op_slots[i].src.size() - su.op_slots[i].ne;
        soff[i] = (int)sgn.size();
        nsv[i] = op_ns[i];
        sgn.insert(sgn.end(), slot_sign[i].begin(), slot_sign[i].end());
      }
      DBuf<long long> dmo, dao;
      DBuf<int> dns, dld, dnc, dso;
      DBuf<double> dsg;
      dmo.upload(op_moff, st); dao.upload(ao, st); dns.upload(nsv, st); dld.upload(op_ld, st);
      dnc.upload(ncv, st); dso.upload(soff, st); dsg.upload(sgn, st);
      k_fold_signs<<<dim3(64, nsl), kThreads, 0, st>>>(dmo.p, dns.p, dld.p, dao.p, dnc.p, dso.p, dsg.p,
                                                      d_opmat.p, d_abc.p);
      LAUNCH_CHECK();
      std::vector<double> ones(h.coef.size(), 1.0);
      for (size_t i = 0; i < h.rows.size(); ++i)
        if (h.rows[i] < 0) ones[i] = 0.0;
      d_opcoef_apply.upload(ones, st);
      CK(cudaStreamSynchronize(st));
      folded = true;
      // K5's cp.async fast path copies 16-byte chunks of F'' and A'' rows:
      // every slot needs even n_s (no chunk straddles F'' and its padding),
      // even n_c and an even A'' offset (16-byte aligned A'' rows).  A
      // one-direction support at a partition vertex (odd n_c) or on an edge
      // (odd n_s) takes the general kernel.
      blk_aligned = true;
      for (int i = 0; i < nsl; ++i)
        if ((nsv[i] & 1) || (ncv[i] & 1) || (ao[i] & 1) || (op_moff[i] & 1) || (op_ld[i] & 1)) blk_aligned = false;
    }
  }
  ptimer.mark("coarse problem + folding", st);
  // ---- scratch
  const size_t m = std::max(1, su.m);
  d_v1.alloc(m); d_v2.alloc(m); d_v3.alloc(m);
  d_g.alloc(3 * (size_t)Ns + 8); d_h.alloc(3 * (size_t)Ns + 8);
  d_partial.alloc(4 * kDotBlocks);
  d_counter.alloc(1);
  d_counter.zero(st);
  d_counter2.alloc(1);
  d_counter2.zero(st);
  d_d.alloc(m); d_lam0.alloc(m);

  // ---- GEMV row split: aim for >= 4 CTAs per SM when subdomains are few
  rsplit = std::max(1, std::min(8, (4 * 148 + Ns - 1) / Ns));
  pc_rsplit = rsplit;
  // ---- symmetric-packed copy of F_s for the single-vector apply (K4)
  const char* nosym = getenv("FETIGPU_NO_SYM");
  const char* forcesym = getenv("FETIGPU_FORCE_SYM");
  const bool want_sym = rsplit == 1 || (forcesym && forcesym[0] == '1');
  if (want_sym && !(nosym && nosym[0] == '1')) {
    const int nsl = (int)su.op_slots.size();
    std::vector<long long> toff(nsl);
    long long tt = 0;
    int nbmax = 0;
    for (int i = 0; i < nsl; ++i) {
      const int nb = (op_ns[i] + 31) / 32;
      toff[i] = tt;
      tt += (long long)nb * (nb + 1) / 2 * 1024;
      nbmax = std::max(nbmax, nb);
    }
    d_symtiles.alloc(tt);
    DBuf<long long> dmo, dto;
    DBuf<int> dns, dld;
    dmo.upload(op_moff, st); dto.upload(toff, st); dns.upload(op_ns, st); dld.upload(op_ld, st);
    k_pack_sym<<<dim3(64, nsl), kThreads, 0, st>>>(dmo.p, dns.p, dld.p, dto.p, d_opmat.p, d_symtiles.p);
    LAUNCH_CHECK();
    std::vector<SymSub> ss(Ns);
    sym_bytes = 0;
    for (int s = 0; s < Ns; ++s) {
      const int sl = su.subs[s].op_slot;
      const int nb = (op_ns[sl] + 31) / 32;
      ss[s] = {toff[sl], op_ns[sl], nb, h.ops[s].map_off, 0};
      sym_bytes += (double)nb * (nb + 1) / 2 * 1024 * 8;
    }
    d_sym.upload(ss, st);
    sym_smem = nbmax * 32 * (1 + kSymWarps) * 8;
    raise_smem_limit(k_sym_gemv_scatter<1, true>, sym_smem);
    raise_smem_limit(k_sym_gemv_scatter<3, false>, sym_smem);
    CK(cudaStreamSynchronize(st));
    use_sym = true;
    // same packing for the (symmetric) preconditioner blocks S~_s / K_TT
    const int npc2 = (int)pc_moff.size();
    std::vector<long long> ptoff(npc2);
    std::vector<int> pns(npc2);
    long long pt = 0;
    int pnbmax = 0;
    for (int i = 0; i < npc2; ++i) {
      pns[i] = su.precond == FETIGPU_DIRICHLET ? (int)(su.pc_slots[i].src.size() - su.pc_slots[i].ne)
                                               : (int)su.pc_lumped_T[i].size();
      const int nb = (pns[i] + 31) / 32;
      ptoff[i] = pt;
      pt += (long long)nb * (nb + 1) / 2 * 1024;
      pnbmax = std::max(pnbmax, nb);
    }
    d_pcsymtiles.alloc(pt);
    DBuf<long long> pmo, pto;
    DBuf<int> pnsd, pldd;
    pmo.upload(pc_moff, st); pto.upload(ptoff, st); pnsd.upload(pns, st); pldd.upload(pc_ld, st);
    k_pack_sym<<<dim3(64, npc2), kThreads, 0, st>>>(pmo.p, pnsd.p, pldd.p, pto.p, d_pcmat.p, d_pcsymtiles.p);
    LAUNCH_CHECK();
    std::vector<SymSub> pss(Ns);
    for (int s = 0; s < Ns; ++s) {
      const int sl = su.subs[s].pc_slot;
      pss[s] = {ptoff[sl], pns[sl], (pns[sl] + 31) / 32, h.pcs[s].map_off, 0};
    }
    d_pcsym.upload(pss, st);
    pc_sym_smem = pnbmax * 32 * (1 + kSymWarps) * 8;
    raise_smem_limit(k_sym_gemv_scatter<1, false>, pc_sym_smem);
    raise_smem_limit(k_sym_gemv_scatter<3, false>, pc_sym_smem);
    CK(cudaStreamSynchronize(st));
    pc_sym = true;
    // TMA ring form (k_sym_gemv_tma): persistent grid, a private ring of 8 KB slots per warp
    {
      const char* e = getenv("FETIGPU_SYM_TMA");
      const char* er = getenv("FETIGPU_SYM_RING");
      int dev = 0, sms = 0, per_sm = 0, optin = 0;
      CK(cudaGetDevice(&dev));
      CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
      CK(cudaDeviceGetAttribute(&per_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev));
      CK(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
      // slots per warp: 2 CTAs per SM if one slot per warp fits beside x_s and the partials, else 1 CTA
      const char* ec = getenv("FETIGPU_SYM_CTAS");
      int ctas = ec && ec[0] == '1' ? 1 : 2;
      auto ring_for = [&](int npad) {
        const long long budget = std::min<long long>(optin, per_sm / ctas - 1024);
        const long long left = budget - (long long)sym_tma_smem(0, npad);
        int r = (int)std::max<long long>(0, left / (kSymWarps * kSymTileBytes));
        r = std::min(r, kSymRingMax);
        if (er && atoi(er) > 0) r = std::min(r, atoi(er));
        return r;
      };
      if (ring_for(nbmax * 32) < 1 || ring_for(pnbmax * 32) < 1) ctas = 1;
      if (const char* ef = getenv("FETIGPU_SYM_FLAGS")) sym_flags = atoi(ef);
      sym_npad = nbmax * 32;
      pc_sym_npad = pnbmax * 32;
      sym_ring = ring_for(sym_npad);
      pc_sym_ring = ring_for(pc_sym_npad);
      sym_tma = !(e && e[0] == '0') && sym_ring >= 1 && pc_sym_ring >= 1;
      if (sym_tma) {
        sym_tma_bytes = sym_tma_smem(sym_ring, sym_npad);
        pc_sym_tma_bytes = sym_tma_smem(pc_sym_ring, pc_sym_npad);
        const size_t mx = std::max(sym_tma_bytes, pc_sym_tma_bytes);
        raise_smem_limit(k_sym_gemv_tma<1, true>, mx);
        raise_smem_limit(k_sym_gemv_tma<1, false>, mx);
        raise_smem_limit(k_sym_gemv_tma<3, false>, mx);
        sym_grid = ctas * sms;
      }
    }
  }
  ptimer.mark("symmetric packing", st);
  setup_pipe();
  // ---- work per apply
  double sn2 = 0, snc = 0, sns = 0;
  for (int s = 0; s < Ns; ++s) {
    const double ns = (double)su.subs[s].Top.size();
    sn2 += ns * ns;
    sns += ns;
    if (dp) snc += ns * (double)su.subs[s].c.size();
  }
  double ld_bytes = 0;
  for (int s = 0; s < Ns; ++s) ld_bytes += 8.0 * op_ns[su.subs[s].op_slot] * op_ld[su.subs[s].op_slot];
  op_bytes = 8 * sn2 + (dp ? 16 * snc + 8.0 * su.Nc * su.Nc : 0) + 16.0 * su.m + 8 * sns;
  op_flops = 2 * sn2 + (dp ? 4 * snc + 2.0 * su.Nc * su.Nc : 0);
  main_bytes = 8 * sn2;
  (void)ld_bytes;
}

void Ctx::build_coarse(const SlotOut& so, const std::vector<int>& osub, const std::vector<int>& oloc) {
  const int Nc = su.Nc;
  if (Nc == 0) return;
  // Kbar_cc = sum_s B_c^T Kbar_cc^s B_c, owners in ascending subdomain order
  std::vector<long long> kco(su.Ns);
  std::vector<int> ncs(su.Ns);
  for (int s = 0; s < su.Ns; ++s) {
    kco[s] = so.kcc_off[su.subs[s].op_slot];
    ncs[s] = (int)su.subs[s].c.size();
  }
  DBuf<long long> dkco;
  DBuf<int> dncs, dos, dol;
  dkco.upload(kco, st); dncs.upload(ncs, st); dos.upload(osub, st); dol.upload(oloc, st);
  DBuf<double> K;
  K.alloc((size_t)Nc * Nc);
  launch_kcc_assemble(d_optr.p, dos.p, dol.p, dkco.p, dncs.p, d_kccs.p, Nc, K.p);
  // blocked right-looking Cholesky: diagonal blocks by k_front_elim_large,
  // panel L21 = A21 L11^{-T} through the inverted diagonal block, trailing
  // update A22 -= L21 L21^T on the lower tiles (DMMA GEMMs, dla.cuh)
  const int NBc = 256;
  DBuf<double> Xd, Pt, Tw;
  Xd.alloc((size_t)NBc * NBc);
  Pt.alloc((size_t)std::max(1, Nc - std::min(NBc, Nc)) * NBc);
  Tw.alloc(tri_inv_workspace(std::max(Nc, NBc)));
  for (int k0 = 0; k0 < Nc; k0 += NBc) {
    const int kb = std::min(NBc, Nc - k0);
    std::vector<FrontDesc> f{{(long long)k0 * Nc + k0, kb, kb, Nc, FETIGPU_E_SINGULAR_COARSE}};
    DBuf<FrontDesc> df;
    df.upload(f, st);
    k_front_elim_large<<<1, kThreads, 0, st>>>(df.p, K.p, d_status.p);
    LAUNCH_CHECK();
    CK(cudaStreamSynchronize(st));
    const int rest = Nc - k0 - kb;
    if (rest > 0) {
      double* L11 = K.p + (size_t)k0 * Nc + k0;
      double* A21 = L11 + kb;
      tri_inv_lower(st, L11, Nc, kb, Xd.p, kb, Tw.p);
      CK(cudaMemcpy2DAsync(Pt.p, (size_t)rest * 8, A21, (size_t)Nc * 8, (size_t)rest * 8, kb,
                           cudaMemcpyDeviceToDevice, st));
      // L21 = A21 X11^T (X11 lower: column c of X11^T ends at row c)
      gemm(st, false, true, rest, kb, kb, 1.0, Pt.p, rest, Xd.p, kb, 0.0, A21, Nc, kGemmKEndByCol);
      gemm(st, false, true, rest, rest, kb, -1.0, A21, Nc, A21, Nc, 1.0, A21 + (size_t)kb * Nc, Nc,
           kGemmLowerTiles);
    }
  }
  check_status();
  // inverse: X = L^{-1}, Kinv = X^T X (lower tiles, then mirrored)
  DBuf<double> X;
  X.alloc((size_t)Nc * Nc);
  tri_inv_lower(st, K.p, Nc, Nc, X.p, Nc, Tw.p);
  d_Kinv.alloc((size_t)Nc * Nc);
  gemm(st, true, false, Nc, Nc, Nc, 1.0, X.p, Nc, X.p, Nc, 0.0, d_Kinv.p, Nc, kGemmLowerTiles | kGemmKStartByCol);
  launch_symmetrize(d_Kinv.p, Nc);
  // fused-gather target + arrival counters (always); symmetric-packed copy
  // of the inverse for the single-vector apply when it is large
  d_gc.alloc(Nc);
  d_gcnt.alloc(Nc);
  d_gcnt.zero(st);
  d_cgather.upload(std::vector<CoarseGather>{{d_gc.p, d_gcnt.p, d_optr.p, d_oidx.p, d_cmap.p}}, st);
  use_csym = Nc > 2048;
  if (!use_csym) {
    CK(cudaStreamSynchronize(st));
    return;
  }
  kinv_nb = (Nc + 31) / 32;
  const size_t ntiles = (size_t)kinv_nb * (kinv_nb + 1) / 2;
  d_kinv_tiles.alloc(ntiles * 1024);
  d_crow.alloc(ntiles * 32);
  d_ccol.alloc(ntiles * 32);
  {
    DBuf<long long> mo, to;
    DBuf<int> ns, ld;
    mo.upload(std::vector<long long>{0}, st); to.upload(std::vector<long long>{0}, st);
    ns.upload(std::vector<int>{Nc}, st); ld.upload(std::vector<int>{Nc}, st);
    k_pack_sym<<<dim3(grid_for((long long)ntiles * 1024), 1), kThreads, 0, st>>>(mo.p, ns.p, ld.p, to.p, d_Kinv.p,
                                                                              d_kinv_tiles.p);
    LAUNCH_CHECK();
    CK(cudaStreamSynchronize(st));
  }
  int dev = 0, sms = 0, per_sm = 0;
  CK(cudaGetDevice(&dev));
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_csym_tiles, 128, 0));
  csym_grid = (int)std::max<long long>(1, std::min<long long>((long long)sms * std::max(1, per_sm),
                                                              ((long long)ntiles + 3) / 4));
}

void Ctx::build() {
  ptimer = PhaseTimer();
  SlotOut so;
  plan_op_slots(so);
  // host index maps on a worker thread, overlapped with the device ND tree
  std::future<HostMaps> maps = std::async(std::launch::async, [this, &so] { return host_maps(so); });
  struct Join {  // never leave the worker running past this frame (e.g. on a build error)
    std::future<HostMaps>& f;
    ~Join() { if (f.valid()) f.wait(); }
  } join{maps};
  CK(cudaEventRecord(ev0, st));
  CK(cudaMemcpyToSymbolAsync(c_kunit, su.kunit, sizeof(su.kunit), 0, cudaMemcpyHostToDevice, st));
  build_nd();
  ptimer.mark("nested dissection", st);
  CK(cudaEventRecord(ev1, st));
  nd_ms = elapsed(ev0, ev1);
  build_ops(so, maps);
  CK(cudaEventRecord(ev2, st));
  CK(cudaStreamSynchronize(st));
  scratch.release(kScWs);
  slot_ms = elapsed(ev1, ev2);
  build_ms = elapsed(ev0, ev2);
  built = true;
}

}  // namespace fg
