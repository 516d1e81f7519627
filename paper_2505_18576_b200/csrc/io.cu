// io.cu -- amgf_export / amgf_import: the AMGF preconditioner as raw little-endian files.
//
// The format (include/amgf.h) is what the oracle writes too (oracle/__init__.py Oracle.export), so a
// hierarchy built on the CPU can be applied by these kernels unchanged: the north star's "single
// preconditioner applies on an identical exported hierarchy".  Import recomputes nothing numeric: it uploads
// the stored operators, l1 diagonals, transfer operators and factors and rebuilds only the solve-side
// layouts (SELL-32 packing, the thin S[:, Z] rows, the nested-dissection block table, band copies of the
// factors), checking that the stored data fit those layouts exactly.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <map>
#include <sstream>
#include <string>
#include <vector>

#include "common.cuh"
#include "nd_kernels.cuh"

namespace amgf {
namespace {

constexpr const char *kManifest = "amgf_hierarchy.txt";

std::string path_of(const std::string &dir, const std::string &name) { return dir + "/" + name; }

void write_bytes(const std::string &path, const void *p, size_t bytes) {
  FILE *f = fopen(path.c_str(), "wb");
  REQUIRE(f, AMGF_ERR_ARG, "export: cannot open " + path + " for writing");
  const size_t w = bytes ? fwrite(p, 1, bytes, f) : 0;
  const int cl = fclose(f);
  REQUIRE(w == bytes && cl == 0, AMGF_ERR_ARG, "export: short write to " + path);
}

template <class T>
std::vector<T> read_vec(const std::string &path, size_t count) {
  FILE *f = fopen(path.c_str(), "rb");
  REQUIRE(f, AMGF_ERR_FORMAT, "import: missing " + path);
  fseek(f, 0, SEEK_END);
  const long size = ftell(f);
  fseek(f, 0, SEEK_SET);
  REQUIRE(size == (long)(count * sizeof(T)), AMGF_ERR_FORMAT,
          "import: " + path + " has " + std::to_string(size) + " bytes, expected " + std::to_string(count * sizeof(T)));
  std::vector<T> v(count);
  const size_t r = count ? fread(v.data(), sizeof(T), count, f) : 0;
  fclose(f);
  REQUIRE(r == count, AMGF_ERR_FORMAT, "import: short read of " + path);
  return v;
}

template <class T>
std::vector<T> d2h(Ctx &c, const T *src, size_t count) {
  std::vector<T> v(count);
  if (count) CK(cudaMemcpyAsync(v.data(), src, count * sizeof(T), cudaMemcpyDeviceToHost, c.stream));
  CK(cudaStreamSynchronize(c.stream));
  return v;
}

template <class T>
T *h2d_new(Ctx &c, const std::vector<T> &v) {
  T *d = c.alloc<T>(v.size());
  if (!v.empty()) CK(cudaMemcpyAsync(d, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, c.stream));
  CK(cudaStreamSynchronize(c.stream));  // the host vectors go out of scope
  return d;
}

// Dense lower factor of a band store Lrow (row i: L_ik at Lrow[i*W + bw - (i-k)]).
void band_to_dense(const std::vector<double> &band, int n, int bw, int W, std::vector<double> &L) {
  for (int i = 0; i < n; i++)
    for (int t = 0; t <= bw && t <= i; t++) L[(size_t)i * n + (i - t)] = band[(size_t)i * W + bw - t];
}

struct Manifest {
  std::map<std::string, std::string> kv;
  struct Lev { long nodes, b, nnzb, nnzb_P, n_agg; };
  std::vector<Lev> lev;
  long get(const std::string &k) const {
    auto it = kv.find(k);
    REQUIRE(it != kv.end(), AMGF_ERR_FORMAT, "import: manifest lacks '" + k + "'");
    return std::stol(it->second);
  }
  bool has(const std::string &k) const { return kv.count(k) != 0; }
};

Manifest read_manifest(const std::string &dir) {
  std::ifstream f(path_of(dir, kManifest));
  REQUIRE(f.good(), AMGF_ERR_FORMAT, "import: missing " + path_of(dir, kManifest));
  Manifest M;
  std::string line;
  REQUIRE(std::getline(f, line) && line.rfind("amgf_hierarchy 1", 0) == 0, AMGF_ERR_FORMAT,
          "import: not an amgf_hierarchy 1 manifest");
  while (std::getline(f, line)) {
    std::istringstream is(line);
    std::string key;
    if (!(is >> key)) continue;
    if (key == "level") {
      long l;
      Manifest::Lev v{};
      REQUIRE(bool(is >> l >> v.nodes >> v.b >> v.nnzb >> v.nnzb_P >> v.n_agg) && l == (long)M.lev.size(),
              AMGF_ERR_FORMAT, "import: bad level line '" + line + "'");
      M.lev.push_back(v);
    } else {
      std::string val;
      is >> val;
      M.kv[key] = val;
    }
  }
  return M;
}

// BSR consistency: ptr from 0 to nnzb, nondecreasing; columns in range and strictly ascending per row.
void check_bsr(const std::vector<int> &ptr, const std::vector<int> &col, long nbc, const std::string &what) {
  REQUIRE(!ptr.empty() && ptr[0] == 0 && ptr.back() == (long)col.size(), AMGF_ERR_FORMAT, "import: " + what + " ptr");
  for (size_t i = 0; i + 1 < ptr.size(); i++) {
    REQUIRE(ptr[i] <= ptr[i + 1], AMGF_ERR_FORMAT, "import: " + what + " ptr not monotone");
    for (int k = ptr[i]; k < ptr[i + 1]; k++)
      REQUIRE(col[k] >= 0 && col[k] < nbc && (k == ptr[i] || col[k] > col[k - 1]), AMGF_ERR_FORMAT,
              "import: " + what + " columns out of range or not ascending in row " + std::to_string(i));
  }
}

void load_bsr(Ctx &c, Bsr &A, const std::string &dir, const std::string &stem, int nbr, int nbc, int br, int bc,
              long nnzb) {
  auto ptr = read_vec<int>(path_of(dir, stem + "_ptr.i32"), (size_t)nbr + 1);
  auto col = read_vec<int>(path_of(dir, stem + "_col.i32"), (size_t)nnzb);
  auto val = read_vec<double>(path_of(dir, stem + "_val.f64"), (size_t)nnzb * br * bc);
  check_bsr(ptr, col, nbc, stem);
  A.nbr = nbr; A.nbc = nbc; A.br = br; A.bc = bc; A.nnzb = nnzb;
  A.ptr = h2d_new(c, ptr);
  A.col = h2d_new(c, col);
  A.val = h2d_new(c, val);
}

void save_bsr(Ctx &c, const Bsr &A, const std::string &dir, const std::string &stem) {
  auto ptr = d2h(c, A.ptr, (size_t)A.nbr + 1);
  auto col = d2h(c, A.col, (size_t)A.nnzb);
  auto val = d2h(c, A.val, (size_t)A.nnzb * A.br * A.bc);
  write_bytes(path_of(dir, stem + "_ptr.i32"), ptr.data(), ptr.size() * 4);
  write_bytes(path_of(dir, stem + "_col.i32"), col.data(), col.size() * 4);
  write_bytes(path_of(dir, stem + "_val.f64"), val.data(), val.size() * 8);
}

}  // namespace

// --------------------------------------------------------------------------- export
static void export_impl(Ctx &c, const std::string &dir) {
  REQUIRE(c.cfg.filter_basis == 0, AMGF_ERR_ARG, "export: the exchange format holds the identity filter basis only");
  REQUIRE(c.cfg.smoother != 2, AMGF_ERR_ARG, "export: the exchange format holds no block-smoother factors");
  CK(cudaStreamSynchronize(c.stream));
  {
    std::ofstream f(path_of(dir, kManifest));
    REQUIRE(f.good(), AMGF_ERR_ARG, "export: cannot write " + path_of(dir, kManifest));
    char ratio[64];
    snprintf(ratio, sizeof ratio, "%.17g", c.cfg.cheb_ratio);
    f << "amgf_hierarchy 1\n"
      << "nodes " << c.nodes << "\nnlev " << c.nlev << "\nnc " << c.nc << "\nbw " << c.bw << "\nnco " << c.nco
      << "\npre_sweeps " << c.cfg.pre_sweeps << "\npost_sweeps " << c.cfg.post_sweeps << "\nsmoother "
      << c.cfg.smoother << "\ncheb_degree " << c.cfg.cheb_degree << "\ncheb_ratio " << ratio << "\nnd_levels "
      << c.cfg.nd_levels << "\ncoarsest_size " << c.cfg.coarsest_size << "\nmax_levels " << c.cfg.max_levels
      << "\npower_iters " << c.cfg.power_iters << "\nagg_seed " << c.cfg.agg_seed << "\n";
    for (int l = 0; l < c.nlev; l++) {
      const Level &L = c.lev[l];
      const bool co = l == c.nlev - 1;
      f << "level " << l << " " << L.nodes << " " << L.b << " " << L.A.nnzb << " " << (co ? 0 : L.P.nnzb) << " "
        << (co ? 0 : L.n_agg) << "\n";
    }
    REQUIRE(f.good(), AMGF_ERR_ARG, "export: manifest write failed");
  }
  for (int l = 0; l < c.nlev; l++) {
    Level &L = c.lev[l];
    const std::string p = "L" + std::to_string(l);
    save_bsr(c, L.A, dir, p + "_A");
    auto d = d2h(c, L.dl1, (size_t)L.n);
    write_bytes(path_of(dir, p + "_l1.f64"), d.data(), d.size() * 8);
    if (l < c.nlev - 1) {
      save_bsr(c, L.P, dir, p + "_P");
      save_bsr(c, L.R, dir, p + "_R");
    }
  }
  auto Z = d2h(c, c.Z, (size_t)c.nc);
  write_bytes(path_of(dir, "Z.i32"), Z.data(), Z.size() * 4);
  const int nc = c.nc;
  std::vector<int> pi(nc);
  std::vector<double> Lw((size_t)nc * nc, 0.0);
  if (nc > 0) {
    pi = d2h(c, c.pi_z, (size_t)nc);
    const int W = band_stride(c.bw);
    band_to_dense(d2h(c, c.Lrow, (size_t)nc * W), nc, c.bw, W, Lw);
    auto blk = d2h(c, (const NdBlk *)c.nd_blk, (size_t)c.nd_nblocks);
    auto off = d2h(c, c.Loff, (size_t)c.loff_size);
    for (const NdBlk &b : blk)
      if (b.kind == 1)
        for (int s = 0; s < b.len; s++)
          for (int k = b.t0; k < b.p0; k++) Lw[(size_t)(b.p0 + s) * nc + k] = off[b.off + (size_t)s * b.rs + (k - b.t0)];
  }
  write_bytes(path_of(dir, "pi.i32"), pi.data(), pi.size() * 4);
  write_bytes(path_of(dir, "Lw.f64"), Lw.data(), Lw.size() * 8);
  const int nco = c.nco, Wc = band_stride(nco - 1);
  std::vector<double> Lc((size_t)nco * nco, 0.0);
  band_to_dense(d2h(c, c.Lc_row, (size_t)nco * Wc), nco, nco - 1, Wc, Lc);
  write_bytes(path_of(dir, "Lc.f64"), Lc.data(), Lc.size() * 8);
}

// --------------------------------------------------------------------------- import
static void import_impl(Ctx &c, const std::string &dir, void *stream) {
  const Manifest M = read_manifest(dir);
  amgf_default_config(&c.cfg);
  auto cfgi = [&](const char *k, int32_t &dst) { if (M.has(k)) dst = (int32_t)M.get(k); };
  cfgi("pre_sweeps", c.cfg.pre_sweeps);
  cfgi("post_sweeps", c.cfg.post_sweeps);
  cfgi("smoother", c.cfg.smoother);
  cfgi("cheb_degree", c.cfg.cheb_degree);
  cfgi("nd_levels", c.cfg.nd_levels);
  cfgi("coarsest_size", c.cfg.coarsest_size);
  cfgi("max_levels", c.cfg.max_levels);
  cfgi("power_iters", c.cfg.power_iters);
  if (M.has("cheb_ratio")) c.cfg.cheb_ratio = std::stod(M.kv.at("cheb_ratio"));
  if (M.has("agg_seed")) c.cfg.agg_seed = std::stoull(M.kv.at("agg_seed"), nullptr, 0);
  ctx_init(c, stream);
  c.imported = true;
  c.nodes = (int)M.get("nodes");
  c.n = 3L * c.nodes;
  c.m = 0;
  c.nlev = (int)M.get("nlev");
  REQUIRE(c.nodes > 0 && c.nlev >= 1 && c.nlev <= MAXLEV && (int)M.lev.size() == c.nlev, AMGF_ERR_FORMAT,
          "import: inconsistent nodes / nlev / level lines");
  c.dot_part = c.alloc<double>(nblk(c.n) + 1);
  // ---- levels
  for (int l = 0; l < c.nlev; l++) {
    const Manifest::Lev &v = M.lev[l];
    Level &L = c.lev[l];
    const bool co = l == c.nlev - 1;
    REQUIRE(v.b == (l == 0 ? 3 : 6) && v.nodes > 0 && v.nnzb > 0, AMGF_ERR_FORMAT, "import: level " + std::to_string(l));
    REQUIRE(l > 0 || v.nodes == c.nodes, AMGF_ERR_FORMAT, "import: level 0 size differs from nodes");
    REQUIRE(l == 0 || v.nodes == M.lev[l - 1].n_agg, AMGF_ERR_FORMAT, "import: level sizes do not chain");
    L.b = (int)v.b;
    L.nodes = (int)v.nodes;
    L.n = (long)v.nodes * v.b;
    const std::string p = "L" + std::to_string(l);
    load_bsr(c, L.A, dir, p + "_A", L.nodes, L.nodes, L.b, L.b, v.nnzb);
    L.dl1 = h2d_new(c, read_vec<double>(path_of(dir, p + "_l1.f64"), (size_t)L.n));
    if (!co) {
      REQUIRE(v.n_agg > 0 && v.nnzb_P > 0, AMGF_ERR_FORMAT, "import: level " + std::to_string(l) + " transfer sizes");
      L.n_agg = (int)v.n_agg;
      load_bsr(c, L.P, dir, p + "_P", L.nodes, L.n_agg, L.b, 6, v.nnzb_P);
      load_bsr(c, L.R, dir, p + "_R", L.n_agg, L.nodes, 6, L.b, v.nnzb_P);
      if (L.b == 3) r_interleave(c, L.R);
    }
  }
  Level &L0 = c.lev[0];
  // ---- Z, pos
  c.nc = (int)M.get("nc");
  REQUIRE(c.nc >= 0 && c.nc <= c.n, AMGF_ERR_FORMAT, "import: nc");
  {
    auto Z = read_vec<int>(path_of(dir, "Z.i32"), (size_t)c.nc);
    std::vector<int> pos((size_t)c.n, -1);
    for (int a = 0; a < c.nc; a++) {
      REQUIRE(Z[a] >= 0 && Z[a] < c.n && pos[Z[a]] < 0, AMGF_ERR_FORMAT, "import: Z out of range or duplicate");
      pos[Z[a]] = a;
    }
    c.Z = h2d_new(c, Z);
    c.pos = h2d_new(c, pos);
  }
  // ---- A_w factor into the nested-dissection layout (filter.cu)
  if (c.nc > 0) {
    const int nc = c.nc;
    c.nf = nc;
    c.bw = band_width(c);
    REQUIRE(c.bw == M.get("bw"), AMGF_ERR_FORMAT,
            "import: bw " + std::to_string(M.get("bw")) + " is not the band width of S[Z,Z] (" + std::to_string(c.bw) + ")");
    nd_symbolic(c);
    auto pi_ref = d2h(c, c.pi_z, (size_t)nc);
    REQUIRE(read_vec<int>(path_of(dir, "pi.i32"), (size_t)nc) == pi_ref, AMGF_ERR_FORMAT,
            "import: pi is not the nested-dissection order of (nc, bw, nd_levels)");
    const auto Lw = read_vec<double>(path_of(dir, "Lw.f64"), (size_t)nc * nc);
    const int W = band_stride(c.bw);
    auto blk = d2h(c, (const NdBlk *)c.nd_blk, (size_t)c.nd_nblocks);
    std::vector<double> band((size_t)nc * W, 0.0), off((size_t)c.loff_size, 0.0);
    std::vector<char> used((size_t)nc * nc, 0);  // entries the layout holds (the rest must be zero)
    for (const NdBlk &b : blk) {
      for (int i = b.p0; i < b.p0 + b.len; i++)
        for (int k = std::max(b.p0, i - c.bw); k <= i; k++) {
          band[(size_t)i * W + c.bw - (i - k)] = Lw[(size_t)i * nc + k];
          used[(size_t)i * nc + k] = 1;
        }
      if (b.kind == 1)
        for (int s = 0; s < b.len; s++)
          for (int k = b.t0; k < b.p0; k++) {
            off[b.off + (size_t)s * b.rs + (k - b.t0)] = Lw[(size_t)(b.p0 + s) * nc + k];
            used[(size_t)(b.p0 + s) * nc + k] = 1;
          }
    }
    for (size_t q = 0; q < Lw.size(); q++)
      REQUIRE(used[q] || Lw[q] == 0.0, AMGF_ERR_FORMAT,
              "import: the A_w factor has a nonzero outside the nested-dissection structure (row " +
                  std::to_string(q / nc) + ", column " + std::to_string(q % nc) + ")");
    for (int i = 0; i < nc; i++)
      REQUIRE(Lw[(size_t)i * nc + i] > 0.0, AMGF_ERR_FORMAT, "import: non-positive A_w factor diagonal");
    CK(cudaMemcpyAsync(c.Lrow, band.data(), band.size() * 8, cudaMemcpyHostToDevice, c.stream));
    if (c.loff_size) CK(cudaMemcpyAsync(c.Loff, off.data(), off.size() * 8, cudaMemcpyHostToDevice, c.stream));
    band_finish(c, nc, c.bw, c.Lrow, c.Lcol, c.Lrev, c.Ldinv);
    CK(cudaStreamSynchronize(c.stream));
    build_thin(c);
  }
  // ---- solve layouts of the levels (as setup_all)
  for (int l = 0; l + 1 < c.nlev; l++) {
    Level &L = c.lev[l];
    const bool sort_level = l > 0 && L.n > 16384;
    build_sell(c, L.A, L.As, true, l > 0, sort_level);
    build_sell(c, L.P, L.Ps, true, l > 0, l == 0 || sort_level);
  }
  // ---- coarsest factor
  {
    c.nco = (int)c.lev[c.nlev - 1].n;
    REQUIRE(c.nco == M.get("nco") && c.nco <= 16384, AMGF_ERR_FORMAT, "import: coarsest size");
    const int nco = c.nco, bw = nco - 1, W = band_stride(bw);
    const auto Lc = read_vec<double>(path_of(dir, "Lc.f64"), (size_t)nco * nco);
    std::vector<double> band((size_t)nco * W, 0.0);
    for (int i = 0; i < nco; i++) {
      REQUIRE(Lc[(size_t)i * nco + i] > 0.0, AMGF_ERR_FORMAT, "import: non-positive coarsest factor diagonal");
      for (int k = 0; k <= i; k++) band[(size_t)i * W + bw - (i - k)] = Lc[(size_t)i * nco + k];
      for (int k = i + 1; k < nco; k++)
        REQUIRE(Lc[(size_t)i * nco + k] == 0.0, AMGF_ERR_FORMAT, "import: coarsest factor not lower triangular");
    }
    coarsest_alloc(c);
    CK(cudaMemcpyAsync(c.Lc_row, band.data(), band.size() * 8, cudaMemcpyHostToDevice, c.stream));
    band_finish(c, nco, bw, c.Lc_row, c.Lc_col, c.Lc_rev, c.Lc_dinv);
    CK(cudaStreamSynchronize(c.stream));
  }
  (void)L0;
  alloc_workspaces(c);
  CK(cudaStreamSynchronize(c.stream));
  tail_plan(c);
}

}  // namespace amgf

using namespace amgf;

extern "C" {

amgf_status amgf_export(amgf_handle h, const char *dir) {
  if (!h || !dir) { set_error("null argument"); return AMGF_ERR_ARG; }
  return guarded([&]() -> amgf_status {
    export_impl(*h, dir);
    return AMGF_OK;
  });
}

amgf_status amgf_import(const char *dir, void *stream, amgf_handle *out) {
  if (!out) { set_error("out is NULL"); return AMGF_ERR_ARG; }
  *out = nullptr;
  if (!dir) { set_error("null dir"); return AMGF_ERR_ARG; }
  amgf_ctx *c = new amgf_ctx();
  const auto t0 = std::chrono::steady_clock::now();
  amgf_status st = guarded([&]() -> amgf_status {
    import_impl(*c, dir, stream);
    return AMGF_OK;
  });
  if (st != AMGF_OK) {
    cudaStreamSynchronize((cudaStream_t)stream);
    delete c;
    return st;
  }
  c->last_setup_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  *out = c;
  return AMGF_OK;
}

}  // extern "C"
