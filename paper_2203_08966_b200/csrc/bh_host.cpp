// bh_host.cpp -- host-side helpers of libbh.so for initial conditions (not the
// hot path).  They restate the reference's scalar generators operation for
// operation so that ICs are bit-identical to nbsim.initcond for a given seed:
// the Philox stream itself is drawn by numpy (the caller passes the doubles),
// and libm's pow/sqrt/sin/cos are the ones numpy's scalar paths call.
// Compiled with -ffp-contract=off (the reference never fuses multiply-adds).
#include <math.h>
#include <stdint.h>

extern "C" {

// initcond.py:62-77 plummer_cluster, consuming pre-drawn uniforms.
// Generates up to n bodies; stops early (returning the bodies completed) if
// the draw buffer runs out mid-body.  *used = draws consumed by the completed
// bodies.  pos/vel are [n][3].
int64_t bh_ic_plummer(const double *u, int64_t nu, int64_t n, double total_mass,
                      double *pos, double *vel, int64_t *used) {
  int64_t k = 0, done = 0;
  const double kPi2 = 2.0 * M_PI;
  const double vscale = sqrt(2.0 * total_mass);
  for (int64_t i = 0; i < n; ++i) {
    int64_t k0 = k;
    double r;
    // _radius (initcond.py:42-50)
    for (;;) {
      if (k >= nu) goto out;
      double a = u[k++];
      if (a == 0.0) continue;
      r = 1.0 / sqrt(pow(a, -2.0 / 3.0) - 1.0);
      if (r < 10.0) break;
    }
    {
      // _unit_vector (initcond.py:32-37)
      if (k + 2 > nu) { k = k0; goto out; }
      double z = 2.0 * u[k++] - 1.0;
      double phi = kPi2 * u[k++];
      double t = 1.0 - z * z;
      double s = sqrt(t > 0.0 ? t : 0.0);
      double ux = s * cos(phi), uy = s * sin(phi), uz = z;
      double v_esc = vscale * pow(1.0 + r * r, -0.25);
      // _speed_fraction (initcond.py:53-59)
      double q;
      for (;;) {
        if (k + 2 > nu) { k = k0; goto out; }
        q = u[k++];
        double g = 0.1 * u[k++];
        if (g < q * q * pow(1.0 - q * q, 3.5)) break;
      }
      double qv = q * v_esc;
      if (k + 2 > nu) { k = k0; goto out; }
      double z2 = 2.0 * u[k++] - 1.0;
      double phi2 = kPi2 * u[k++];
      double t2 = 1.0 - z2 * z2;
      double s2 = sqrt(t2 > 0.0 ? t2 : 0.0);
      pos[3 * i] = r * ux; pos[3 * i + 1] = r * uy; pos[3 * i + 2] = r * uz;
      vel[3 * i] = qv * (s2 * cos(phi2));
      vel[3 * i + 1] = qv * (s2 * sin(phi2));
      vel[3 * i + 2] = qv * z2;
      done = i + 1;
    }
  }
out:
  *used = k;
  return done;
}

// physics.py:273-285 _potential_pairs in its sequential pair order (used by
// initcond.standardize so that standardised ICs match the reference bitwise).
double bh_host_potential_pairs(const double *mass, const double *pos, int64_t n, double eps) {
  const double e2 = eps * eps;
  double pot = 0.0;
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = i + 1; j < n; ++j) {
      double dx = pos[3 * i] - pos[3 * j], dy = pos[3 * i + 1] - pos[3 * j + 1],
             dz = pos[3 * i + 2] - pos[3 * j + 2];
      double r2 = dx * dx + dy * dy + dz * dz;
      pot -= mass[i] * mass[j] / sqrt(r2 + e2);
    }
  return pot;
}
}

// ---------------------------------------------------------------------------
// Distributed build, host side: the top of the global tree from every rank's
// branch nodes (hashed.py:719-786 recombination), laid out for
// the walk.  Replaces a Python dict assembly that cost ~9 ms per step at 8
// ranks on cfg3.  Branch rows are the int32 rows decomposition._pack_branches
// allgathers: key (2), level, count (2), moments (10 doubles: mass, com[3],
// quad[6]), record index, first body, walk record (16).
//
// Output: the breadth-first top region, one 16-int walk record per entry.
//   kind 0  top cell: record built here (first child, nchild)
//   kind 1  bucket-sized top cell: record built here, bodies at its first
//           branch-body position
//   kind 2  branch node: the row's own record, unpatched (the caller redirects
//           its children / bodies to wherever that subtree lives)
// row_of[e] is the branch row of a kind-2 entry (else -1); bb[r] is the
// position of row r's bodies in the [own | bucket-sized branch bodies] list
// (bucket-sized rows only, else -1).  Combine arithmetic is _moments_kernel's
// (flattree.py:201-252), in the same expression order (-ffp-contract=off).
#include <algorithm>
#include <cstring>
#include <vector>

namespace {
constexpr int kBrInts = 2 + 1 + 2 + 20 + 1 + 1 + 16;
struct Mom {
  double m, c[3], q[6];
  int64_t count, bb;
};
inline int bitlen(uint64_t k) { return 64 - __builtin_clzll(k); }
inline int32_t fbits(float f) {
  int32_t i;
  memcpy(&i, &f, 4);
  return i;
}
}  // namespace

extern "C" int64_t bh_top_tree(const int32_t *rows, int64_t nrows, int64_t n_own, int leaf, double R,
                               double theta, int32_t *region, int32_t *kind, int32_t *row_of, int64_t *bb,
                               int64_t cap) {
  const int64_t BIG = int64_t(1) << 62;
  std::vector<uint64_t> rkey(nrows);
  std::vector<Mom> rmom(nrows);
  int64_t bbpos = n_own;
  for (int64_t r = 0; r < nrows; ++r) {
    const int32_t *w = rows + r * kBrInts;
    uint64_t key;
    int64_t count;
    memcpy(&key, w, 8);
    memcpy(&count, w + 3, 8);
    double mom[10];
    memcpy(mom, w + 5, 80);
    rkey[r] = key;
    Mom &M = rmom[r];
    M.m = mom[0];
    for (int a = 0; a < 3; ++a) M.c[a] = mom[1 + a];
    for (int a = 0; a < 6; ++a) M.q[a] = mom[4 + a];
    M.count = count;
    if (count <= leaf) {
      M.bb = bbpos;
      bb[r] = bbpos;
      bbpos += count;
    } else {
      M.bb = BIG;
      bb[r] = -1;
    }
  }
  // top cells: every proper ancestor of a branch node
  std::vector<uint64_t> top;
  top.reserve(nrows * 8);
  for (int64_t r = 0; r < nrows; ++r)
    for (uint64_t k = rkey[r] >> 3; k >= 1; k >>= 3) top.push_back(k);
  std::sort(top.begin(), top.end());
  top.erase(std::unique(top.begin(), top.end()), top.end());
  // every node (top cells and branch rows) sorted by key: the children of p
  // are the nodes with keys in [8p, 8p + 8), in slot order
  struct Node {
    uint64_t key;
    int64_t row;  // >= 0: a branch row; -1 - t: top cell t
  };
  std::vector<Node> nodes;
  nodes.reserve(top.size() + nrows);
  for (size_t t = 0; t < top.size(); ++t) nodes.push_back({top[t], -1 - (int64_t)t});
  for (int64_t r = 0; r < nrows; ++r) nodes.push_back({rkey[r], r});
  std::sort(nodes.begin(), nodes.end(), [](const Node &a, const Node &b) { return a.key < b.key; });
  auto child_range = [&](uint64_t p, size_t &b, size_t &e) {
    const uint64_t lo = p << 3, hi = lo + 8;
    b = std::lower_bound(nodes.begin(), nodes.end(), lo, [](const Node &x, uint64_t v) { return x.key < v; }) -
        nodes.begin();
    e = std::lower_bound(nodes.begin() + b, nodes.end(), hi, [](const Node &x, uint64_t v) { return x.key < v; }) -
        nodes.begin();
  };
  std::vector<Mom> tmom(top.size());
  auto mom_of = [&](const Node &x) -> const Mom & { return x.row >= 0 ? rmom[x.row] : tmom[-1 - x.row]; };
  // deepest first (hashed.py:719-786): children are final before their parent
  std::vector<size_t> order(top.size());
  for (size_t t = 0; t < top.size(); ++t) order[t] = t;
  std::stable_sort(order.begin(), order.end(),
                   [&](size_t a, size_t b) { return bitlen(top[a]) > bitlen(top[b]); });
  for (size_t t : order) {
    size_t b, e;
    child_range(top[t], b, e);
    double total = 0.0, cx = 0.0, cy = 0.0, cz = 0.0;
    int64_t count = 0, bbmin = BIG;
    for (size_t i = b; i < e; ++i) {
      const Mom &c = mom_of(nodes[i]);
      count += c.count;
      bbmin = std::min(bbmin, c.bb);
      if (c.m == 0.0) continue;
      total += c.m;
      cx += c.m * c.c[0];
      cy += c.m * c.c[1];
      cz += c.m * c.c[2];
    }
    Mom &M = tmom[t];
    M.count = count;
    M.bb = bbmin;
    for (int a = 0; a < 6; ++a) M.q[a] = 0.0;
    if (total == 0.0) {
      M.m = 0.0;
      M.c[0] = M.c[1] = M.c[2] = 0.0;
      continue;
    }
    cx /= total;
    cy /= total;
    cz /= total;
    double q[6] = {0, 0, 0, 0, 0, 0};
    for (size_t i = b; i < e; ++i) {
      const Mom &c = mom_of(nodes[i]);
      const double m = c.m;
      if (m == 0.0) continue;
      const double dx = c.c[0] - cx, dy = c.c[1] - cy, dz = c.c[2] - cz;
      const double d2 = dx * dx + dy * dy + dz * dz;
      q[0] += c.q[0] + m * (3.0 * (dx * dx) - d2);
      q[1] += c.q[1] + m * (3.0 * (dx * dy) - 0.0);
      q[2] += c.q[2] + m * (3.0 * (dx * dz) - 0.0);
      q[3] += c.q[3] + m * (3.0 * (dy * dy) - d2);
      q[4] += c.q[4] + m * (3.0 * (dy * dz) - 0.0);
      q[5] += c.q[5] + m * (3.0 * (dz * dz) - d2);
    }
    M.m = total;
    M.c[0] = cx;
    M.c[1] = cy;
    M.c[2] = cz;
    for (int a = 0; a < 6; ++a) M.q[a] = q[a];
  }
  // breadth-first layout, each cell's children contiguous in slot order
  auto record = [&](int64_t e, const Mom &M, uint64_t key, int32_t d0, int32_t nchild) {
    const int level = (bitlen(key) - 1) / 3;
    double mac2 = 1.0 / 0.0;
    if (theta != 0.0) {
      const double rr = ldexp(2.0 * R, -level) / theta;
      mac2 = rr * rr;
    }
    int32_t *o = region + e * 16;
    o[0] = fbits((float)-M.c[0]);
    o[1] = fbits((float)-M.c[1]);
    o[2] = fbits((float)-M.c[2]);
    o[3] = fbits((float)mac2);
    o[4] = fbits((float)M.q[0]);
    o[5] = fbits((float)M.q[1]);
    o[6] = fbits((float)M.q[1]);
    o[7] = fbits((float)M.q[3]);
    o[8] = fbits((float)M.q[2]);
    o[9] = fbits((float)M.q[4]);
    o[10] = fbits((float)M.m);
    o[11] = fbits((float)M.q[5]);
    o[12] = d0;
    o[13] = (int32_t)M.count;
    o[14] = nchild;
    o[15] = level;
  };
  auto put_branch = [&](int64_t e, int64_t r) {
    memcpy(region + e * 16, rows + r * kBrInts + 27, 16 * sizeof(int32_t));
    kind[e] = 2;
    row_of[e] = (int32_t)r;
  };
  int64_t ne = 0;
  if (top.empty()) {
    if (nrows == 0) return 0;
    if (cap < 1) return -1;
    put_branch(0, 0);
    return 1;
  }
  if (cap < 1) return -1;
  ne = 1;  // the root's slot
  struct Q {
    uint64_t key;
    int64_t at;
    size_t t;
  };
  std::vector<Q> queue;
  queue.push_back({1, 0, (size_t)(std::lower_bound(top.begin(), top.end(), (uint64_t)1) - top.begin())});
  for (size_t qi = 0; qi < queue.size(); ++qi) {
    const Q cur = queue[qi];
    const Mom &M = tmom[cur.t];
    if (cur.key != 1 && M.count <= leaf) {  // a bucket spanning ranks
      record(cur.at, M, cur.key, (int32_t)M.bb, 0);
      kind[cur.at] = 1;
      row_of[cur.at] = -1;
      continue;
    }
    size_t b, e;
    child_range(cur.key, b, e);
    const int64_t first = ne;
    for (size_t i = b; i < e; ++i) {
      if (ne >= cap) return -1;
      const Node &x = nodes[i];
      if (x.row >= 0) {
        put_branch(ne, x.row);
      } else {
        queue.push_back({x.key, ne, (size_t)(-1 - x.row)});
      }
      ++ne;
    }
    record(cur.at, M, cur.key, (int32_t)first, (int32_t)(e - b));
    kind[cur.at] = 0;
    row_of[cur.at] = -1;
  }
  return ne;
}
