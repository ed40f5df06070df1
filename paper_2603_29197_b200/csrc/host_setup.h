// Host-side (CPU, run once per problem) structure building: CSC transposes, KKT
// pattern + index maps, fill-reducing ordering and the supernodal symbolic
// analysis that drives the GPU LDL' factorisation.  Nothing here runs per
// iteration.
#pragma once
#include <stdint.h>

#include <string>
#include <vector>

typedef long long i64;

// ---- CSC <-> CSR ---------------------------------------------------------
// (tp, ti, tx) = transpose of the rows x cols CSC matrix (p, i, x); stable, so
// indices inside each output column ascend.
void hs_transpose(i64 rows, i64 cols, const i64* p, const i64* i, const double* x, i64* tp, i64* ti, double* tx);

// ---- KKT assembly (reference: kkt.py:55-135) ------------------------------
struct KktDims {
  i64 n, p, m, l, nsoc;
  const i64* q;  // [nsoc]
};
i64 hs_kkt_nnz(const KktDims& d, const i64* Pp, const i64* Pi, i64 nnzA, i64 nnzG);
i64 hs_slot_count(const KktDims& d);
// Ar/Gr are the CSR views (transposes) of A and G.  Outputs sized by hs_kkt_nnz
// / hs_slot_count; positions/slot arrays may be null.
void hs_kkt_assemble(const KktDims& d, const i64* Pp, const i64* Pi, const double* Px, const i64* Arp, const i64* Ari,
                     const double* Arx, const i64* Grp, const i64* Gri, const double* Grx, i64* Kp, i64* Ki,
                     double* Kx, i64* positions, i64* slot_offsets, i64* soc_slot_starts);

// Kp = column pointers of the full KKT matrix; (Kcp, Kci) = its pattern without the off-diagonal entries of the
// dense SOC blocks (what hs_symbolic_cliques needs next to the clique ranges).  O(N + nnz(P, A, G)).
void hs_kkt_pattern(const KktDims& d, const i64* Pp, const i64* Pi, const i64* Arp, const i64* Ari, const i64* Grp,
                    const i64* Gri, i64* Kp, std::vector<i64>* Kcp, std::vector<i64>* Kci);

// ---- symbolic analysis ------------------------------------------------------
struct Symbolic {
  i64 N = 0;
  std::vector<int> perm;   // perm[new] = old   (fill-reducing order composed with the postorder)
  std::vector<int> iperm;  // iperm[old] = new
  int nsup = 0;
  std::vector<int> col0;      // [nsup+1] first pivot column (new numbering) of each supernode
  std::vector<int> sup_of;    // [N] supernode of a (new) column
  std::vector<i64> rowptr;    // [nsup+1]
  std::vector<int> rowidx;    // front row lists: pivot columns first, then the update rows, ascending
  std::vector<int> parent;    // [nsup] parent supernode or -1
  std::vector<int> childptr;  // [nsup+1]
  std::vector<int> child;     // children, ascending
  std::vector<i64> relptr;    // [nsup+1] start of rel(s) (length nu(s))
  std::vector<int> rel;       // position of each update row of s inside the parent's row list
  std::vector<i64> Loff;      // [nsup+1] panel storage offsets (nr x ns, column major)
  std::vector<i64> Uoff;      // [nsup+1] update-matrix storage offsets (nu x nu)
  std::vector<i64> Boff;      // [nsup+1] solve contribution vector offsets (nu)
  int nlevels = 0;
  std::vector<int> levelptr;  // [nlevels+1]
  std::vector<int> levelsup;  // supernodes by level (leaves first)
  i64 lnz = 0;                // entries of L including the diagonal
  double flops = 0.0;
  int max_nr = 0, max_ns = 0;
};

// Pattern = upper-triangular CSC (Kp, Ki) of dimension N.  order: 0 natural,
// 1 AMD (own implementation, amd_order below), 2 user permutation in user_perm
// (user_perm[new] = old).  relax: amalgamate a chain child into its parent while
// the extra explicit zeros stay below relax_zeros_frac of the merged panel.
// Returns empty string on success, else the error text.
std::string hs_symbolic(i64 N, const i64* Kp, const i64* Ki, int order, const i64* user_perm, Symbolic* out);
// Same, told that the index ranges [clique_start[c], clique_start[c]+clique_size[c])
// are full cliques of the pattern (the dense SOC blocks): the ordering takes them
// as initial quotient-graph elements and the tree/count passes as stars, so the
// analysis costs O(nnz(P,A,G) + m) instead of O(nnz(K)).
std::string hs_symbolic_cliques(i64 N, const i64* Kp, const i64* Ki, int order, const i64* user_perm, i64 ncliques,
                                const i64* clique_start, const i64* clique_size, Symbolic* out);

// Approximate-minimum-degree ordering of the symmetric pattern given by its
// upper triangle.  perm[new] = old.
void amd_order(i64 N, const i64* Kp, const i64* Ki, std::vector<int>* perm);
