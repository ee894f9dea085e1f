// Reference tetrahedron for the nodal DG operators (library side, fp64).
// PAPER.md P:407-414 (Appendix A): orthonormal polynomial basis on each element
// (mass matrix = multiple of I).  The library builds the nodal operators from
// that basis -- the orthonormal Dubiner/PKDO polynomials on the reference tet,
// evaluated with normalised Jacobi recurrences -- entirely in fp64, a route
// independent of the oracle's (shifted monomials + 50-digit mpmath).
#pragma once
#include <string>
#include <vector>

namespace dgb {

struct RefElem {
  int N = 0, Np = 0, Nfp = 0;
  std::vector<double> r, s, t;          // Np node coordinates (ABI order)
  std::vector<double> Dr, Ds, Dt;       // Np x Np row-major
  std::vector<double> LIFT;             // Np x 4Nfp row-major, columns face-major
  std::vector<int> Fmask;               // 4 x Nfp ascending node ids per face
  // face-local lattice coordinates of each face node: for face f node i, the
  // integer weights (over N) of the face's three vertices FACE_VERTS[f]
  std::vector<int> face_lat;            // 4 x Nfp x 3
  // nbr_local[((f*4 + f2)*6 + sigma)*Nfp + i]: face-local index j on neighbour
  // face f2 of my face node i when my face vertex m matches neighbour face
  // vertex PERM[sigma][m]
  std::vector<int> nbr_local;
  std::vector<double> Vinv;             // Np x Np inverse Vandermonde (orthonormal basis)
};

extern const int FACE_VERTS[4][3];
extern const int PERM6[6][3];

inline int n_nodes(int N) { return (N + 1) * (N + 2) * (N + 3) / 6; }
inline int n_face_nodes(int N) { return (N + 1) * (N + 2) / 2; }

// Builds everything above; returns false (with msg) on numerical failure.
bool build_reference(int N, RefElem& R, std::string* msg);

// Tables of the paper's modal-quadrature scheme (reading A23):
// orthonormal PKDO basis psi (the same polynomials as the nodal operators), collapsed
// Gauss-Jacobi rules with n = p+1 points per direction (exact to degree 2p+1) on the tet
// and on each face triangle.  Face points are those of the face's owner (smaller global
// element id): Pstd[f] evaluates psi at the standard rule of face f, Pmap[fa][fb][sigma] at
// the standard points of face fa carried onto face fb when face vertex m of fa matches
// face vertex PERM6[sigma][m] of fb.
struct ModalTables {
  int p = 0, Np = 0, NQ = 0, NQF = 0;
  std::vector<double> wq;               // NQ volume weights
  std::vector<double> Vq;               // NQ x Np   psi at the volume points
  std::vector<double> Dq;               // 3 x Np x NQ   w_q dpsi_i/d(r,s,t)
  std::vector<double> wf;               // NQF face weights (parameter measure, area 2)
  std::vector<double> Pstd;             // 4 x NQF x Np
  std::vector<double> Pmap;             // 4 x 4 x 6 x NQF x Np
  std::vector<double> V, Vinv;          // Np x Np nodal <-> modal (V_nm = psi_m(x_n))
};
bool build_modal(const RefElem& R, ModalTables& T, std::string* msg);
extern const int PERM6_INV[6];

// Nodal interpolation weights at a reference point: w_i = l_i(r,s,t) = sum_j Vinv[j][i] psi_j(r,s,t).
void interp_weights(const RefElem& R, double r, double s, double t, double* w);

}  // namespace dgb
