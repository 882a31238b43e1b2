// elastic.cuh — Neo-Hookean tet energy / gradient / F-space-projected Hessian (closed form) and the
// ABD orthogonality energy.  P:L86, P:L358 (NH with Young's modulus and Poisson ratio); density
// Ψ = μ/2(tr FᵀF − 3) − μ ln J + λ/2 (ln J)² (reading R3).  Projection: clamp negative eigenvalues
// of ∂²Ψ/∂F² to 0 (reading R4), using the analytic eigensystem in the SVD frame of F:
//   3 "scaling" modes from A_ij = μδ_ij + λ/(σ_iσ_j) + kδ_ij/σ_i², k = μ − λ ln J,
//   6 "twist/flip" modes μ ± k/(σ_iσ_j) with Q = U (e_ie_jᵀ ± e_je_iᵀ) Vᵀ/√2.
// The 12×12 block is Δt²V_e Bᵀ H⁺ B with B = ∂vec F/∂x; with β_k the rows of ∂F/∂x (β_0 =
// −Σβ_k) and h_k = F⁻ᵀβ_k:  H[(k,c),(l,d)] = μ(β_k·β_l)δ_cd + λ h_k[c]h_l[d] + k h_l[c]h_k[d]
//   − Σ_{λ_m<0} λ_m (Q_mβ_k)_c (Q_mβ_l)_d.
#pragma once
#include "common.cuh"

namespace tac {

// Cyclic Jacobi eigen-decomposition of a symmetric 3×3 (row-major A, destroyed).  Eigenvalues in
// w, eigenvectors as COLUMNS of V (row-major).
HD void sym3_eig(double* A, double* w, double* V) {
  for (int i = 0; i < 9; ++i) V[i] = (i % 4 == 0) ? 1.0 : 0.0;
  for (int sweep = 0; sweep < 20; ++sweep) {
    double off = A[1] * A[1] + A[2] * A[2] + A[5] * A[5];
    double dg = A[0] * A[0] + A[4] * A[4] + A[8] * A[8];
    if (off <= 1e-34 * dg || off == 0.0) break;
    for (int pq = 0; pq < 3; ++pq) {
      int p = (pq == 2) ? 1 : 0, q = (pq == 0) ? 1 : 2;
      double apq = A[3 * p + q];
      if (apq == 0.0) continue;
      double app = A[3 * p + p], aqq = A[3 * q + q];
      double tau = (aqq - app) / (2.0 * apq);
      double t = (tau >= 0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
      double c = 1.0 / sqrt(1.0 + t * t), s = t * c;
      for (int k = 0; k < 3; ++k) {  // A ← A J (columns p, q)
        double akp = A[3 * k + p], akq = A[3 * k + q];
        A[3 * k + p] = c * akp - s * akq;
        A[3 * k + q] = s * akp + c * akq;
      }
      for (int k = 0; k < 3; ++k) {  // A ← Jᵀ A (rows p, q)
        double apk = A[3 * p + k], aqk = A[3 * q + k];
        A[3 * p + k] = c * apk - s * aqk;
        A[3 * q + k] = s * apk + c * aqk;
      }
      for (int k = 0; k < 3; ++k) {  // V ← V J
        double vkp = V[3 * k + p], vkq = V[3 * k + q];
        V[3 * k + p] = c * vkp - s * vkq;
        V[3 * k + q] = s * vkp + c * vkq;
      }
    }
  }
  w[0] = A[0]; w[1] = A[4]; w[2] = A[8];
}

// Deformation gradient F = D_s D_m⁻¹ (D_s columns x1−x0, x2−x0, x3−x0); Dmi row-major.
HD void deformation_gradient(const v3* x, const double* Dmi, double* F) {
  v3 c0 = x[1] - x[0], c1 = x[2] - x[0], c2 = x[3] - x[0];
  for (int a = 0; a < 3; ++a) {
    double r0 = comp(c0, a), r1 = comp(c1, a), r2 = comp(c2, a);
    for (int b = 0; b < 3; ++b) F[3 * a + b] = r0 * Dmi[b] + r1 * Dmi[3 + b] + r2 * Dmi[6 + b];
  }
}

// Energy only (line search); returns +inf-flag through *inverted when det F <= 0.
HD double nh_energy(const v3* x, const double* Dmi, double mu, double lam, bool* inverted) {
  double F[9];
  deformation_gradient(x, Dmi, F);
  double J = det33(F);
  if (!(J > 0.0)) { *inverted = true; return 0.0; }
  double lnJ = log(J), I = 0.0;
  for (int i = 0; i < 9; ++i) I += F[i] * F[i];
  return 0.5 * mu * (I - 3.0) - mu * lnJ + 0.5 * lam * lnJ * lnJ;
}

// Gradient g[12] (slot-major: 3*k + c) and packed-upper projected Hessian H[78] of scale·Ψ(F(x)).
// Outputs go through store functors: gst(i, value) for the 12 gradient entries, hst(r, s, value) for r ≤ s
// for the 78 Hessian entries (k_tets stores straight to its SoA buffer, no local arrays)
template <class GStore, class HStore>
HD void nh_grad_hess_t(const v3* x, const double* Dmi, double mu, double lam, double scale, double* psi_out,
                       GStore gst, HStore hst, bool project) {
  double F[9];
  deformation_gradient(x, Dmi, F);
  double J = det33(F);
  double lnJ = log(J);
  double Fi[9];
  inv33(F, Fi);  // F⁻¹; F⁻ᵀ[a][b] = Fi[b][a]
  double I = 0.0;
  for (int i = 0; i < 9; ++i) I += F[i] * F[i];
  if (psi_out) *psi_out = 0.5 * mu * (I - 3.0) - mu * lnJ + 0.5 * lam * lnJ * lnJ;
  // β_k: rows of D_m⁻¹ (k=1..3), β_0 = −Σ
  v3 beta[4];
  beta[1] = ld3(Dmi); beta[2] = ld3(Dmi + 3); beta[3] = ld3(Dmi + 6);
  beta[0] = -(beta[1] + beta[2] + beta[3]);
  // P = μF + (λ ln J − μ) F⁻ᵀ ; gradient (k,c) = (P β_k)_c
  double P[9];
  double cP = lam * lnJ - mu;
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) P[3 * a + b] = mu * F[3 * a + b] + cP * Fi[3 * b + a];
  for (int k = 0; k < 4; ++k) {
    const v3 gk = scale * mul33(P, beta[k]);
    gst(3 * k, gk.x); gst(3 * k + 1, gk.y); gst(3 * k + 2, gk.z);
  }
  // h_k = F⁻ᵀ β_k
  v3 h[4];
  for (int k = 0; k < 4; ++k) h[k] = mul33T(Fi, beta[k]);
  const double kk = mu - lam * lnJ;
  // negative modes: collect up to 9 (λ_m, Q_m) and subtract (projected Hessians only; the exact
  // Hessian of the default LM Newton, R14c, needs no singular values)
  double negl[9]; double negQ[9][9]; int nneg = 0;
  if (project) {
    // SVD via eig(FᵀF): F = U Σ Vᵀ
    double C[9], sig2[3], Vm[9];
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) C[3 * a + b] = F[a] * F[b] + F[3 + a] * F[3 + b] + F[6 + a] * F[6 + b];
    sym3_eig(C, sig2, Vm);
    double sg[3];
    for (int i = 0; i < 3; ++i) sg[i] = sqrt(fmax(sig2[i], 0.0));
    double U[9];  // U = F V Σ⁻¹ (columns)
    for (int i = 0; i < 3; ++i) {
      v3 vi = mk(Vm[i], Vm[3 + i], Vm[6 + i]);
      v3 ui = (1.0 / sg[i]) * mul33(F, vi);
      U[i] = ui.x; U[3 + i] = ui.y; U[6 + i] = ui.z;
    }
    double A3[9];
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j)
        A3[3 * i + j] = lam / (sg[i] * sg[j]) + ((i == j) ? (mu + kk / (sg[i] * sg[i])) : 0.0);
    double w3[3], Q3[9];
    sym3_eig(A3, w3, Q3);
    for (int m = 0; m < 3; ++m) {
      if (w3[m] < 0.0) {
        // Q = U diag(q) Vᵀ, q = column m of Q3
        for (int a = 0; a < 3; ++a)
          for (int b = 0; b < 3; ++b) {
            double s = 0.0;
            for (int i = 0; i < 3; ++i) s += U[3 * a + i] * Q3[3 * i + m] * Vm[3 * b + i];
            negQ[nneg][3 * a + b] = s;
          }
        negl[nneg++] = w3[m];
      }
    }
    const int pi[3] = {0, 0, 1}, pj[3] = {1, 2, 2};
    const double r2 = 0.70710678118654752440;
    for (int t = 0; t < 3; ++t) {
      int i = pi[t], j = pj[t];
      double off = kk / (sg[i] * sg[j]);
      for (int sgn = -1; sgn <= 1; sgn += 2) {
        double lm = mu + sgn * off;
        if (lm < 0.0) {
          // Q = U (e_i e_jᵀ + sgn e_j e_iᵀ) Vᵀ / √2
          for (int a = 0; a < 3; ++a)
            for (int b = 0; b < 3; ++b)
              negQ[nneg][3 * a + b] = r2 * (U[3 * a + i] * Vm[3 * b + j] + sgn * U[3 * a + j] * Vm[3 * b + i]);
          negl[nneg++] = lm;
        }
      }
    }
  }
  // assemble packed upper 12×12
  v3 qb[9][4];
  for (int m = 0; m < nneg; ++m)
    for (int k = 0; k < 4; ++k) qb[m][k] = mul33(negQ[m], beta[k]);
#pragma unroll
  for (int r = 0; r < 12; ++r) {
    int k = r / 3, c = r % 3;
#pragma unroll
    for (int s = r; s < 12; ++s) {
      int l = s / 3, d = s % 3;
      double v = lam * comp(h[k], c) * comp(h[l], d) + kk * comp(h[l], c) * comp(h[k], d);
      if (c == d) v += mu * dot(beta[k], beta[l]);
      for (int m = 0; m < nneg; ++m) v -= negl[m] * comp(qb[m][k], c) * comp(qb[m][l], d);
      hst(r, s, scale * v);
    }
  }
}
HD void nh_grad_hess(const v3* x, const double* Dmi, double mu, double lam, double scale, double* psi_out,
                     double* g, double* H, bool project = true) {
  nh_grad_hess_t(x, Dmi, mu, lam, scale, psi_out, [&](int i, double v) { g[i] = v; },
                 [&](int r, int s, double v) { H[sym_idx(r, s, 12)] = v; }, project);
}

// ABD orthogonality energy E = κ V ‖AAᵀ − I‖²_F (reading R9 of the garbled ARAP term P:L116):
// gradient 4κV (AAᵀ−I)A and Hessian 4κV[δ_ac (AᵀA)_db + A_ad A_cb + G_ac δ_bd] on A row-major.
HD double ortho_energy(const double* A, double kv) {
  double e = 0.0;
  for (int a = 0; a < 3; ++a)
    for (int c = 0; c < 3; ++c) {
      double G = A[3 * a] * A[3 * c] + A[3 * a + 1] * A[3 * c + 1] + A[3 * a + 2] * A[3 * c + 2] - (a == c ? 1.0 : 0.0);
      e += G * G;
    }
  return kv * e;
}
HD void ortho_grad(const double* A, double kv, double* g9) {
  double G[9];
  for (int a = 0; a < 3; ++a)
    for (int c = 0; c < 3; ++c)
      G[3 * a + c] = A[3 * a] * A[3 * c] + A[3 * a + 1] * A[3 * c + 1] + A[3 * a + 2] * A[3 * c + 2] - (a == c ? 1.0 : 0.0);
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) g9[3 * a + b] = 4.0 * kv * (G[3 * a] * A[b] + G[3 * a + 1] * A[3 + b] + G[3 * a + 2] * A[6 + b]);
}
HD double ortho_hess_entry(const double* A, double kv, int r, int s) {
  int a = r / 3, b = r % 3, c = s / 3, d = s % 3;
  double AtA_db = A[d] * A[b] + A[3 + d] * A[3 + b] + A[6 + d] * A[6 + b];
  double G_ac = A[3 * a] * A[3 * c] + A[3 * a + 1] * A[3 * c + 1] + A[3 * a + 2] * A[3 * c + 2] - (a == c ? 1.0 : 0.0);
  double v = A[3 * a + d] * A[3 * c + b];
  if (a == c) v += AtA_db;
  if (b == d) v += G_ac;
  return 4.0 * kv * v;
}

}  // namespace tac
