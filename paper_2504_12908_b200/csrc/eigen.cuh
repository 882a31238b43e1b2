// eigen.cuh — PSD projection of a symmetric n×n (n ≤ 12) by parallel cyclic Jacobi, executed by
// one warp on a matrix in shared memory (round-robin pairing: 6 disjoint rotations per round,
// 11 rounds per sweep).  The same code runs on the host with lane_begin=0, lane_stride=1 (used
// only by a dev check), so the device path is the only product path.
//   H⁺ = Q max(Λ, 0) Qᵀ   (clamp negative eigenvalues to 0: readings R4/R6/R12)
#pragma once
#include "common.cuh"

namespace tac {

#ifdef __CUDA_ARCH__
#define TAC_SYNCWARP() __syncwarp()
#else
#define TAC_SYNCWARP()
#endif

struct JacobiScratch {   // per-warp shared scratch
  double A[144];         // 12×12 row-major
  double Q[144];         // eigenvectors (columns)
  double c[6], s[6];
  int p[6], q[6];
  double red[32];
};

// round-robin pairs for 12 players: round r, k = 0..5
HD void rr_pair(int r, int k, int* p, int* q) {
  if (k == 0) { *p = 11; *q = r; return; }
  int a = (r + k) % 11, b = (r - k + 11) % 11;
  *p = a < b ? a : b; *q = a < b ? b : a;
}

// Input: S.A holds a symmetric 12×12 (pad unused rows/cols with zeros).  Output: S.A = H⁺.
HD void jacobi12_psd(JacobiScratch& S, int lane, int stride) {
  for (int i = lane; i < 144; i += stride) S.Q[i] = (i % 13 == 0) ? 1.0 : 0.0;
  TAC_SYNCWARP();
  for (int sweep = 0; sweep < 16; ++sweep) {
    // convergence test: off-diagonal mass vs diagonal mass
    double off = 0.0, dg = 0.0;
    for (int i = lane; i < 144; i += stride) {
      int r = i / 12, c = i % 12;
      double v = S.A[i] * S.A[i];
      if (r == c) dg += v; else off += v;
    }
#ifdef __CUDA_ARCH__
    for (int o = 16; o > 0; o >>= 1) {
      off += __shfl_xor_sync(0xffffffffu, off, o);
      dg += __shfl_xor_sync(0xffffffffu, dg, o);
    }
#endif
    if (off <= 1e-32 * dg || off == 0.0) break;
    for (int r = 0; r < 11; ++r) {
      for (int k = lane; k < 6; k += stride) {
        int p, q;
        rr_pair(r, k, &p, &q);
        double apq = S.A[12 * p + q], app = S.A[12 * p + p], aqq = S.A[12 * q + q];
        double c = 1.0, s = 0.0;
        if (apq != 0.0 && fabs(apq) > 1e-300) {
          double tau = (aqq - app) / (2.0 * apq);
          double t = (tau >= 0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
          c = 1.0 / sqrt(1.0 + t * t);
          s = t * c;
        }
        S.p[k] = p; S.q[k] = q; S.c[k] = c; S.s[k] = s;
      }
      TAC_SYNCWARP();
      // columns: A ← A J, Q ← Q J  (6 pairs × 12 rows each)
      for (int i = lane; i < 72; i += stride) {
        int k = i / 12, row = i % 12;
        int p = S.p[k], q = S.q[k];
        double c = S.c[k], s = S.s[k];
        double ap = S.A[12 * row + p], aq = S.A[12 * row + q];
        S.A[12 * row + p] = c * ap - s * aq;
        S.A[12 * row + q] = s * ap + c * aq;
        double qp = S.Q[12 * row + p], qq = S.Q[12 * row + q];
        S.Q[12 * row + p] = c * qp - s * qq;
        S.Q[12 * row + q] = s * qp + c * qq;
      }
      TAC_SYNCWARP();
      // rows: A ← Jᵀ A
      for (int i = lane; i < 72; i += stride) {
        int k = i / 12, col = i % 12;
        int p = S.p[k], q = S.q[k];
        double c = S.c[k], s = S.s[k];
        double ap = S.A[12 * p + col], aq = S.A[12 * q + col];
        S.A[12 * p + col] = c * ap - s * aq;
        S.A[12 * q + col] = s * ap + c * aq;
      }
      TAC_SYNCWARP();
    }
  }
  // eigenvalues on the diagonal; reconstruct H⁺ = Q max(Λ,0) Qᵀ into the upper triangle, then mirror
  double lam[12];
  for (int k = 0; k < 12; ++k) lam[k] = fmax(S.A[13 * k], 0.0);
  TAC_SYNCWARP();
  for (int i = lane; i < 144; i += stride) {
    int r = i / 12, c = i % 12;
    double v = 0.0;
    for (int k = 0; k < 12; ++k) v += S.Q[12 * r + k] * lam[k] * S.Q[12 * c + k];
    S.A[i] = v;
  }
  TAC_SYNCWARP();
  // exact symmetry: keep the upper triangle
  for (int i = lane; i < 144; i += stride) {
    int r = i / 12, c = i % 12;
    if (r > c) S.A[i] = S.A[12 * c + r];
  }
  TAC_SYNCWARP();
}

}  // namespace tac
