// geometry.cuh — point-triangle / edge-edge closest-point classification, squared distances and
// their closed-form first/second derivatives (hand-derived; the oracle uses autograd instead).
//
// Contact pairs are PT and EE pairs of surface primitives; the barrier acts on their
// distance.  Classification rules (readings R10/R11):
//   PT: interior iff projected barycentrics all >= 0 -> point-plane; else min over edges
//       e0=(t0,t1), e1=(t1,t2), e2=(t2,t0) of the clamped point-segment distance, ties to the
//       lowest edge.  types 0 P-T, 1..3 P-E0..2, 4..6 P-V0..2.
//   EE: Ericson clamped closest points (parallel iff a*e - b^2 <= 1e-14*a*e -> s = 0);
//       type = 3*state(s) + state(t), state 0 = endpoint 0, 1 = interior, 2 = endpoint 1.
// Slots of a pair: PT (p, t0, t1, t2); EE (a0, a1, b0, b1).
#pragma once
#include "common.cuh"

namespace tac {

enum { PT_T = 0, PT_E0 = 1, PT_V0 = 4, EE_LL = 4 };

HD double d2_pp(v3 p, v3 q) { v3 d = p - q; return dot(d, d); }
HD double d2_pl(v3 p, v3 a, v3 b) { v3 e = b - a; v3 c = cross(p - a, e); return dot(c, c) / dot(e, e); }
HD double d2_tri(v3 w, v3 e1, v3 e2) { v3 n = cross(e1, e2); double u = dot(w, n); return u * u / dot(n, n); }

HD int pt_classify(v3 p, v3 t0, v3 t1, v3 t2, double* d2) {
  v3 e1 = t1 - t0, e2 = t2 - t0, w = p - t0;
  double a11 = dot(e1, e1), a12 = dot(e1, e2), a22 = dot(e2, e2), b1 = dot(e1, w), b2 = dot(e2, w);
  double det = a11 * a22 - a12 * a12;
  double be1 = (a22 * b1 - a12 * b2) / det;
  double be2 = (a11 * b2 - a12 * b1) / det;
  double be0 = 1.0 - be1 - be2;
  if (be0 >= 0.0 && be1 >= 0.0 && be2 >= 0.0) { *d2 = d2_tri(w, e1, e2); return PT_T; }
  v3 T[3] = {t0, t1, t2};
  double best = 1.0e300; int bt = 0;
  for (int i = 0; i < 3; ++i) {
    v3 a = T[i], b = T[(i + 1) % 3];
    v3 e = b - a;
    double s = dot(p - a, e) / dot(e, e);
    double d; int ty;
    if (s <= 0.0) { d = d2_pp(p, a); ty = PT_V0 + i; }
    else if (s >= 1.0) { d = d2_pp(p, b); ty = PT_V0 + (i + 1) % 3; }
    else { d = d2_pl(p, a, b); ty = PT_E0 + i; }
    if (d < best) { best = d; bt = ty; }
  }
  *d2 = best;
  return bt;
}

HD int ee_classify(v3 a0, v3 a1, v3 b0, v3 b1, double* d2) {
  v3 d1 = a1 - a0, d2v = b1 - b0, r = a0 - b0;
  double A = dot(d1, d1), E = dot(d2v, d2v), F = dot(d2v, r), C = dot(d1, r), B = dot(d1, d2v);
  double denom = A * E - B * B;
  double s = 0.0;
  if (!(denom <= 1e-14 * A * E)) s = fmin(fmax((B * F - C * E) / denom, 0.0), 1.0);
  double t = (B * s + F) / E;
  if (t < 0.0) { t = 0.0; s = fmin(fmax(-C / A, 0.0), 1.0); }
  else if (t > 1.0) { t = 1.0; s = fmin(fmax((B - C) / A, 0.0), 1.0); }
  int ss = (s == 0.0) ? 0 : (s == 1.0 ? 2 : 1);
  int ts = (t == 0.0) ? 0 : (t == 1.0 ? 2 : 1);
  int ty = 3 * ss + ts;
  v3 pa[3] = {a0, a0, a1}, pb[3] = {b0, b0, b1};
  if (ss == 1 && ts == 1) *d2 = d2_tri(a0 - b0, d1, d2v);
  else if (ss == 1) *d2 = d2_pl(pb[ts], a0, a1);
  else if (ts == 1) *d2 = d2_pl(pa[ss], b0, b1);
  else *d2 = d2_pp(pa[ss], pb[ts]);
  return ty;
}

HD int classify(int kind, const v3* X, double* d2) {
  return kind == 0 ? pt_classify(X[0], X[1], X[2], X[3], d2) : ee_classify(X[0], X[1], X[2], X[3], d2);
}

// ----------------------------------------------------------------------------------------------
// Sub-distance derivative evaluator.  A sub-distance is a function of up to three "variable"
// vectors (w, e1/e, e2), each a ±1 combination of the 4 slots (coef[var][slot]).  gradient and
// Hessian entries are evaluated entry-by-entry so a warp can split the 12x12 among lanes.
// ----------------------------------------------------------------------------------------------
enum { SUB_PP = 0, SUB_PL = 1, SUB_TRI = 2 };

struct SubDist {
  int sub;
  signed char coef[3][4];
  v3 w, e1, e2;         // PP: w; PL: w, e1(=e); TRI: w, e1, e2
  // cached scalars
  double s;             // squared distance
  double N, D, we, ww;  // PL
  v3 n; double u;       // TRI: n = e1×e2, u = w·n, D = n·n
  double iD, iD2, iD3;  // 1/D, 1/D², 1/D³ (derivatives multiply instead of divide)
};

HD void sd_zero(SubDist& S) {
  for (int a = 0; a < 3; ++a) for (int b = 0; b < 4; ++b) S.coef[a][b] = 0;
}

HD v3 slot_combo(const signed char* c, const v3* X) {
  v3 r = mk(0, 0, 0);
  for (int k = 0; k < 4; ++k) if (c[k]) r += (double)c[k] * X[k];
  return r;
}

HD void sd_finish(SubDist& S, const v3* X) {
  S.w = slot_combo(S.coef[0], X);
  S.e1 = slot_combo(S.coef[1], X);
  S.e2 = slot_combo(S.coef[2], X);
  if (S.sub == SUB_PP) {
    S.s = dot(S.w, S.w);
  } else if (S.sub == SUB_PL) {
    S.ww = dot(S.w, S.w); S.D = dot(S.e1, S.e1); S.we = dot(S.w, S.e1);
    v3 c = cross(S.w, S.e1);
    S.N = dot(c, c);
    S.s = S.N / S.D;
    S.iD = 1.0 / S.D; S.iD2 = S.iD * S.iD; S.iD3 = S.iD2 * S.iD;
  } else {
    S.n = cross(S.e1, S.e2); S.u = dot(S.w, S.n); S.D = dot(S.n, S.n);
    S.s = S.u * S.u / S.D;
    S.iD = 1.0 / S.D; S.iD2 = S.iD * S.iD; S.iD3 = S.iD2 * S.iD;
  }
}

// Build the sub-distance of a classified pair.
HD void sd_make(SubDist& S, int kind, int type, const v3* X) {
  sd_zero(S);
  if (kind == 0) {
    if (type == PT_T) {
      S.sub = SUB_TRI;
      S.coef[0][0] = 1; S.coef[0][1] = -1;
      S.coef[1][2] = 1; S.coef[1][1] = -1;
      S.coef[2][3] = 1; S.coef[2][1] = -1;
    } else if (type < PT_V0) {
      int i = type - PT_E0, a = 1 + i, b = 1 + (i + 1) % 3;
      S.sub = SUB_PL;
      S.coef[0][0] = 1; S.coef[0][a] = -1;
      S.coef[1][b] = 1; S.coef[1][a] = -1;
    } else {
      S.sub = SUB_PP;
      S.coef[0][0] = 1; S.coef[0][1 + type - PT_V0] = -1;
    }
  } else {
    int ss = type / 3, ts = type % 3;
    if (ss == 1 && ts == 1) {
      S.sub = SUB_TRI;
      S.coef[0][0] = 1; S.coef[0][2] = -1;          // w  = a0 - b0
      S.coef[1][1] = 1; S.coef[1][0] = -1;          // e1 = a1 - a0
      S.coef[2][3] = 1; S.coef[2][2] = -1;          // e2 = b1 - b0
    } else if (ss == 1) {                           // point b(ts) vs line a0a1
      int p = ts == 0 ? 2 : 3;
      S.sub = SUB_PL;
      S.coef[0][p] = 1; S.coef[0][0] = -1;
      S.coef[1][1] = 1; S.coef[1][0] = -1;
    } else if (ts == 1) {                           // point a(ss) vs line b0b1
      int p = ss == 0 ? 0 : 1;
      S.sub = SUB_PL;
      S.coef[0][p] = 1; S.coef[0][2] = -1;
      S.coef[1][3] = 1; S.coef[1][2] = -1;
    } else {
      S.sub = SUB_PP;
      S.coef[0][ss == 0 ? 0 : 1] = 1; S.coef[0][ts == 0 ? 2 : 3] = -1;
    }
  }
  sd_finish(S, X);
}

// The EE mollifier argument c = ‖(a1−a0)×(b1−b0)‖² as a TRI-style D with e1, e2 (w unused).
HD void sd_make_cross(SubDist& S, const v3* X) {
  sd_zero(S);
  S.sub = SUB_TRI;
  S.coef[1][1] = 1; S.coef[1][0] = -1;
  S.coef[2][3] = 1; S.coef[2][2] = -1;
  sd_finish(S, X);
}

// skew(a)[r][c] such that skew(a) b = a × b
HD double skew(v3 a, int r, int c) {
  if (r == c) return 0.0;
  if (r == 0) return c == 1 ? -a.z : a.y;
  if (r == 1) return c == 0 ? a.z : -a.x;
  return c == 0 ? -a.y : a.x;
}

// ---- variable-space first derivatives (var index 0=w, 1=e1, 2=e2), component a ----
// PL: N = |w|^2 D - (w.e)^2, D = e.e
HD double pl_N1(const SubDist& S, int v, int a) {
  return v == 0 ? 2.0 * (S.D * comp(S.w, a) - S.we * comp(S.e1, a)) : 2.0 * (S.ww * comp(S.e1, a) - S.we * comp(S.w, a));
}
HD double pl_D1(const SubDist& S, int v, int a) { return v == 1 ? 2.0 * comp(S.e1, a) : 0.0; }
HD double pl_N2(const SubDist& S, int v, int a, int u, int b) {
  double dab = (a == b) ? 1.0 : 0.0;
  if (v == 0 && u == 0) return 2.0 * (S.D * dab - comp(S.e1, a) * comp(S.e1, b));
  if (v == 1 && u == 1) return 2.0 * (S.ww * dab - comp(S.w, a) * comp(S.w, b));
  if (v == 0 && u == 1) return 2.0 * (2.0 * comp(S.w, a) * comp(S.e1, b) - comp(S.e1, a) * comp(S.w, b) - S.we * dab);
  /* v == 1 && u == 0 */ return 2.0 * (2.0 * comp(S.w, b) * comp(S.e1, a) - comp(S.e1, b) * comp(S.w, a) - S.we * dab);
}
HD double pl_D2(int v, int a, int u, int b) { return (v == 1 && u == 1 && a == b) ? 2.0 : 0.0; }

// TRI: u = w.n, n = e1×e2, D = n.n
HD double tri_u1(const SubDist& S, int v, int a) {
  if (v == 0) return comp(S.n, a);
  if (v == 1) return comp(cross(S.e2, S.w), a);
  return comp(cross(S.w, S.e1), a);
}
HD double tri_u2(const SubDist& S, int v, int a, int u, int b) {
  if (v == u) return 0.0;
  if (v == 0 && u == 1) return -skew(S.e2, a, b);
  if (v == 1 && u == 0) return -skew(S.e2, b, a);
  if (v == 0 && u == 2) return skew(S.e1, a, b);
  if (v == 2 && u == 0) return skew(S.e1, b, a);
  if (v == 1 && u == 2) return -skew(S.w, a, b);
  /* v == 2 && u == 1 */ return -skew(S.w, b, a);
}
HD double tri_D1(const SubDist& S, int v, int a) {
  if (v == 1) return 2.0 * comp(cross(S.e2, S.n), a);
  if (v == 2) return 2.0 * comp(cross(S.n, S.e1), a);
  return 0.0;
}
// ∂n_i/∂var_v[a]: J1 = −[e2]×, J2 = [e1]×
HD double tri_Jn(const SubDist& S, int v, int i, int a) {
  if (v == 1) return -skew(S.e2, i, a);
  if (v == 2) return skew(S.e1, i, a);
  return 0.0;
}
HD double tri_D2(const SubDist& S, int v, int a, int u, int b) {
  if (v == 0 || u == 0) return 0.0;
  double r = 0.0;
  for (int i = 0; i < 3; ++i) r += tri_Jn(S, v, i, a) * tri_Jn(S, u, i, b);
  r *= 2.0;
  if (v == 1 && u == 2) r += -2.0 * skew(S.n, a, b);
  if (v == 2 && u == 1) r += -2.0 * skew(S.n, b, a);
  return r;
}

// variable-space derivatives of s
HD double sd_var1(const SubDist& S, int v, int a) {
  if (S.sub == SUB_PP) return v == 0 ? 2.0 * comp(S.w, a) : 0.0;
  if (S.sub == SUB_PL) return pl_N1(S, v, a) * S.iD - S.N * pl_D1(S, v, a) * S.iD2;
  return 2.0 * S.u * tri_u1(S, v, a) * S.iD - S.u * S.u * tri_D1(S, v, a) * S.iD2;
}
HD double sd_var2(const SubDist& S, int v, int a, int u, int b) {
  if (S.sub == SUB_PP) return (v == 0 && u == 0 && a == b) ? 2.0 : 0.0;
  if (S.sub == SUB_PL) {
    const double N = S.N;
    return pl_N2(S, v, a, u, b) * S.iD - (pl_N1(S, v, a) * pl_D1(S, u, b) + pl_D1(S, v, a) * pl_N1(S, u, b)) * S.iD2 -
           N * pl_D2(v, a, u, b) * S.iD2 + 2.0 * N * pl_D1(S, v, a) * pl_D1(S, u, b) * S.iD3;
  }
  const double U = S.u;
  double ua = tri_u1(S, v, a), ub = tri_u1(S, u, b), Da = tri_D1(S, v, a), Db = tri_D1(S, u, b);
  return 2.0 * (ua * ub + U * tri_u2(S, v, a, u, b)) * S.iD - 2.0 * U * (ua * Db + Da * ub) * S.iD2 -
         U * U * tri_D2(S, v, a, u, b) * S.iD2 + 2.0 * U * U * Da * Db * S.iD3;
}
// cross-product magnitude c = D of an sd_make_cross evaluator, and its derivatives
HD double sc_var1(const SubDist& S, int v, int a) { return tri_D1(S, v, a); }
HD double sc_var2(const SubDist& S, int v, int a, int u, int b) { return tri_D2(S, v, a, u, b); }

// slot-space entries: r = 3*slot + comp
HD double sd_grad(const SubDist& S, int r, bool cross_c = false) {
  int k = r / 3, a = r % 3;
  double g = 0.0;
  for (int v = 0; v < 3; ++v)
    if (S.coef[v][k]) g += (double)S.coef[v][k] * (cross_c ? sc_var1(S, v, a) : sd_var1(S, v, a));
  return g;
}
HD double sd_hess(const SubDist& S, int r, int c, bool cross_c = false) {
  int k = r / 3, a = r % 3, l = c / 3, b = c % 3;
  double h = 0.0;
  for (int v = 0; v < 3; ++v) {
    if (!S.coef[v][k]) continue;
    for (int u = 0; u < 3; ++u) {
      if (!S.coef[u][l]) continue;
      h += (double)(S.coef[v][k] * S.coef[u][l]) * (cross_c ? sc_var2(S, v, a, u, b) : sd_var2(S, v, a, u, b));
    }
  }
  return h;
}

// ---- barrier b(d) = −(d−d̂)² ln(d/d̂) on (0, d̂) and its s-derivatives, s = d² ----
HD void barrier_s(double s, double dhat, double* B, double* B1, double* B2) {
  double d = sqrt(s);
  if (!(d < dhat)) { *B = 0; *B1 = 0; *B2 = 0; return; }
  double lg = log(d / dhat), dm = d - dhat;
  double b = -dm * dm * lg;
  double b1 = -2.0 * dm * lg - dm * dm / d;
  double b2 = -2.0 * lg - 4.0 * dm / d + dm * dm / (d * d);
  *B = b;
  *B1 = b1 / (2.0 * d);
  *B2 = (b2 - b1 / d) / (4.0 * s);
}
// EE mollifier m(c) = (2 − c/ε)(c/ε) for c < ε else 1
HD void mollifier(double c, double eps, double* m, double* m1, double* m2) {
  if (c < eps) {
    double r = c / eps;
    *m = (2.0 - r) * r; *m1 = 2.0 / eps - 2.0 * c / (eps * eps); *m2 = -2.0 / (eps * eps);
  } else { *m = 1.0; *m1 = 0.0; *m2 = 0.0; }
}

}  // namespace tac
