// Device linearization of the plant models (sqp.linearize, sqp.py:105-147).
//
// One CTA per (stage, instance).  Jacobians are exact: analytic for the
// Dubins car and the synthetic legged plants, forward-mode dual numbers
// pushed through the RK4 map / the pendulum's mass-matrix solve for the rest
// (thread t carries tangent e_t, so the n+m threads produce the n+m columns of
// [A | B]).  Model formulas mirror paper_2604_07644_b200/models.py (the host
// specification), which in turn mirrors the reference fixtures
// (models.py:130-448).  Everything is evaluated in float64; matrices are
// stored float32, vectors float64 (include/gsls.h precision split).
#include <algorithm>
#include <cmath>

#include "ctx.h"
#include "prof.h"

namespace gsls {

enum { M_DUBINS = 1, M_PLANAR = 2, M_PENDULUM = 3, M_QUAD12 = 4, M_SYNTH = 5 };
constexpr double kG = 9.81;

struct Dual {
  double v, d;
  __device__ Dual() : v(0), d(0) {}
  __device__ Dual(double a) : v(a), d(0) {}
  __device__ Dual(double a, double b) : v(a), d(b) {}
};
__device__ inline Dual operator+(Dual a, Dual b) { return {a.v + b.v, a.d + b.d}; }
__device__ inline Dual operator-(Dual a, Dual b) { return {a.v - b.v, a.d - b.d}; }
__device__ inline Dual operator-(Dual a) { return {-a.v, -a.d}; }
__device__ inline Dual operator*(Dual a, Dual b) { return {a.v * b.v, a.d * b.v + a.v * b.d}; }
__device__ inline Dual operator/(Dual a, Dual b) { return {a.v / b.v, (a.d * b.v - a.v * b.d) / (b.v * b.v)}; }
__device__ inline Dual sin(Dual a) { return {::sin(a.v), a.d * ::cos(a.v)}; }
__device__ inline Dual cos(Dual a) { return {::cos(a.v), -a.d * ::sin(a.v)}; }
__device__ inline double sin(double a) { return ::sin(a); }
__device__ inline double cos(double a) { return ::cos(a); }
__device__ inline double val(double a) { return a; }
__device__ inline double val(Dual a) { return a.v; }

// ---- planar quadrotor (models.py:204-299) ----------------------------------
template <class T>
__device__ void fc_planar(const double* P, const T* x, const T* u, T* o) {
  const double m = P[0], L = P[1], J = P[2];
  const T th = u[0] + u[1];
  o[0] = x[3];
  o[1] = x[4];
  o[2] = x[5];
  o[3] = -(th * sin(x[2])) / T(m);
  o[4] = th * cos(x[2]) / T(m) - T(kG);
  o[5] = T(L) * (u[1] - u[0]) / T(J);
}

// ---- 12D quadrotor (models.py Quadrotor12) ----------------------------------
template <class T>
__device__ void fc_quad12(const double* P, const T* x, const T* u, T* o) {
  const double mass = P[0], arm = P[1], Jx = P[2], Jy = P[3], Jz = P[4], kap = P[5];
  const T sf = sin(x[3]), cf = cos(x[3]), st = sin(x[4]), ct = cos(x[4]), sp = sin(x[5]), cp = cos(x[5]);
  const T p = x[9], q = x[10], r = x[11];
  const T Th = u[0] + u[1] + u[2] + u[3];
  const T tx = T(arm) * (u[1] - u[3]);
  const T ty = T(arm) * (u[2] - u[0]);
  const T tz = T(kap) * (u[0] - u[1] + u[2] - u[3]);
  const T tt = st / ct;
  const T Tm = Th / T(mass);
  o[0] = x[6];
  o[1] = x[7];
  o[2] = x[8];
  o[3] = p + sf * tt * q + cf * tt * r;
  o[4] = cf * q - sf * r;
  o[5] = (sf * q + cf * r) / ct;
  o[6] = Tm * (cf * st * cp + sf * sp);
  o[7] = Tm * (cf * st * sp - sf * cp);
  o[8] = Tm * (cf * ct) - T(kG);
  o[9] = (tx - T(Jz - Jy) * q * r) / T(Jx);
  o[10] = (ty - T(Jx - Jz) * p * r) / T(Jy);
  o[11] = (tz - T(Jy - Jx) * p * q) / T(Jz);
}

template <class T, int NX, class F>
__device__ void rk4(F fc, const double* P, const T* x, const T* u, double dt, T* xn) {
  T k1[NX], k2[NX], k3[NX], k4[NX], y[NX];
  fc(P, x, u, k1);
  for (int i = 0; i < NX; ++i) y[i] = x[i] + T(0.5 * dt) * k1[i];
  fc(P, y, u, k2);
  for (int i = 0; i < NX; ++i) y[i] = x[i] + T(0.5 * dt) * k2[i];
  fc(P, y, u, k3);
  for (int i = 0; i < NX; ++i) y[i] = x[i] + T(dt) * k3[i];
  fc(P, y, u, k4);
  for (int i = 0; i < NX; ++i) xn[i] = x[i] + T(dt / 6.0) * (k1[i] + T(2.0) * k2[i] + T(2.0) * k3[i] + k4[i]);
}

// ---- n-link pendulum, semi-implicit Euler (models.py:302-448) ----------------
constexpr int kMaxLinks = 10;
template <class T>
__device__ void step_pendulum(const double* P, const T* x, const T* u, T* xn) {
  const int nl = (int)P[0];
  const double dt = P[1];
  const double* kap = P + 2;
  const double* inert = kap + nl * nl;
  const double* glev = inert + nl;
  T M[kMaxLinks][kMaxLinks + 1];
  for (int i = 0; i < nl; ++i) {
    T bias = T(0.0);
    for (int j = 0; j < nl; ++j) {
      const T d = x[i] - x[j];
      M[i][j] = T(kap[i * nl + j]) * cos(d) + T(i == j ? inert[i] : 0.0);
      bias = bias + T(kap[i * nl + j]) * sin(d) * (x[nl + j] * x[nl + j]);
    }
    bias = bias + T(glev[i]) * sin(x[i]);
    // input map T': row i = u_i - u_{i+1}
    T tau = u[i];
    if (i + 1 < nl) tau = tau - u[i + 1];
    M[i][nl] = tau - bias;
  }
  // Gaussian elimination (M is SPD)
  for (int k = 0; k < nl; ++k)
    for (int i = k + 1; i < nl; ++i) {
      const T f = M[i][k] / M[k][k];
      for (int j = k; j <= nl; ++j) M[i][j] = M[i][j] - f * M[k][j];
    }
  T acc[kMaxLinks];
  for (int i = nl - 1; i >= 0; --i) {
    T s = M[i][nl];
    for (int j = i + 1; j < nl; ++j) s = s - M[i][j] * acc[j];
    acc[i] = s / M[i][i];
  }
  for (int i = 0; i < nl; ++i) {
    xn[nl + i] = x[nl + i] + T(dt) * acc[i];
    xn[i] = x[i] + T(dt) * xn[nl + i];
  }
}

// ---- linearization kernel -------------------------------------------------------

struct LinArgs {
  int model;
  const double* P;      // model parameters (models.py device_spec)
  const double* cons;   // constraint block: n_obs, lo[m], hi[m], obs[3*n_obs]
  const double *x, *u;  // (B,N+1,n), (B,N,m)
  const double *h, *hf; // (B,N,c), (B,nf) or null
  const double* xbar0;  // (B,n) or null
  const double *Qw, *Rw, *QNw;  // (n,n), (m,m), (n,n)
  const double *xref, *uref;    // (N+1,n), (N,m)
  const double* Eco;    // constant disturbance (n,n) or null
  int write_weights;
  // outputs
  float *A, *B, *Q, *R, *S, *QN, *C, *D, *CN, *E;
  double *b, *q, *r, *qN, *f, *fN, *dx0;
  ErrSlot* err;
  int n, m, c, nf, N;
};

__device__ inline void constraints(const LinArgs& a, const double* x, const double* u, int stage, int inst,
                                   bool terminal) {
  const int n = a.n, m = a.m, c = a.c, nf = a.nf;
  const int nobs = (int)a.cons[0];
  const double* lo = a.cons + 1;
  const double* hi = lo + m;
  const double* obs = hi + m;
  if (!terminal) {
    const size_t st = (size_t)inst * a.N + stage;
    float* C = a.C + st * c * n;
    float* D = a.D + st * c * m;
    double* f = a.f + st * c;
    const double* h = a.h ? a.h + st * c : nullptr;
    for (int e = threadIdx.x; e < c * n; e += blockDim.x) {
      const int r = e / n, i = e - r * n;
      float v = 0.f;
      if (r >= 2 * m && i < 2) {
        const double* o = obs + 3 * (r - 2 * m);
        v = (float)(-2.0 * (x[i] - o[i]));
      }
      C[e] = v;
    }
    for (int e = threadIdx.x; e < c * m; e += blockDim.x) {
      const int r = e / m, l = e - r * m;
      D[e] = (r < m && l == r) ? 1.f : (r >= m && r < 2 * m && l == r - m) ? -1.f : 0.f;
    }
    for (int r = threadIdx.x; r < c; r += blockDim.x) {
      double g;
      if (r < m) g = u[r] - hi[r];
      else if (r < 2 * m) g = lo[r - m] - u[r - m];
      else {
        const double* o = obs + 3 * (r - 2 * m);
        g = o[2] * o[2] - (x[0] - o[0]) * (x[0] - o[0]) - (x[1] - o[1]) * (x[1] - o[1]);
      }
      if (!isfinite(g)) raise_err(a.err + inst, GSLS_ERR_NONFINITE, stage, -1, GSLS_LABEL_NONFINITE_CON);
      f[r] = -g - (h ? h[r] : 0.0);
    }
  } else {
    float* CN = a.CN + (size_t)inst * nf * n;
    double* fN = a.fN + (size_t)inst * nf;
    for (int e = threadIdx.x; e < nf * n; e += blockDim.x) {
      const int r = e / n, i = e - r * n;
      const double* o = obs + 3 * r;
      CN[e] = (i < 2) ? (float)(-2.0 * (x[i] - o[i])) : 0.f;
    }
    for (int r = threadIdx.x; r < nf; r += blockDim.x) {
      const double* o = obs + 3 * r;
      const double g = o[2] * o[2] - (x[0] - o[0]) * (x[0] - o[0]) - (x[1] - o[1]) * (x[1] - o[1]);
      fN[r] = -g - (a.hf ? a.hf[(size_t)inst * nf + r] : 0.0);
    }
  }
  (void)nobs;
}

template <int NX>
__device__ void dual_jac(const LinArgs& a, const double* x, const double* u, double* fval, float* A, float* B) {
  const int n = a.n, m = a.m;
  const int t = threadIdx.x;
  if (t < n + m) {
    Dual xd[NX], ud[NX], xn[NX];
    for (int i = 0; i < n; ++i) xd[i] = Dual(x[i], (t == i) ? 1.0 : 0.0);
    for (int l = 0; l < m; ++l) ud[l] = Dual(u[l], (t == n + l) ? 1.0 : 0.0);
    if (a.model == M_PLANAR) rk4<Dual, NX>(fc_planar<Dual>, a.P, xd, ud, a.P[3], xn);
    else if (a.model == M_QUAD12) rk4<Dual, NX>(fc_quad12<Dual>, a.P, xd, ud, a.P[6], xn);
    else step_pendulum<Dual>(a.P, xd, ud, xn);
    for (int i = 0; i < n; ++i) {
      if (t < n) A[i * n + t] = (float)xn[i].d;
      else B[i * m + (t - n)] = (float)xn[i].d;
    }
    if (t == 0)
      for (int i = 0; i < n; ++i) fval[i] = xn[i].v;
  }
}

__global__ void __launch_bounds__(128) k_linearize(LinArgs a) {
  const int k = blockIdx.x, inst = blockIdx.y;
  const int n = a.n, m = a.m, N = a.N;
  const double* x = a.x + ((size_t)inst * (N + 1) + k) * n;
  __shared__ double fval[kMaxN];
  if (k == N) {
    constraints(a, x, nullptr, k, inst, true);
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      double s = 0.0;
      for (int j = 0; j < n; ++j) s = fma(a.QNw[i * n + j], x[j] - a.xref[(size_t)N * n + j], s);
      a.qN[(size_t)inst * n + i] = s;
      const double* x0 = a.x + (size_t)inst * (N + 1) * n;
      a.dx0[(size_t)inst * n + i] = a.xbar0 ? a.xbar0[(size_t)inst * n + i] - x0[i] : 0.0;
    }
    if (a.write_weights)
      for (int e = threadIdx.x; e < n * n; e += blockDim.x) a.QN[(size_t)inst * n * n + e] = (float)a.QNw[e];
    return;
  }
  const double* u = a.u + ((size_t)inst * N + k) * m;
  const size_t st = (size_t)inst * N + k;
  float* A = a.A + st * n * n;
  float* B = a.B + st * n * m;
  if (a.model == M_DUBINS) {
    const double v = a.P[0], dt = a.P[1];
    if (threadIdx.x == 0) {
      fval[0] = x[0] + v * ::cos(x[2]) * dt;
      fval[1] = x[1] + v * ::sin(x[2]) * dt;
      fval[2] = x[2] + u[0] * dt;
    }
    for (int e = threadIdx.x; e < 9; e += blockDim.x) {
      const int i = e / 3, j = e % 3;
      float val = (i == j) ? 1.f : 0.f;
      if (i == 0 && j == 2) val = (float)(-v * ::sin(x[2]) * dt);
      if (i == 1 && j == 2) val = (float)(v * ::cos(x[2]) * dt);
      A[e] = val;
    }
    if (threadIdx.x < 3) B[threadIdx.x] = (threadIdx.x == 2) ? (float)dt : 0.f;
  } else if (a.model == M_SYNTH) {
    const double dt = a.P[0], cpl = a.P[1];
    const double* A0 = a.P + 2;
    const double* B0 = A0 + n * n;
    const double* W = B0 + n * m;
    __shared__ double th[kMaxN];
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      double s = 0.0, fa = 0.0, fb = 0.0;
      for (int j = 0; j < n; ++j) {
        s = fma(W[i * n + j], x[j], s);
        fa = fma(A0[i * n + j], x[j], fa);
      }
      for (int l = 0; l < m; ++l) fb = fma(B0[i * m + l], u[l], fb);
      const double t = ::tanh(s);
      th[i] = t;
      fval[i] = x[i] + dt * (fa + fb + cpl * t);
    }
    __syncthreads();
    for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
      const int i = e / n, j = e - i * n;
      const double sd = 1.0 - th[i] * th[i];
      A[e] = (float)(((i == j) ? 1.0 : 0.0) + dt * (A0[e] + cpl * sd * W[e]));
    }
    for (int e = threadIdx.x; e < n * m; e += blockDim.x) B[e] = (float)(dt * B0[e]);
  } else if (a.model == M_PENDULUM) {
    dual_jac<2 * kMaxLinks>(a, x, u, fval, A, B);
  } else if (a.model == M_PLANAR) {
    dual_jac<6>(a, x, u, fval, A, B);
  } else {
    dual_jac<12>(a, x, u, fval, A, B);
  }
  __syncthreads();
  const double* xn = x + n;  // traj.x[k+1]
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    if (!isfinite(fval[i])) raise_err(a.err + inst, GSLS_ERR_NONFINITE, k, -1, GSLS_LABEL_NONFINITE_DYN);
    a.b[st * n + i] = fval[i] - xn[i];
    double s = 0.0;
    for (int j = 0; j < n; ++j) s = fma(a.Qw[i * n + j], x[j] - a.xref[(size_t)k * n + j], s);
    a.q[st * n + i] = s;
  }
  for (int l = threadIdx.x; l < m; l += blockDim.x) {
    double s = 0.0;
    for (int j = 0; j < m; ++j) s = fma(a.Rw[l * m + j], u[j] - a.uref[(size_t)k * m + j], s);
    a.r[st * m + l] = s;
  }
  constraints(a, x, u, k, inst, false);
  if (a.write_weights) {
    for (int e = threadIdx.x; e < n * n; e += blockDim.x) a.Q[st * n * n + e] = (float)a.Qw[e];
    for (int e = threadIdx.x; e < m * m; e += blockDim.x) a.R[st * m * m + e] = (float)a.Rw[e];
    for (int e = threadIdx.x; e < m * n; e += blockDim.x) a.S[st * m * n + e] = 0.f;
    if (a.E && a.Eco)
      for (int e = threadIdx.x; e < n * n; e += blockDim.x) a.E[st * n * n + e] = (float)a.Eco[e];
  }
}

int linearize(Ctx* c, const gsls_linearize_args_t* in, gsls_qp_t* out_qp, float* E, cudaStream_t st) {
  const gsls_dims_t& d = c->dims;
  if (in->model_id == M_PENDULUM && d.nx > 2 * kMaxLinks) return GSLS_ERR_TOO_LARGE;
  if ((in->model_id == M_PLANAR && d.nx != 6) || (in->model_id == M_QUAD12 && d.nx != 12) ||
      (in->model_id == M_DUBINS && d.nx != 3) || in->model_id < 1 || in->model_id > 5)
    return GSLS_ERR_ARG;
  LinArgs a{};
  a.model = in->model_id;
  a.P = in->params;
  a.cons = in->params + in->cons_offset;
  a.x = in->x; a.u = in->u; a.h = in->h; a.hf = in->hf; a.xbar0 = in->xbar0;
  a.Qw = in->Qw; a.Rw = in->Rw; a.QNw = in->QNw; a.xref = in->xref; a.uref = in->uref; a.Eco = in->E_const;
  a.write_weights = in->write_weights;
  a.A = (float*)out_qp->A; a.B = (float*)out_qp->B; a.Q = (float*)out_qp->Q; a.R = (float*)out_qp->R;
  a.S = (float*)out_qp->S; a.QN = (float*)out_qp->QN; a.C = (float*)out_qp->C; a.D = (float*)out_qp->D;
  a.CN = (float*)out_qp->CN; a.E = E;
  a.b = (double*)out_qp->b; a.q = (double*)out_qp->q; a.r = (double*)out_qp->r; a.qN = (double*)out_qp->qN;
  a.f = (double*)out_qp->f; a.fN = (double*)out_qp->fN; a.dx0 = (double*)out_qp->dx0;
  a.err = c->dev.err;
  a.n = d.nx; a.m = d.nu; a.c = d.nc; a.nf = d.nf; a.N = d.N;
  ProfScope ps(P_LINEARIZE, st, (double)(d.N + 1) * d.batch);
  k_linearize<<<dim3(d.N + 1, d.batch), 128, 0, st>>>(a);
  GSLS_CUDA_CHECK(cudaGetLastError());
  return GSLS_OK;
}

}  // namespace gsls

namespace gsls {

// f <- f - h, fN <- fN - hf (the tightened re-linearization of sqp.py:136,
// :140; A, B, C, D are identical between the two linearizations of an RTI step).
__global__ void k_apply_tightening(double* f, double* fN, const double* h, const double* hf, long long nstage,
                                   long long nterm) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < nstage + nterm;
       e += (long long)gridDim.x * blockDim.x) {
    if (e < nstage) f[e] -= h[e];
    else fN[e - nstage] -= hf[e - nstage];
  }
}

int apply_tightening(Ctx* c, double* f, double* fN, const double* h, const double* hf, cudaStream_t st) {
  const gsls_dims_t& d = c->dims;
  const long long ns = (long long)d.batch * d.N * d.nc, nt = (long long)d.batch * d.nf;
  if (ns + nt == 0) return GSLS_OK;
  const int blocks = (int)std::min<long long>((ns + nt + 255) / 256, 148 * 8);
  ProfScope ps(P_RTI_MISC, st, (double)d.batch);
  k_apply_tightening<<<blocks, 256, 0, st>>>(f, fN, h, hf, ns, nt);
  GSLS_CUDA_CHECK(cudaGetLastError());
  return GSLS_OK;
}

// plan = previous + (dx, du) (sqp.py:293), warm start = plan shifted by one
// stage with the last entry duplicated (sqp.py:40-43), u0, and the tracking
// cost of the plan (models.py:85-93).
__global__ void k_rti_apply(int n, int m, int N, const double* px, const double* pu, const double* dx,
                            const double* du, double* plan_x, double* plan_u, double* warm_x, double* warm_u,
                            double* u0, const double* Qw, const double* Rw, const double* QNw, const double* xref,
                            const double* uref, double* cost) {
  const int inst = blockIdx.x;
  const size_t bx = (size_t)inst * (N + 1) * n, bu = (size_t)inst * N * m;
  for (int e = threadIdx.x; e < (N + 1) * n; e += blockDim.x) plan_x[bx + e] = px[bx + e] + dx[bx + e];
  for (int e = threadIdx.x; e < N * m; e += blockDim.x) plan_u[bu + e] = pu[bu + e] + du[bu + e];
  __syncthreads();
  for (int e = threadIdx.x; e < (N + 1) * n; e += blockDim.x) {
    const int k = e / n, i = e - k * n;
    warm_x[bx + e] = plan_x[bx + (size_t)(k < N ? k + 1 : N) * n + i];
  }
  for (int e = threadIdx.x; e < N * m; e += blockDim.x) {
    const int k = e / m, i = e - k * m;
    warm_u[bu + e] = plan_u[bu + (size_t)(k + 1 < N ? k + 1 : N - 1) * m + i];
  }
  for (int i = threadIdx.x; i < m; i += blockDim.x) u0[(size_t)inst * m + i] = plan_u[bu + i];
  if (cost) {
    __shared__ double red[32];
    double s = 0.0;
    for (int e = threadIdx.x; e < (N + 1) * n; e += blockDim.x) {
      const int k = e / n, i = e - k * n;
      const double* W = (k < N) ? Qw : QNw;
      const double* xk = plan_x + bx + (size_t)k * n;
      const double* rk = xref + (size_t)k * n;
      double wi = 0.0;
      for (int j = 0; j < n; ++j) wi = fma(W[i * n + j], xk[j] - rk[j], wi);
      s += 0.5 * (xk[i] - rk[i]) * wi;
    }
    for (int e = threadIdx.x; e < N * m; e += blockDim.x) {
      const int k = e / m, i = e - k * m;
      const double* uk = plan_u + bu + (size_t)k * m;
      const double* rk = uref + (size_t)k * m;
      double wi = 0.0;
      for (int j = 0; j < m; ++j) wi = fma(Rw[i * m + j], uk[j] - rk[j], wi);
      s += 0.5 * (uk[i] - rk[i]) * wi;
    }
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
      cost[inst] = t;
    }
  }
}

int rti_apply(Ctx* c, const double* px, const double* pu, const double* dx, const double* du, double* plan_x,
              double* plan_u, double* warm_x, double* warm_u, double* u0, const double* Qw, const double* Rw,
              const double* QNw, const double* xref, const double* uref, double* cost, cudaStream_t st) {
  const gsls_dims_t& d = c->dims;
  ProfScope ps(P_RTI_MISC, st, (double)d.batch);
  k_rti_apply<<<d.batch, 256, 0, st>>>(d.nx, d.nu, d.N, px, pu, dx, du, plan_x, plan_u, warm_x, warm_u, u0, Qw, Rw,
                                       QNw, xref, uref, cost);
  GSLS_CUDA_CHECK(cudaGetLastError());
  return GSLS_OK;
}

}  // namespace gsls

namespace gsls {

// value-only one-step map f(x, u) for models with small n (one thread per stage)
__device__ void step_value(const LinArgs& a, const double* x, const double* u, double* xn) {
  if (a.model == M_DUBINS) {
    const double v = a.P[0], dt = a.P[1];
    xn[0] = x[0] + v * ::cos(x[2]) * dt;
    xn[1] = x[1] + v * ::sin(x[2]) * dt;
    xn[2] = x[2] + u[0] * dt;
  } else if (a.model == M_PLANAR) {
    rk4<double, 6>(fc_planar<double>, a.P, x, u, a.P[3], xn);
  } else if (a.model == M_QUAD12) {
    rk4<double, 12>(fc_quad12<double>, a.P, x, u, a.P[6], xn);
  } else if (a.model == M_PENDULUM) {
    step_pendulum<double>(a.P, x, u, xn);
  }
}

// Per-instance trajectory terms used by the SQP loop (sqp.py:150-187):
// out[inst*8 + ...] = {J, defect_inf, defect_l1, viol_max, viol_pos_l1, x0dev_l1, x0dev_inf, 0}.
__global__ void __launch_bounds__(256) k_traj_eval(LinArgs a, double* out) {
  const int inst = blockIdx.x;
  const int n = a.n, m = a.m, c = a.c, nf = a.nf, N = a.N;
  const double* X = a.x + (size_t)inst * (N + 1) * n;
  const double* U = a.u + (size_t)inst * N * m;
  const int nobs = (int)a.cons[0];
  const double* lo = a.cons + 1;
  const double* hi = lo + m;
  const double* obs = hi + m;
  double J = 0.0, dinf = 0.0, dl1 = 0.0, vmax = 0.0, vpos = 0.0;
  __shared__ double fx[kMaxN];
  // defect
  if (a.model == M_SYNTH) {
    const double dt = a.P[0], cpl = a.P[1];
    const double* A0 = a.P + 2;
    const double* B0 = A0 + n * n;
    const double* W = B0 + n * m;
    for (int e = threadIdx.x; e < N * n; e += blockDim.x) {
      const int k = e / n, i = e - k * n;
      const double* x = X + (size_t)k * n;
      const double* u = U + (size_t)k * m;
      double s = 0.0, fa = 0.0, fb = 0.0;
      for (int j = 0; j < n; ++j) { s = fma(W[i * n + j], x[j], s); fa = fma(A0[i * n + j], x[j], fa); }
      for (int l = 0; l < m; ++l) fb = fma(B0[i * m + l], u[l], fb);
      const double d = fabs(X[(size_t)(k + 1) * n + i] - (x[i] + dt * (fa + fb + cpl * ::tanh(s))));
      dinf = fmax(dinf, d);
      dl1 += d;
    }
  } else {
    for (int k = threadIdx.x; k < N; k += blockDim.x) {
      double xn[2 * kMaxLinks > 12 ? 2 * kMaxLinks : 12];
      step_value(a, X + (size_t)k * n, U + (size_t)k * m, xn);
      for (int i = 0; i < n; ++i) {
        const double d = fabs(X[(size_t)(k + 1) * n + i] - xn[i]);
        dinf = fmax(dinf, d);
        dl1 += d;
      }
    }
  }
  (void)fx;
  // constraints (with tightenings) and tracking cost
  for (int e = threadIdx.x; e < N * c; e += blockDim.x) {
    const int k = e / c, r = e - k * c;
    const double* x = X + (size_t)k * n;
    const double* u = U + (size_t)k * m;
    double g;
    if (r < m) g = u[r] - hi[r];
    else if (r < 2 * m) g = lo[r - m] - u[r - m];
    else {
      const double* o = obs + 3 * (r - 2 * m);
      g = o[2] * o[2] - (x[0] - o[0]) * (x[0] - o[0]) - (x[1] - o[1]) * (x[1] - o[1]);
    }
    if (a.h) g += a.h[((size_t)inst * N + k) * c + r];
    vmax = fmax(vmax, g);
    vpos += fmax(g, 0.0);
  }
  for (int r = threadIdx.x; r < nf; r += blockDim.x) {
    const double* x = X + (size_t)N * n;
    const double* o = obs + 3 * r;
    double g = o[2] * o[2] - (x[0] - o[0]) * (x[0] - o[0]) - (x[1] - o[1]) * (x[1] - o[1]);
    if (a.hf) g += a.hf[(size_t)inst * nf + r];
    vmax = fmax(vmax, g);
    vpos += fmax(g, 0.0);
  }
  for (int e = threadIdx.x; e < (N + 1) * n; e += blockDim.x) {
    const int k = e / n, i = e - k * n;
    const double* W = (k < N) ? a.Qw : a.QNw;
    const double* xk = X + (size_t)k * n;
    const double* rk = a.xref + (size_t)k * n;
    double wi = 0.0;
    for (int j = 0; j < n; ++j) wi = fma(W[i * n + j], xk[j] - rk[j], wi);
    J += 0.5 * (xk[i] - rk[i]) * wi;
  }
  for (int e = threadIdx.x; e < N * m; e += blockDim.x) {
    const int k = e / m, i = e - k * m;
    const double* uk = U + (size_t)k * m;
    const double* rk = a.uref + (size_t)k * m;
    double wi = 0.0;
    for (int j = 0; j < m; ++j) wi = fma(a.Rw[i * m + j], uk[j] - rk[j], wi);
    J += 0.5 * (uk[i] - rk[i]) * wi;
  }
  double x1 = 0.0, xinf = 0.0;
  if (a.xbar0)
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      const double d = fabs(X[i] - a.xbar0[(size_t)inst * n + i]);
      x1 += d;
      xinf = fmax(xinf, d);
    }
  // block reductions (sum: J, dl1, vpos, x1; max: dinf, vmax, xinf)
  __shared__ double red[7][32];
  double v[7] = {J, dinf, dl1, vmax, vpos, x1, xinf};
  const bool is_max[7] = {false, true, false, true, false, false, true};
  for (int q = 0; q < 7; ++q)
    for (int o = 16; o > 0; o >>= 1) {
      const double w = __shfl_xor_sync(0xffffffffu, v[q], o);
      v[q] = is_max[q] ? fmax(v[q], w) : v[q] + w;
    }
  if ((threadIdx.x & 31) == 0)
    for (int q = 0; q < 7; ++q) red[q][threadIdx.x >> 5] = v[q];
  __syncthreads();
  if (threadIdx.x < 7) {
    const int q = threadIdx.x;
    double r = is_max[q] ? (q == 3 ? -1e300 : 0.0) : 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) r = is_max[q] ? fmax(r, red[q][w]) : r + red[q][w];
    out[(size_t)inst * 8 + q] = r;
  }
  if (threadIdx.x == 7) out[(size_t)inst * 8 + 7] = (double)nobs;
}

int traj_eval(Ctx* c, const gsls_linearize_args_t* in, double* out, cudaStream_t st) {
  const gsls_dims_t& d = c->dims;
  LinArgs a{};
  a.model = in->model_id;
  a.P = in->params;
  a.cons = in->params + in->cons_offset;
  a.x = in->x; a.u = in->u; a.h = in->h; a.hf = in->hf; a.xbar0 = in->xbar0;
  a.Qw = in->Qw; a.Rw = in->Rw; a.QNw = in->QNw; a.xref = in->xref; a.uref = in->uref;
  a.n = d.nx; a.m = d.nu; a.c = d.nc; a.nf = d.nf; a.N = d.N;
  k_traj_eval<<<d.batch, 256, 0, st>>>(a, out);
  GSLS_CUDA_CHECK(cudaGetLastError());
  return GSLS_OK;
}

}  // namespace gsls

namespace gsls {

// ---- closed-loop rollouts (rollout.py:47-93) -------------------------------------
//
// One CTA per (rollout, instance).  The horizon is sequential; inside a stage the
// CTA evaluates the feedback u_k = v_k + sum_{j<k} Phi^u_{k,j} w_hat_j (one warp per
// input row over the flattened (j, i) range), the model step, the disturbed state
// x_{k+1} = f(x_k, u_k) + E d_k, the reconstruction w_hat_k = E^+ (x_{k+1} - f) and the
// constraint / tube checks.  E is state-independent for every device model, so E and
// its range-restricted pseudo-inverse (rollout.py:41-44) arrive precomputed.
struct RolloutArgs {
  int model;
  const double* P;
  const double* cons;
  int n, m, c, nf, N, S;
  const double *x, *u;      // nominal (B,N+1,n), (B,N,m)
  const float* phiu;        // (B, N(N+1)/2, m, n) cell layout, or null (open loop)
  const double *E, *Epinv;  // (n,n)
  const double* dist;       // (B,S,N,n)
  const double* h;          // (B,N,c) or null: no tube check
  double tol_lin;
  double *ox, *ou, *ow, *og, *ogf, *omargin, *omaxw;
  int* oflags;              // (B,S,3): safe, tube_ok, disturbance_model_violated
};

__device__ inline double stage_con(const double* cons, int m, const double* x, const double* u, int r) {
  const double* lo = cons + 1;
  const double* hi = lo + m;
  if (r < m) return u[r] - hi[r];
  if (r < 2 * m) return lo[r - m] - u[r - m];
  const double* o = hi + m + 3 * (r - 2 * m);
  return o[2] * o[2] - (x[0] - o[0]) * (x[0] - o[0]) - (x[1] - o[1]) * (x[1] - o[1]);
}

__device__ inline double block_sum128(double v, double* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double r = 0.0;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) r += red[w];
  return r;
}

__device__ inline double block_min128(double v, double* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double r = INFINITY;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) r = fmin(r, red[w]);
  return r;
}

__global__ void __launch_bounds__(128, 8) k_rollout(RolloutArgs a) {
  const int s = blockIdx.x, inst = blockIdx.y;
  const int n = a.n, m = a.m, c = a.c, nf = a.nf, N = a.N, S = a.S;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  extern __shared__ double smr[];
  double* x = smr;           // realized x_k
  double* nom = x + n;       // f(x_k, u_k)
  double* xn = nom + n;      // x_{k+1}
  double* u = xn + n;        // u_k
  double* wh = u + m;        // w_hat (N, n)
  double* red = wh + (size_t)N * n;  // 32
  const long long rs = (long long)inst * S + s;
  const double* xnom = a.x + (size_t)inst * (N + 1) * n;
  const double* unom = a.u + (size_t)inst * N * m;
  const double* d = a.dist + (size_t)rs * N * n;
  const double* h = a.h ? a.h + (size_t)inst * N * c : nullptr;
  const int ncell = N * (N + 1) / 2;
  const float* phiu = a.phiu ? a.phiu + (size_t)inst * ncell * m * n : nullptr;
  double* ox = a.ox + (size_t)rs * (N + 1) * n;
  LinArgs la{};
  la.model = a.model;
  la.P = a.P;
  for (int i = tid; i < n; i += blockDim.x) {
    x[i] = xnom[i];
    ox[i] = xnom[i];
  }
  bool safe = true, tube_ok = true, violated = false;
  double maxw = 0.0;
  __syncthreads();
  for (int k = 0; k < N; ++k) {
    // u_k = v_k + sum_{j<k} Phi^u_{k,j} w_hat_j  (rollout.py:69-73)
    for (int l = warp; l < m; l += nw) {
      double acc = 0.0;
      if (phiu)
        for (int j = 0; j < k; ++j) {  // row l of Phi^u_{k,j} (contiguous) against w_hat_j
          const float* pr = phiu + ((size_t)(j * N - j * (j - 1) / 2 + (k - j - 1)) * m + l) * n;
          const double* wj = wh + (size_t)j * n;
          for (int i = lane; i < n; i += 32) acc = fma((double)pr[i], wj[i], acc);
        }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      if (lane == 0) u[l] = unom[(size_t)k * m + l] + acc;
    }
    __syncthreads();
    // nominal_next = f(x_k, u_k)
    if (a.model == M_SYNTH) {
      const double dt = a.P[0], cpl = a.P[1];
      const double* A0 = a.P + 2;
      const double* B0 = A0 + n * n;
      const double* W = B0 + n * m;
      for (int i = tid; i < n; i += blockDim.x) {
        double sw = 0.0, fa = 0.0, fb = 0.0;
        for (int j = 0; j < n; ++j) {
          sw = fma(W[i * n + j], x[j], sw);
          fa = fma(A0[i * n + j], x[j], fa);
        }
        for (int l = 0; l < m; ++l) fb = fma(B0[i * m + l], u[l], fb);
        nom[i] = x[i] + dt * (fa + fb + cpl * ::tanh(sw));
      }
    } else if (tid == 0) {
      step_value(la, x, u, nom);
    }
    __syncthreads();
    // x_{k+1} = f + E d_k  (rollout.py:75-76)
    for (int i = tid; i < n; i += blockDim.x) {
      double v = nom[i];
      for (int j = 0; j < n; ++j) v = fma(a.E[i * n + j], d[(size_t)k * n + j], v);
      xn[i] = v;
    }
    __syncthreads();
    // w_hat_k = E^+ (x_{k+1} - f)  (rollout.py:77)
    double sq = 0.0;
    for (int i = tid; i < n; i += blockDim.x) {
      double v = 0.0;
      for (int j = 0; j < n; ++j) v = fma(a.Epinv[i * n + j], xn[j] - nom[j], v);
      wh[(size_t)k * n + i] = v;
      sq = fma(v, v, sq);
    }
    const double wn = sqrt(block_sum128(sq, red));
    if (wn > 1.0 + 1e-9) violated = true;  // rollout.py:78-79 (WNORM_TOL)
    maxw = fmax(maxw, wn);
    // stage constraints at (x_k, u_k) and the tube slack against the nominal + h_k (rollout.py:80-85)
    double slack = INFINITY;
    bool ok = true;
    for (int r = tid; r < c; r += blockDim.x) {
      const double g = stage_con(a.cons, m, x, u, r);
      a.og[((size_t)rs * N + k) * c + r] = g;
      ok = ok && (g <= 0.0);
      if (h) slack = fmin(slack, stage_con(a.cons, m, xnom + (size_t)k * n, unom + (size_t)k * m, r) + h[(size_t)k * c + r] +
                                     a.tol_lin - g);
    }
    const int all_ok = __syncthreads_and(ok);
    safe = safe && all_ok;
    if (h && c > 0) {
      const double sl = block_min128(slack, red);
      if (tid == 0) a.omargin[(size_t)rs * N + k] = sl;
      tube_ok = tube_ok && (sl >= 0.0);
    } else if (tid == 0) {
      a.omargin[(size_t)rs * N + k] = INFINITY;
    }
    for (int i = tid; i < n; i += blockDim.x) {
      a.ow[((size_t)rs * N + k) * n + i] = wh[(size_t)k * n + i];
      ox[(size_t)(k + 1) * n + i] = xn[i];
    }
    for (int l = tid; l < m; l += blockDim.x) a.ou[((size_t)rs * N + k) * m + l] = u[l];
    __syncthreads();
    for (int i = tid; i < n; i += blockDim.x) x[i] = xn[i];
    __syncthreads();
  }
  // terminal constraints (obstacles) at x_N (rollout.py:86-87)
  bool okf = true;
  const int nobs = (int)a.cons[0];
  for (int r = tid; r < nf; r += blockDim.x) {
    double g = 0.0;
    if (r < nobs) {
      const double* o = a.cons + 1 + 2 * m + 3 * r;
      g = o[2] * o[2] - (x[0] - o[0]) * (x[0] - o[0]) - (x[1] - o[1]) * (x[1] - o[1]);
    }
    a.ogf[(size_t)rs * nf + r] = g;
    okf = okf && (g <= 0.0);
  }
  const int all_okf = __syncthreads_and(okf);
  safe = safe && all_okf;
  if (tid == 0) {
    a.oflags[rs * 3 + 0] = safe;
    a.oflags[rs * 3 + 1] = tube_ok;
    a.oflags[rs * 3 + 2] = violated;
    a.omaxw[rs] = maxw;
  }
}

int rollout(Ctx* c, const gsls_rollout_args_t* in, const gsls_rollout_out_t* out, cudaStream_t st) {
  const gsls_dims_t& d = c->dims;
  if ((in->model_id == M_PLANAR && d.nx != 6) || (in->model_id == M_QUAD12 && d.nx != 12) ||
      (in->model_id == M_DUBINS && d.nx != 3) || in->model_id < 1 || in->model_id > 5 || in->rollouts < 0)
    return GSLS_ERR_ARG;
  if (in->model_id == M_PENDULUM && d.nx > 2 * kMaxLinks) return GSLS_ERR_TOO_LARGE;
  if (d.batch == 0 || in->rollouts == 0 || d.N == 0) return GSLS_OK;
  RolloutArgs a{};
  a.model = in->model_id;
  a.P = in->params;
  a.cons = in->params + in->cons_offset;
  a.n = d.nx; a.m = d.nu; a.c = d.nc; a.nf = d.nf; a.N = d.N; a.S = in->rollouts;
  a.x = in->x; a.u = in->u; a.phiu = in->phi_u; a.E = in->E; a.Epinv = in->E_pinv; a.dist = in->disturbances;
  a.h = in->h; a.tol_lin = in->tol_lin;
  a.ox = out->x; a.ou = out->u; a.ow = out->w; a.og = out->stage_g; a.ogf = out->terminal_g;
  a.omargin = out->tube_margin; a.omaxw = out->max_w_norm; a.oflags = out->flags;
  const size_t smem = (size_t)(3 * d.nx + d.nu + (size_t)d.N * d.nx + 32) * sizeof(double);
  if (smem > 48 * 1024) {
    if (smem > 227 * 1024) return GSLS_ERR_TOO_LARGE;
    GSLS_CUDA_CHECK(cudaFuncSetAttribute((const void*)k_rollout, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  }
  ProfScope ps(P_ROLLOUT, st, (double)in->rollouts * d.batch);
  k_rollout<<<dim3(in->rollouts, d.batch), 128, smem, st>>>(a);
  GSLS_CUDA_CHECK(cudaGetLastError());
  return GSLS_OK;
}

}  // namespace gsls
