// How far does an order-preserving hybrid arithmetic drift from the fp32
// reference over a leapfrog run?  The reference evaluates
//   acc = c0*u; acc = acc + c_k*u_k   (every product and sum rounded)
// in term order.  The hybrid keeps that order and every sum, but fuses the
// product of the taps at distance >= K0 into the sum (fmaf): those taps carry
// small coefficients, so dropping the product's rounding perturbs the sum by a
// small fraction of its own rounding error.  K0 = R+1 is the reference itself.
//   hybrid_drift nz ny nx R steps coef.bin u0.bin u1.bin m.bin
// Inputs as for fp64_leapfrog.cpp.  Prints max|hybrid - reference| / max|reference|
// over the final two levels for K0 = 1 .. R.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

static long nz, ny, nx, Py, Px;
static int R;
static size_t idx(long z, long y, long x) { return ((size_t)(z + R) * Py + (y + R)) * Px + (x + R); }

static void run(int K0, int steps, const std::vector<float>& c, const std::vector<float>& u0,
                const std::vector<float>& u1, const std::vector<float>& mf, std::vector<float>& o0,
                std::vector<float>& o1) {
  const size_t PN = (size_t)(nz + 2 * R) * Py * Px;
  std::vector<float> a(PN, 0.f), b(PN, 0.f), d(PN, 0.f);
  for (long z = 0; z < nz; ++z)
    for (long y = 0; y < ny; ++y)
      for (long x = 0; x < nx; ++x) {
        const size_t i = ((size_t)z * ny + y) * nx + x;
        a[idx(z, y, x)] = u0[i];
        b[idx(z, y, x)] = u1[i];
      }
  const long sz = Py * Px, sy = Px;
  float *um = a.data(), *uc = b.data(), *un = d.data();
  for (int t = 0; t < steps; ++t) {
#pragma omp parallel for schedule(static)
    for (long z = 0; z < nz; ++z)
      for (long y = 0; y < ny; ++y)
        for (long x = 0; x < nx; ++x) {
          const size_t p = idx(z, y, x);
          float acc = c[0] * uc[p];
          int k = 1;
          for (long s : {sz, sy, 1L})
            for (int r = 1; r <= R; ++r) {
              if (r >= K0) {
                acc = std::fmaf(c[k], uc[p - r * s], acc); ++k;
                acc = std::fmaf(c[k], uc[p + r * s], acc); ++k;
              } else {
                float pr = c[k++] * uc[p - r * s];
                acc = acc + pr;
                pr = c[k++] * uc[p + r * s];
                acc = acc + pr;
              }
            }
          const float two = uc[p] + uc[p];
          const float bb = two - um[p];
          const float mm = mf[((size_t)z * ny + y) * nx + x] * acc;
          un[p] = bb + mm;
        }
    float* tmp = um; um = uc; uc = un; un = tmp;
  }
  o0.assign(um, um + PN);
  o1.assign(uc, uc + PN);
}

int main(int argc, char** argv) {
  if (argc != 10) { std::fprintf(stderr, "usage\n"); return 2; }
  nz = atol(argv[1]); ny = atol(argv[2]); nx = atol(argv[3]);
  R = atoi(argv[4]);
  const int steps = atoi(argv[5]);
  Py = ny + 2 * R; Px = nx + 2 * R;
  auto readf = [](const char* p, size_t n) {
    std::vector<float> v(n);
    FILE* f = std::fopen(p, "rb");
    if (!f || std::fread(v.data(), 4, n, f) != n) { std::fprintf(stderr, "read %s\n", p); std::exit(1); }
    std::fclose(f);
    return v;
  };
  const size_t N = (size_t)nz * ny * nx;
  auto c = readf(argv[6], 1 + 6 * R), u0 = readf(argv[7], N), u1 = readf(argv[8], N), mf = readf(argv[9], N);
  std::vector<float> r0, r1, h0, h1;
  run(R + 1, steps, c, u0, u1, mf, r0, r1);
  double scale = 0;
  for (float v : r1) scale = std::fmax(scale, std::fabs((double)v));
  for (float v : r0) scale = std::fmax(scale, std::fabs((double)v));
  std::printf("reference max|u| = %.5g\n", scale);
  for (int K0 = R; K0 >= 1; --K0) {
    run(K0, steps, c, u0, u1, mf, h0, h1);
    double e = 0;
    for (size_t i = 0; i < r0.size(); ++i) {
      e = std::fmax(e, std::fabs((double)h0[i] - r0[i]));
      e = std::fmax(e, std::fabs((double)h1[i] - r1[i]));
    }
    std::printf("taps at distance >= %d fused (%d of %d products): max rel err vs reference %.3e\n", K0,
                6 * (R - K0 + 1), 6 * R + 1, e / scale);
  }
  return 0;
}
