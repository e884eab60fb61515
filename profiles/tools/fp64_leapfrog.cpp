// fp64 leapfrog of a 3-D star wave (the executor's wave model evaluated in
// double, same term order): the "exact" solution of the discrete scheme for
// the float inputs, used to measure how far the fp32 reference and FAST
// arithmetic each drift from it (profiles/tools/fp64_drift.py).
//   fp64_leapfrog nz ny nx R steps coef.bin u0.bin u1.bin m.bin out.bin
// u0/u1/m: float32 interiors (z, y, x); coef: float32 [1 + 6R] in canonical
// star order (centre, then per axis -1, +1, -2, +2, ...); zero halo of width R.
// out: the final two levels (float64 interiors).
#include <cstdio>
#include <cstdlib>
#include <vector>

int main(int argc, char** argv) {
  if (argc != 11) { std::fprintf(stderr, "usage\n"); return 2; }
  const long nz = atol(argv[1]), ny = atol(argv[2]), nx = atol(argv[3]);
  const int R = atoi(argv[4]), steps = atoi(argv[5]);
  auto readf = [](const char* p, size_t n) {
    std::vector<float> v(n);
    FILE* f = std::fopen(p, "rb");
    if (!f || std::fread(v.data(), 4, n, f) != n) { std::fprintf(stderr, "read %s\n", p); std::exit(1); }
    std::fclose(f);
    return v;
  };
  const long Pz = nz + 2 * R, Py = ny + 2 * R, Px = nx + 2 * R;
  const size_t N = (size_t)nz * ny * nx, PN = (size_t)Pz * Py * Px;
  std::vector<float> cf = readf(argv[6], 1 + 6 * R);
  std::vector<double> c(cf.begin(), cf.end());
  std::vector<float> u0f = readf(argv[7], N), u1f = readf(argv[8], N), mf = readf(argv[9], N);
  std::vector<double> a(PN, 0.0), b(PN, 0.0), d(PN, 0.0);   // u^{n-1}, u^n, scratch
  auto idx = [&](long z, long y, long x) { return ((size_t)(z + R) * Py + (y + R)) * Px + (x + R); };
  for (long z = 0; z < nz; ++z)
    for (long y = 0; y < ny; ++y)
      for (long x = 0; x < nx; ++x) {
        const size_t i = ((size_t)z * ny + y) * nx + x;
        a[idx(z, y, x)] = u0f[i];
        b[idx(z, y, x)] = u1f[i];
      }
  const long sz = (long)Py * Px, sy = Px;
  double *um = a.data(), *uc = b.data(), *un = d.data();
  for (int t = 0; t < steps; ++t) {
#pragma omp parallel for schedule(static)
    for (long z = 0; z < nz; ++z)
      for (long y = 0; y < ny; ++y)
        for (long x = 0; x < nx; ++x) {
          const size_t p = idx(z, y, x);
          double acc = c[0] * uc[p];
          int k = 1;
          for (long s : {sz, sy, 1L})
            for (int r = 1; r <= R; ++r) {
              acc = acc + c[k++] * uc[p - r * s];
              acc = acc + c[k++] * uc[p + r * s];
            }
          un[p] = (2.0 * uc[p] - um[p]) + (double)mf[((size_t)z * ny + y) * nx + x] * acc;
        }
    double* tmp = um;
    um = uc;
    uc = un;
    un = tmp;
  }
  FILE* f = std::fopen(argv[10], "wb");
  for (double* lv : {um, uc})
    for (long z = 0; z < nz; ++z)
      for (long y = 0; y < ny; ++y) std::fwrite(lv + idx(z, y, 0), 8, nx, f);
  std::fclose(f);
  return 0;
}
