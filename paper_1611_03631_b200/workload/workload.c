/* Seeded synthetic workloads for BASELINE.json configs[0..4].
 *
 * BENCH / TEST INFRASTRUCTURE: the paper's datasets (EuRoC, KITTI, Cow) are not
 * in this image, so analytic scenes rendered here stand in for them with the
 * shapes, sizes and noise models BASELINE.json states. Depth is rendered by
 * exact ray-primitive intersection in fp64 (room interior, axis-aligned boxes,
 * spheres, vertical cylinders, ground plane), then noised and emitted as
 * sensor-frame float32 points in row-major pixel order (the scan order, hence
 * the simple-mode ray order), with optional uniform uint8 RGB.
 *
 * Randomness is the reference's splitmix64 Rng (proj/include/vxf/core.h:89-125)
 * used counter-style: every pixel draws from Rng(mix(seed, frame, pixel)), so
 * the output is identical for any OpenMP thread count.
 * Seeds: scene=1, trajectory=2, noise=3, colour=4, invalidation=5.
 */
#include <math.h>
#include <stdint.h>
#include <string.h>

#define WL_BOX 0
#define WL_SPHERE 1
#define WL_CYL 2    /* vertical cylinder: axis along `up` */
#define WL_ROOM 3   /* inside of an AABB */
#define WL_PLANE 4  /* horizontal ground plane at height a[0] along `up` */

typedef struct wl_prim {
  int32_t kind;
  int32_t up; /* up axis index for cylinders / planes */
  double a[6];
} wl_prim;

/* ------------------------------------------------------------------ RNG */
static inline uint64_t sm64_next(uint64_t* s) {
  uint64_t z = (*s += 0x9e3779b97f4a7c15ULL);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
static inline double sm64_uniform(uint64_t* s) { return (double)(sm64_next(s) >> 11) * 0x1.0p-53; }
static inline uint64_t rng_seed(uint64_t seed) { return seed ? seed : 0x9e3779b97f4a7c15ULL; }
static inline uint64_t mix3(uint64_t seed, uint64_t a, uint64_t b) {
  uint64_t s = seed * 0x9e3779b97f4a7c15ULL ^ (a + 0x632be59bd9b4e019ULL) * 0xbf58476d1ce4e5b9ULL;
  s ^= (b + 0x2545f4914f6cdd1dULL) * 0x94d049bb133111ebULL;
  uint64_t t = s;
  return rng_seed(sm64_next(&t));
}
static inline double gauss(uint64_t* s) { /* Box-Muller on Rng::uniform */
  double u1 = sm64_uniform(s), u2 = sm64_uniform(s);
  if (u1 < 1e-300) u1 = 1e-300;
  return sqrt(-2.0 * log(u1)) * cos(2.0 * M_PI * u2);
}

/* -------------------------------------------------------- intersections */
static double hit_prim(const wl_prim* p, const double o[3], const double d[3]) {
  const double inf = 1e300;
  switch (p->kind) {
    case WL_ROOM: {
      double t = inf;
      for (int i = 0; i < 3; ++i) {
        if (d[i] > 0) { double ti = (p->a[3 + i] - o[i]) / d[i]; if (ti < t) t = ti; }
        else if (d[i] < 0) { double ti = (p->a[i] - o[i]) / d[i]; if (ti < t) t = ti; }
      }
      return t > 1e-9 ? t : inf;
    }
    case WL_BOX: {
      double tmin = -inf, tmax = inf;
      for (int i = 0; i < 3; ++i) {
        const double lo = p->a[i] - p->a[3 + i], hi = p->a[i] + p->a[3 + i];
        if (d[i] == 0.0) {
          if (o[i] < lo || o[i] > hi) return inf;
        } else {
          double t1 = (lo - o[i]) / d[i], t2 = (hi - o[i]) / d[i];
          if (t1 > t2) { double tt = t1; t1 = t2; t2 = tt; }
          if (t1 > tmin) tmin = t1;
          if (t2 < tmax) tmax = t2;
        }
      }
      if (tmax < tmin || tmax <= 1e-9) return inf;
      return tmin > 1e-9 ? tmin : inf;
    }
    case WL_SPHERE: {
      const double oc[3] = {o[0] - p->a[0], o[1] - p->a[1], o[2] - p->a[2]};
      const double A = d[0] * d[0] + d[1] * d[1] + d[2] * d[2];
      const double B = 2.0 * (oc[0] * d[0] + oc[1] * d[1] + oc[2] * d[2]);
      const double C = oc[0] * oc[0] + oc[1] * oc[1] + oc[2] * oc[2] - p->a[3] * p->a[3];
      const double disc = B * B - 4 * A * C;
      if (disc < 0) return inf;
      const double sq = sqrt(disc);
      double t = (-B - sq) / (2 * A);
      if (t <= 1e-9) t = (-B + sq) / (2 * A);
      return t > 1e-9 ? t : inf;
    }
    case WL_CYL: { /* a = (c0, c1 horizontal centre, r, h_lo, h_hi) */
      const int u = p->up, h0 = (u + 1) % 3, h1 = (u + 2) % 3;
      const double ox = o[h0] - p->a[0], oy = o[h1] - p->a[1];
      const double A = d[h0] * d[h0] + d[h1] * d[h1];
      double best = inf;
      if (A > 0) {
        const double B = 2 * (ox * d[h0] + oy * d[h1]);
        const double C = ox * ox + oy * oy - p->a[2] * p->a[2];
        const double disc = B * B - 4 * A * C;
        if (disc >= 0) {
          const double sq = sqrt(disc);
          const double ts[2] = {(-B - sq) / (2 * A), (-B + sq) / (2 * A)};
          for (int k = 0; k < 2; ++k) {
            const double t = ts[k];
            if (t > 1e-9 && t < best) {
              const double h = o[u] + t * d[u];
              if (h >= p->a[3] && h <= p->a[4]) best = t;
            }
          }
        }
      }
      if (d[u] != 0.0) { /* caps */
        const double caps[2] = {p->a[3], p->a[4]};
        for (int k = 0; k < 2; ++k) {
          const double t = (caps[k] - o[u]) / d[u];
          if (t > 1e-9 && t < best) {
            const double x = ox + t * d[h0], y = oy + t * d[h1];
            if (x * x + y * y <= p->a[2] * p->a[2]) best = t;
          }
        }
      }
      return best;
    }
    case WL_PLANE: {
      const int u = p->up;
      if (d[u] == 0.0) return inf;
      const double t = (p->a[0] - o[u]) / d[u];
      return t > 1e-9 ? t : inf;
    }
  }
  return inf;
}

static double cast_scene(const wl_prim* prims, int n, const double o[3], const double d[3]) {
  double best = 1e300;
  for (int i = 0; i < n; ++i) {
    const double t = hit_prim(&prims[i], o, d);
    if (t < best) best = t;
  }
  return best;
}

/* ------------------------------------------------------------- scenes */
static double dist_point_prim_bound(const wl_prim* p, const double q[3]) {
  /* conservative distance from q to the primitive's bounding sphere */
  double c[3], r;
  if (p->kind == WL_BOX) {
    c[0] = p->a[0]; c[1] = p->a[1]; c[2] = p->a[2];
    r = sqrt(p->a[3] * p->a[3] + p->a[4] * p->a[4] + p->a[5] * p->a[5]);
  } else if (p->kind == WL_SPHERE) {
    c[0] = p->a[0]; c[1] = p->a[1]; c[2] = p->a[2];
    r = p->a[3];
  } else if (p->kind == WL_CYL) {
    const int u = p->up;
    c[(u + 1) % 3] = p->a[0]; c[(u + 2) % 3] = p->a[1];
    c[u] = 0.5 * (p->a[3] + p->a[4]);
    const double hh = 0.5 * (p->a[4] - p->a[3]);
    r = sqrt(p->a[2] * p->a[2] + hh * hh);
  } else {
    return 1e300;
  }
  const double dx = q[0] - c[0], dy = q[1] - c[1], dz = q[2] - c[2];
  return sqrt(dx * dx + dy * dy + dz * dz) - r;
}

/* Keep-out test against the sensor path of each config. */
static int too_close(int cfg, const wl_prim* p, double scale) {
  const double clearance = 0.5 * scale;
  if (cfg == 0 || cfg == 1 || cfg == 4) {
    const double o[3] = {0, 0, 0};
    if (dist_point_prim_bound(p, o) < clearance) return 1;
    const double radius = (cfg == 4) ? 4.0 : 1.0;
    for (int k = 0; k < 64; ++k) { /* the circular camera path */
      const double th = 2 * M_PI * k / 64.0;
      const double q[3] = {radius * cos(th), 0, radius * sin(th)};
      if (dist_point_prim_bound(p, q) < clearance + 0.15) return 1;
    }
  }
  return 0;
}

/* cfg 0/1/4: room x in [-3,3], y in [-1.5,1.5] (vertical), z in [-3,3] (cfg4:
 * 20x20x5). 20 AABBs + 10 spheres. cfg2: 10x10x5 room with boxes and vertical
 * cylinders. cfg3: ground plane + box buildings + poles along a 1 km road. */
int wl_make_scene(int cfg, uint64_t seed, wl_prim* out, int cap) {
  uint64_t s = rng_seed(seed);
  int n = 0;
#define PUSH(pr) do { if (n < cap) out[n] = (pr); ++n; } while (0)
  if (cfg == 0 || cfg == 1 || cfg == 4) {
    const double hx = cfg == 4 ? 10.0 : 3.0, hy = cfg == 4 ? 2.5 : 1.5, hz = cfg == 4 ? 10.0 : 3.0;
    const double scale = cfg == 4 ? 2.0 : 1.0;
    wl_prim room = {WL_ROOM, 1, {-hx, -hy, -hz, hx, hy, hz}};
    PUSH(room);
    int boxes = 0, spheres = 0, guard = 0;
    while ((boxes < 20 || spheres < 10) && guard++ < 100000) {
      wl_prim p;
      memset(&p, 0, sizeof p);
      if (boxes < 20) {
        p.kind = WL_BOX;
        p.a[0] = (sm64_uniform(&s) * 2 - 1) * hx;
        p.a[1] = (sm64_uniform(&s) * 2 - 1) * hy;
        p.a[2] = (sm64_uniform(&s) * 2 - 1) * hz;
        for (int k = 0; k < 3; ++k) p.a[3 + k] = (0.1 + 0.4 * sm64_uniform(&s)) * scale;
      } else {
        p.kind = WL_SPHERE;
        p.a[0] = (sm64_uniform(&s) * 2 - 1) * hx;
        p.a[1] = (sm64_uniform(&s) * 2 - 1) * hy;
        p.a[2] = (sm64_uniform(&s) * 2 - 1) * hz;
        p.a[3] = (0.1 + 0.3 * sm64_uniform(&s)) * scale;
      }
      if (too_close(cfg, &p, scale)) continue;
      PUSH(p);
      if (p.kind == WL_BOX) ++boxes; else ++spheres;
    }
  } else if (cfg == 2) {
    wl_prim room = {WL_ROOM, 1, {-5, -2.5, -5, 5, 2.5, 5}};
    PUSH(room);
    int boxes = 0, cyls = 0, guard = 0;
    while ((boxes < 25 || cyls < 15) && guard++ < 100000) {
      wl_prim p;
      memset(&p, 0, sizeof p);
      if (boxes < 25) {
        p.kind = WL_BOX;
        p.a[0] = (sm64_uniform(&s) * 2 - 1) * 5;
        p.a[1] = (sm64_uniform(&s) * 2 - 1) * 2.5;
        p.a[2] = (sm64_uniform(&s) * 2 - 1) * 5;
        for (int k = 0; k < 3; ++k) p.a[3 + k] = 0.15 + 0.6 * sm64_uniform(&s);
      } else {
        p.kind = WL_CYL;
        p.up = 1;
        p.a[0] = (sm64_uniform(&s) * 2 - 1) * 5; /* x */
        p.a[1] = (sm64_uniform(&s) * 2 - 1) * 5; /* z  (h0 = 2, h1 = 0 for up=1) */
        p.a[2] = 0.1 + 0.3 * sm64_uniform(&s);
        p.a[3] = -2.5;
        p.a[4] = -2.5 + 0.5 + 4.5 * sm64_uniform(&s);
      }
      /* keep the central flight corridor (|x|,|z| < 3 ring) mostly free */
      const double cx = p.kind == WL_CYL ? p.a[1] : p.a[0];
      const double cz = p.kind == WL_CYL ? p.a[0] : p.a[2];
      const double rr = sqrt(cx * cx + cz * cz);
      if (rr > 1.8 && rr < 3.6) continue;
      PUSH(p);
      if (p.kind == WL_BOX) ++boxes; else ++cyls;
    }
  } else if (cfg == 3) {
    wl_prim ground = {WL_PLANE, 2, {0, 0, 0, 0, 0, 0}};
    PUSH(ground);
    /* road along +x from 0 to 1000 m, gentle sinusoidal y(x) */
    for (double x = -40; x < 1040; x += 0) {
      wl_prim b;
      memset(&b, 0, sizeof b);
      b.kind = WL_BOX;
      const double len = 6 + 14 * sm64_uniform(&s);
      const double side = sm64_uniform(&s) < 0.5 ? -1 : 1;
      const double off = 9 + 20 * sm64_uniform(&s);
      const double cy = 15.0 * sin(x / 160.0) + side * (off + 4);
      const double h = 3 + 17 * sm64_uniform(&s);
      b.a[0] = x + 0.5 * len; b.a[1] = cy; b.a[2] = 0.5 * h;
      b.a[3] = 0.5 * len; b.a[4] = 2 + 4 * sm64_uniform(&s); b.a[5] = 0.5 * h;
      PUSH(b);
      x += len + 2 + 6 * sm64_uniform(&s);
    }
    for (double x = 0; x < 1040; x += 12 + 6 * sm64_uniform(&s)) {
      for (int side = -1; side <= 1; side += 2) {
        wl_prim c;
        memset(&c, 0, sizeof c);
        c.kind = WL_CYL;
        c.up = 2;
        c.a[0] = x; /* h0 = 0 (x) */
        c.a[1] = 15.0 * sin(x / 160.0) + side * 6.5; /* h1 = 1 (y) */
        c.a[2] = 0.12 + 0.1 * sm64_uniform(&s);
        c.a[3] = 0; c.a[4] = 5 + 3 * sm64_uniform(&s);
        PUSH(c);
      }
    }
  }
#undef PUSH
  return n;
}

/* -------------------------------------------------------------- poses */
static void rodrigues(const double w[3], double R[9]) {
  const double th = sqrt(w[0] * w[0] + w[1] * w[1] + w[2] * w[2]);
  if (th < 1e-15) { memset(R, 0, 9 * sizeof(double)); R[0] = R[4] = R[8] = 1; return; }
  const double k[3] = {w[0] / th, w[1] / th, w[2] / th};
  const double c = cos(th), s = sin(th), v = 1 - c;
  R[0] = k[0] * k[0] * v + c;        R[1] = k[0] * k[1] * v - k[2] * s; R[2] = k[0] * k[2] * v + k[1] * s;
  R[3] = k[1] * k[0] * v + k[2] * s; R[4] = k[1] * k[1] * v + c;        R[5] = k[1] * k[2] * v - k[0] * s;
  R[6] = k[2] * k[0] * v - k[1] * s; R[7] = k[2] * k[1] * v + k[0] * s; R[8] = k[2] * k[2] * v + c;
}
static void matmul3(const double A[9], const double B[9], double C[9]) {
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) C[3 * i + j] = A[3 * i] * B[j] + A[3 * i + 1] * B[3 + j] + A[3 * i + 2] * B[6 + j];
}
/* camera frame: x right, y down, z forward; columns of R are the camera axes in world */
static void look_frame(const double fwd[3], const double up_hint[3], double R[9]) {
  double z[3] = {fwd[0], fwd[1], fwd[2]};
  double nz = sqrt(z[0] * z[0] + z[1] * z[1] + z[2] * z[2]);
  for (int i = 0; i < 3; ++i) z[i] /= nz;
  /* y = down = -up projected */
  double y[3] = {-up_hint[0], -up_hint[1], -up_hint[2]};
  double dp = y[0] * z[0] + y[1] * z[1] + y[2] * z[2];
  for (int i = 0; i < 3; ++i) y[i] -= dp * z[i];
  double ny = sqrt(y[0] * y[0] + y[1] * y[1] + y[2] * y[2]);
  for (int i = 0; i < 3; ++i) y[i] /= ny;
  const double x[3] = {y[1] * z[2] - y[2] * z[1], y[2] * z[0] - y[0] * z[2], y[0] * z[1] - y[1] * z[0]};
  for (int i = 0; i < 3; ++i) { R[3 * i] = x[i]; R[3 * i + 1] = y[i]; R[3 * i + 2] = z[i]; }
}

/* Sensor->world pose of frame f for config cfg, 3x4 row-major float [R | t]. */
void wl_pose(int cfg, int frame, int n_frames, uint64_t seed, float pose_out[12]) {
  double R[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1}, t[3] = {0, 0, 0};
  if (n_frames < 1) n_frames = 1;
  if (cfg == 1 || cfg == 4) {
    const double radius = cfg == 4 ? 4.0 : 1.0;
    const double th = 2 * M_PI * frame / n_frames;
    const double up[3] = {0, 1, 0};
    const double fwd[3] = {-sin(th), 0, cos(th)}; /* yaw tangent to the circle */
    double Rb[9];
    look_frame(fwd, up, Rb);
    uint64_t s = mix3(seed, 0x7001, (uint64_t)frame);
    const double jr = 0.5 * M_PI / 180.0;
    const double w[3] = {jr * gauss(&s), jr * gauss(&s), jr * gauss(&s)};
    double Rj[9];
    rodrigues(w, Rj);
    matmul3(Rb, Rj, R);
    t[0] = radius * cos(th) + 0.01 * gauss(&s);
    t[1] = 0.01 * gauss(&s);
    t[2] = radius * sin(th) + 0.01 * gauss(&s);
  } else if (cfg == 2) {
    /* smooth 6-DoF flight: Lissajous ring through the free corridor (r in 1.8..3.6)
     * with seeded phase/amplitudes, looking along the velocity, rolling slightly */
    uint64_t s = mix3(seed, 0x7002, 0);
    const double ph = 2 * M_PI * sm64_uniform(&s), ay = 0.6 + 0.4 * sm64_uniform(&s);
    const double u = 2 * M_PI * frame / n_frames;
    const double r = 2.7 + 0.5 * sin(3 * u + ph);
    t[0] = r * cos(u); t[2] = r * sin(u); t[1] = ay * sin(2 * u + ph);
    const double u2 = u + 1e-3;
    const double r2 = 2.7 + 0.5 * sin(3 * u2 + ph);
    const double fwd[3] = {r2 * cos(u2) - t[0], ay * sin(2 * u2 + ph) - t[1], r2 * sin(u2) - t[2]};
    const double up[3] = {0, 1, 0};
    double Rb[9];
    look_frame(fwd, up, Rb);
    const double roll = 0.15 * sin(5 * u + ph);
    const double w[3] = {0, 0, roll}; /* roll about the camera z axis */
    double Rr[9];
    rodrigues(w, Rr);
    matmul3(Rb, Rr, R);
  } else if (cfg == 3) {
    /* 1 km drive along x, ~2 m per scan, sensor 1.7 m above ground; LiDAR frame
     * x forward, y left, z up */
    const double x = 1000.0 * frame / (n_frames > 1 ? n_frames - 1 : 1);
    const double y = 15.0 * sin(x / 160.0);
    const double dy = 15.0 / 160.0 * cos(x / 160.0);
    const double yaw = atan(dy);
    R[0] = cos(yaw); R[1] = -sin(yaw); R[2] = 0;
    R[3] = sin(yaw); R[4] = cos(yaw);  R[5] = 0;
    R[6] = 0;        R[7] = 0;         R[8] = 1;
    t[0] = x; t[1] = y; t[2] = 1.7;
  }
  for (int i = 0; i < 3; ++i) {
    for (int j = 0; j < 3; ++j) pose_out[4 * i + j] = (float)R[3 * i + j];
    pose_out[4 * i + 3] = (float)t[i];
  }
}

/* Pinhole depth frame (cfg 0/1/2/4). noise sigma = noise_k * z^2 on the
 * z-depth; each pixel is dropped with probability drop_prob (cfg2). Points are
 * sensor-frame ((u-cx) z/fx, (v-cy) z/fy, z). Returns the point count. */
int64_t wl_render_pinhole(const wl_prim* prims, int n_prims, const float pose[12], int width, int height,
                          double fx, double fy, double cx, double cy, double max_range, double noise_k,
                          double drop_prob, uint64_t seed, uint32_t frame, float* xyz, uint8_t* rgb) {
  double R[9], o[3];
  for (int i = 0; i < 3; ++i) {
    for (int j = 0; j < 3; ++j) R[3 * i + j] = pose[4 * i + j];
    o[i] = pose[4 * i + 3];
  }
  const int64_t npx = (int64_t)width * height;
  /* pass 1: per-pixel depth (or <0 = no point), in parallel */
  int64_t count = 0;
#pragma omp parallel for schedule(static) reduction(+ : count)
  for (int64_t i = 0; i < npx; ++i) {
    const int u = (int)(i % width), v = (int)(i / width);
    const double dc[3] = {(u - cx) / fx, (v - cy) / fy, 1.0};
    const double dw[3] = {R[0] * dc[0] + R[1] * dc[1] + R[2] * dc[2], R[3] * dc[0] + R[4] * dc[1] + R[5] * dc[2],
                          R[6] * dc[0] + R[7] * dc[1] + R[8] * dc[2]};
    double z = cast_scene(prims, n_prims, o, dw); /* z-depth since dc.z == 1 */
    int valid = z < 1e299 && z * sqrt(dc[0] * dc[0] + dc[1] * dc[1] + 1.0) <= max_range;
    if (valid && drop_prob > 0) {
      uint64_t sd = mix3(seed + 5, frame, (uint64_t)i);
      if (sm64_uniform(&sd) < drop_prob) valid = 0;
    }
    if (valid) {
      uint64_t sn = mix3(seed + 3, frame, (uint64_t)i);
      z += noise_k * z * z * gauss(&sn);
      if (!(z > 0)) valid = 0;
    }
    xyz[3 * i + 2] = valid ? (float)z : -1.0f;
    if (valid) {
      xyz[3 * i + 0] = (float)(dc[0] * z);
      xyz[3 * i + 1] = (float)(dc[1] * z);
      if (rgb) {
        uint64_t sc = mix3(seed + 4, frame, (uint64_t)i);
        const uint64_t r = sm64_next(&sc);
        rgb[3 * i + 0] = (uint8_t)(r & 0xff);
        rgb[3 * i + 1] = (uint8_t)((r >> 8) & 0xff);
        rgb[3 * i + 2] = (uint8_t)((r >> 16) & 0xff);
      }
      ++count;
    }
  }
  /* pass 2: stable compaction (row-major order preserved) */
  int64_t k = 0;
  for (int64_t i = 0; i < npx; ++i) {
    if (xyz[3 * i + 2] < 0.0f) continue;
    if (k != i) {
      xyz[3 * k + 0] = xyz[3 * i + 0];
      xyz[3 * k + 1] = xyz[3 * i + 1];
      xyz[3 * k + 2] = xyz[3 * i + 2];
      if (rgb) {
        rgb[3 * k + 0] = rgb[3 * i + 0];
        rgb[3 * k + 1] = rgb[3 * i + 1];
        rgb[3 * k + 2] = rgb[3 * i + 2];
      }
    }
    ++k;
  }
  return k;
}

/* 64-beam spinning LiDAR (cfg3): elevations linspace(elev_lo, elev_hi, beams),
 * azimuth step az_step_deg over 360 deg, returns <= max_range, range noise
 * N(0, noise_sigma). Point order: azimuth-major, beam-minor. Culls primitives
 * beyond max_range + 30 m of the sensor before casting. */
int64_t wl_render_lidar(const wl_prim* prims, int n_prims, const float pose[12], int beams, double elev_lo_deg,
                        double elev_hi_deg, double az_step_deg, double max_range, double noise_sigma,
                        uint64_t seed, uint32_t frame, float* xyz, wl_prim* scratch) {
  double R[9], o[3];
  for (int i = 0; i < 3; ++i) {
    for (int j = 0; j < 3; ++j) R[3 * i + j] = pose[4 * i + j];
    o[i] = pose[4 * i + 3];
  }
  int nn = 0;
  for (int i = 0; i < n_prims; ++i) {
    if (prims[i].kind == WL_PLANE || dist_point_prim_bound(&prims[i], o) < max_range + 30.0) scratch[nn++] = prims[i];
  }
  const int steps = (int)ceil(360.0 / az_step_deg - 1e-9);
  const int64_t nrays = (int64_t)steps * beams;
  int64_t count = 0;
#pragma omp parallel for schedule(static) reduction(+ : count)
  for (int64_t i = 0; i < nrays; ++i) {
    const int a = (int)(i / beams), b = (int)(i % beams);
    const double az = a * az_step_deg * M_PI / 180.0;
    const double el = (elev_lo_deg + (elev_hi_deg - elev_lo_deg) * b / (beams - 1)) * M_PI / 180.0;
    const double dc[3] = {cos(el) * cos(az), cos(el) * sin(az), sin(el)};
    const double dw[3] = {R[0] * dc[0] + R[1] * dc[1] + R[2] * dc[2], R[3] * dc[0] + R[4] * dc[1] + R[5] * dc[2],
                          R[6] * dc[0] + R[7] * dc[1] + R[8] * dc[2]};
    double r = cast_scene(scratch, nn, o, dw);
    int valid = r <= max_range;
    if (valid) {
      uint64_t sn = mix3(seed + 3, frame, (uint64_t)i);
      r += noise_sigma * gauss(&sn);
      if (!(r > 0) || r > max_range) valid = 0;
    }
    if (valid) {
      xyz[3 * i + 0] = (float)(dc[0] * r);
      xyz[3 * i + 1] = (float)(dc[1] * r);
      xyz[3 * i + 2] = (float)(dc[2] * r);
      ++count;
    } else {
      xyz[3 * i + 0] = NAN;
    }
  }
  int64_t k = 0;
  for (int64_t i = 0; i < nrays; ++i) {
    if (isnan(xyz[3 * i + 0])) continue;
    if (k != i) {
      xyz[3 * k + 0] = xyz[3 * i + 0];
      xyz[3 * k + 1] = xyz[3 * i + 1];
      xyz[3 * k + 2] = xyz[3 * i + 2];
    }
    ++k;
  }
  return k;
}
