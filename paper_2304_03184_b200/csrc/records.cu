// Motion-prior ingestion: the CFMP v1 stream the tracker
// appends per frame (records.py:98-147) decoded natively into caller-owned host
// arrays (pinned, for one upload into the device LUT), its encoder, and the
// per-frame forward kinematics of the skeleton on the device, batched over all
// frames of the stream (skinning_transforms, skeleton.py:121-139).
//
// CFMP v1 (little-endian): "CFMP" | u32 version=1 | u32 n_nodes | u32 n_theta,
// then per frame: i64 frame_id | array(dqs n_nodes*8) | array(theta n_theta) |
// array(rotation 9) | array(translation 3), with array(x) = u32 count | count
// float64 (records.py:27-36,106-113).
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "common.cuh"

namespace {

constexpr char kMagic[4] = {'C', 'F', 'M', 'P'};
constexpr uint32_t kVersion = 1;

struct File {
  FILE* f = nullptr;
  explicit File(const char* path, const char* mode) : f(std::fopen(path, mode)) {}
  ~File() {
    if (f) std::fclose(f);
  }
};

// little-endian host assumed (x86-64 / aarch64), as the format is
bool read_exact(FILE* f, void* dst, size_t n) { return std::fread(dst, 1, n, f) == n; }

int fmt_error(const char* path, const std::string& what) {
  return cf::fail(CF_E_FORMAT, std::string(path) + ": " + what);
}

// header -> (n_nodes, n_theta); the error strings follow records.py:134-137
int read_header(FILE* f, const char* path, uint32_t* n_nodes, uint32_t* n_theta) {
  char magic[4];
  if (!read_exact(f, magic, 4) || std::memcmp(magic, kMagic, 4) != 0)
    return fmt_error(path, "not a motion prior stream");
  uint32_t h[3];
  if (!read_exact(f, h, sizeof(h))) return fmt_error(path, "truncated header");
  if (h[0] != kVersion) return fmt_error(path, "unsupported version " + std::to_string(h[0]));
  *n_nodes = h[1];
  *n_theta = h[2];
  return CF_OK;
}

// one length-prefixed float64 array of exactly `expect` values (records.py:33-36)
int read_array(FILE* f, const char* path, uint64_t expect, double* dst, int64_t frame, const char* what) {
  uint32_t n;
  if (!read_exact(f, &n, 4)) return fmt_error(path, "truncated frame " + std::to_string(frame));
  if (n != expect)
    return fmt_error(path, std::string(what) + " of frame " + std::to_string(frame) + " has " + std::to_string(n) +
                               " values, expected " + std::to_string(expect));
  if (dst) {
    if (!read_exact(f, dst, 8 * (size_t)n)) return fmt_error(path, "truncated frame " + std::to_string(frame));
  } else if (std::fseek(f, 8 * (long)n, SEEK_CUR) != 0) {
    return fmt_error(path, "truncated frame " + std::to_string(frame));
  }
  return CF_OK;
}

// Walk the frames; with dst pointers, decode frames [first, first + count).
int walk(const char* path, cf_mp_info* info, int64_t first, int64_t count, int64_t* fids, double* dqs, double* theta,
         double* rot, double* trans) {
  if (!path) return cf::fail(CF_E_BAD_ARG, "cf_mp: null path");
  File F(path, "rb");
  if (!F.f) return cf::fail(CF_E_BAD_ARG, std::string(path) + ": cannot open");
  uint32_t nn, nt;
  if (int rc = read_header(F.f, path, &nn, &nt)) return rc;
  std::fseek(F.f, 0, SEEK_END);
  const long size = std::ftell(F.f);
  std::fseek(F.f, 16, SEEK_SET);
  const uint64_t nd = 8ull * nn;
  int64_t fr = 0;
  for (;;) {
    int64_t fid;
    const size_t got = std::fread(&fid, 1, 8, F.f);
    if (got == 0) break;  // clean end of stream (records.py:141-142)
    if (got != 8) return fmt_error(path, "truncated frame " + std::to_string(fr));
    const bool want = fids && fr >= first && fr < first + count;
    if (!want) {
      // frames outside the range: validate the four array lengths, skip the payload
      if (int rc = read_array(F.f, path, nd, nullptr, fr, "dqs")) return rc;
      if (int rc = read_array(F.f, path, nt, nullptr, fr, "theta")) return rc;
      if (int rc = read_array(F.f, path, 9, nullptr, fr, "rotation")) return rc;
      if (int rc = read_array(F.f, path, 3, nullptr, fr, "translation")) return rc;
      if (std::ftell(F.f) > size) return fmt_error(path, "truncated frame " + std::to_string(fr));
    } else {
      const int64_t i = fr - first;
      fids[i] = fid;
      if (int rc = read_array(F.f, path, nd, dqs + i * nd, fr, "dqs")) return rc;
      if (int rc = read_array(F.f, path, nt, theta + i * nt, fr, "theta")) return rc;
      if (int rc = read_array(F.f, path, 9, rot + i * 9, fr, "rotation")) return rc;
      if (int rc = read_array(F.f, path, 3, trans + i * 3, fr, "translation")) return rc;
    }
    ++fr;
    if (fids && fr >= first + count) break;
  }
  if (info) {
    info->n_frames = fr;
    info->n_nodes = (int32_t)nn;
    info->n_theta = (int32_t)nt;
    info->bytes = size;
  }
  if (fids && fr < first + count) return cf::fail(CF_E_BAD_ARG, std::string(path) + ": frame range beyond the stream");
  return CF_OK;
}

// ------------------------------------------------------------ device FK
// One warp per frame. Lanes compute the joints' rotation matrices in parallel
// (quat_from_rotvec + quat_to_matrix, transforms.py:66-84, numpy's operation
// order), then walk the chain: lanes 0..11 own entry (r, c), r < 3, of
// G_j = G_parent L_j (skeleton.py:121-132); the rest pose G_j(0) = [I | c_j]
// with c_j = c_parent + offset_j exactly, whose inverse is exactly [I | -c_j],
// so A_j = G_j(theta) G_j(0)^-1 = [R_j | t_j - R_j c_j] (skeleton.py:135-139).
constexpr int kMaxJ = 64;
constexpr int kFkWarps = 2;  // frames per CTA

struct Rig {  // kernel parameter (validated on the host: parents[j] < j)
  int32_t parents[kMaxJ];
  double offsets[kMaxJ][3];
};

__global__ void __launch_bounds__(32 * kFkWarps) fk_kernel(const double* __restrict__ theta, int64_t n_frames,
                                                           const __grid_constant__ Rig rig, int J,
                                                           double* __restrict__ A) {
  __shared__ double sR[kFkWarps][kMaxJ][9];
  __shared__ double sG[kFkWarps][kMaxJ][12];
  __shared__ double sC[kFkWarps][kMaxJ][3];
  const int w = threadIdx.x / 32, lane = threadIdx.x & 31;
  const int64_t fr = (int64_t)blockIdx.x * kFkWarps + w;
  if (fr >= n_frames) return;
  const double* th = theta + fr * 3 * J;
  for (int j = lane; j < J; j += 32) {
    const double rx = th[3 * j], ry = th[3 * j + 1], rz = th[3 * j + 2];
    // np.linalg.norm: sqrt(x*x + y*y + z*z) summed left to right
    const double ang = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(rx, rx), __dmul_rn(ry, ry)), __dmul_rn(rz, rz)));
    const double half = __dmul_rn(0.5, ang);
    double k;
    if (ang < 1e-12)
      k = __dsub_rn(0.5, __ddiv_rn(__dmul_rn(ang, ang), 48.0));
    else
      k = __ddiv_rn(sin(half), ang);
    const double qw = cos(half), qx = __dmul_rn(k, rx), qy = __dmul_rn(k, ry), qz = __dmul_rn(k, rz);
    double* R = sR[w][j];
    R[0] = __dsub_rn(1.0, __dmul_rn(2.0, __dadd_rn(__dmul_rn(qy, qy), __dmul_rn(qz, qz))));
    R[1] = __dmul_rn(2.0, __dsub_rn(__dmul_rn(qx, qy), __dmul_rn(qw, qz)));
    R[2] = __dmul_rn(2.0, __dadd_rn(__dmul_rn(qx, qz), __dmul_rn(qw, qy)));
    R[3] = __dmul_rn(2.0, __dadd_rn(__dmul_rn(qx, qy), __dmul_rn(qw, qz)));
    R[4] = __dsub_rn(1.0, __dmul_rn(2.0, __dadd_rn(__dmul_rn(qx, qx), __dmul_rn(qz, qz))));
    R[5] = __dmul_rn(2.0, __dsub_rn(__dmul_rn(qy, qz), __dmul_rn(qw, qx)));
    R[6] = __dmul_rn(2.0, __dsub_rn(__dmul_rn(qx, qz), __dmul_rn(qw, qy)));
    R[7] = __dmul_rn(2.0, __dadd_rn(__dmul_rn(qy, qz), __dmul_rn(qw, qx)));
    R[8] = __dsub_rn(1.0, __dmul_rn(2.0, __dadd_rn(__dmul_rn(qx, qx), __dmul_rn(qy, qy))));
  }
  __syncwarp();
  const int r = lane / 4, c = lane % 4;
  for (int j = 0; j < J; ++j) {
    const int p = rig.parents[j];
    const double* R = sR[w][j];
    const double* o = rig.offsets[j];
    if (lane < 12) {
      // L_j = [[R, o], [0, 0, 0, 1]]; column c of L
      const double l0 = c < 3 ? R[c] : o[0], l1 = c < 3 ? R[3 + c] : o[1], l2 = c < 3 ? R[6 + c] : o[2];
      double v;
      if (p < 0) {
        v = r == 0 ? l0 : (r == 1 ? l1 : l2);
      } else {
        const double* G = sG[w][p];
        v = __dadd_rn(__dadd_rn(__dmul_rn(G[4 * r], l0), __dmul_rn(G[4 * r + 1], l1)), __dmul_rn(G[4 * r + 2], l2));
        if (c == 3) v = __dadd_rn(v, G[4 * r + 3]);  // + G[r][3] * 1
      }
      sG[w][j][4 * r + c] = v;
    } else if (lane < 15) {
      const int a = lane - 12;
      sC[w][j][a] = p < 0 ? o[a] : __dadd_rn(sC[w][p][a], o[a]);
    }
    __syncwarp();
  }
  // A_j = [R_j | t_j - R_j c_j], bottom row (0, 0, 0, 1)
  double* out = A + fr * 16 * J;
  for (int e = lane; e < 16 * J; e += 32) {
    const int j = e / 16, rr = (e % 16) / 4, cc = e % 4;
    double v;
    if (rr == 3) {
      v = cc == 3 ? 1.0 : 0.0;
    } else if (cc < 3) {
      v = sG[w][j][4 * rr + cc];
    } else {
      const double* G = sG[w][j];
      const double* C = sC[w][j];
      v = __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(G[4 * rr], -C[0]), __dmul_rn(G[4 * rr + 1], -C[1])),
                              __dmul_rn(G[4 * rr + 2], -C[2])),
                    G[4 * rr + 3]);
    }
    out[e] = v;
  }
}

// DeformNet layer-1 pose term of a frame (theta folded into a per-frame bias,
// DESIGN.md §3): out[i] = sum_j W[i, col0 + j] * (float)theta[j], fp32, j ascending.
__global__ void pose_bias_kernel(const float* __restrict__ W, int ldw, int col0, int n_out,
                                 const double* __restrict__ theta, int n_theta, float* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_out) return;
  float acc = 0.0f;
  for (int j = 0; j < n_theta; ++j) acc = __fadd_rn(acc, __fmul_rn(W[(int64_t)i * ldw + col0 + j], (float)theta[j]));
  out[i] = acc;
}

}  // namespace

extern "C" {

int cf_mp_scan(const char* path, cf_mp_info* info) {
  if (!info) return cf::fail(CF_E_BAD_ARG, "cf_mp_scan: null info");
  return walk(path, info, 0, 0, nullptr, nullptr, nullptr, nullptr, nullptr);
}

int cf_mp_read(const char* path, int64_t first, int64_t count, int64_t* frame_ids, double* dqs, double* theta,
               double* rot, double* trans) {
  if (first < 0 || count < 0) return cf::fail(CF_E_BAD_ARG, "cf_mp_read: bad frame range");
  if (count == 0) return CF_OK;
  if (!frame_ids || !dqs || !theta || !rot || !trans) return cf::fail(CF_E_BAD_ARG, "cf_mp_read: null output");
  return walk(path, nullptr, first, count, frame_ids, dqs, theta, rot, trans);
}

int cf_mp_write(const char* path, int create, int32_t n_nodes, int32_t n_theta, int64_t count,
                const int64_t* frame_ids, const double* dqs, const double* theta, const double* rot,
                const double* trans) {
  if (!path || n_nodes < 0 || n_theta < 0 || count < 0) return cf::fail(CF_E_BAD_ARG, "cf_mp_write: bad args");
  if (count > 0 && (!frame_ids || !dqs || !theta || !rot || !trans))
    return cf::fail(CF_E_BAD_ARG, "cf_mp_write: null input");
  if (!create) {  // appending: the stream's shape must match (MotionPriorWriter keeps one shape)
    cf_mp_info info;
    if (int rc = cf_mp_scan(path, &info)) return rc;
    if (info.n_nodes != n_nodes || info.n_theta != n_theta)
      return cf::fail(CF_E_BAD_ARG, std::string(path) + ": stream shape differs from the appended frames");
  }
  File F(path, create ? "wb" : "ab");
  if (!F.f) return cf::fail(CF_E_BAD_ARG, std::string(path) + ": cannot open for writing");
  bool ok = true;
  if (create) {
    const uint32_t h[3] = {kVersion, (uint32_t)n_nodes, (uint32_t)n_theta};
    ok = std::fwrite(kMagic, 1, 4, F.f) == 4 && std::fwrite(h, 4, 3, F.f) == 3;
  }
  auto put = [&](const double* src, uint32_t n) {
    ok = ok && std::fwrite(&n, 4, 1, F.f) == 1 && std::fwrite(src, 8, n, F.f) == n;
  };
  const uint32_t nd = 8u * (uint32_t)n_nodes;
  for (int64_t i = 0; i < count && ok; ++i) {
    ok = std::fwrite(&frame_ids[i], 8, 1, F.f) == 1;
    put(dqs + i * nd, nd);
    put(theta + i * n_theta, (uint32_t)n_theta);
    put(rot + i * 9, 9);
    put(trans + i * 3, 3);
  }
  ok = ok && std::fflush(F.f) == 0;
  return ok ? CF_OK : cf::fail(CF_E_BAD_ARG, std::string(path) + ": write failed");
}

int cf_pose_bias(const float* W, int ldw, int col0, int n_out, const double* theta, int n_theta, float* out,
                 void* stream) {
  if (!W || !theta || !out || n_out < 0 || n_theta < 0 || ldw < col0 + n_theta)
    return cf::fail(CF_E_BAD_ARG, "cf_pose_bias: bad args");
  if (n_out == 0) return CF_OK;
  pose_bias_kernel<<<(unsigned)((n_out + 127) / 128), 128, 0, cf::as_stream(stream)>>>(W, ldw, col0, n_out, theta,
                                                                                       n_theta, out);
  return cf::check_launch("cf_pose_bias");
}

int cf_skinning_transforms(const double* theta, int64_t n_frames, const int32_t* parents, const double* offsets,
                           int32_t n_joints, double* A, void* stream) {
  if (n_frames < 0 || n_joints <= 0 || n_joints > kMaxJ || !theta || !parents || !offsets || !A)
    return cf::fail(CF_E_BAD_ARG, "cf_skinning_transforms: bad args (1 <= J <= 64)");
  Rig rig = {};
  for (int j = 0; j < n_joints; ++j) {
    if (parents[j] >= j || parents[j] < -1)
      return cf::fail(CF_E_BAD_ARG, "cf_skinning_transforms: parents must precede their children");
    rig.parents[j] = parents[j];
    for (int a = 0; a < 3; ++a) rig.offsets[j][a] = offsets[3 * j + a];
  }
  if (n_frames == 0) return CF_OK;
  fk_kernel<<<(unsigned)((n_frames + kFkWarps - 1) / kFkWarps), 32 * kFkWarps, 0, cf::as_stream(stream)>>>(
      theta, n_frames, rig, n_joints, A);
  return cf::check_launch("cf_skinning_transforms");
}

}  // extern "C"
