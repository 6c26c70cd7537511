// gs_project kernel — Eq. 2-3, O1.
// Compiled with -fmad=false: depth key, radius, rect and tile count must match the oracle bit for
// bit, so every binary operation is rounded separately in the fixed order of DESIGN.md O1, and
// '/' and sqrtf are the IEEE (correctly rounded) versions.
#include "gs_internal.cuh"

namespace gs {

__device__ __forceinline__ int clamp_tile(float v, int hi) {
    if (!(v > 0.f)) return 0;   // NaN -> 0
    if (v > float(hi)) return hi;
    return int(v);
}

// One Gaussian: the DESIGN.md O1 steps on its 14 parameter values p (rows 11-13: RGB or SH constant
// terms), writing its record, depth key, rect, radius and tile count.
__device__ __forceinline__ void project_one(
    const float (&p)[14], int64_t i, const float* __restrict__ params, int64_t ld, const uint8_t* __restrict__ mask,
    const float* V, const gs_camera& cam, int GX, int GY, int sh, int orad, float4* __restrict__ rec,
    uint32_t* __restrict__ depth_key, short4* __restrict__ rect, int32_t* __restrict__ radius_out,
    uint32_t* __restrict__ tiles_out) {

    float4 r0 = make_float4(0.f, 0.f, 0.f, 0.f), r1 = r0, r2 = r0;
    int radius = 0;
    short4 rc = make_short4(0, 0, 0, 0);
    uint32_t tiles = 0;
    // 1. X^c = W X + t
    const float xc = ((V[0] * p[0] + V[1] * p[1]) + V[2] * p[2]) + V[3];
    const float yc = ((V[4] * p[0] + V[5] * p[1]) + V[6] * p[2]) + V[7];
    const float zc = ((V[8] * p[0] + V[9] * p[1]) + V[10] * p[2]) + V[11];
    const uint32_t dkey = __float_as_uint(zc);
    bool ok = zc > cam.znear && (mask == nullptr || mask[i] != 0);   // 2. near-plane cull (NaN fails)
    float qr = 0.f, qi = 0.f, qj = 0.f, qk = 0.f;
    if (ok) {   // 3. normalise q
        const float n2 = ((p[6] * p[6] + p[7] * p[7]) + p[8] * p[8]) + p[9] * p[9];
        ok = n2 > 0.f;
        const float nq = sqrtf(n2);
        qr = p[6] / nq; qi = p[7] / nq; qj = p[8] / nq; qk = p[9] / nq;
    }
    if (ok) {
        // 4. R(q) per Eq. S1
        float R[3][3];
        R[0][0] = 1.f - 2.f * (qj * qj + qk * qk);
        R[0][1] = 2.f * (qi * qj - qr * qk);
        R[0][2] = 2.f * (qi * qk + qr * qj);
        R[1][0] = 2.f * (qi * qj + qr * qk);
        R[1][1] = 1.f - 2.f * (qi * qi + qk * qk);
        R[1][2] = 2.f * (qj * qk - qr * qi);
        R[2][0] = 2.f * (qi * qk - qr * qj);
        R[2][1] = 2.f * (qj * qk + qr * qi);
        R[2][2] = 1.f - 2.f * (qi * qi + qj * qj);
        // 5. Sigma = M M^T, M = R diag(s)   (Eq. 2)
        float M[3][3];
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
            for (int k = 0; k < 3; ++k) M[a][k] = R[a][k] * p[3 + k];
        float S[3][3];
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
            for (int b = a; b < 3; ++b) {
                S[a][b] = (M[a][0] * M[b][0] + M[a][1] * M[b][1]) + M[a][2] * M[b][2];
                S[b][a] = S[a][b];
            }
        // 6. Sigma' = E Sigma E^T + dil I,  E = J W   (Eq. 3)
        const float tx = xc / zc, ty = yc / zc;
        const float j00 = cam.fx / zc, j11 = cam.fy / zc;
        const float j02 = -(j00 * tx), j12 = -(j11 * ty);
        float E[2][3];
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            E[0][k] = j00 * V[k] + j02 * V[8 + k];
            E[1][k] = j11 * V[4 + k] + j12 * V[8 + k];
        }
        float U[2][3];
#pragma unroll
        for (int a = 0; a < 2; ++a)
#pragma unroll
            for (int k = 0; k < 3; ++k) U[a][k] = (E[a][0] * S[0][k] + E[a][1] * S[1][k]) + E[a][2] * S[2][k];
        const float A = ((U[0][0] * E[0][0] + U[0][1] * E[0][1]) + U[0][2] * E[0][2]) + cam.cov2d_dilation;
        const float B = (U[0][0] * E[1][0] + U[0][1] * E[1][1]) + U[0][2] * E[1][2];
        const float C = ((U[1][0] * E[1][0] + U[1][1] * E[1][1]) + U[1][2] * E[1][2]) + cam.cov2d_dilation;
        // 7. conic
        const float det = A * C - B * B;
        if (det > 0.f) {
            const float inv = 1.f / det;
            const float ca = C * inv, cb = -(B * inv), cc = A * inv;
            // 8. radius: 3 sigma, or the alpha >= 1/255 reach (GS_FLAG_OPACITY_RADIUS, reading C33):
            //    q <= q_m = 2 ln(255 o) + 2e-3 (margin over the renderer's fp32 skip test); the
            //    ellipse's bounding box is |x| <= sqrt(q_m A), |y| <= sqrt(q_m C)
            const float mid = 0.5f * (A + C);
            const float lam1 = mid + sqrtf(fmaxf(0.1f, mid * mid - det));
            float rf, rx = 0.f, ry = 0.f;
            bool reach = true;
            if (orad) {
                const float qo = float(2.0 * log(255.0 * double(p[10])));
                reach = qo > 0.f;
                const float qm = qo + 2e-3f;
                rf = ceilf(sqrtf(qm * lam1));
                rx = sqrtf(qm * A);
                ry = sqrtf(qm * C);
            } else {
                rf = ceilf(3.f * sqrtf(lam1));
            }
            if (!(rf < 16777216.f)) rf = 16777216.f;
            radius = reach ? int(rf) : 0;
            // 9. mean
            const float mx = cam.fx * tx + cam.cx;
            const float my = cam.fy * ty + cam.cy;
            // 10. rect: the 3DGS tile box of the radius, or (C33) the tiles holding the integer pixels
            //     of the bounding box [ceil(m - r), floor(m + r)]
            int xlo, xhi, ylo, yhi;
            if (orad) {
                xlo = clamp_tile(floorf(ceilf(mx - rx) / 16.f), GX);
                xhi = clamp_tile(floorf(floorf(mx + rx) / 16.f) + 1.f, GX);
                ylo = clamp_tile(floorf(ceilf(my - ry) / 16.f), GY);
                yhi = clamp_tile(floorf(floorf(my + ry) / 16.f) + 1.f, GY);
            } else {
                const float r = float(radius);
                xlo = clamp_tile(floorf((mx - r) / 16.f), GX);
                xhi = clamp_tile(floorf(((mx + r) + 15.f) / 16.f), GX);
                ylo = clamp_tile(floorf((my - r) / 16.f), GY);
                yhi = clamp_tile(floorf(((my + r) + 15.f) / 16.f), GY);
            }
            if (reach) {
                rc = make_short4(short(xlo), short(xhi), short(ylo), short(yhi));
                tiles = uint32_t(max(0, xhi - xlo)) * uint32_t(max(0, yhi - ylo));
            }
            // exactly scaled conic for the blend: A = -a/2, B = -b, C = -c/2 (gs_internal.cuh)
            r0 = make_float4(mx, my, -0.5f * ca, -cb);
            // r1.w: squared Mahalanobis reach q_max = 2 ln(255 o), where o exp(-q/2) = 1/255, plus a
            // margin (render.cu can_reach; no decision uses it, so it is outside reading R1's order)
            r1 = make_float4(-0.5f * cc, p[10], zc, 2.f * (logf(255.f * p[10]) + 1e-4f) + 2e-4f);
            if (sh == 1) {
                // degree-1 SH colour at the view direction (gs.h gs_project_sh, reading C29), in the
                // oracle's fp32 order: camera centre c = -W^T t, u = (X - c)/|X - c|,
                // rgb = max(0, 1/2 + C0 Y0 + C1 (-u_y Y1 + u_z Y2 - u_x Y3)); rows 11 + 3k + c
                const float cwx = -((V[0] * V[3] + V[4] * V[7]) + V[8] * V[11]);
                const float cwy = -((V[1] * V[3] + V[5] * V[7]) + V[9] * V[11]);
                const float cwz = -((V[2] * V[3] + V[6] * V[7]) + V[10] * V[11]);
                const float dx = p[0] - cwx, dy = p[1] - cwy, dz = p[2] - cwz;
                const float len = sqrtf((dx * dx + dy * dy) + dz * dz);
                const float ux = dx / len, uy = dy / len, uz = dz / len;
                float rgb[3];
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    const float y1 = __ldg(params + (14 + c) * ld + i), y2 = __ldg(params + (17 + c) * ld + i),
                                y3 = __ldg(params + (20 + c) * ld + i);
                    const float lin = (-(uy * y1) + uz * y2) - ux * y3;
                    const float v = (0.28209479177387814f * p[11 + c] + 0.4886025119029199f * lin) + 0.5f;
                    rgb[c] = v > 0.f ? v : 0.f;
                }
                r2 = make_float4(rgb[0], rgb[1], rgb[2], 0.f);
            } else {
                r2 = make_float4(p[11], p[12], p[13], 0.f);
            }
        } else {
            radius = 0;
        }
    }
    rec[3 * i + 0] = r0;
    rec[3 * i + 1] = r1;
    rec[3 * i + 2] = r2;
    depth_key[i] = dkey;
    rect[i] = rc;
    radius_out[i] = radius;
    tiles_out[i] = tiles;
}

// kG Gaussians per thread (i, i + 256, ...): all their parameter loads are issued before any of the
// (long, division-heavy) projection chains, so each warp keeps kG x 14 loads in flight.
constexpr int kProjG = 2;
__global__ void __launch_bounds__(256) project_kernel(
    const float* __restrict__ params, int64_t n, int64_t ld, const uint8_t* __restrict__ mask,
    const float* __restrict__ viewmat, gs_camera cam, int GX, int GY, int sh, int orad,
    float4* __restrict__ rec, uint32_t* __restrict__ depth_key, short4* __restrict__ rect,
    int32_t* __restrict__ radius_out, uint32_t* __restrict__ tiles_out) {
    griddep_wait();   // PDL: the previous kernel's writes (and its reads of what this one writes) are done
    __shared__ float V[12];
    if (threadIdx.x < 12) V[threadIdx.x] = viewmat[threadIdx.x];
    __syncthreads();
    const int64_t i0 = int64_t(blockIdx.x) * blockDim.x * kProjG + threadIdx.x;
    float p[kProjG][14];
#pragma unroll
    for (int g = 0; g < kProjG; ++g) {
        const int64_t i = i0 + int64_t(g) * blockDim.x;
        // a masked-out Gaussian (tracking's fine stage) needs only its position (its depth key is
        // still written); the other 11 rows are not read
        const bool on = i < n && (mask == nullptr || mask[i] != 0);
#pragma unroll
        for (int k = 0; k < 14; ++k) p[g][k] = (k < 3 ? i < n : on) ? __ldg(params + k * ld + i) : 0.f;
    }
#pragma unroll
    for (int g = 0; g < kProjG; ++g) {
        const int64_t i = i0 + int64_t(g) * blockDim.x;
        if (i < n)
            project_one(p[g], i, params, ld, mask, V, cam, GX, GY, sh, orad, rec, depth_key, rect, radius_out,
                        tiles_out);
    }
}

void launch_project(WsState* s, const float* params, int64_t n, int64_t ld, const uint8_t* mask,
                    const float* viewmat, const gs_camera& cam, cudaStream_t st) {
    const int GX = (cam.width + kTile - 1) / kTile, GY = (cam.height + kTile - 1) / kTile;
    if (n == 0) return;
    const int blocks = int((n + 256 * kProjG - 1) / (256 * kProjG));
    KTimer kt(s, KID_PROJECT, st);
    launch_pdl(project_kernel, dim3(blocks), dim3(256), 0, st, params, n, ld, mask, viewmat, cam, GX, GY, s->sh_degree,
                                           s->opacity_radius, at<float4>(s, s->rec),
                                           at<uint32_t>(s, s->depth_key), at<short4>(s, s->rect),
                                           at<int32_t>(s, s->radius), at<uint32_t>(s, s->tiles));
}

}  // namespace gs
