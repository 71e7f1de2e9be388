// metrics.cu -- the tuner's sampling statistics and the quality metrics on
// the GPU, bit-identical to the reference's numpy / scipy
// arithmetic:
//  * analyze_samples (tuner.py:86-124): per-axis linear / cubic prediction
//    residuals at the strided interior sample (grid.py:198-219), summed in
//    numpy's pairwise order (np.mean = pairwise sum / n, divided on the host);
//  * psnr (metrics.py:36-51): pairwise sum of (x - y)^2;
//  * ssim (metrics.py:64-94): scipy.ndimage.uniform_filter (reflect mode,
//    one running-sum 1-D pass per axis, scipy's NI_UniformFilter1D order),
//    the elementwise SSIM terms at every second full-window centre, and a
//    pairwise mean.
// Every product / sum is a separately rounded f64 operation (-fmad=false).
#include <cstdio>

#include "common.cuh"
#include "pairwise.cuh"

namespace hpez {

constexpr int kRedD = 12;  // 4096 partial subtrees for long reductions

template <typename T>
__device__ __forceinline__ double ld64(const void *p, int64_t i) {
    return (double)reinterpret_cast<const T *>(p)[i];
}

// ------------------------------------------------------- analyze_samples --
struct SampleGeom {
    int32_t rank;
    int32_t is_f64;
    int64_t dims[kMaxRank];
    int64_t estr[kMaxRank];
    int64_t lo[kMaxRank];
    int64_t size[kMaxRank];
    int64_t m, n;
};

// residual^2 of sample i along `axis`: kind 0 = linear, 1 = cubic
struct SampleResidual {
    const void *grid;
    SampleGeom g;
    int axis, kind;
    __device__ double val(int64_t idx) const {
        return g.is_f64 ? ld64<double>(grid, idx) : ld64<float>(grid, idx);
    }
    __device__ double operator()(int64_t i) const {
        // flat = (i * m) // n over the row-major interior box (grid.py:213-219)
        int64_t rem = i * g.m / g.n;  // < n * m, far below 2^63
        int64_t idx = 0;
        for (int a = kMaxRank - 1; a >= 0; a--) {
            if (a < g.rank) {
                const int64_t c = rem % g.size[a] + g.lo[a];
                rem /= g.size[a];
                idx += c * g.estr[a];
            }
        }
        const int64_t st = g.estr[axis];
        const double v = val(idx);
        double pred;
        if (kind == 0) {  // vals - 0.5 * (nb(-1) + nb(1))
            pred = __dmul_rn(0.5, __dadd_rn(val(idx - st), val(idx + st)));
        } else {  // sum(c * nb(o) for o, c in _CUBIC), starting from int 0
            pred = __dadd_rn(0.0, __dmul_rn(-1.0 / 16, val(idx - 3 * st)));
            pred = __dadd_rn(pred, __dmul_rn(9.0 / 16, val(idx - st)));
            pred = __dadd_rn(pred, __dmul_rn(9.0 / 16, val(idx + st)));
            pred = __dadd_rn(pred, __dmul_rn(-1.0 / 16, val(idx + 3 * st)));
        }
        const double d = __dsub_rn(v, pred);
        return __dmul_rn(d, d);
    }
};

// (x - y)^2 of two grids (psnr's mse numerator)
struct SqDiff {
    const void *a, *b;
    int a64, b64;
    __device__ double operator()(int64_t i) const {
        const double x = a64 ? ld64<double>(a, i) : ld64<float>(a, i);
        const double y = b64 ? ld64<double>(b, i) : ld64<float>(b, i);
        const double d = __dsub_rn(x, y);
        return __dmul_rn(d, d);
    }
};

template <typename F>
static cudaError_t pairwise_sum_f(const F &f, int64_t n, double *out, double *scratch, cudaStream_t st) {
    // scratch: (1 << kRedD) doubles then (1 << kRedD) bytes
    int8_t *leaf = reinterpret_cast<int8_t *>(scratch + (1 << kRedD));
    np_pairwise_partials_kernel<kRedD, F><<<(1 << kRedD) / 256, 256, 0, st>>>(f, n, scratch, leaf);
    const size_t smem = (size_t)(1 << kRedD) * 9;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(np_pairwise_finish_kernel<kRedD>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem);
        attr = true;
    }
    np_pairwise_finish_kernel<kRedD><<<1, 1024, smem, st>>>(scratch, leaf, out);
    return cudaGetLastError();
}

// ----------------------------------------------------------------- ssim --
// scipy.ndimage.uniform_filter1d(mode="reflect") along one axis: one thread
// per line, the running sum of NI_UniformFilter1D:
//   tmp = sum(line[-size1 .. size2]);  out[0] = tmp / w
//   tmp += line[l - 1 + w - size1] - line[l - 1 - size1];  out[l] = tmp / w
// with reflected (half-sample symmetric) extensions, w <= line length.
__global__ void __launch_bounds__(256) uniform1d_kernel(const double *__restrict__ in, double *__restrict__ out,
                                                        int64_t L, int64_t inner, int64_t nlines, int w) {
    const int64_t id = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (id >= nlines) return;
    const int64_t base = (id / inner) * L * inner + (id % inner);
    const int size1 = w / 2;
    auto at = [&](int64_t p) {
        const int64_t q = p < 0 ? -p - 1 : (p >= L ? 2 * L - p - 1 : p);
        return in[base + q * inner];
    };
    const double fw = (double)w;
    double tmp = 0.0;
    for (int l = 0; l < w; l++) tmp = __dadd_rn(tmp, at(l - size1));
    out[base] = __ddiv_rn(tmp, fw);
    for (int64_t l = 1; l < L; l++) {
        tmp = __dadd_rn(tmp, __dsub_rn(at(l - 1 + w - size1), at(l - 1 - size1)));
        out[base + l * inner] = __ddiv_rn(tmp, fw);
    }
}

// x, y, x*x, y*y, x*y as f64 arrays
__global__ void ssim_prep_kernel(const void *a, int a64, const void *b, int b64, int64_t n, double *x, double *y,
                                 double *xx, double *yy, double *xy) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double u = a64 ? ld64<double>(a, i) : ld64<float>(a, i);
    const double v = b64 ? ld64<double>(b, i) : ld64<float>(b, i);
    x[i] = u;
    y[i] = v;
    xx[i] = __dmul_rn(u, u);
    yy[i] = __dmul_rn(v, v);
    xy[i] = __dmul_rn(u, v);
}

struct SelGeom {
    int32_t rank;
    int64_t estr[kMaxRank];
    int64_t lo[kMaxRank];
    int64_t cnt[kMaxRank];
    int64_t n;
};

// num / den at the selected centres (metrics.py:86-93), compact row-major
__global__ void ssim_terms_kernel(const double *mu_x, const double *mu_y, const double *xx, const double *yy,
                                  const double *xy, SelGeom g, double c1, double c2, double *out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= g.n) return;
    int64_t rem = i, idx = 0;
    for (int a = kMaxRank - 1; a >= 0; a--) {
        if (a < g.rank) {
            idx += (g.lo[a] + 2 * (rem % g.cnt[a])) * g.estr[a];
            rem /= g.cnt[a];
        }
    }
    const double mx = mu_x[idx], my = mu_y[idx];
    const double var_x = __dsub_rn(xx[idx], __dmul_rn(mx, mx));
    const double var_y = __dsub_rn(yy[idx], __dmul_rn(my, my));
    const double cov = __dsub_rn(xy[idx], __dmul_rn(mx, my));
    const double num = __dmul_rn(__dadd_rn(__dmul_rn(__dmul_rn(2.0, mx), my), c1), __dadd_rn(__dmul_rn(2.0, cov), c2));
    const double den = __dmul_rn(__dadd_rn(__dadd_rn(__dmul_rn(mx, mx), __dmul_rn(my, my)), c1),
                                 __dadd_rn(__dadd_rn(var_x, var_y), c2));
    out[i] = __ddiv_rn(num, den);
}

static int status(cudaError_t e) {
    if (e == cudaSuccess) return HPEZ_OK;
    fprintf(stderr, "hpez_b200: CUDA error %s\n", cudaGetErrorString(e));
    return HPEZ_CUDA_ERROR;
}

}  // namespace hpez

using namespace hpez;

extern "C" {

int64_t hpez_reduce_scratch_bytes(void) { return (int64_t)(1 << kRedD) * 9 + 256; }

int hpez_pairwise_sum(const double *a, int64_t n, double *out, void *scratch, void *stream) {
    if (n < 0 || (n > 0 && !a) || !out || !scratch) return HPEZ_BAD_ARGUMENT;
    if (n == 0) return status(cudaMemsetAsync(out, 0, sizeof(double), (cudaStream_t)stream));
    return status(pairwise_sum_f(ArrayAt{a}, n, out, (double *)scratch, (cudaStream_t)stream));
}

int hpez_sample_stats(const void *grid, int32_t is_f64, int32_t rank, const int64_t *dims, const int64_t *lo,
                      const int64_t *size, int64_t n, uint32_t lin_mask, uint32_t cub_mask, double *sums,
                      void *scratch, void *stream) {
    if (!grid || !dims || !lo || !size || !sums || !scratch || rank < 1 || rank > kMaxRank || n < 1)
        return HPEZ_BAD_ARGUMENT;
    SampleGeom g{};
    g.rank = rank;
    g.is_f64 = is_f64;
    int64_t e = 1, m = 1;
    for (int a = rank - 1; a >= 0; a--) {
        g.dims[a] = dims[a];
        g.estr[a] = e;
        e *= dims[a];
        g.lo[a] = lo[a];
        g.size[a] = size[a];
        m *= size[a];
    }
    g.m = m;
    g.n = n;
    cudaStream_t st = (cudaStream_t)stream;
    for (int a = 0; a < rank; a++)
        for (int k = 0; k < 2; k++) {
            if (!((k == 0 ? lin_mask : cub_mask) >> a & 1)) continue;
            SampleResidual f{grid, g, a, k};
            cudaError_t err = pairwise_sum_f(f, n, sums + 2 * a + k, (double *)scratch, st);
            if (err) return status(err);
        }
    return HPEZ_OK;
}

int hpez_sq_diff_sum(const void *a, int32_t a_f64, const void *b, int32_t b_f64, int64_t n, double *out,
                     void *scratch, void *stream) {
    if (!a || !b || !out || !scratch || n < 1) return HPEZ_BAD_ARGUMENT;
    return status(pairwise_sum_f(SqDiff{a, b, a_f64, b_f64}, n, out, (double *)scratch, (cudaStream_t)stream));
}

int hpez_uniform_filter1d(const double *in, double *out, int32_t rank, const int64_t *dims, int32_t axis,
                          int32_t size, void *stream) {
    if (!in || !out || in == out || !dims || rank < 1 || rank > kMaxRank || axis < 0 || axis >= rank || size < 1)
        return HPEZ_BAD_ARGUMENT;
    int64_t inner = 1, total = 1;
    for (int a = 0; a < rank; a++) total *= dims[a];
    for (int a = axis + 1; a < rank; a++) inner *= dims[a];
    const int64_t L = dims[axis];
    if (size > L) return HPEZ_BAD_ARGUMENT;  // one reflection per side
    const int64_t nlines = total / L;
    uniform1d_kernel<<<(unsigned)((nlines + 255) / 256), 256, 0, (cudaStream_t)stream>>>(in, out, L, inner, nlines,
                                                                                         size);
    return status(cudaGetLastError());
}

int hpez_ssim_prep(const void *a, int32_t a_f64, const void *b, int32_t b_f64, int64_t n, double *x, double *y,
                   double *xx, double *yy, double *xy, void *stream) {
    if (!a || !b || !x || !y || !xx || !yy || !xy || n < 1) return HPEZ_BAD_ARGUMENT;
    ssim_prep_kernel<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(a, a_f64, b, b_f64, n, x, y,
                                                                                    xx, yy, xy);
    return status(cudaGetLastError());
}

int hpez_ssim_terms(const double *mu_x, const double *mu_y, const double *xx, const double *yy, const double *xy,
                    int32_t rank, const int64_t *dims, const int64_t *lo, const int64_t *cnt, double c1, double c2,
                    double *out, void *stream) {
    if (!mu_x || !mu_y || !xx || !yy || !xy || !out || !dims || !lo || !cnt || rank < 1 || rank > kMaxRank)
        return HPEZ_BAD_ARGUMENT;
    SelGeom g{};
    g.rank = rank;
    int64_t e = 1, n = 1;
    for (int a = rank - 1; a >= 0; a--) {
        g.estr[a] = e;
        e *= dims[a];
        g.lo[a] = lo[a];
        g.cnt[a] = cnt[a];
        n *= cnt[a];
    }
    g.n = n;
    if (n == 0) return HPEZ_OK;
    ssim_terms_kernel<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(mu_x, mu_y, xx, yy, xy, g, c1,
                                                                                     c2, out);
    return status(cudaGetLastError());
}

}  // extern "C"
