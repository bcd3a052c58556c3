// spmv_work_oriented.cu — work_oriented (merge-path) schedule.
//
// Schedule (reference schedules.py:63-110): the merge path over
// (row boundaries x atoms) has rows+nnz items; lane k of P owns diagonals
// [min(k*items, total), min((k+1)*items, total)) with items = ceil(total/P), i.e.
// exactly merge_path_partition(ts, P). Ties consume the row boundary first, so an
// empty row costs one item (schedules.py:81).
//
// Device mapping. A lane is one thread. Three kernels, all stream-ordered:
//  1. k_merge_path_search: one binary search per CTA boundary (or per lane for
//     the direct variant) over off[t]+t; the same search lw_merge_path_partition
//     exports, bit-exact with schedules.merge_path_partition.
//  2. k_wo_staged<IPT> (items <= IPT): a CTA of NT lanes owns NT*items
//     consecutive diagonals. Its row ends and its contiguous atom range are staged
//     through shared memory with coalesced loads (values*x[col] formed during the
//     staging pass so all gathers of the CTA are in flight together); every thread
//     then re-runs the merge-path search inside shared memory for its own diagonal
//     and consumes its items sequentially. Rows completed inside a thread are
//     assigned directly; the partial row a thread starts in is finished with a
//     block-wide segmented scan of thread carries (deterministic order), and the
//     CTA's trailing partial becomes one carry-out.
//     k_wo_direct (items > IPT, i.e. caller-chosen small lane counts): each lane
//     walks its slice straight from global memory, the reference loop verbatim
//     in semantics (_fast.py:31-52), one carry per lane.
//  3. k_carry_fixup: adds carry-outs to their rows in lane/CTA order — the
//     device form of the serial fix-up kernels.py:90-91 / fixup_combine
//     (executor.py:212-221). Runs of carries into one row are summed in order,
//     so results are run-to-run reproducible (no float atomics).
#include "lw_common.cuh"

namespace lw {

constexpr int WO_NT = 256;          // lanes per CTA
constexpr int WO_IPT_AUTO = 8;      // items per lane when lanes are auto-sized
constexpr unsigned WO_PHASE_PARTITION = 1, WO_PHASE_SPMV = 2, WO_PHASE_FIXUP = 4;

// ---- 1. partition ---------------------------------------------------------
template <class OffT>
__global__ void k_merge_path_search(const OffT* __restrict__ off, int64_t rows, int64_t nnz,
                                    int64_t n_bounds, int64_t span,
                                    int64_t* __restrict__ out_tile,
                                    int64_t* __restrict__ out_coords) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n_bounds) return;
    const int64_t total = rows + nnz;
    const int64_t d = min(k * span, total);
    int64_t lo = max((int64_t)0, d - nnz), hi = min(d, rows);
    // greatest t with off[t] <= d - t  (off[t]+t strictly increasing)
    while (lo < hi) {
        const int64_t mid = (lo + hi + 1) >> 1;
        if (ld_off(off + mid) <= d - mid) lo = mid;
        else hi = mid - 1;
    }
    if (out_tile) out_tile[k] = lo;
    if (out_coords) {
        out_coords[2 * k] = lo;
        out_coords[2 * k + 1] = d - lo;
    }
}

// ---- 2a. staged even-share SpMV ------------------------------------------------
struct WoScan {
    int key[WO_NT / kWarp];
    double val[WO_NT / kWarp];
    int pkey[WO_NT / kWarp];      // inclusive scan of warp aggregates
    double pval[WO_NT / kWarp];
};

template <class OffT, class ValT, int IPT, bool PROBE>
__global__ void __launch_bounds__(WO_NT)
    k_wo_staged(Csr<OffT, ValT> A, const ValT* __restrict__ x, ValT* __restrict__ y,
                int64_t lanes, int64_t items, const int64_t* __restrict__ cta_tile,
                int64_t* __restrict__ carry_tile, double* __restrict__ carry_val,
                Probe probe) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double* s_prod = reinterpret_cast<double*>(smem_raw);                // [NT*IPT]
    int32_t* s_end = reinterpret_cast<int32_t*>(s_prod + WO_NT * IPT);    // [NT*IPT]
    __shared__ WoScan scan;

    const int tid = threadIdx.x;
    const int lane = tid & (kWarp - 1), warp = tid >> 5;
    const int64_t c = blockIdx.x;
    const int64_t total = A.rows + A.nnz;
    const int64_t span = WO_NT * items;
    const int64_t d0 = min(c * span, total), d1 = min((c + 1) * span, total);
    const int64_t t0 = cta_tile[c], t1 = cta_tile[c + 1];
    const int64_t a0 = d0 - t0, a1 = d1 - t1;
    const int n_rows = (int)(t1 - t0), n_atoms = (int)(a1 - a0);

    // stage row ends (relative to a0): s_end[i] = off[t0+1+i] - a0
    for (int i = tid; i < n_rows; i += WO_NT) s_end[i] = (int32_t)(ld_off(A.off + t0 + 1 + i) - a0);

    // stage products: coalesced streaming loads, then all gathers in flight
    {
        int32_t cidx[IPT];
        ValT v[IPT];
#pragma unroll
        for (int k = 0; k < IPT; ++k) {
            const int j = k * WO_NT + tid;
            if (j < n_atoms) {
                cidx[k] = ld_stream(A.col + a0 + j);
                v[k] = ld_stream(A.val + a0 + j);
            }
        }
#pragma unroll
        for (int k = 0; k < IPT; ++k) {
            const int j = k * WO_NT + tid;
            if (j < n_atoms) s_prod[j] = (double)v[k] * (double)ld_gather(x + cidx[k]);
        }
    }
    __syncthreads();

    // this lane's local coordinates: search inside shared memory
    const int n_total = n_rows + n_atoms;
    const int dl = (int)min((int64_t)tid * items, (int64_t)n_total);
    const int dl_end = (int)min((int64_t)dl + items, (int64_t)n_total);
    int lo = max(0, dl - n_atoms), hi = min(dl, n_rows);
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (s_end[mid - 1] <= dl - mid) lo = mid;
        else hi = mid - 1;
    }
    int i = lo, j = dl - lo;
    const int i_first = i, j_first = j;
    const int64_t glane = c * WO_NT + tid;

    double acc = 0.0, head = 0.0;
    bool done_any = false;
    for (int step = dl; step < dl_end; ++step) {
        if (i < n_rows && s_end[i] <= j) {           // row boundary first on ties
            if (!done_any) { head = acc; done_any = true; }
            else y[t0 + i] = (ValT)acc;
            acc = 0.0;
            ++i;
        } else {
            acc += s_prod[j];
            if (PROBE) probe_atom(probe, a0 + j, glane, t0 + i);
            ++j;
        }
    }
    if (PROBE && probe.lane_atoms && glane < lanes)
        probe.lane_atoms[glane] = j - j_first;

    // block-wide inclusive segmented scan of (tail row, tail partial)
    int key = i;
    double val = acc;
#pragma unroll
    for (int d = 1; d < kWarp; d <<= 1) {
        const double ov = shfl_up(val, d);
        const int ok = shfl_up(key, d);
        if (lane >= d && ok == key) val += ov;
    }
    if (lane == kWarp - 1) { scan.key[warp] = key; scan.val[warp] = val; }
    __syncthreads();
    if (tid == 0) {
        int pk = scan.key[0];
        double pv = scan.val[0];
        scan.pkey[0] = pk; scan.pval[0] = pv;
        for (int w = 1; w < WO_NT / kWarp; ++w) {
            const int k2 = scan.key[w];
            pv = (k2 == pk) ? pv + scan.val[w] : scan.val[w];
            pk = k2;
            scan.pkey[w] = pk; scan.pval[w] = pv;
        }
    }
    __syncthreads();
    if (warp > 0 && scan.pkey[warp - 1] == key) val += scan.pval[warp - 1];
    // carry into this thread = inclusive value of the previous thread
    double carry_in = shfl_up(val, 1);
    if (lane == 0) carry_in = (warp > 0) ? scan.pval[warp - 1] : 0.0;
    if (done_any) y[t0 + i_first] = (ValT)(head + carry_in);

    if (tid == WO_NT - 1) {
        // the CTA's trailing partial belongs to row t1 (if that row has atoms here)
        const bool tail = (t1 < A.rows) && n_atoms > 0 &&
                          (n_rows == 0 || s_end[n_rows - 1] < n_atoms);
        carry_tile[c] = tail ? t1 : -1;
        carry_val[c] = tail ? val : 0.0;
    }
}

// ---- 2b. direct per-lane SpMV (large item counts) ------------------------------
template <class OffT, class ValT, bool PROBE>
__global__ void __launch_bounds__(256)
    k_wo_direct(Csr<OffT, ValT> A, const ValT* __restrict__ x, ValT* __restrict__ y,
                int64_t lanes, int64_t items, const int64_t* __restrict__ lane_tile,
                int64_t* __restrict__ carry_tile, double* __restrict__ carry_val,
                Probe probe) {
    const int64_t l = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (l >= lanes) return;
    const int64_t total = A.rows + A.nnz;
    int64_t t = lane_tile[l];
    int64_t a = min(l * items, total) - t;
    const int64_t t_end = lane_tile[l + 1];
    const int64_t a_end = min((l + 1) * items, total) - t_end;
    const int64_t a_begin = a;
    double acc = 0.0;
    for (; t < t_end; ++t) {
        const int64_t re = ld_off(A.off + t + 1);
        for (; a < re; ++a) {
            acc = fma((double)__ldg(A.val + a), (double)ld_gather(x + __ldg(A.col + a)), acc);
            if (PROBE) probe_atom(probe, a, l, t);
        }
        y[t] = (ValT)acc;
        acc = 0.0;
    }
    const bool tail = a < a_end;
    for (; a < a_end; ++a) {
        acc = fma((double)__ldg(A.val + a), (double)ld_gather(x + __ldg(A.col + a)), acc);
        if (PROBE) probe_atom(probe, a, l, t_end);
    }
    carry_tile[l] = tail ? t_end : -1;
    carry_val[l] = acc;
    if (PROBE && probe.lane_atoms) probe.lane_atoms[l] = a_end - a_begin;
}

// ---- 3. ordered carry fix-up -----------------------------------------------------
template <class ValT>
__global__ void k_carry_fixup(const int64_t* __restrict__ carry_tile,
                              const double* __restrict__ carry_val, int64_t n,
                              ValT* __restrict__ y, int64_t rows) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    const int64_t r = carry_tile[k];
    if (r < 0 || r >= rows) return;
    if (k > 0 && carry_tile[k - 1] == r) return;   // not the head of its run
    double s = 0.0;
    for (int64_t m = k; m < n && carry_tile[m] == r; ++m) s += carry_val[m];
    y[r] = (ValT)((double)y[r] + s);
}

// ---- host side -------------------------------------------------------------------
struct WoPlan {
    int64_t total, lanes, items;
    int ipt;          // 8, 16 = staged variant; 0 = direct
    int64_t n_units;  // CTAs (staged) or lanes (direct): carry slots
};

static WoPlan wo_plan(int64_t rows, int64_t nnz, int64_t lanes) {
    WoPlan p{};
    p.total = rows + nnz;
    if (lanes <= 0) lanes = p.total > 0 ? ceil_div(p.total, WO_IPT_AUTO) : 1;
    p.lanes = lanes;
    p.items = p.total > 0 ? ceil_div(p.total, lanes) : 0;
    if (p.items <= 8) p.ipt = 8;
    else if (p.items <= 16) p.ipt = 16;
    else p.ipt = 0;
    p.n_units = p.ipt ? ceil_div(lanes, WO_NT) : lanes;
    return p;
}

static size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

size_t wo_workspace(int64_t rows, int64_t nnz, int64_t lanes) {
    const WoPlan p = wo_plan(rows, nnz, lanes);
    const size_t n = (size_t)p.n_units;
    return align_up((n + 1) * 8, 256) + align_up(n * 8, 256) + align_up(n * 8, 256);
}

template <class OffT>
static int launch_search(const OffT* off, int64_t rows, int64_t nnz, int64_t n_bounds,
                         int64_t span, int64_t* out_tile, int64_t* out_coords,
                         cudaStream_t s) {
    const int NT = 256;
    k_merge_path_search<OffT><<<ceil_div(n_bounds, NT), NT, 0, s>>>(off, rows, nnz, n_bounds, span,
                                                                 out_tile, out_coords);
    LW_LAUNCH_CHECK();
    return LW_OK;
}

int merge_path_partition(int64_t rows, int64_t nnz, const void* off, int bits, int64_t lanes,
                         int64_t* coords, cudaStream_t s) {
    if (lanes < 1 || rows < 0 || nnz < 0 || !coords || (!off && rows > 0)) return LW_E_INVALID_ARG;
    const int64_t total = rows + nnz;
    const int64_t items = total > 0 ? ceil_div(total, lanes) : 0;
    if (bits == 32)
        return launch_search<int32_t>((const int32_t*)off, rows, nnz, lanes + 1, items, nullptr, coords, s);
    return launch_search<int64_t>((const int64_t*)off, rows, nnz, lanes + 1, items, nullptr, coords, s);
}

template <class OffT, class ValT>
static int launch_wo(const lw_csr_t* A, const void* x, void* y, const WoPlan& p, void* ws,
                     const lw_probe_t* probe, unsigned phases, cudaStream_t s) {
    Csr<OffT, ValT> a{A->rows, A->cols, A->nnz, (const OffT*)A->row_offsets,
                      A->col_indices, (const ValT*)A->values};
    const size_t n = (size_t)p.n_units;
    unsigned char* w = (unsigned char*)ws;
    int64_t* tiles = (int64_t*)w;
    int64_t* c_tile = (int64_t*)(w + align_up((n + 1) * 8, 256));
    double* c_val = (double*)(w + align_up((n + 1) * 8, 256) + align_up(n * 8, 256));
    Probe pr{};
    if (probe) pr = Probe{probe->lane_atoms, probe->atom_lane, probe->atom_tile, probe->atom_visits};
    if (n > 0x7fffffff) return LW_E_UNSUPPORTED;

    if (phases & WO_PHASE_PARTITION) {
        // CTA boundaries (staged) or lane boundaries (direct)
        const int64_t span = p.ipt ? (int64_t)WO_NT * p.items : p.items;
        int rc = launch_search<OffT>(a.off, a.rows, a.nnz, n + 1, span, tiles, nullptr, s);
        if (rc) return rc;
    }
    if (phases & WO_PHASE_SPMV) {
        if (probe && pr.lane_atoms) LW_TRY(cudaMemsetAsync(pr.lane_atoms, 0, p.lanes * 8, s));
        if (p.ipt) {
            const size_t smem = (size_t)WO_NT * p.ipt * (sizeof(double) + sizeof(int32_t));
#define LW_WO_LAUNCH(IPT, PR)                                                                  \
    do {                                                                                       \
        auto kern = k_wo_staged<OffT, ValT, IPT, PR>;                                          \
        static bool attr_set = false;                                                          \
        if (!attr_set && smem > 48 * 1024) {                                                   \
            LW_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,     \
                                        (int)(WO_NT * IPT * 12)));                            \
            attr_set = true;                                                                   \
        }                                                                                      \
        kern<<<(unsigned)n, WO_NT, smem, s>>>(a, (const ValT*)x, (ValT*)y, p.lanes, p.items, tiles, \
                                            c_tile, c_val, pr);                                \
    } while (0)
            if (p.ipt == 8) { if (probe) LW_WO_LAUNCH(8, true); else LW_WO_LAUNCH(8, false); }
            else            { if (probe) LW_WO_LAUNCH(16, true); else LW_WO_LAUNCH(16, false); }
#undef LW_WO_LAUNCH
        } else {
            const int NT = 256;
            if (probe)
                k_wo_direct<OffT, ValT, true><<<ceil_div(n, NT), NT, 0, s>>>(a, (const ValT*)x, (ValT*)y, p.lanes, p.items, tiles, c_tile, c_val, pr);
            else
                k_wo_direct<OffT, ValT, false><<<ceil_div(n, NT), NT, 0, s>>>(a, (const ValT*)x, (ValT*)y, p.lanes, p.items, tiles, c_tile, c_val, pr);
        }
        LW_LAUNCH_CHECK();
    }
    if (phases & WO_PHASE_FIXUP) {
        k_carry_fixup<ValT><<<ceil_div(n, 256), 256, 0, s>>>(c_tile, c_val, (int64_t)n, (ValT*)y, a.rows);
        LW_LAUNCH_CHECK();
    }
    return LW_OK;
}

int spmv_work_oriented(const lw_csr_t* A, const void* x, void* y, int64_t lanes, void* ws,
                       size_t ws_bytes, const lw_probe_t* probe, unsigned phases,
                       cudaStream_t s) {
    const WoPlan p = wo_plan(A->rows, A->nnz, lanes);
    if (A->rows == 0) return LW_OK;
    if (!ws || ws_bytes < wo_workspace(A->rows, A->nnz, lanes)) return LW_E_WORKSPACE;
    const bool o32 = A->offset_bits == 32;
    if (A->dtype == LW_F32)
        return o32 ? launch_wo<int32_t, float>(A, x, y, p, ws, probe, phases, s)
                   : launch_wo<int64_t, float>(A, x, y, p, ws, probe, phases, s);
    return o32 ? launch_wo<int32_t, double>(A, x, y, p, ws, probe, phases, s)
               : launch_wo<int64_t, double>(A, x, y, p, ws, probe, phases, s);
}

int64_t wo_lanes(int64_t rows, int64_t nnz, int64_t lanes) { return wo_plan(rows, nnz, lanes).lanes; }

}  // namespace lw
