/*
 * smlm_oracle.c -- plain, slow, obviously-correct fp64 CPU oracle for SMLM.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg may load this library.  The product path
 * (paper_2511_00101_b200/) never links, imports or calls it, and shares no code with it.
 *
 * What it computes (the plain definition of Segmented Multi-LoRA Multiplication):
 *   PAPER.md P:379-384 (§3.3 "Unified computation flow management and SMLM kernel"):
 *     one call computes every row's LoRA-augmented projection with a per-segment adapter,
 *     LoRA weights processed "one linear layer at a time", static scaling or a dynamic
 *     per-request scale, four request kinds (fine-tune, eval, prefill, decode).
 *   PAPER.md P:415-422 (§3.3): fine-tune rows get gradients; each trainer updates only its
 *     own adapter (masking); one shared backward over all fine-tune jobs.
 *   Layout/notation: SURVEY.md §8 "Math and layout" (nn.Linear / PEFT convention):
 *     X [S,in], W [out,in], A_a [r,in], B_a [out,r], Y [S,out].
 *
 * For a row t in segment g, adapter a = slot[g], s = slot_scale[a] * seg_scale[g]:
 *     v      = A_a x_t                              (rank-r intermediate)
 *     y_t    = W x_t + s B_a v                      (a = -1: y_t = W x_t)
 *   fine-tune rows only (backward):
 *     u      = B_a^T dy_t
 *     dx_t   = W^T dy_t + s A_a^T u
 *     dA_a  += s u x_t^T ,   dB_a += s dy_t v^T     (only for adapters that have grads)
 *
 * LoRA dropout (f2; App. D Table 5 "lora_dropout 0.05"; reading R13):
 * with the PEFT LoRA definition y = W x + s B A dropout(x), dropout acting in training mode only,
 * i.e. on FINETUNE rows.  The mask is an INPUT here (keep [S,in], 1 = kept, NULL = no dropout):
 *     x~_t   = keep_t * x_t * keep_scale            (keep_scale = 1/(1-p), inverted dropout)
 *     v      = A_a x~_t ,   y_t = W x_t + s B_a v
 *     dx_t   = W^T dy_t + s keep_t * keep_scale * (A_a^T u)
 *     dA_a  += s u x~_t^T ,  dB_a += s dy_t v^T
 * for fine-tune rows with an adapter; every other row is unchanged.
 *
 * Every sum is a straight loop in ascending index order with an fp64 accumulator.
 * No blocking, no fusion, no reordering.  OpenMP only splits independent rows/entries.
 */
#include <stdlib.h>
#include <string.h>

#define SMLM_FINETUNE 0

/* row -> segment map; returns 0 on success, nonzero on malformed offsets */
static int row_segments(int S, int G, const int *off, int *seg_of_row)
{
    if (off[0] != 0 || off[G] != S) return 1;
    for (int g = 0; g < G; ++g) {
        if (off[g + 1] < off[g]) return 1;
        for (int t = off[g]; t < off[g + 1]; ++t) seg_of_row[t] = g;
    }
    return 0;
}

static double eff_scale(int g, int a, const double *slot_scale, const double *seg_scale)
{
    double s = (a >= 0) ? slot_scale[a] : 0.0;
    if (seg_scale) s *= seg_scale[g];
    return s;
}

/*
 * Forward over the selected rows (rows == NULL: all S rows).
 * W == NULL: Y holds the base output on entry and the LoRA term is added in place.
 * Vsave (optional): v for fine-tune rows with an adapter.
 */
int oracle_forward(int S, int in_f, int out_f, int r, int G,
                   const int *off, const int *slot, const signed char *mode,
                   const double *seg_scale, const double *slot_scale,
                   const double *A, const double *B,
                   const double *X, const double *W, double *Y, double *Vsave,
                   int n_rows, const long *rows, const unsigned char *keep, double keep_scale)
{
    int *seg = (int *)malloc(sizeof(int) * (S > 0 ? S : 1));
    if (row_segments(S, G, off, seg)) { free(seg); return 1; }
    int n = rows ? n_rows : S;
#pragma omp parallel for schedule(dynamic, 4)
    for (int i = 0; i < n; ++i) {
        long t = rows ? rows[i] : i;
        int g = seg[t];
        int a = slot[g];
        double s = eff_scale(g, a, slot_scale, seg_scale);
        const double *x = X + (size_t)t * in_f;
        const unsigned char *kp = (keep && mode[g] == SMLM_FINETUNE) ? keep + (size_t)t * in_f : NULL;
        double v[256];
        if (a >= 0) {
            const double *Aa = A + (size_t)a * r * in_f;
            for (int j = 0; j < r; ++j) {
                double acc = 0.0;
                for (int k = 0; k < in_f; ++k) {
                    double xk = kp ? (kp[k] ? x[k] * keep_scale : 0.0) : x[k];   /* dropout(x) */
                    acc += Aa[(size_t)j * in_f + k] * xk;
                }
                v[j] = acc;
            }
        }
        for (int o = 0; o < out_f; ++o) {
            double base;
            if (W) {
                base = 0.0;
                for (int k = 0; k < in_f; ++k) base += W[(size_t)o * in_f + k] * x[k];
            } else {
                base = Y[(size_t)t * out_f + o];
            }
            double lora = 0.0;
            if (a >= 0) {
                const double *Ba = B + (size_t)a * out_f * r;
                for (int j = 0; j < r; ++j) lora += Ba[(size_t)o * r + j] * v[j];
            }
            Y[(size_t)t * out_f + o] = base + s * lora;
        }
        if (Vsave && a >= 0 && mode[g] == SMLM_FINETUNE)
            for (int j = 0; j < r; ++j) Vsave[(size_t)t * r + j] = v[j];
    }
    free(seg);
    return 0;
}

/*
 * Backward for fine-tune rows.
 *   dX (optional): written for the selected fine-tune rows (rows == NULL: all rows; non
 *   fine-tune rows are skipped and left untouched).  W == NULL omits the base term.
 *   dA [n_slots,r,in], dB [n_slots,out,r]: for every slot a with has_grad[a] != 0 that owns
 *   at least one fine-tune row, dA_a/dB_a are set (accumulate == 0) or incremented
 *   (accumulate != 0) with the sum over ALL of a's fine-tune rows (never sampled).
 *   Slots with no fine-tune rows in this batch are untouched.
 */
int oracle_backward(int S, int in_f, int out_f, int r, int G,
                    const int *off, const int *slot, const signed char *mode,
                    const double *seg_scale, int n_slots, const double *slot_scale,
                    const double *A, const double *B, const double *X, const double *W,
                    const double *dY, double *dX, double *dA, double *dB,
                    const int *has_grad, int accumulate, int n_rows, const long *rows,
                    const unsigned char *keep, double keep_scale)
{
    int *seg = (int *)malloc(sizeof(int) * (S > 0 ? S : 1));
    if (row_segments(S, G, off, seg)) { free(seg); return 1; }

    /* ---- dX over the selected fine-tune rows ---- */
    if (dX) {
        int n = rows ? n_rows : S;
#pragma omp parallel for schedule(dynamic, 4)
        for (int i = 0; i < n; ++i) {
            long t = rows ? rows[i] : i;
            int g = seg[t];
            if (mode[g] != SMLM_FINETUNE) continue;
            int a = slot[g];
            double s = eff_scale(g, a, slot_scale, seg_scale);
            const double *dy = dY + (size_t)t * out_f;
            double u[256];
            if (a >= 0) {
                const double *Ba = B + (size_t)a * out_f * r;
                for (int j = 0; j < r; ++j) {
                    double acc = 0.0;
                    for (int o = 0; o < out_f; ++o) acc += dy[o] * Ba[(size_t)o * r + j];
                    u[j] = acc;
                }
            }
            for (int k = 0; k < in_f; ++k) {
                double base = 0.0;
                if (W)
                    for (int o = 0; o < out_f; ++o) base += dy[o] * W[(size_t)o * in_f + k];
                double lora = 0.0;
                if (a >= 0) {
                    const double *Aa = A + (size_t)a * r * in_f;
                    for (int j = 0; j < r; ++j) lora += u[j] * Aa[(size_t)j * in_f + k];
                    if (keep) lora *= keep[(size_t)t * in_f + k] ? keep_scale : 0.0;   /* d dropout(x) / dx */
                }
                dX[(size_t)t * in_f + k] = base + s * lora;
            }
        }
    }

    /* ---- dA / dB per adapter, full sum over that adapter's fine-tune rows ---- */
    if (dA || dB) {
        long *trows = (long *)malloc(sizeof(long) * (S > 0 ? S : 1));
        double *U = (double *)malloc(sizeof(double) * (size_t)(S > 0 ? S : 1) * r);
        double *V = (double *)malloc(sizeof(double) * (size_t)(S > 0 ? S : 1) * r);
        double *sc = (double *)malloc(sizeof(double) * (S > 0 ? S : 1));
        for (int a = 0; a < n_slots; ++a) {
            if (!has_grad || !has_grad[a]) continue;
            int T = 0;
            for (int t = 0; t < S; ++t) {
                int g = seg[t];
                if (mode[g] == SMLM_FINETUNE && slot[g] == a) {
                    trows[T] = t;
                    sc[T] = eff_scale(g, a, slot_scale, seg_scale);
                    ++T;
                }
            }
            if (T == 0) continue; /* untouched */
            const double *Aa = A + (size_t)a * r * in_f;
            const double *Ba = B + (size_t)a * out_f * r;
#pragma omp parallel for schedule(static)
            for (int i = 0; i < T; ++i) {
                const double *x = X + (size_t)trows[i] * in_f;
                const double *dy = dY + (size_t)trows[i] * out_f;
                const unsigned char *kp = keep ? keep + (size_t)trows[i] * in_f : NULL;
                for (int j = 0; j < r; ++j) {
                    double uv = 0.0, vv = 0.0;
                    for (int o = 0; o < out_f; ++o) uv += dy[o] * Ba[(size_t)o * r + j];
                    for (int k = 0; k < in_f; ++k)
                        vv += Aa[(size_t)j * in_f + k] * (kp ? (kp[k] ? x[k] * keep_scale : 0.0) : x[k]);
                    U[(size_t)i * r + j] = uv;
                    V[(size_t)i * r + j] = vv;
                }
            }
            if (dA) {
                double *dAa = dA + (size_t)a * r * in_f;
#pragma omp parallel for schedule(static)
                for (long e = 0; e < (long)r * in_f; ++e) {
                    int j = (int)(e / in_f), k = (int)(e % in_f);
                    double acc = 0.0;
                    for (int i = 0; i < T; ++i) {
                        double xk = X[(size_t)trows[i] * in_f + k];
                        if (keep) xk = keep[(size_t)trows[i] * in_f + k] ? xk * keep_scale : 0.0;   /* x~ */
                        acc += sc[i] * U[(size_t)i * r + j] * xk;
                    }
                    dAa[e] = accumulate ? dAa[e] + acc : acc;
                }
            }
            if (dB) {
                double *dBa = dB + (size_t)a * out_f * r;
#pragma omp parallel for schedule(static)
                for (long e = 0; e < (long)out_f * r; ++e) {
                    int o = (int)(e / r), j = (int)(e % r);
                    double acc = 0.0;
                    for (int i = 0; i < T; ++i)
                        acc += sc[i] * dY[(size_t)trows[i] * out_f + o] * V[(size_t)i * r + j];
                    dBa[e] = accumulate ? dBa[e] + acc : acc;
                }
            }
        }
        free(trows); free(U); free(V); free(sc);
    }
    free(seg);
    return 0;
}

int oracle_num_threads(void)
{
#ifdef _OPENMP
    extern int omp_get_max_threads(void);
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* Thread count of the row-parallel loops (bench.py times the oracle at 1 thread and at all host
 * cores); n <= 0 restores the OpenMP default.  No effect on results (rows are independent and
 * every sum runs in a fixed order inside one thread). */
void oracle_set_num_threads(int n)
{
#ifdef _OPENMP
    extern void omp_set_num_threads(int);
    extern int omp_get_num_procs(void);
    omp_set_num_threads(n > 0 ? n : omp_get_num_procs());
#else
    (void)n;
#endif
}
