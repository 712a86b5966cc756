/*
 * amtc_oracle.c -- CPU ORACLE.  TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  The product path
 * (paper_1110_2477_b200/) never links, imports or calls it, and shares no code,
 * header, table or constant with it.
 *
 * What it computes (citations: P:n = /root/reference/PAPER.md line n):
 *
 *   - The ask and bid prices of an American option under proportional
 *     transaction costs k, by the Roux-Zastawniak seller/buyer recursions over
 *     piecewise-linear (PWL) functions of the share holding y, exactly in the
 *     order of Sec. 3 on the recombining CRR tree of Sec. 4.1,
 *     including the extra time instant t = N+1 with payoff (0,0) (P:159,
 *     Alg. 1 lines 2-5 at P:219-227) and no costs at t = 0.
 *   - The frictionless CRR American / European price by scalar backward
 *     induction (Appendix), no extra level.
 *   - The European CRR price as the closed-form binomial sum (textbook; used
 *     only as an independent pin of the scalar induction).
 *
 * Style: plain and slow on purpose.  Every PWL operation allocates its result;
 * there is no blocking, fusion or reordering beyond what the definitions state.
 * Floating point is IEEE fp64; build with -O2 -ffp-contract=off (no FMA
 * contraction, no fast-math).
 *
 * PWL representation (oracle only): a continuous PWL function f on the real
 * line is given by n >= 1 vertices (x[i], f[i]) with x strictly increasing,
 * linear interpolation between vertices, and two tail slopes sl (left of x[0])
 * and sr (right of x[n-1]).  A line is one anchor vertex with sl == sr.
 *
 * Readings of the paper taken here (listed in DESIGN.md "Readings"):
 *   R7  slope restriction of a possibly non-convex f to [lo, hi] is the
 *       infimal convolution v(y) = inf_y' [ f(y') + c(y - y') ] with the
 *       rebalancing cost c(d) = lo*d (d <= 0, buy at ask -lo) and hi*d (d >= 0,
 *       sell at bid -hi); computed as min(A, B), A = "buy" branch (y' >= y),
 *       B = "sell" branch (y' <= y).  For convex f it is slope clipping, as in
 *       the P:118 example.
 *   R9  the buyer's w is the max of the children ("similar").
 *   R6  payoffs: put (K,-1) physical; call (-K,+1) physical;
 *       bull spread cash ((S-K1)^+ - (S-K2)^+, 0).
 *   R8  bid = -z'_0(0) where z' is the buyer's function.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define OR_OK 0
#define OR_EINVAL 1
#define OR_EARBITRAGE 2
#define OR_EUNBOUNDED 4
#define OR_ENOMEM 7

#define OR_PUT 0
#define OR_CALL 1
#define OR_BULL 2


/* ------------------------------------------------------------------------- */
/* PWL functions                                                              */
/* ------------------------------------------------------------------------- */

typedef struct {
    int n;     /* number of vertices, >= 1 */
    int cap;
    double *x; /* abscissae, strictly increasing */
    double *f; /* values at the vertices */
    double sl; /* slope on (-inf, x[0]) */
    double sr; /* slope on (x[n-1], +inf) */
} pwl;

/*
 * Operation counters (instrumentation only; never part of any result).
 * The SURVEY 8(d) cost model of "algorithmic FP64 ops" is applied to them in
 * oracle_price_tc_stats():
 *   merge visit (one candidate abscissa of max/min: evaluate the other
 *                function there and compare)                      = 3
 *   crossing    (2 DADD + 1 DDIV + 1 DFMA)                           = 4
 *   restriction visit (one vertex of f = w/r in one scan pass):
 *                2 when f is convex (clip compares), 4 when not      = 2 | 4
 *   scaling by 1/r, per vertex of w                                  = 2
 *   max/min with the expense function u                              = as merge
 * The counts follow the DEFINITION of each step (union of both vertex sets
 * for an envelope, one visit per vertex per scan pass), not the oracle's
 * allocation pattern; the min(A, B) that closes the restriction is part of
 * the restriction's definition (its candidates are not merge visits; its
 * crossings are crossings).
 */
typedef struct {
    int64_t vertices_out;    /* sum of output vertex counts of every z */
    int64_t crossings;       /* crossing points solved (one division each) */
    int64_t merge_visits;    /* candidate abscissae of max(z^u,z^d) and of max/min(u,v) */
    int64_t restrict_cvx;    /* restriction scan steps on a convex f */
    int64_t restrict_ncvx;   /* restriction scan steps on a non-convex f */
    int64_t scale_visits;    /* vertices of w scaled by 1/r */
    int in_restrict;         /* set while min(A,B) of a restriction runs */
} counters;

static int pwl_init(pwl *p, int cap)
{
    if (cap < 1) cap = 1;
    p->n = 0;
    p->cap = cap;
    p->x = (double *)malloc(sizeof(double) * (size_t)cap);
    p->f = (double *)malloc(sizeof(double) * (size_t)cap);
    p->sl = p->sr = 0.0;
    return (p->x && p->f) ? OR_OK : OR_ENOMEM;
}

static void pwl_free(pwl *p)
{
    free(p->x);
    free(p->f);
    p->x = p->f = NULL;
    p->n = p->cap = 0;
}

static void pwl_push(pwl *p, double x, double f)
{
    /* callers size cap generously; grow if not */
    if (p->n == p->cap) {
        p->cap *= 2;
        p->x = (double *)realloc(p->x, sizeof(double) * (size_t)p->cap);
        p->f = (double *)realloc(p->f, sizeof(double) * (size_t)p->cap);
    }
    p->x[p->n] = x;
    p->f[p->n] = f;
    p->n++;
}

/* slope of the piece between vertices i and i+1 */
static double pwl_piece_slope(const pwl *p, int i)
{
    return (p->f[i + 1] - p->f[i]) / (p->x[i + 1] - p->x[i]);
}

/* f(y) */
static double pwl_eval(const pwl *p, double y)
{
    int n = p->n;
    if (y <= p->x[0]) return p->f[0] + p->sl * (y - p->x[0]);
    if (y >= p->x[n - 1]) return p->f[n - 1] + p->sr * (y - p->x[n - 1]);
    /* find the piece [x_i, x_{i+1}] containing y by bisection */
    int i = 0, hi = n - 1; /* invariant: x[i] < y <= x[hi] */
    while (hi - i > 1) {
        int mid = (i + hi) / 2;
        if (p->x[mid] < y) i = mid;
        else hi = mid;
    }
    double t = (y - p->x[i]) / (p->x[i + 1] - p->x[i]);
    return p->f[i] + t * (p->f[i + 1] - p->f[i]);
}

/*
 * Canonical form (reading R10, SPEC "canonicalize"): drop every vertex that is
 * not a kink.  "Not a kink" is decided on VALUES, not on difference-quotient
 * slopes (which are noisy on short pieces): vertex i is dropped when it, and
 * the first vertex of the run of dropped vertices before it, lie within
 * CANON_ATOL * max(1, max|f|) of the chord that replaces them -- the segment
 * from the last kept vertex to vertex i+1, or, at either end, the tail line
 * (whose slope is kept) through the kept neighbour.
 * The function keeps at least one vertex (a line is one anchor vertex).
 */
#define CANON_ATOL 1e-14

/* value at x of the chord replacing the vertices strictly between a and b;
   a = -1 means the left tail (slope sl through vertex b), b = n the right
   tail (slope sr through vertex a) */
static double chord_at(const pwl *p, int a, int b, double x)
{
    if (a < 0) return p->f[b] + p->sl * (x - p->x[b]);
    if (b >= p->n) return p->f[a] + p->sr * (x - p->x[a]);
    double t = (x - p->x[a]) / (p->x[b] - p->x[a]);
    return p->f[a] + t * (p->f[b] - p->f[a]);
}

static void pwl_canonicalize(pwl *p)
{
    int n = p->n;
    if (n <= 1) return;
    double fmaxabs = 1.0;
    for (int i = 0; i < n; i++) fmaxabs = fmax(fmaxabs, fabs(p->f[i]));
    double tol = CANON_ATOL * fmaxabs;
    int *keep = (int *)malloc(sizeof(int) * (size_t)n);
    int prev = -1; /* last kept vertex, -1 = left tail */
    for (int i = 0; i < n; i++) {
        int next = i + 1; /* == n means the right tail */
        int droppable = 1;
        if (prev < 0 && next >= n) {
            /* dropping the last remaining vertex: only a line may do that,
               and a line keeps its anchor anyway */
            droppable = 0;
        } else {
            /* vertex i and the first vertex of the current run of dropped
               vertices must both lie on the replacing chord (O(1) per vertex) */
            if (fabs(p->f[i] - chord_at(p, prev, next, p->x[i])) > tol) droppable = 0;
            if (prev + 1 < i && fabs(p->f[prev + 1] - chord_at(p, prev, next, p->x[prev + 1])) > tol)
                droppable = 0;
        }
        keep[i] = !droppable;
        if (keep[i]) prev = i;
    }
    int m = 0;
    for (int i = 0; i < n; i++) {
        if (!keep[i]) continue;
        p->x[m] = p->x[i];
        p->f[m] = p->f[i];
        m++;
    }
    free(keep);
    p->n = m;
}

/* the number of kinks (breakpoints) of a canonical function */
static int pwl_kinks(const pwl *p)
{
    if (p->n == 1 && p->sl == p->sr) return 0;
    return p->n;
}

/* c * f, c > 0 ("discounted by r" uses c = 1/r, done as f / r below) */
static int pwl_div(const pwl *p, double r, pwl *out)
{
    if (pwl_init(out, p->n) != OR_OK) return OR_ENOMEM;
    for (int i = 0; i < p->n; i++) pwl_push(out, p->x[i], p->f[i] / r);
    out->sl = p->sl / r;
    out->sr = p->sr / r;
    return OR_OK;
}

/*
 * Pointwise max (want_max = 1) or min (want_max = 0) of f and g
 * (P:118 w = max(z^u, z^d); P:119 z = max(u, v); P:142 z = min(u, v)).
 * Candidate abscissae are the union of both vertex sets; between two
 * consecutive candidates, and on the two tails, both functions are affine, so
 * the difference d = f - g changes sign at most once there; each sign change
 * is a crossing vertex.
 */
static int pwl_envelope(const pwl *f, const pwl *g, int want_max, pwl *out, counters *cnt)
{
    int nc = 0;
    double *X = (double *)malloc(sizeof(double) * (size_t)(f->n + g->n));
    if (!X) return OR_ENOMEM;
    {   /* sorted union */
        int i = 0, j = 0;
        while (i < f->n || j < g->n) {
            double c;
            if (j >= g->n || (i < f->n && f->x[i] < g->x[j])) c = f->x[i++];
            else if (i >= f->n || g->x[j] < f->x[i]) c = g->x[j++];
            else { c = f->x[i]; i++; j++; }
            X[nc++] = c;
        }
    }
    if (pwl_init(out, 2 * nc + 2) != OR_OK) { free(X); return OR_ENOMEM; }
    if (cnt && !cnt->in_restrict) cnt->merge_visits += nc;

    double *D = (double *)calloc((size_t)nc, sizeof(double));
    double *F = (double *)malloc(sizeof(double) * (size_t)nc);
    double *G = (double *)malloc(sizeof(double) * (size_t)nc);
    for (int i = 0; i < nc; i++) {
        F[i] = pwl_eval(f, X[i]);
        G[i] = pwl_eval(g, X[i]);
        D[i] = F[i] - G[i];
    }
#define PICK(a, b) (want_max ? fmax((a), (b)) : fmin((a), (b)))
    /* left tail: d(y) = D0 + (f.sl - g.sl)(y - X0) for y <= X0 */
    {
        double ds = f->sl - g->sl;
        if (ds != 0.0 && D[0] != 0.0 && ((D[0] > 0.0) == (ds > 0.0))) {
            double yc = X[0] - D[0] / ds;
            pwl_push(out, yc, pwl_eval(f, yc));
            if (cnt) cnt->crossings++;
        }
    }
    for (int i = 0; i < nc; i++) {
        pwl_push(out, X[i], PICK(F[i], G[i]));
        if (i + 1 < nc && ((D[i] > 0.0 && D[i + 1] < 0.0) || (D[i] < 0.0 && D[i + 1] > 0.0))) {
            double yc = X[i] + (X[i + 1] - X[i]) * (D[i] / (D[i] - D[i + 1]));
            pwl_push(out, yc, pwl_eval(f, yc));
            if (cnt) cnt->crossings++;
        }
    }
    /* right tail: d(y) = Dn + (f.sr - g.sr)(y - Xn) for y >= Xn */
    {
        double ds = f->sr - g->sr;
        double Dn = D[nc - 1];
        if (ds != 0.0 && Dn != 0.0 && ((Dn > 0.0) != (ds > 0.0))) {
            double yc = X[nc - 1] - Dn / ds;
            pwl_push(out, yc, pwl_eval(f, yc));
            if (cnt) cnt->crossings++;
        }
    }
#undef PICK
    /* tails: the max is eventually the steeper-from-the-left / steeper-to-the-right line */
    if (want_max) {
        out->sl = fmin(f->sl, g->sl);
        out->sr = fmax(f->sr, g->sr);
    } else {
        out->sl = fmax(f->sl, g->sl);
        out->sr = fmin(f->sr, g->sr);
    }
    free(X); free(D); free(F); free(G);
    pwl_canonicalize(out);
    return OR_OK;
}

/* f~(t) = f(-t) */
static int pwl_reflect(const pwl *p, pwl *out)
{
    if (pwl_init(out, p->n) != OR_OK) return OR_ENOMEM;
    for (int i = p->n - 1; i >= 0; i--) pwl_push(out, -p->x[i], p->f[i]);
    out->sl = -p->sr;
    out->sr = -p->sl;
    return OR_OK;
}

/* f(y) + a*y */
static int pwl_add_linear(const pwl *p, double a, pwl *out)
{
    if (pwl_init(out, p->n) != OR_OK) return OR_ENOMEM;
    for (int i = 0; i < p->n; i++) pwl_push(out, p->x[i], p->f[i] + a * p->x[i]);
    out->sl = p->sl + a;
    out->sr = p->sr + a;
    return OR_OK;
}

/*
 * G(y) = inf_{y' >= y} g(y')   (suffix infimum).
 * Finite iff g's right tail slope >= 0 (otherwise g -> -inf).
 * On each piece, walked right to left with m = G(right end):
 *   slope < 0  -> G = m on the piece;
 *   slope >= 0 -> G = min(g, m), with one crossing if g(left) < m < g(right).
 */
static int pwl_suffix_inf(const pwl *g, pwl *out, counters *cnt)
{
    int n = g->n;
    if (!(g->sr >= 0.0)) return OR_EUNBOUNDED;
    pwl rev; /* vertices collected right-to-left */
    if (pwl_init(&rev, 2 * n + 2) != OR_OK) return OR_ENOMEM;
    double m = g->f[n - 1];
    pwl_push(&rev, g->x[n - 1], m);
    for (int i = n - 2; i >= 0; i--) {
        double s = pwl_piece_slope(g, i);
        if (s < 0.0) {
            pwl_push(&rev, g->x[i], m);
        } else {
            if (g->f[i] < m && m < g->f[i + 1]) {
                double yc = g->x[i] + (m - g->f[i]) / s;
                pwl_push(&rev, yc, m);
                if (cnt) cnt->crossings++;
            }
            m = fmin(g->f[i], m);
            pwl_push(&rev, g->x[i], m);
        }
    }
    /* left tail */
    double sl_out;
    if (g->sl > 0.0) {
        if (g->f[0] > m) { /* g(y) falls below m left of x0 */
            double yc = g->x[0] - (g->f[0] - m) / g->sl;
            pwl_push(&rev, yc, m);
            if (cnt) cnt->crossings++;
        }
        sl_out = g->sl;
    } else {
        sl_out = 0.0; /* g is non-increasing to the right on the tail: G = m */
    }
    if (pwl_init(out, rev.n) != OR_OK) { pwl_free(&rev); return OR_ENOMEM; }
    for (int i = rev.n - 1; i >= 0; i--) pwl_push(out, rev.x[i], rev.f[i]);
    out->sl = sl_out;
    out->sr = g->sr;
    pwl_free(&rev);
    pwl_canonicalize(out);
    return OR_OK;
}

/*
 * Slope restriction ("the slopes of this discounted function w_t/r must
 * be restricted within the interval [-S^a_t, -S^b_t]"), reading R7:
 *   v(y) = inf_{y'} [ f(y') + c(y - y') ],  c(d) = lo*d (d<=0), hi*d (d>=0)
 *        = min( A(y), B(y) ),
 *   A(y) = inf_{y' >= y} [ f(y') - lo*y' ] + lo*y     (buy y'-y shares at -lo)
 *   B(y) = inf_{y' <= y} [ f(y') - hi*y' ] + hi*y     (sell y-y' shares at -hi)
 * B is computed as the reflection of a suffix infimum.
 */
/* f is convex iff its slopes (tails included) are non-decreasing */
static int pwl_is_convex(const pwl *p)
{
    double prev = p->sl;
    for (int i = 0; i + 1 < p->n; i++) {
        double s = pwl_piece_slope(p, i);
        if (s < prev) return 0;
        prev = s;
    }
    return p->sr >= prev;
}

static int pwl_restrict(const pwl *f, double lo, double hi, pwl *out, counters *cnt)
{
    int st;
    pwl g, G, A, h, hr, Hr, H, B;
    if (cnt) { /* two scan passes over the vertices of f (cost model above) */
        if (pwl_is_convex(f)) cnt->restrict_cvx += 2 * (int64_t)f->n;
        else cnt->restrict_ncvx += 2 * (int64_t)f->n;
    }
    /* A */
    if ((st = pwl_add_linear(f, -lo, &g)) != OR_OK) return st;
    st = pwl_suffix_inf(&g, &G, cnt);
    pwl_free(&g);
    if (st != OR_OK) return st;
    st = pwl_add_linear(&G, lo, &A);
    pwl_free(&G);
    if (st != OR_OK) return st;
    /* B: inf over y' <= y of h(y') = suffix-inf of h(-t) at t = -y */
    if ((st = pwl_add_linear(f, -hi, &h)) != OR_OK) { pwl_free(&A); return st; }
    st = pwl_reflect(&h, &hr);
    pwl_free(&h);
    if (st != OR_OK) { pwl_free(&A); return st; }
    st = pwl_suffix_inf(&hr, &Hr, cnt);
    pwl_free(&hr);
    if (st != OR_OK) { pwl_free(&A); return st; }
    st = pwl_reflect(&Hr, &H);
    pwl_free(&Hr);
    if (st != OR_OK) { pwl_free(&A); return st; }
    st = pwl_add_linear(&H, hi, &B);
    pwl_free(&H);
    if (st != OR_OK) { pwl_free(&A); return st; }
    if (cnt) cnt->in_restrict = 1;
    st = pwl_envelope(&A, &B, 0, out, cnt);
    if (cnt) cnt->in_restrict = 0;
    pwl_free(&A);
    pwl_free(&B);
    return st;
}

/* seller's expense function, Eq. (1): u(y) = xi + (y-zeta)^- Sa - (y-zeta)^+ Sb */
static int seller_expense(double xi, double zeta, double Sa, double Sb, pwl *out)
{
    if (pwl_init(out, 1) != OR_OK) return OR_ENOMEM;
    pwl_push(out, zeta, xi);
    out->sl = -Sa;
    out->sr = -Sb;
    pwl_canonicalize(out);
    return OR_OK;
}

/* buyer's expense function, Eq. (6): u(y) = -xi + (y+zeta)^- Sa - (y+zeta)^+ Sb */
static int buyer_expense(double xi, double zeta, double Sa, double Sb, pwl *out)
{
    if (pwl_init(out, 1) != OR_OK) return OR_ENOMEM;
    pwl_push(out, -zeta, -xi);
    out->sl = -Sa;
    out->sr = -Sb;
    pwl_canonicalize(out);
    return OR_OK;
}

/* ------------------------------------------------------------------------- */
/* Model                                                                      */
/* ------------------------------------------------------------------------- */

typedef struct {
    double S0, K, K2, T, sigma, R, k;
    int32_t kind;
    int32_t american; /* 1 = American (default), 0 = European: no exercise before N
                         (TC reading: z_t = v_t for t < N) */
    int32_t cash;     /* 1 = put / call settled in cash ((K-S)^+ or (S-K)^+, 0)
                         instead of physically (NEXT #3, P:35 settlement-agnostic) */
    int32_t cost_t0;  /* 1 = proportional costs also at t = 0 (variant of P:159's
                         convention, NEXT #3): S^a_0 = (1+k) S0, S^b_0 = (1-k) S0 */
} or_option;

typedef struct {
    double ask, bid;
    int32_t status;
    int32_t max_kinks_ask, max_kinks_bid;
    int32_t pad;
    int64_t sum_kinks_ask, sum_kinks_bid; /* over all nodes t <= N */
    int64_t crossings;
    /* root hedge: the share position y* the seller /
       buyer takes at t = 0, argmin_y [ w_0(y)/r + S0 y ] over the vertices of
       w_0 = max(z_{1,0}, z_{1,1}) (no costs at t = 0, so v_0 is the line
       min_y'[w_0(y')/r + S0 y'] - S0 y, derived A.4); smallest minimiser */
    double hedge_ask, hedge_bid;
    /* SURVEY 8(d) cost model (instrumentation; see "Operation counters"):
       fp64_ops = 3 merge_visits + 4 crossings + 2 restrict_cvx
                  + 4 restrict_ncvx + 2 scale_visits, over every node t <= N */
    int64_t fp64_ops, merge_visits, restrict_cvx, restrict_ncvx, scale_visits;
    int64_t fp64_ops_party[2]; /* fp64_ops split by party: [0] seller (ask), [1] buyer (bid) */
} or_quote;

/*
 * Per-level kink statistics (instrumentation), accumulated (max / +=) into a
 * caller-owned int64 array of 2 x (N+1) x OR_LVL_STRIDE entries so a caller
 * can aggregate a batch: entry [party][t][0] = max kinks over the level's
 * nodes, [1] = sum of kinks, [2 + b] = number of nodes whose kink count falls
 * in bin b (or_kink_bin: exact below 128, then 8 bins per octave).
 */
#define OR_HBINS 240
#define OR_LVL_STRIDE (2 + OR_HBINS)

static int or_kink_bin(int c)
{
    if (c < 128) return c;
    int e = 0;
    while ((c >> (e + 1)) != 0) e++; /* e = floor(log2 c) >= 7 */
    int b = 128 + 8 * (e - 7) + ((c >> (e - 3)) - 8);
    return b < OR_HBINS ? b : OR_HBINS - 1;
}

int oracle_kink_bin_hi(int b) /* largest kink count of bin b */
{
    if (b < 128) return b;
    int e = 7 + (b - 128) / 8, sub = (b - 128) % 8;
    return ((9 + sub) << (e - 3)) - 1;
}

/* Sec. 4.1: u = exp(sigma sqrt(T/N)), d = 1/u, r = exp(RT/N) */
static int calibrate(const or_option *o, int N, double *u, double *d, double *r)
{
    if (!(o->S0 > 0) || !(o->T > 0) || !(o->sigma > 0) || N < 1) return OR_EINVAL;
    if (!(o->k >= 0.0 && o->k < 1.0)) return OR_EINVAL;
    if (o->kind != OR_PUT && o->kind != OR_CALL && o->kind != OR_BULL) return OR_EINVAL;
    if (o->kind != OR_BULL && !(o->K > 0)) return OR_EINVAL;
    if (o->kind == OR_BULL && !(o->K < o->K2)) return OR_EINVAL;
    *u = exp(o->sigma * sqrt(o->T / N));
    *d = 1.0 / *u;
    *r = exp(o->R * o->T / N);
    if (!(*d < *r && *r < *u)) return OR_EARBITRAGE;
    return OR_OK;
}

/* stock price at node (t, j), j = number of down-moves: S0 u^(t-j) d^j */
static double node_price(double S0, double u, double d, int t, int j)
{
    return S0 * pow(u, (double)(t - j)) * pow(d, (double)j);
}

/* payoff process (xi, zeta) at a node with stock price S, t <= N (R6) */
static void payoff(const or_option *o, double S, double *xi, double *zeta)
{
    switch (o->kind) {
    case OR_PUT:
        if (o->cash) { *xi = fmax(o->K - S, 0.0); *zeta = 0.0; }  /* cash ((K-S)^+, 0) */
        else { *xi = o->K; *zeta = -1.0; }                          /* (K, -1) P:94 */
        break;
    case OR_CALL:
        if (o->cash) { *xi = fmax(S - o->K, 0.0); *zeta = 0.0; }  /* cash ((S-K)^+, 0) */
        else { *xi = -o->K; *zeta = 1.0; }                          /* (-K, +1) */
        break;
    default: /* bull spread, cash */
        *xi = fmax(S - o->K, 0.0) - fmax(S - o->K2, 0.0);
        *zeta = 0.0;
        break;
    }
}

/* one node of the seller (party 0) or buyer (party 1) recursion */
/* exercisable = 0: a European node before expiry, z = v (NEXT #3 reading) */
static int node_update_x(int party, const pwl *zu, const pwl *zd, double r, double Sa, double Sb,
                         double xi, double zeta, int exercisable, pwl *z, counters *cnt)
{
    int st;
    pwl w, f, v, u;
    if ((st = pwl_envelope(zu, zd, 1, &w, cnt)) != OR_OK) return st; /* w = max(z^u, z^d) */
    st = pwl_div(&w, r, &f);                                        /* w / r */
    if (cnt) cnt->scale_visits += w.n;
    pwl_free(&w);
    if (st != OR_OK) return st;
    st = pwl_restrict(&f, -Sa, -Sb, &v, cnt);                       /* v */
    pwl_free(&f);
    if (st != OR_OK) return st;
    if (!exercisable) { *z = v; return OR_OK; }
    st = (party == 0) ? seller_expense(xi, zeta, Sa, Sb, &u) : buyer_expense(xi, zeta, Sa, Sb, &u);
    if (st != OR_OK) { pwl_free(&v); return st; }
    st = pwl_envelope(&u, &v, party == 0 ? 1 : 0, z, cnt);          /* max / min (u, v) */
    pwl_free(&u);
    pwl_free(&v);
    return st;
}

static int node_update(int party, const pwl *zu, const pwl *zd, double r, double Sa, double Sb,
                       double xi, double zeta, pwl *z, counters *cnt)
{
    return node_update_x(party, zu, zd, r, Sa, Sb, xi, zeta, 1, z, cnt);
}

/*
 * Ask and bid of an American option under proportional costs k (Sec. 3, 4.1).
 * kinks_out (optional): 2 * (N+1)(N+2)/2 ints, node (t,j) at index
 * 2*(t(t+1)/2 + j) + party, the kink count of z at that node.
 */
int oracle_price_tc_stats(const or_option *o, int N, or_quote *q, int32_t *kinks_out,
                          int64_t *lvl_stats)
{
    double u, d, r;
    memset(q, 0, sizeof *q);
    q->ask = q->bid = NAN;
    q->hedge_ask = q->hedge_bid = NAN;
    int st = calibrate(o, N, &u, &d, &r);
    if (st != OR_OK) { q->status = st; return st; }
    counters cntp[2]; /* per party */
    memset(cntp, 0, sizeof cntp);
    pwl *z[2];
    z[0] = (pwl *)calloc((size_t)N + 2, sizeof(pwl));
    z[1] = (pwl *)calloc((size_t)N + 2, sizeof(pwl));
    /* t = N+1: payoff (0,0) for both parties (Alg. 1 line 5) */
    for (int j = 0; j <= N + 1; j++) {
        double S = node_price(o->S0, u, d, N + 1, j);
        double Sa = (1.0 + o->k) * S, Sb = (1.0 - o->k) * S;
        seller_expense(0.0, 0.0, Sa, Sb, &z[0][j]);
        buyer_expense(0.0, 0.0, Sa, Sb, &z[1][j]);
    }
    for (int t = N; t >= 0 && st == OR_OK; t--) {
        for (int j = 0; j <= t && st == OR_OK; j++) {
            double S = node_price(o->S0, u, d, t, j);
            double Sa, Sb;
            if (t == 0 && !o->cost_t0) { Sa = Sb = S; } /* no costs at t = 0 */
            else { Sa = (1.0 + o->k) * S; Sb = (1.0 - o->k) * S; }
            double xi, zeta;
            payoff(o, S, &xi, &zeta);
            for (int party = 0; party < 2 && st == OR_OK; party++) {
                if (t == 0 && !o->cost_t0) {
                    /* root hedge: argmin over the vertices of w_0 of w_0(x)/r + S0 x (A.4) */
                    pwl w;
                    if ((st = pwl_envelope(&z[party][0], &z[party][1], 1, &w, NULL)) != OR_OK) break;
                    double best = INFINITY, bx = NAN;
                    for (int i = 0; i < w.n; i++) {
                        double g = w.f[i] / r + S * w.x[i];
                        if (g < best) { best = g; bx = w.x[i]; }
                    }
                    pwl_free(&w);
                    if (party == 0) q->hedge_ask = bx;
                    else q->hedge_bid = bx;
                }
                pwl znew;
                st = node_update_x(party, &z[party][j], &z[party][j + 1], r, Sa, Sb, xi, zeta,
                                   o->american || t == N, &znew, &cntp[party]);
                if (st != OR_OK) break;
                /* z[party][j] is read only by nodes j-1 (done) and j (this one) */
                pwl_free(&z[party][j]);
                z[party][j] = znew;
                int kk = pwl_kinks(&znew);
                if (party == 0) {
                    q->sum_kinks_ask += kk;
                    if (kk > q->max_kinks_ask) q->max_kinks_ask = kk;
                } else {
                    q->sum_kinks_bid += kk;
                    if (kk > q->max_kinks_bid) q->max_kinks_bid = kk;
                }
                if (kinks_out) kinks_out[2 * ((int64_t)t * (t + 1) / 2 + j) + party] = kk;
                if (lvl_stats) {
                    int64_t *L = lvl_stats + ((int64_t)party * (N + 1) + t) * OR_LVL_STRIDE;
                    if (kk > L[0]) L[0] = kk;
                    L[1] += kk;
                    L[2 + or_kink_bin(kk)] += 1;
                }
            }
        }
    }
    if (st == OR_OK) {
        q->ask = pwl_eval(&z[0][0], 0.0);  /* pi^a_0 = z_0(0) */
        q->bid = -pwl_eval(&z[1][0], 0.0); /* pi^b_0 = -z'_0(0) */
    }
    for (int p = 0; p < 2; p++) {
        const counters *c = &cntp[p];
        q->crossings += c->crossings;
        q->merge_visits += c->merge_visits;
        q->restrict_cvx += c->restrict_cvx;
        q->restrict_ncvx += c->restrict_ncvx;
        q->scale_visits += c->scale_visits;
        q->fp64_ops_party[p] = 3 * c->merge_visits + 4 * c->crossings + 2 * c->restrict_cvx
                               + 4 * c->restrict_ncvx + 2 * c->scale_visits;
    }
    q->fp64_ops = q->fp64_ops_party[0] + q->fp64_ops_party[1];
    q->status = st;
    for (int p = 0; p < 2; p++) {
        for (int j = 0; j <= N + 1; j++) pwl_free(&z[p][j]);
        free(z[p]);
    }
    return st;
}

int oracle_price_tc(const or_option *o, int N, or_quote *q, int32_t *kinks_out)
{
    return oracle_price_tc_stats(o, N, q, kinks_out, NULL);
}

/* frictionless exercise value P(S) (P_t = max(K - S_t, 0) for the put) */
static double exercise_value(const or_option *o, double S)
{
    double xi, zeta;
    payoff(o, S, &xi, &zeta);
    return fmax(xi + zeta * S, 0.0);
}

/*
 * Frictionless CRR price by backward induction (Appendix: no extra
 * level, scalar max).  p = (r-d)/(u-d); pi_N = P_N;
 * pi_t = max(P_t, (p pi^u + (1-p) pi^d)/r)  (American) or without the max.
 */
int oracle_price_crr(const or_option *o, int N, double *price)
{
    double u, d, r;
    or_option o0 = *o;
    o0.k = 0.0;
    *price = NAN;
    int st = calibrate(&o0, N, &u, &d, &r);
    if (st != OR_OK) return st;
    double p = (r - d) / (u - d);
    double *V = (double *)malloc(sizeof(double) * ((size_t)N + 1));
    if (!V) return OR_ENOMEM;
    for (int j = 0; j <= N; j++) V[j] = exercise_value(o, node_price(o->S0, u, d, N, j));
    for (int t = N - 1; t >= 0; t--) {
        for (int j = 0; j <= t; j++) {
            double cont = (p * V[j] + (1.0 - p) * V[j + 1]) / r;
            V[j] = o->american ? fmax(exercise_value(o, node_price(o->S0, u, d, t, j)), cont) : cont;
        }
    }
    *price = V[0];
    free(V);
    return OR_OK;
}

/*
 * European CRR price as the closed-form binomial sum (textbook):
 *   r^-N sum_j C(N,j) p^(N-j) (1-p)^j P(S0 u^(N-j) d^j),
 * each weight evaluated in log space (lgamma) since C(N, N/2) overflows fp64.
 */
int oracle_price_euro_closed(const or_option *o, int N, double *price)
{
    double u, d, r;
    or_option o0 = *o;
    o0.k = 0.0;
    *price = NAN;
    int st = calibrate(&o0, N, &u, &d, &r);
    if (st != OR_OK) return st;
    double p = (r - d) / (u - d);
    double lp = log(p), lq = log1p(-p), lr = log(r);
    double sum = 0.0;
    for (int j = 0; j <= N; j++) {
        double P = exercise_value(o, node_price(o->S0, u, d, N, j));
        if (P == 0.0) continue;
        double lw = lgamma(N + 1.0) - lgamma(j + 1.0) - lgamma(N - j + 1.0) + (N - j) * lp + j * lq - N * lr;
        sum += exp(lw) * P;
    }
    *price = sum;
    return OR_OK;
}

/* ------------------------------------------------------------------------- */
/* Exposed PWL algebra (for the oracle's own unit pins)                       */
/* A function crosses the ctypes boundary as (n, x[], f[], sl, sr).           */
/* ------------------------------------------------------------------------- */

static int to_pwl(int n, const double *x, const double *f, double sl, double sr, pwl *p)
{
    if (n < 1 || pwl_init(p, n) != OR_OK) return OR_EINVAL;
    for (int i = 0; i < n; i++) pwl_push(p, x[i], f[i]);
    p->sl = sl;
    p->sr = sr;
    return OR_OK;
}

static int from_pwl(const pwl *p, int cap, int *n, double *x, double *f, double *sl, double *sr)
{
    if (p->n > cap) return OR_EINVAL;
    *n = p->n;
    memcpy(x, p->x, sizeof(double) * (size_t)p->n);
    memcpy(f, p->f, sizeof(double) * (size_t)p->n);
    *sl = p->sl;
    *sr = p->sr;
    return OR_OK;
}

/* op: 0 = max, 1 = min, 2 = restrict(lo=a, hi=b), 3 = divide by a, 4 = canonicalize */
int oracle_pwl_op(int op, int n1, const double *x1, const double *f1, double sl1, double sr1,
                  int n2, const double *x2, const double *f2, double sl2, double sr2,
                  double a, double b, int cap, int *n, double *x, double *f, double *sl, double *sr)
{
    pwl p1, p2, out;
    int st = to_pwl(n1, x1, f1, sl1, sr1, &p1);
    if (st != OR_OK) return st;
    switch (op) {
    case 0:
    case 1:
        if ((st = to_pwl(n2, x2, f2, sl2, sr2, &p2)) != OR_OK) { pwl_free(&p1); return st; }
        st = pwl_envelope(&p1, &p2, op == 0, &out, NULL);
        pwl_free(&p2);
        break;
    case 2: st = pwl_restrict(&p1, a, b, &out, NULL); break;
    case 3: st = pwl_div(&p1, a, &out); break;
    case 4:
        st = to_pwl(n1, x1, f1, sl1, sr1, &out);
        if (st == OR_OK) pwl_canonicalize(&out);
        break;
    default: st = OR_EINVAL;
    }
    pwl_free(&p1);
    if (st != OR_OK) return st;
    st = from_pwl(&out, cap, n, x, f, sl, sr);
    pwl_free(&out);
    return st;
}

/* evaluate a PWL function at m points */
int oracle_pwl_eval(int n, const double *x, const double *f, double sl, double sr, int m,
                    const double *y, double *out)
{
    pwl p;
    int st = to_pwl(n, x, f, sl, sr, &p);
    if (st != OR_OK) return st;
    for (int i = 0; i < m; i++) out[i] = pwl_eval(&p, y[i]);
    pwl_free(&p);
    return OR_OK;
}

/* one node update exposed (the P:100-144 one-step worked examples) */
int oracle_node_update(int party, int n1, const double *x1, const double *f1, double sl1, double sr1,
                       int n2, const double *x2, const double *f2, double sl2, double sr2,
                       double r, double Sa, double Sb, double xi, double zeta,
                       int cap, int *n, double *x, double *f, double *sl, double *sr)
{
    pwl zu, zd, z;
    int st = to_pwl(n1, x1, f1, sl1, sr1, &zu);
    if (st != OR_OK) return st;
    if ((st = to_pwl(n2, x2, f2, sl2, sr2, &zd)) != OR_OK) { pwl_free(&zu); return st; }
    st = node_update(party, &zu, &zd, r, Sa, Sb, xi, zeta, &z, NULL);
    pwl_free(&zu);
    pwl_free(&zd);
    if (st != OR_OK) return st;
    st = from_pwl(&z, cap, n, x, f, sl, sr);
    pwl_free(&z);
    return st;
}

int oracle_abi_version(void) { return 2; }
int oracle_lvl_stride(void) { return OR_LVL_STRIDE; }
