// Host-side orbit planners of the chain layouts (included by lq_api.cu inside
// its anonymous namespace; no device code, no CUDA calls): prime n
// (DESIGN.md §4.1b), n = 2^k levels (§4.1d) and composite n by divisor
// classes (§4.1f).  Plans are cached per (n, a, chain length, kernel form).
#pragma once
// ------------------------------------------------------------ Korobov orbits
// Host plan of k_orbit (lq_kernels.cu): primality of n, the order o of a in
// (Z/n)^*, a primitive root g, the coset/exponent enumeration of half of the
// nonzero points (the mirrors n - i cover the other half) and the start tables.
uint32_t powmod32(uint64_t b, uint64_t e, uint32_t n) {
    uint64_t r = 1 % n;
    b %= n;
    while (e) {
        if (e & 1) r = r * b % n;
        b = b * b % n;
        e >>= 1;
    }
    return (uint32_t)r;
}

bool is_prime32(uint32_t n) {
    if (n < 2) return false;
    for (uint32_t p : {2u, 3u, 5u, 7u, 11u, 13u}) {
        if (n % p == 0) return n == p;
    }
    uint32_t d = n - 1;
    int s = 0;
    while (!(d & 1)) { d >>= 1; ++s; }
    for (uint32_t b : {2u, 3u, 5u, 7u}) {   // deterministic below 3.2e9
        uint64_t x = powmod32(b, d, n);
        if (x == 1 || x == n - 1) continue;
        bool comp = true;
        for (int r = 1; r < s && comp; ++r) {
            x = x * x % n;
            if (x == n - 1) comp = false;
        }
        if (comp) return false;
    }
    return true;
}

struct OrbPlan {
    uint64_t id = 0;
    uint32_t n = 0, a = 0, as = 0, qc = 0, h = 0;
    uint64_t units = 0;
    int m = 0;
    bool mirror = true;
    bool zero = true;             // the launch covering unit 0 also adds the point x = 0
    std::vector<uint32_t> G, Alo, Ahi;
    std::vector<uint32_t> apow;   // FFT plans: (a^t mod n, Shoup constant) pairs, t < kFftN
    std::vector<uint32_t> starts; // FFT plans: first point of every chain (no divisions on the device)
};

// Chain starts of an FFT plan: starts[u] = G[u / qc] a^(m (u mod qc)) mod n.
void fill_chain_starts(OrbPlan& p) {
    const uint64_t n = p.n;
    uint64_t am = 1;
    for (int i = 0; i < p.m; ++i) am = am * p.a % n;
    p.starts.resize(p.units);
    size_t u = 0;
    for (size_t cs = 0; cs < p.G.size(); ++cs) {
        uint64_t t = p.G[cs];
        for (uint32_t q = 0; q < p.qc; ++q, ++u) {
            p.starts[u] = (uint32_t)t;
            t = t * am % n;
        }
    }
}

constexpr uint32_t kOrbMaxCosets = 4096;

// nullptr when the rule is not a Korobov rule over a prime modulus the orbit
// kernel can enumerate (caller then uses the per-index kernels).
// mirror: enumerate half of the nonzero points (their mirrors n - i are summed
// with them); otherwise every nonzero point once (product family).
// relaxed (composite-n levels): chains may be shorter than m and the cosets
// many (kOrbMaxCosetsLevel); the kernels mask a chain's tail either way.
constexpr uint32_t kOrbMaxCosetsLevel = 1u << 20;
std::shared_ptr<const OrbPlan> build_orbit_plan(uint32_t n, uint32_t a, int m, bool mirror, bool relaxed = false) {
    if (!is_prime32(n) || a < 1 || a >= n) return nullptr;
    std::vector<uint32_t> primes;
    uint32_t rest = n - 1;
    for (uint32_t p = 2; (uint64_t)p * p <= rest; ++p)
        if (rest % p == 0) {
            primes.push_back(p);
            while (rest % p == 0) rest /= p;
        }
    if (rest > 1) primes.push_back(rest);
    uint32_t o = n - 1;
    for (uint32_t p : primes)
        while (o % p == 0 && powmod32(a, o / p, n) == 1) o /= p;
    uint32_t g = 2;
    for (;; ++g) {
        bool prim = true;
        for (uint32_t p : primes)
            if (powmod32(g, (n - 1) / p, n) == 1) { prim = false; break; }
        if (prim) break;
    }
    const uint32_t C = (n - 1) / o;
    uint32_t cosets, h;
    if (!mirror) { cosets = C; h = o; }                 // every coset, every exponent
    else if (o % 2 == 0) { cosets = C; h = o / 2; }     // -1 lies in <a>: half of each coset
    else { cosets = C / 2; h = o; }                     // -coset(s) = coset(s + C/2)
    if (cosets < 1 || cosets > (relaxed ? kOrbMaxCosetsLevel : kOrbMaxCosets) || h < (relaxed ? 1u : (uint32_t)m))
        return nullptr;
    static std::atomic<uint64_t> next_id{1};
    auto p = std::make_shared<OrbPlan>();
    p->id = next_id++;
    p->n = n; p->a = a; p->m = m; p->h = h; p->mirror = mirror;
    p->as = (uint32_t)(((uint64_t)a << 32) / n);
    p->qc = (h + m - 1) / m;
    p->units = (uint64_t)cosets * p->qc;
    p->G.resize(cosets);
    const uint32_t gC = powmod32(g, 1, n);
    uint64_t gs = 1;
    for (uint32_t s = 0; s < cosets; ++s) { p->G[s] = (uint32_t)gs; gs = gs * gC % n; }
    const uint32_t am = powmod32(a, (uint64_t)m, n);
    p->Alo.resize(4096);
    uint64_t t = 1;
    for (int q = 0; q < 4096; ++q) { p->Alo[q] = (uint32_t)t; t = t * am % n; }
    const uint32_t am4096 = (uint32_t)t;
    p->Ahi.resize(p->qc / 4096 + 1);
    t = 1;
    for (size_t q = 0; q < p->Ahi.size(); ++q) { p->Ahi[q] = (uint32_t)t; t = t * am4096 % n; }
    return p;
}

std::shared_ptr<const OrbPlan> orbit_plan(uint32_t n, uint32_t a, int m, bool mirror, bool fft = false) {
    static std::mutex mu;
    static std::map<std::tuple<uint32_t, uint32_t, int, bool, bool>, std::shared_ptr<const OrbPlan>> cache;
    std::lock_guard<std::mutex> lk(mu);
    auto key = std::make_tuple(n, a, m, mirror, fft);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
    auto p = build_orbit_plan(n, a, m, mirror);
    if (p && fft) {
        auto q = std::make_shared<OrbPlan>(*p);
        q->apow.resize(2 * lq::kFftN);
        uint64_t t = 1 % n;
        for (int k = 0; k < lq::kFftN; ++k) {
            q->apow[2 * k] = (uint32_t)t;
            q->apow[2 * k + 1] = (uint32_t)((t << 32) / n);
            t = t * a % n;
        }
        fill_chain_starts(*q);
        p = q;
    }
    if (cache.size() > 64) cache.clear();
    cache[key] = p;
    return p;
}

// ---- Korobov rules with n = 2^k.  Point i = 2^v u (u odd) has residues
// 2^v (u a^(j-1) mod 2^m), m = k - v: level m is the unit group mod 2^m, whose
// mirror classes {u, -u} are the cyclic group <5> (order 2^(m-2)); a = +-5^alpha
// moves a class by alpha, so the chains i0 a^t of a level run along the cosets
// 5^e <5^alpha> (e < 2^tau, tau = v2(alpha)).  Each level is an orbit sum with
// modulus 2^m; the levels too short for chains, and the point 0, form the
// lattice with modulus 2^m0, summed by the per-index kernel.
uint64_t inv_pow2(uint64_t x, int m) {   // x odd: x^-1 mod 2^m (Newton)
    uint64_t y = x;
    for (int i = 0; i < 6; ++i) y *= 2 - x * y;
    return m >= 64 ? y : (y & ((1ull << m) - 1));
}

std::shared_ptr<const OrbPlan> build_orbit_plan_pow2(int m, uint32_t a_full, int len, bool fft) {
    if (m < 3 || m > 31) return nullptr;
    const uint64_t n = 1ull << m, mask = n - 1;
    const uint64_t a = a_full & mask;
    if (!(a & 1)) return nullptr;
    const uint64_t b = (a & 3) == 1 ? a : (n - a) & mask;   // the <5> part of +-a
    // discrete log of b to base 5 in <5> mod 2^m, bit by bit (5^(2^i) = 1 + 2^(i+2) mod 2^(i+3))
    uint64_t alpha = 0, cur = b, p5 = 5;   // cur = b 5^-alpha
    for (int i = 0; i < m - 2; ++i) {
        if ((cur & ((1ull << (i + 3)) - 1)) != 1) {
            alpha |= 1ull << i;
            cur = (cur * inv_pow2(p5, 64)) & mask;
        }
        p5 = (p5 * p5) & mask;
    }
    if (alpha == 0) return nullptr;                          // a = +-1 mod 2^m: no chains
    int tau = 0;
    while (!((alpha >> tau) & 1)) ++tau;
    const uint64_t L = 1ull << (m - 2 - tau);                 // class-cycle length
    const uint64_t cosets = 1ull << tau;
    if (cosets > kOrbMaxCosets || L < (uint64_t)len) return nullptr;
    static std::atomic<uint64_t> next_id{1ull << 40};
    auto p = std::make_shared<OrbPlan>();
    p->id = next_id++;
    p->n = (uint32_t)n; p->a = (uint32_t)a; p->m = len; p->h = (uint32_t)L; p->mirror = true; p->zero = false;
    p->as = (uint32_t)((a << 32) / n);
    p->qc = (uint32_t)((L + len - 1) / len);
    p->units = cosets * p->qc;
    p->G.resize(cosets);
    uint64_t g = 1;
    for (uint64_t e = 0; e < cosets; ++e) { p->G[e] = (uint32_t)g; g = (g * 5) & mask; }
    auto mulm = [&](uint64_t x, uint64_t y) { return (x * y) & mask; };
    uint64_t am = 1;
    for (int i = 0; i < len; ++i) am = mulm(am, a);
    p->Alo.resize(4096);
    uint64_t t = 1;
    for (int q = 0; q < 4096; ++q) { p->Alo[q] = (uint32_t)t; t = mulm(t, am); }
    const uint64_t am4096 = t;
    p->Ahi.resize(p->qc / 4096 + 1);
    t = 1;
    for (size_t q = 0; q < p->Ahi.size(); ++q) { p->Ahi[q] = (uint32_t)t; t = mulm(t, am4096); }
    if (fft) {
        p->apow.resize(2 * lq::kFftN);
        t = 1;
        for (int k = 0; k < lq::kFftN; ++k) {
            p->apow[2 * k] = (uint32_t)t;
            p->apow[2 * k + 1] = (uint32_t)((t << 32) / n);
            t = mulm(t, a);
        }
        fill_chain_starts(*p);
    }
    return p;
}

// Levels + small lattice (n = 2^k here; composite n below, DivPlan): every
// level is the orbit sum of one class of points (a unit group mod its own
// modulus), and the small lattice -- modulus small_n, the per-index kernel --
// holds the classes too short for chains and the point 0.
struct Pow2Plan {
    int k = 0, m0 = 0;                                  // levels m0+1 .. k; small lattice mod 2^m0
    bool fft = false;
    uint64_t small_n = 1;                               // modulus of the small lattice
    std::vector<std::shared_ptr<const OrbPlan>> levels; // m = k, k-1, ..., m0+1
};

std::shared_ptr<const Pow2Plan> pow2_plan(uint32_t a, int k, int len, bool fft) {
    static std::mutex mu;
    static std::map<std::tuple<uint32_t, int, int, bool>, std::shared_ptr<const Pow2Plan>> cache;
    std::lock_guard<std::mutex> lk(mu);
    auto key = std::make_tuple(a, k, len, fft);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
    auto P = std::make_shared<Pow2Plan>();
    P->k = k;
    P->fft = fft;
    int m = k;
    for (; m >= 3; --m) {
        auto lp = build_orbit_plan_pow2(m, a, len, fft);
        if (!lp) break;
        P->levels.push_back(lp);
    }
    P->m0 = m;
    P->small_n = 1ull << m;
    std::shared_ptr<const Pow2Plan> out = P->levels.empty() ? nullptr : P;
    if (cache.size() > 64) cache.clear();
    cache[key] = out;
    return out;
}

// ---- Korobov rules with composite n.  Point i with
// gcd(i, n) = n/m is (n/m) u, u a unit mod m, and its coordinates are
// frac(u a^(j-1) / m): the class is the unit group U(m) of the Korobov lattice
// mod m.  U(m) is a product of cyclic groups (a primitive root per odd prime
// power, -1 and 5 for 2^e); in those exponent coordinates <a> (with -1 for the
// mirror pairs) is a subgroup, and the box of a triangular (Hermite) basis of
// the relation lattice is a complete set of coset representatives.
struct UnitComp {
    uint64_t q;      // prime-power modulus of the component
    uint64_t ord;    // cyclic order
    uint64_t gen;    // generator mod q
    int two;         // 0 odd prime power; 1 the -1 factor of 2^e; 2 the <5> factor of 2^e
};

uint64_t mulmod64(uint64_t x, uint64_t y, uint64_t m) { return (uint64_t)((unsigned __int128)x * y % m); }
uint64_t powmod64(uint64_t b, uint64_t e, uint64_t m) {
    uint64_t r = 1 % m;
    b %= m;
    for (; e; e >>= 1, b = mulmod64(b, b, m))
        if (e & 1) r = mulmod64(r, b, m);
    return r;
}
uint64_t gcd64(uint64_t x, uint64_t y) { while (y) { uint64_t t = x % y; x = y; y = t; } return x; }

std::vector<std::pair<uint64_t, int>> factor64(uint64_t n) {
    std::vector<std::pair<uint64_t, int>> out;
    for (uint64_t p = 2; p * p <= n; ++p)
        if (n % p == 0) {
            int e = 0;
            while (n % p == 0) { n /= p; ++e; }
            out.push_back({p, e});
        }
    if (n > 1) out.push_back({n, 1});
    return out;
}

// discrete log of x to base g in the cyclic group of order ord mod q (baby-step
// giant-step); ord < 2^32
uint64_t dlog_bsgs(uint64_t g, uint64_t x, uint64_t ord, uint64_t q) {
    const uint64_t s = (uint64_t)std::ceil(std::sqrt((double)ord)) + 1;
    std::unordered_map<uint64_t, uint64_t> baby;
    baby.reserve(2 * s);
    uint64_t cur = 1 % q;
    for (uint64_t j = 0; j < s; ++j) {
        baby.emplace(cur, j);
        cur = mulmod64(cur, g, q);
    }
    const uint64_t ginv_s = powmod64(powmod64(g, ord - 1, q), s, q);   // g^-s
    cur = x % q;
    for (uint64_t i = 0; i <= s; ++i) {
        auto it = baby.find(cur);
        if (it != baby.end()) return (i * s + it->second) % ord;
        cur = mulmod64(cur, ginv_s, q);
    }
    return UINT64_MAX;
}

uint64_t primitive_root_pe(uint64_t p, int e) {
    const uint64_t pm1 = p - 1;
    auto fs = factor64(pm1);
    for (uint64_t g = 2;; ++g) {
        bool prim = true;
        for (auto& f : fs)
            if (powmod64(g, pm1 / f.first, p) == 1) { prim = false; break; }
        if (!prim) continue;
        if (e >= 2 && powmod64(g, pm1, p * p) == 1) continue;   // lifts to p^e unless g^(p-1) = 1 mod p^2
        return g;
    }
}

// Orbit plan of the unit group U(m) (m composite or a prime power) under
// multiplication by a, mirror pairs u, -u summed together; nullptr when the
// chains would be shorter than len or the cosets too many.
std::shared_ptr<const OrbPlan> build_orbit_plan_units(uint32_t m, uint32_t a_full, int len, bool fft) {
    if (m < 3) return nullptr;
    const uint64_t a = a_full % m;
    if (gcd64(a, m) != 1) return nullptr;
    // cyclic components and the exponent vectors of a and -1
    std::vector<UnitComp> comp;
    std::vector<uint64_t> al, be;
    for (auto& pe : factor64(m)) {
        uint64_t q = 1;
        for (int i = 0; i < pe.second; ++i) q *= pe.first;
        if (pe.first == 2) {
            if (pe.second == 1) {            // U(2) is trivial, but u must still be odd (CRT)
                comp.push_back({2, 1, 1, 1});
                al.push_back(0);
                be.push_back(0);
                continue;
            }
            const uint64_t ar = a % q;
            const bool neg = (ar & 3) == 3;
            comp.push_back({q, 2, q - 1, 1});
            al.push_back(neg ? 1 : 0);
            be.push_back(1);
            if (pe.second >= 3) {
                const int e = pe.second;
                const uint64_t ord5 = q >> 2, b = neg ? (q - ar) % q : ar;   // +-a = 5^k
                uint64_t k = 0, cur = b, p5 = 5;
                for (int i = 0; i < e - 2; ++i) {
                    if ((cur & ((1ull << (i + 3)) - 1)) != 1) {
                        k |= 1ull << i;
                        cur = mulmod64(cur, inv_pow2(p5, 64) & (q - 1), q);
                    }
                    p5 = mulmod64(p5, p5, q);
                }
                comp.push_back({q, ord5, 5, 2});
                al.push_back(k);
                be.push_back(0);
            }
        } else {
            const uint64_t ord = q / pe.first * (pe.first - 1);
            // (generator, log of a) per prime power, shared by every divisor
            // of n that contains it (div_plan builds ~all of them)
            static std::mutex dl_mu;
            static std::map<std::pair<uint64_t, uint64_t>, std::pair<uint64_t, uint64_t>> dl_cache;
            uint64_t g, k;
            {
                std::lock_guard<std::mutex> lk(dl_mu);
                auto key = std::make_pair(q, a % q);
                auto hit = dl_cache.find(key);
                if (hit != dl_cache.end()) {
                    g = hit->second.first;
                    k = hit->second.second;
                } else {
                    g = primitive_root_pe(pe.first, pe.second);
                    k = dlog_bsgs(g, a % q, ord, q);
                    if (dl_cache.size() > 4096) dl_cache.clear();
                    dl_cache[key] = {g, k};
                }
            }
            if (k == UINT64_MAX) return nullptr;
            comp.push_back({q, ord, g, 0});
            al.push_back(k);
            be.push_back(ord / 2);          // -1 = g^(ord/2)
        }
    }
    const int r = (int)comp.size();
    if (r == 0) return nullptr;
    uint64_t o = 1, phi = 1;                  // ord(a), |U(m)|
    for (int c = 0; c < r; ++c) {
        const uint64_t oc = comp[c].ord / gcd64(comp[c].ord, al[c]);
        o = o / gcd64(o, oc) * oc;
        phi *= comp[c].ord;
    }
    const bool neg_in = (o % 2 == 0) && powmod64(a, o / 2, m) == m - 1;
    const uint64_t h = neg_in ? o / 2 : o;
    const uint64_t hsize = neg_in ? o : 2 * o;   // |H|, H = <a> or <a, -1>
    if (phi % hsize) return nullptr;
    const uint64_t cosets = phi / hsize;
    if (cosets > kOrbMaxCosetsLevel || h < 1) return nullptr;
    // triangular basis of the relation lattice span{ord_c e_c, alpha (, beta)}
    std::vector<std::vector<int64_t>> rows;
    rows.push_back(std::vector<int64_t>(al.begin(), al.end()));
    if (!neg_in) rows.push_back(std::vector<int64_t>(be.begin(), be.end()));
    auto modc = [&](int64_t v, int c) { const int64_t M = (int64_t)comp[c].ord; v %= M; return v < 0 ? v + M : v; };
    std::vector<int64_t> diag(r);
    for (int c = 0; c < r; ++c) {
        std::vector<int64_t> piv(r, 0);
        piv[c] = (int64_t)comp[c].ord;        // the relation ord_c e_c
        for (auto& R : rows) {
            if (R[c] == 0) continue;
            // extended gcd of (piv[c], R[c]): [piv; R] <- [[s, t], [-R_c/g, piv_c/g]] [piv; R]
            int64_t x0 = piv[c], x1 = R[c], s0 = 1, s1 = 0, t0 = 0, t1 = 1;
            while (x1) {
                const int64_t qq = x0 / x1;
                int64_t tmp = x0 - qq * x1; x0 = x1; x1 = tmp;
                tmp = s0 - qq * s1; s0 = s1; s1 = tmp;
                tmp = t0 - qq * t1; t0 = t1; t1 = tmp;
            }
            const int64_t g = x0, u = piv[c] / g, v = R[c] / g;
            std::vector<int64_t> np(r), nr(r);
            for (int k = 0; k < r; ++k) {
                const __int128 pk = piv[k], rk = R[k];
                const __int128 a1 = (__int128)s0 * pk + (__int128)t0 * rk, a2 = -(__int128)v * pk + (__int128)u * rk;
                if (k == c) { np[k] = (int64_t)a1; nr[k] = (int64_t)a2; continue; }
                const __int128 M = (__int128)comp[k].ord;
                __int128 b1 = a1 % M, b2 = a2 % M;
                np[k] = (int64_t)(b1 < 0 ? b1 + M : b1);
                nr[k] = (int64_t)(b2 < 0 ? b2 + M : b2);
            }
            piv.swap(np);
            R.swap(nr);
        }
        // piv is the basis vector b_c = (0, .., 0, g, *, ..); every remaining
        // row now has a zero in column c
        diag[c] = piv[c] < 0 ? -piv[c] : piv[c];
    }
    uint64_t box = 1;
    for (int c = 0; c < r; ++c) {
        if (diag[c] < 1) return nullptr;
        box *= (uint64_t)diag[c];
    }
    if (box != cosets) return nullptr;        // the basis must index exactly |U(m)/H| cosets
    // representatives: x in the box -> prod_c gen_c^(x_c), CRT over the prime powers
    static std::atomic<uint64_t> next_id{1ull << 50};
    auto p = std::make_shared<OrbPlan>();
    p->id = next_id++;
    p->n = m; p->a = (uint32_t)a; p->m = len; p->h = (uint32_t)h; p->mirror = true; p->zero = false;
    p->as = (uint32_t)((a << 32) / m);
    p->qc = (uint32_t)((h + len - 1) / len);
    p->units = cosets * p->qc;
    p->G.resize(cosets);
    // CRT idempotents e_q (e_q = 1 mod q, 0 mod the other prime powers) and
    // the per-component powers gen_c^(x_c), advanced incrementally with the
    // mixed-radix counter over the box
    std::vector<uint64_t> qs, eq;
    std::vector<int> comp_q(r);
    for (int c = 0; c < r; ++c) {
        if (c == 0 || comp[c].q != comp[c - 1].q) qs.push_back(comp[c].q);
        comp_q[c] = (int)qs.size() - 1;
    }
    for (uint64_t q : qs) {
        const uint64_t Mq = m / q;
        int64_t e0 = (int64_t)(Mq % q), e1 = (int64_t)q, s0 = 1, s1 = 0;
        while (e1) { const int64_t qq = e0 / e1; int64_t tmp = e0 - qq * e1; e0 = e1; e1 = tmp; tmp = s0 - qq * s1; s0 = s1; s1 = tmp; }
        const uint64_t inv = (uint64_t)((s0 % (int64_t)q + (int64_t)q) % (int64_t)q);
        eq.push_back(mulmod64(Mq % m, inv, m));
    }
    std::vector<int64_t> x(r, 0);
    std::vector<uint64_t> pw(r, 1);   // gen_c^(x_c) mod q_c
    for (int c = 0; c < r; ++c) pw[c] = 1 % comp[c].q;
    for (uint64_t idx = 0; idx < cosets; ++idx) {
        uint64_t u = 0;
        size_t c = 0;
        for (size_t qi = 0; qi < qs.size(); ++qi) {
            const uint64_t q = qs[qi];
            uint64_t v = 1 % q;
            for (; c < (size_t)r && comp[c].q == q; ++c) v = v * pw[c] % q;
            u = (u + v * eq[qi]) % m;
        }
        p->G[idx] = (uint32_t)u;
        for (int k = r - 1; k >= 0; --k) {   // mixed-radix increment over the box
            if (++x[k] < diag[k]) { pw[k] = pw[k] * comp[k].gen % comp[k].q; break; }
            x[k] = 0;
            pw[k] = 1 % comp[k].q;
        }
    }
    (void)comp_q;
    auto mulm = [&](uint64_t xx, uint64_t yy) { return xx * yy % m; };   // operands < m < 2^32
    uint64_t am = 1;
    for (int i = 0; i < len; ++i) am = mulm(am, a);
    p->Alo.resize(4096);
    uint64_t t = 1;
    for (int q = 0; q < 4096; ++q) { p->Alo[q] = (uint32_t)t; t = mulm(t, am); }
    const uint64_t am4096 = t;
    p->Ahi.resize(p->qc / 4096 + 1);
    t = 1;
    for (size_t q = 0; q < p->Ahi.size(); ++q) { p->Ahi[q] = (uint32_t)t; t = mulm(t, am4096); }
    if (fft) {
        p->apow.resize(2 * lq::kFftN);
        t = 1;
        for (int k = 0; k < lq::kFftN; ++k) {
            p->apow[2 * k] = (uint32_t)t;
            p->apow[2 * k + 1] = (uint32_t)((t << 32) / m);
            t = mulm(t, a);
        }
        fill_chain_starts(*p);
    }
    return p;
}

// Composite n: a level for every divisor m of n whose unit group has chains
// (the prime plan for prime m), the small lattice mod m0 for the rest.  m0 is
// grown (lcm) by every divisor without a plan, so its divisors are exactly the
// classes left to the per-index kernel.  nullptr when m0 would exceed n / 4.
std::shared_ptr<const Pow2Plan> div_plan(uint32_t n, uint32_t a, int len, bool fft, int len_direct) {
    static std::mutex mu;
    static std::map<std::tuple<uint32_t, uint32_t, int, bool, int>, std::shared_ptr<const Pow2Plan>> cache;
    std::lock_guard<std::mutex> lk(mu);
    auto key = std::make_tuple(n, a, len, fft, len_direct);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
    std::vector<uint64_t> divs{1};
    for (auto& pe : factor64(n)) {
        const size_t k = divs.size();
        uint64_t q = 1;
        for (int e = 1; e <= pe.second; ++e) {
            q *= pe.first;
            for (size_t i = 0; i < k; ++i) divs.push_back(divs[i] * q);
        }
    }
    std::sort(divs.rbegin(), divs.rend());
    std::map<uint64_t, std::shared_ptr<const OrbPlan>> plans;
    // one class: FFT-form chains when its orbits fill at least half a tile,
    // else direct chains (len_direct; 0 = no direct form for this integrand)
    auto build = [&](uint64_t m, int ln, bool f) -> std::shared_ptr<const OrbPlan> {
        std::shared_ptr<const OrbPlan> pl;
        if (is_prime32((uint32_t)m)) {
            auto q = build_orbit_plan((uint32_t)m, (uint32_t)(a % m), ln, true, true);
            if (q) {
                auto w = std::make_shared<OrbPlan>(*q);
                w->zero = false;   // the point 0 belongs to the small lattice
                if (f) {
                    w->apow.resize(2 * lq::kFftN);
                    uint64_t t = 1 % m;
                    for (int k = 0; k < lq::kFftN; ++k) {
                        w->apow[2 * k] = (uint32_t)t;
                        w->apow[2 * k + 1] = (uint32_t)((t << 32) / m);
                        t = t * (a % m) % m;
                    }
                    fill_chain_starts(*w);
                }
                pl = w;
            }
        } else {
            pl = build_orbit_plan_units((uint32_t)m, a, ln, f);
        }
        return pl;
    };
    // a global bound on the chains of all levels (short orbits on many
    // classes: one unit per few points) -- past it the whole plan is refused
    // and the paired index kernel runs; it also bounds the host tables
    const uint64_t unit_budget = 4 * ((uint64_t)n / (uint64_t)std::max(len, 1) + 1) + (1u << 20);
    uint64_t units_total = 0;
    bool over = false;
    auto plan_of = [&](uint64_t m) -> std::shared_ptr<const OrbPlan> {
        auto hit = plans.find(m);
        if (hit != plans.end()) return hit->second;
        if (over) return nullptr;
        std::shared_ptr<const OrbPlan> pl;
        if (fft) {
            pl = build(m, len, true);
            if (pl && 2 * (uint64_t)pl->h < (uint64_t)len) pl = nullptr;
        }
        if (!pl && len_direct > 0) pl = build(m, len_direct, false);
        if (pl) {
            units_total += pl->units;
            if (units_total > unit_budget) {
                over = true;
                pl = nullptr;
            }
        }
        plans[m] = pl;
        return pl;
    };
    uint64_t m0 = (n % 2 == 0) ? 2 : 1;
    for (bool grew = true; grew;) {
        grew = false;
        for (uint64_t m : divs) {
            if (m0 % m == 0) continue;
            if (!plan_of(m)) {
                m0 = m0 / gcd64(m0, m) * m;
                grew = true;
                break;
            }
        }
        if (m0 > n / 4) break;
    }
    std::shared_ptr<const Pow2Plan> out;
    if (m0 <= n / 4 && !over) {
        auto P = std::make_shared<Pow2Plan>();
        P->small_n = m0;
        for (uint64_t m : divs)
            if (m0 % m) {
                P->levels.push_back(plan_of(m));
                P->fft = P->fft || !P->levels.back()->apow.empty();
            }
        if (!P->levels.empty()) out = P;
    }
    if (cache.size() > 64) cache.clear();
    cache[key] = out;
    return out;
}

