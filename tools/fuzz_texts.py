"""Random integrand texts in the make_golden fuzz grammar (shared by the fuzz tools)."""


def texts(rng, count):
    def index(depth, names):
        if depth > 1 or rng.random() < 0.4:
            return rng.choice([str(rng.randint(1, 3)), "d"] + list(names))
        return f"({index(depth + 1, names)}{rng.choice(['+', '-', '*'])}{index(depth + 1, names)})"

    def real(depth, names):
        r = rng.random()
        if depth > 3 or r < 0.25:
            return rng.choice([f"x[{index(1, names)}]", repr(round(rng.uniform(-2, 2), 3)), "pi", "e"] + list(names))
        if r < 0.55:
            return f"{real(depth + 1, names)} {rng.choice(['+', '-', '*'])} {real(depth + 1, names)}"
        if r < 0.65:
            return f"({real(depth + 1, names)})^{rng.choice(['2', '3', '(1+1)'])}"
        if r < 0.8:
            return f"{rng.choice(['exp', 'sin', 'cos'])}({real(depth + 1, names)})"
        if r < 0.9:
            v = rng.choice(["i", "j", "k"])
            return f"{rng.choice(['sum', 'prod'])}({v}=1..{rng.choice(['d', '2'])}, {real(depth + 1, names | {v})})"
        return f"-{real(depth + 1, names)}"
    return [real(0, frozenset()) for _ in range(count)]
