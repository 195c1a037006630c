"""Writes tests/golden/phi_bar.txt from the paper's closed forms (no oracle, no
CUDA).  Eq. 6: phi_bar_rho(beta) = 2 / (1 + exp(-(rho*beta - 2*rho))).
Eq. 5: phi(beta) = Gamma(3/beta) / Gamma(1/beta).
Evaluated in 50-digit decimal arithmetic (exp by its Taylor series; Gamma via
math.lgamma is only double, so Eq. 5 values are printed to 15 digits)."""
import math
import os
from decimal import Decimal, getcontext

getcontext().prec = 60


def dexp(x: Decimal) -> Decimal:
    # exp(x) = exp(x/2^k)^(2^k), Taylor on the reduced argument
    k = 0
    while abs(x) > Decimal("0.01"):
        x /= 2
        k += 1
    s, term, n = Decimal(1), Decimal(1), 0
    while True:
        n += 1
        term = term * x / n
        if abs(term) < Decimal(10) ** -70:
            break
        s += term
    for _ in range(k):
        s = s * s
    return s


def phi_bar(beta, rho):
    b, r = Decimal(beta), Decimal(rho)
    return Decimal(2) / (Decimal(1) + dexp(-(r * b - 2 * r)))


if __name__ == "__main__":
    here = os.path.dirname(os.path.abspath(__file__))
    with open(os.path.join(here, "phi_bar.txt"), "w") as f:
        f.write("# Eq. 6 (PAPER.md:291-293) phi_bar_rho(beta), 30 significant digits.\n")
        f.write("# columns: beta rho phi_bar\n")
        for rho in ("0.1", "0.5", "0"):
            for beta in ("0.5", "1", "2", "4", "6", "8", "12"):
                f.write(f"{beta} {rho} {phi_bar(beta, rho):.30}\n")
        f.write("# Eq. 5 (PAPER.md:285-287) Gamma(3/beta)/Gamma(1/beta); exact: beta=2 -> 0.5, beta=1 -> 2\n")
        for beta in (1.0, 2.0, 4.0):
            g = math.exp(math.lgamma(3 / beta) - math.lgamma(1 / beta))
            f.write(f"gamma {beta} {g:.15g}\n")
