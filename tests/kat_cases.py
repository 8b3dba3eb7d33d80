"""Known-answer tests taken from the reference's own test suites.

Each case: (name, source, entry, expected flattened output leaves, citation).
The program texts restate the reference tests' programs (whole-file programs
with literals; `entry` is the top-level name whose value is compared).
"""

KATS = [
    ("matmul_2x2",
     "x = [[1.0, 2.0], [3.0, 4.0]]\n"
     "y = [[5.0, 6.0], [7.0, 8.0]]\n"
     "z = for i k.\n"
     "  prods = for j. (x.i.j) * (y.j.k)\n"
     "  sum prods\n",
     "z", [[19.0, 22.0, 43.0, 50.0]], "proj/tests/test_eval.cpp:60-80"),
    ("histogram_5_3",
     "points : (Fin 5) => (Fin 3) = [@0, @1, @0, @2, @0]\n"
     "hist = yieldAccum \\h.\n"
     "  for i. h!(points.i) += 1.0\n",
     "hist", [[3.0, 1.0, 1.0]], "proj/tests/test_eval.cpp:82-92"),
    ("sum_4",
     "xs = [1.0, 2.0, 3.0, 4.0]\n"
     "total = sum xs\n",
     "total", [[10.0]], "proj/tests/test_eval.cpp:46-50 (kSum)"),
    ("grad_square_at_3",
     "g = grad (\\x:Float. x * x) 3.0\n",
     "g", [[6.0]], "proj/tests/test_autodiff.cpp:130-133"),
    ("grad_sumsq",
     "f = \\xs:((Fin 2)=>Float). sum (for i. (xs.i) * (xs.i))\n"
     "g = grad f [1.0, 2.0]\n",
     "g", [[2.0, 4.0]], "proj/tests/test_autodiff.cpp:135-143"),
    ("linearize_square",
     "p = linearize (\\x:Float. x * x) 3.0\n"
     "y = fst p\n"
     "df = snd p\n"
     "dy = df 1.0\n"
     "r = (y, dy)\n",
     "r", [[9.0], [6.0]], "proj/tests/test_autodiff.cpp:145-156"),
    ("grad_stateful_recurrence",
     "f = \\xs:((Fin 3)=>Float). yieldState 0.0 \\s.\n"
     "  for i. s := ((get s) * 2.0) + (xs.i)\n"
     "  ()\n"
     "g = grad f [1.0, 2.0, 3.0]\n",
     "g", [[4.0, 2.0, 1.0]], "proj/tests/test_autodiff.cpp:184-197"),
    ("grad_trace_product",
     "b = [[5.0, 6.0], [7.0, 8.0]]\n"
     "f = \\a:((Fin 2)=>((Fin 2)=>Float)).\n"
     "  m = for i k. sum (for j. (a.i.j) * (b.j.k))\n"
     "  sum (for i. m.i.i)\n"
     "g = grad f [[1.0, 2.0], [3.0, 4.0]]\n",
     "g", [[5.0, 7.0, 6.0, 8.0]], "proj/tests/test_autodiff.cpp:199-220 (d tr(AB)/dA = B^T)"),
    ("transpose_dot",
     "c = [2.0, 3.0, 5.0]\n"
     "t = transpose (\\x:((Fin 3)=>Float). sum (for i. (x.i) * (c.i))) 2.0\n",
     "t", [[4.0, 6.0, 10.0]], "proj/tests/test_autodiff.cpp:234-243"),
    ("transpose_permutation",
     "t = transpose (\\x:((Fin 3)=>Float). for i : Fin 3. (x.(reverse i)) * 2.0) [1.0, 2.0, 3.0]\n",
     "t", [[6.0, 4.0, 2.0]], "proj/tests/test_autodiff.cpp:245-254"),
]
