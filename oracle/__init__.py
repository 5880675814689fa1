"""CPU oracle for the elastostatic BEM / KIFMM hot path of arXiv:1612.04082.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import, call or
execute anything under ``oracle/``.  The product path (the CUDA library under
``paper_1612_04082_b200/``) shares no code with this package and never imports it.

Everything here is plain, slow, fp64 numpy written from PAPER.md:

* ``kernels``  -- the four fundamental solutions U, P, D, S (Sec. 2.1,
                  Eqs. disp_1, disp_2, stress_2, stress_3) and the O(N^2) direct sum
                  of Eq. fmm_summation.
* ``tree``     -- the octree of Sec. 2.2 ("Generation of an octree partitioning of
                  the domain into boxes") built from Morton codes, and the
                  U/V/W/X interaction lists of the adaptive KIFMM.
* ``kifmm``    -- the kernel-independent FMM of Sec. 2.2 ("Kernel-independent fast
                  multipole method" paragraph): equivalent/check surfaces, upward
                  pass, downward pass, near field.
* ``gmres``    -- restarted GMRES (Sec. 2.2, "parallel implementation of GMRES").
* ``bem``      -- the collocation BIE system (Eqs. BIE, num, coef, num2).

Readings of the paper where it is garbled or ambiguous are listed in DESIGN.md
Sec. 3 and cited at the function that takes them.
"""
