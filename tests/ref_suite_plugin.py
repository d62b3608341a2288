"""pytest plugin: route the reference package's entry points through the
B200 drop-in before the reference's own test-suite is imported
(tests/test_reference_suite.py runs that suite with ``-p ref_suite_plugin``)."""

import sketchlpa

from paper_2411_19901_b200.integration import install

install(sketchlpa)
