"""Reference-side integration of the B200 path: the shim a
`multilap` maintainer would add, and the pytest plugin that runs the
reference's own tests through it."""
